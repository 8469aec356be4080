// kern_bin2q.cu -- the quarter-table sweep (kernel templates: kern_bin2q.cuh).
#include "kern_bin2q.cuh"

namespace lcsbk {
namespace {

static bool qp_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LCSB_QP");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// the plain sweep (fp32 Q1 path) for the handle's tile 4^M
template <bool WMODE>
cudaError_t dispatch_q(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms) {
  if (dtype == LCSB_F32) {
    switch (M) {
      case 6:  // A/B: variant 10; with a work counter the producer pipelined three deep
        if (!WMODE && qp_on()) {  // the quarter-pipelined sweep (LCSB_QP=0: bin2q_kernel)
          if (a.K < 7) break;
          return q_dynamic(a, 6) ? launch_qp<3>(a, s, sms) : launch_qp<1>(a, s, sms);
        }
        if (!WMODE && q_dynamic(a, 6))
          return launch_q<float, 6, 1, WMODE, 3, kThreads, 1, false, false, 3>(a, s, sms);
        return launch_q<float, 6, 1, WMODE, 3>(a, s, sms);
      case 5: return launch_q<float, 5, 2, WMODE>(a, s, sms);
      case 4: return launch_q<float, 4, 2, WMODE>(a, s, sms);
      case 3: return launch_q<float, 3, 2, WMODE>(a, s, sms);
      case 2: return launch_q<float, 2, 2, WMODE>(a, s, sms);
      case 1: return launch_q<float, 1, 2, WMODE>(a, s, sms);
    }
  } else {
    switch (M) {
      case 5:  // A/B: variant 9
        if (!WMODE && q_dynamic(a, 5))
          return launch_q<double, 5, 2, WMODE, 2, kThreads, 1, false, false, 3>(a, s, sms);
        return launch_q<double, 5, 2, WMODE, 2>(a, s, sms);
      case 4: return launch_q<double, 4, 2, WMODE>(a, s, sms);
      case 3: return launch_q<double, 3, 2, WMODE>(a, s, sms);
      case 2: return launch_q<double, 2, 2, WMODE>(a, s, sms);
      case 1: return launch_q<double, 1, 2, WMODE>(a, s, sms);
    }
  }
  return cudaErrorInvalidValue;
}

// Sweep variants (tile 4^M, pipeline stages S, min CTAs/SM) for the A/B (tools/ab_bin2q.py);
// 0 = the default of dispatch_q for the handle's M.  Measured on B200 at l = 17 fp32 / l = 16
// fp64: fp32 (6,1,3) 8.27 ms/sweep, (6,1,2) 8.97, (6,2,1) 10.6, M = 5 >= 12.5
// (per-item overhead); fp64 (5,2,2) 4.13, (5,3,2) 4.24, (5,2,3) 4.42, (5,1,2) 4.84.
struct QVariant {
  int m, s, mb;
};
constexpr QVariant kQ32[] = {{0, 0, 0}, {6, 1, 2}, {5, 2, 3}, {5, 3, 2}, {5, 2, 2}, {4, 4, 3},
                             {4, 6, 2}, {5, 4, 1}, {4, 3, 3}, {6, 2, 1}, {6, 1, 3}};
constexpr QVariant kQ64[] = {{0, 0, 0}, {5, 1, 2}, {5, 3, 2}, {4, 8, 3}, {4, 6, 3}, {5, 2, 3},
                             {4, 12, 2}, {4, 4, 3}, {3, 8, 3}, {5, 2, 2}, {4, 3, 3}};
constexpr int kQVariants = 11;

}  // namespace

int bin2q_variant_m(int dtype, int variant) {
  if (variant <= 0 || variant >= kQVariants) return 0;
  return (dtype == LCSB_F32) ? kQ32[variant].m : kQ64[variant].m;
}

cudaError_t launch_bin2q_sweep(const Bin2QArgs& a, int dtype, int M, int variant, cudaStream_t s,
                               int sms) {
  if (a.ost || a.base) return launch_bin2q_sweep_ext(a, dtype, M, s, sms);  // kern_bin2q_ext.cu
  if (variant <= 0) return dispatch_q<false>(a, dtype, M, s, sms);
  if (variant >= kQVariants) return cudaErrorInvalidValue;
#define LCSB_QV(T, M_, S_, MB_) \
  if (d.m == M_ && d.s == S_ && d.mb == MB_) return launch_q<T, M_, S_, false, MB_>(a, s, sms);
  if (dtype == LCSB_F32) {
    const QVariant d = kQ32[variant];
    LCSB_QV(float, 6, 1, 2) LCSB_QV(float, 5, 2, 3) LCSB_QV(float, 5, 3, 2) LCSB_QV(float, 5, 2, 2)
    LCSB_QV(float, 4, 4, 3) LCSB_QV(float, 4, 6, 2) LCSB_QV(float, 5, 4, 1) LCSB_QV(float, 4, 3, 3)
    LCSB_QV(float, 6, 2, 1) LCSB_QV(float, 6, 1, 3)
  } else {
    const QVariant d = kQ64[variant];
    LCSB_QV(double, 5, 1, 2) LCSB_QV(double, 5, 3, 2) LCSB_QV(double, 4, 8, 3)
    LCSB_QV(double, 4, 6, 3) LCSB_QV(double, 5, 2, 3) LCSB_QV(double, 4, 12, 2)
    LCSB_QV(double, 4, 4, 3) LCSB_QV(double, 3, 8, 3) LCSB_QV(double, 5, 2, 2)
    LCSB_QV(double, 4, 3, 3)
  }
#undef LCSB_QV
  return cudaErrorInvalidValue;
}

}  // namespace lcsbk
