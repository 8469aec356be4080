// kern_bin2q_ext.cu -- the quarter-table sweeps with integer offsets (reading R23) and with
// residual storage (R24); kernel templates: kern_bin2q.cuh.
#include "kern_bin2q.cuh"

namespace lcsbk {

cudaError_t launch_bin2q_sweep_ext(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms) {
  constexpr bool WMODE = false;
  if (a.base) {  // residual storage (reading R24): fp32, windows of base and residual, M <= 5
    if (dtype != LCSB_F32 || (!WMODE && !a.ost)) return cudaErrorInvalidValue;
    constexpr int NT = kThreads;
    switch (M < 5 ? M : 5) {
      case 5: return launch_q<float, 5, 2, WMODE, 2, NT, 1, !WMODE, true>(a, s, sms);
      case 4: return launch_q<float, 4, 2, WMODE, 1, NT, 1, !WMODE, true>(a, s, sms);
      case 3: return launch_q<float, 3, 2, WMODE, 1, NT, 1, !WMODE, true>(a, s, sms);
      case 2: return launch_q<float, 2, 2, WMODE, 1, NT, 1, !WMODE, true>(a, s, sms);
      case 1: return launch_q<float, 1, 2, WMODE, 1, NT, 1, !WMODE, true>(a, s, sms);
    }
    return cudaErrorInvalidValue;
  }
  if (!WMODE && a.ost) {  // integer offsets (reading R23): the fp64 Q1 path, shift and min
    constexpr int NT = kThreads;
    if (dtype == LCSB_F32) {
      switch (M) {
        case 6:
          if (q_dynamic(a, 6)) return launch_q<float, 6, 1, false, 3, NT, 1, true, false, 3>(a, s, sms);
          return launch_q<float, 6, 1, false, 3, NT, 1, true>(a, s, sms);
        case 5: return launch_q<float, 5, 2, false, 1, NT, 1, true>(a, s, sms);
        case 4: return launch_q<float, 4, 2, false, 1, NT, 1, true>(a, s, sms);
        case 3: return launch_q<float, 3, 2, false, 1, NT, 1, true>(a, s, sms);
        case 2: return launch_q<float, 2, 2, false, 1, NT, 1, true>(a, s, sms);
        case 1: return launch_q<float, 1, 2, false, 1, NT, 1, true>(a, s, sms);
      }
    } else {
      switch (M) {
        case 5:
          if (q_dynamic(a, 5)) return launch_q<double, 5, 2, false, 2, NT, 1, true, false, 3>(a, s, sms);
          return launch_q<double, 5, 2, false, 2, NT, 1, true>(a, s, sms);
        case 4: return launch_q<double, 4, 2, false, 1, NT, 1, true>(a, s, sms);
        case 3: return launch_q<double, 3, 2, false, 1, NT, 1, true>(a, s, sms);
        case 2: return launch_q<double, 2, 2, false, 1, NT, 1, true>(a, s, sms);
        case 1: return launch_q<double, 1, 2, false, 1, NT, 1, true>(a, s, sms);
      }
    }
    return cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace lcsbk
