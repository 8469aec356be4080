// kern_bin2q_bound.cu -- the quarter table's one-pass bound (reading R21; kernel
// templates: kern_bin2q.cuh), plain and residual storage (R24).
#include "kern_bin2q.cuh"

namespace lcsbk {

cudaError_t launch_bin2q_wpass(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms) {
  constexpr bool WMODE = true;
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
  if (WMODE && dtype == LCSB_F32 && M == 6) {
    static int wv = -1;  // LCSB_BIN2Q_WDIRECT=1 (A/B): the bound pass at 2 CTAs/SM
    if (wv < 0) {
      const char* e = getenv("LCSB_BIN2Q_WDIRECT");
      wv = e ? atoi(e) : 0;
    }
    static int qpw = -1;  // the staged quarter-pipelined pass (default; LCSB_QPW=0: direct loads)
    if (qpw < 0) {
      const char* e = getenv("LCSB_QPW");
      qpw = e ? atoi(e) : 1;
    }
    if (qpw && wv == 0 && a.K >= 7)
      return q_dynamic(a, 6) ? launch_qpw<3>(a, s, sms) : launch_qpw<1>(a, s, sms);
    if (wv == 1) return launch_q<float, 6, 1, true, 2>(a, s, sms);
    // LCSB_BIN2Q_WDIRECT=2 (A/B): one 512-thread CTA per SM with two stages (prefetch overlap)
    if (wv == 2) return launch_q<float, 6, 2, true, 1, 512>(a, s, sms);
    // 3 / 4 / 5: quads unrolled by 2 (3 CTAs/SM), by 4 (2 CTAs/SM), by 2 (2 CTAs/SM)
    if (wv == 3) return launch_q<float, 6, 1, true, 3, kThreads, 2>(a, s, sms);
    if (wv == 4) return launch_q<float, 6, 1, true, 2, kThreads, 4>(a, s, sms);
    if (wv == 5) return launch_q<float, 6, 1, true, 2, kThreads, 2>(a, s, sms);
    return launch_q<float, 6, 1, true, 3>(a, s, sms);
  }
  if (WMODE && dtype == LCSB_F64 && M == 5) return launch_q<double, 5, 1, true, 3>(a, s, sms);
  if (dtype == LCSB_F32) {
    switch (M) {
      case 5: return launch_q<float, 5, 2, true>(a, s, sms);
      case 4: return launch_q<float, 4, 2, true>(a, s, sms);
      case 3: return launch_q<float, 3, 2, true>(a, s, sms);
      case 2: return launch_q<float, 2, 2, true>(a, s, sms);
      case 1: return launch_q<float, 1, 2, true>(a, s, sms);
    }
  } else {
    switch (M) {
      case 4: return launch_q<double, 4, 2, true>(a, s, sms);
      case 3: return launch_q<double, 3, 2, true>(a, s, sms);
      case 2: return launch_q<double, 2, 2, true>(a, s, sms);
      case 1: return launch_q<double, 1, 2, true>(a, s, sms);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace lcsbk
