// kern_bin2q_diff.cu -- the quarter table's tracking sweep (kernel templates: kern_bin2q.cuh):
// a sweep v_n = F(v_{n-1}) whose every stored output x also reads v_{n-1}[x] and reduces
//   R_max, R_min of v_n - v_{n-1}   (Alg. 5 line 7; R of the iterate it writes)
//   D = min(F(v_{n-1}) - v_{n-1})   (F in fp64 before the storage rounding; reading R21)
// into red_out[0..2].  The last sweep before lcsb_bound tracks, so the bound needs only the
// D pass of v_n (no read of v_{n-1}); two tracked sweeps give the whole bound of v_{n-1}
// (lcsb_sweep_bound: Alg. 2's W evaluation of iterate n-1 is the F(u,u) of sweep n, reading R25).
#include "kern_bin2q.cuh"

namespace lcsbk {

static bool qpw_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LCSB_QPW");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

cudaError_t launch_bin2q_diff(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms) {
  if (a.ost || a.base) return cudaErrorInvalidValue;  // plain storage only
  constexpr bool W = false, DF = true;
  constexpr int NT = kThreads;
  const bool dyn = q_dynamic(a, M);
  if (dtype == LCSB_F32) {
    switch (M) {
      case 6:
        // the staged quarter-pipelined pass of the bound in its tracking-sweep form (default;
        // LCSB_QPW=0: the direct-load walks below)
        if (qpw_on() && a.K >= 7)
          return dyn ? launch_qpw<3, true>(a, s, sms) : launch_qpw<1, true>(a, s, sms);
        // the register-lean fp32 walk (pair_quads_w32) at 3 CTAs/SM, like the bound pass
        // (LCSB_DIFF_MINB=2, A/B: 2 CTAs/SM, no register cap spills)
        if (getenv("LCSB_DIFF_MINB") && atoi(getenv("LCSB_DIFF_MINB")) == 2)
          return dyn ? launch_q<float, 6, 1, W, 2, NT, 1, false, false, 3, DF>(a, s, sms)
                     : launch_q<float, 6, 1, W, 2, NT, 1, false, false, 1, DF>(a, s, sms);
        if (dyn) return launch_q<float, 6, 1, W, 3, NT, 1, false, false, 3, DF>(a, s, sms);
        return launch_q<float, 6, 1, W, 3, NT, 1, false, false, 1, DF>(a, s, sms);
      case 5: return launch_q<float, 5, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 4: return launch_q<float, 4, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 3: return launch_q<float, 3, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 2: return launch_q<float, 2, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 1: return launch_q<float, 1, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
    }
  } else {
    switch (M) {
      case 5:
        if (dyn) return launch_q<double, 5, 2, W, 2, NT, 1, false, false, 3, DF>(a, s, sms);
        return launch_q<double, 5, 2, W, 2, NT, 1, false, false, 1, DF>(a, s, sms);
      case 4: return launch_q<double, 4, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 3: return launch_q<double, 3, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 2: return launch_q<double, 2, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
      case 1: return launch_q<double, 1, 2, W, 1, NT, 1, false, false, 1, DF>(a, s, sms);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace lcsbk
