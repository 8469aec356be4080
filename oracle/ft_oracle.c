/*
 * ft_oracle.c -- CPU ORACLE for the Feasible Triplet recurrence of arXiv 2407.10925.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2407_10925_b200/, include/,
 * csrc/) may include, link, load or call this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it (through oracle/ft_oracle.py).
 * It shares no code, header, table or constant with the CUDA path.
 *
 * What it is: a plain, slow, literal transcription of
 *   - Alg. 1 "Calculating F_z"
 *   - Eq. (ineq3)  F = b + max_z F_z
 * over the FULL logical table (no symmetry folding, no row tricks, no blocking), in fp64.
 * The iteration / bound bookkeeping of Alg. 2 / Alg. 5 is driven from
 * oracle/ft_oracle.py, which calls fo_apply_F below once per F evaluation.
 *
 * Readings:
 *   R1  F_z with |N| = k reads the generation k sweeps back (Alg. 1 reads v_{|N|}; Alg. 2 calls
 *       F(v_{d-1},...,v_0), so argument 1 is the 1-back vector).
 *   R3  empty N (all heads equal z) gives F_z = 0.
 *   R4  the options are z in Sigma (masks N_z), not all subsets.
 *   R14 tuple order: idx = sum_k sum_j A_j[k] * sigma^(d(l-1-k) + (d-1-j)), i.e. heads in the
 *       most significant digit group, string 0 most significant inside a group; for
 *       sigma=2,d=2 this is the paper's interleaving (a=1011,b=0010 -> 142).
 *   R16 F_z returns sigma^(-|N|) * r (Alg. 1 line "Return sigma^{-|N|} r"), evaluated as
 *       r * (1.0 / sigma^|N|) with sigma^|N| an exact integer; r accumulates in the loop
 *       order of Alg. 1: c over Sigma^{|N|} lexicographically, c_1 (the lowest string index in
 *       N) most significant.
 *   R20 two-array form for d = 2, any sigma (extension of PAPER.md:400): the drop-both option
 *       (heads differ, N = both strings) is not offered; the others are as in Alg. 1.
 *
 * Storage rounding (dtype = f32) is applied by the caller (ft_oracle.py) after each sweep, as
 * a round-to-nearest-even cast of the fp64 result, which is what storing fp32 does.
 *
 * parity pinned: see tests/test_oracle_pins.py (Table 2, Appendix 3, closed forms,
 * brute-force W_n, exact l=1 rationals, Lemma-1 properties).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FO_MAXD 16
#define FO_MAXL 40

static uint64_t fo_ipow(uint64_t b, int e) {
    uint64_t r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

/* R14: decode x into A[j*ell + k] = character k of string j. */
void fo_decode(int sigma, int d, int ell, uint64_t x, int* A) {
    for (int k = ell - 1; k >= 0; --k)
        for (int j = d - 1; j >= 0; --j) {
            A[j * ell + k] = (int)(x % (uint64_t)sigma);
            x /= (uint64_t)sigma;
        }
}

/* R14: encode A (A[j*ell + k]) into the tuple index. */
uint64_t fo_encode(int sigma, int d, int ell, const int* A) {
    uint64_t x = 0;
    for (int k = 0; k < ell; ++k)
        for (int j = 0; j < d; ++j) x = x * (uint64_t)sigma + (uint64_t)A[j * ell + k];
    return x;
}

/*
 * F at one coordinate x (Eq. ineq3 + Alg. 1).
 *   src[k-1]   : the vector read by F_z when |N| = k (k = 1..d)            (R1)
 *   shift[k-1] : a constant added to every value read from src[k-1]; this is how the W pass
 *                F(v + (d-1)R 1, ..., v + 0 R 1) of Alg. 2 line 6 is formed literally
 *                (value = v[y] + shift, in fp64, before summation).
 *   two_array  : 1 = two-array form with d = 2 and sigma > 2 (reading R20): the option
 *                that drops both heads when they differ (|N| = d with b = 0) is not offered.  For
 *                sigma = 2 that option never exists, so the binary form is unaffected.
 */
static double fo_F_at(int sigma, int d, int ell, const double* const* src, const double* shift,
                      const double* post, int two_array, uint64_t x) {
    int A[FO_MAXD * FO_MAXL];
    int S[FO_MAXD * FO_MAXL];
    int N[FO_MAXD];
    int c[FO_MAXD];
    fo_decode(sigma, d, ell, x, A);

    /* b = 1 iff all strings start with the same character */
    int b = 1;
    for (int j = 1; j < d; ++j)
        if (A[j * ell + 0] != A[0]) b = 0;

    double best = -INFINITY;
    for (int z = 0; z < sigma; ++z) {
        /* N <- ( j | h(s_j) != z ), ascending (Alg. 1 line 3) */
        int nN = 0;
        for (int j = 0; j < d; ++j)
            if (A[j * ell + 0] != z) N[nN++] = j;
        if (two_array && nN == d && !b) continue; /* R20: drop-both not offered */
        double cand;
        if (nN == 0) {
            cand = post ? post[0] : 0.0; /* R3 (offsets, R26: the 0 in stored terms, -o_n) */
        } else {
            double r = 0.0;
            uint64_t combos = fo_ipow((uint64_t)sigma, nN);
            for (uint64_t t = 0; t < combos; ++t) {
                /* (c_1..c_|N|) in lexicographic order, c_1 most significant */
                uint64_t tt = t;
                for (int q = nN - 1; q >= 0; --q) {
                    c[q] = (int)(tt % (uint64_t)sigma);
                    tt /= (uint64_t)sigma;
                }
                memcpy(S, A, sizeof(int) * (size_t)d * (size_t)ell);
                /* s_{N[j]} <- T(s_{N[j]}) c_j  (Alg. 1 lines 5-7) */
                for (int q = 0; q < nN; ++q) {
                    int j = N[q];
                    for (int k = 0; k + 1 < ell; ++k) S[j * ell + k] = A[j * ell + k + 1];
                    S[j * ell + ell - 1] = c[q];
                }
                uint64_t y = fo_encode(sigma, d, ell, S);
                r = r + (src[nN - 1][y] + shift[nN - 1]); /* r <- r + v_{|N|}[s] (line 8) */
            }
            double inv = 1.0 / (double)combos; /* sigma^{-|N|} (R16) */
            cand = inv * r;
            /* integer offsets, KS form (R26): the table |N| sweeps back is read relative to the
             * newest one's offset, F_z(s + p) = F_z(s) + p (Lemma 1 (2)); p is added to the mean */
            if (post) cand = cand + post[nN];
        }
        if (cand > best) best = cand;
    }
    return (double)b + best;
}

/*
 * out = F(src[0], ..., src[d-1]) over all sigma^(d*ell) coordinates.
 * threads <= 0 uses the OpenMP default.  Coordinates are independent, so the
 * thread count does not change any value.
 */
int fo_apply_F(int sigma, int d, int ell, const double* const* src, const double* shift,
               double* out, int threads, int two_array) {
    if (sigma < 2 || d < 2 || ell < 1 || d > FO_MAXD || ell > FO_MAXL) return 1;
    if (two_array && d != 2) return 1;
    uint64_t n = fo_ipow((uint64_t)sigma, d * ell);
    double zero[FO_MAXD] = {0};
    const double* sh = shift ? shift : zero;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t x = 0; x < (int64_t)n; ++x) out[x] = fo_F_at(sigma, d, ell, src, sh, NULL, two_array, (uint64_t)x);
    (void)threads;
    return 0;
}

/* fo_apply_F with post[k] added to every F_z whose |N| = k >= 1, after its mean, and post[0]
 * as the value of the |N| = 0 option instead of R3's 0 (reading R26; d + 1 entries). */
int fo_apply_F_post(int sigma, int d, int ell, const double* const* src, const double* post,
                    double* out, int threads, int two_array) {
    if (sigma < 2 || d < 2 || ell < 1 || d > FO_MAXD || ell > FO_MAXL || !post) return 1;
    if (two_array && d != 2) return 1;
    uint64_t n = fo_ipow((uint64_t)sigma, d * ell);
    double zero[FO_MAXD] = {0};
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t x = 0; x < (int64_t)n; ++x)
        out[x] = fo_F_at(sigma, d, ell, src, zero, post, two_array, (uint64_t)x);
    (void)threads;
    return 0;
}

/* F at a list of coordinates only (used by the sampled mode in ft_oracle.py). */
int fo_apply_F_at(int sigma, int d, int ell, const double* const* src, const double* shift,
                  const uint64_t* idx, int64_t count, double* out, int two_array) {
    if (sigma < 2 || d < 2 || ell < 1 || d > FO_MAXD || ell > FO_MAXL) return 1;
    if (two_array && d != 2) return 1;
    double zero[FO_MAXD] = {0};
    const double* sh = shift ? shift : zero;
    for (int64_t i = 0; i < count; ++i) out[i] = fo_F_at(sigma, d, ell, src, sh, NULL, two_array, idx[i]);
    return 0;
}

/*
 * Sampled mode for large l (l >= 17), where the full table does not fit in host RAM:
 * the value of the table after `sweeps` sweeps at coordinate x, by plain top-down recursion
 * from the all-zero start.  Each level evaluates Eq. (ineq3) exactly as
 * fo_F_at does, reading the previous levels' values through recursion instead of a stored
 * table, and applies the storage rounding (f32) to every level, as a stored table would.
 *   form 1 = KS (Alg. 2/5: |N| = k reads k sweeps back), form 2 = two-array (every |N| reads
 *   the previous sweep).
 * Cost grows like (sigma^d * sigma)^sweeps; intended for sweeps <= 4.
 */
static double fo_value_rec(int sigma, int d, int ell, int form, int f32, int s, uint64_t x);

static double fo_value_rec(int sigma, int d, int ell, int form, int f32, int s, uint64_t x) {
    if (s <= 0) return 0.0;
    int A[FO_MAXD * FO_MAXL];
    int S[FO_MAXD * FO_MAXL];
    int N[FO_MAXD];
    int c[FO_MAXD];
    fo_decode(sigma, d, ell, x, A);
    int b = 1;
    for (int j = 1; j < d; ++j)
        if (A[j * ell + 0] != A[0]) b = 0;
    double best = -INFINITY;
    for (int z = 0; z < sigma; ++z) {
        int nN = 0;
        for (int j = 0; j < d; ++j)
            if (A[j * ell + 0] != z) N[nN++] = j;
        if (form == 2 && nN == d && !b) continue; /* R20 (as in fo_F_at) */
        double cand;
        if (nN == 0) {
            cand = 0.0;
        } else {
            int back = (form == 1) ? nN : 1;
            double r = 0.0;
            uint64_t combos = fo_ipow((uint64_t)sigma, nN);
            for (uint64_t t = 0; t < combos; ++t) {
                uint64_t tt = t;
                for (int q = nN - 1; q >= 0; --q) {
                    c[q] = (int)(tt % (uint64_t)sigma);
                    tt /= (uint64_t)sigma;
                }
                memcpy(S, A, sizeof(int) * (size_t)d * (size_t)ell);
                for (int q = 0; q < nN; ++q) {
                    int j = N[q];
                    for (int k = 0; k + 1 < ell; ++k) S[j * ell + k] = A[j * ell + k + 1];
                    S[j * ell + ell - 1] = c[q];
                }
                uint64_t y = fo_encode(sigma, d, ell, S);
                r = r + fo_value_rec(sigma, d, ell, form, f32, s - back, y);
            }
            double inv = 1.0 / (double)combos;
            cand = inv * r;
        }
        if (cand > best) best = cand;
    }
    double v = (double)b + best;
    if (f32) v = (double)(float)v; /* storage rounding, round-to-nearest-even */
    return v;
}

int fo_sample(int sigma, int d, int ell, int form, int f32, int sweeps, const uint64_t* idx,
              int64_t count, double* out, int threads) {
    if (sigma < 2 || d < 2 || ell < 1 || d > FO_MAXD || ell > FO_MAXL) return 1;
    if (form == 2 && d != 2) return 1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
    for (int64_t i = 0; i < count; ++i)
        out[i] = fo_value_rec(sigma, d, ell, form, f32, sweeps, idx[i]);
    (void)threads;
    return 0;
}

int fo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
