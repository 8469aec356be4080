"""Pins for the CPU oracle (oracle/), against what the paper and the mathematics fix.

Each test names the passage it follows.  None of these calls the CUDA path.
"""
import math
import os
from fractions import Fraction
from itertools import permutations

import numpy as np
import pytest

from oracle import ft_oracle as fo
from tests import brute

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append(line.split())
    return rows


def _in_band(value: float, printed: float) -> bool:
    """Printed values are floored or rounded to 6 decimals (reading R8)."""
    return printed - 5e-7 - 1e-12 <= value < printed + 1e-6 + 1e-12


# ---------------------------------------------------------------- codec

def test_interleave_paper_example():
    # "a = 1011 and b = 0010 is represented as 0...10001110"
    assert fo.interleave_pair("1011", "0010") == 0b10001110 == 142
    assert fo.deinterleave_pair(142, 4) == ("1011", "0010")


def test_complement_index_example():
    # Eq. (comp_eq): j = 2^(2l) - 1 - i decodes to the complemented pair
    j = fo.complement_index(142, 4)
    assert j == 113
    assert fo.deinterleave_pair(j, 4) == ("0100", "1101")
    for ell in range(1, 6):
        for i in range(1 << (2 * ell - 1)):
            j = fo.complement_index(i, ell)
            assert (1 << (2 * ell)) > j >= (1 << (2 * ell - 1))
            a, b = fo.deinterleave_pair(i, ell)
            ca, cb = fo.deinterleave_pair(j, ell)
            flip = str.maketrans("01", "10")
            assert (ca, cb) == (a.translate(flip), b.translate(flip))


def test_general_order_equals_paper_interleave_for_binary():
    for ell in range(1, 5):
        for i in range(1 << (2 * ell)):
            a, b = fo.deinterleave_pair(i, ell)
            assert fo.encode_tuple([a, b], 2, 2, ell) == i


def test_general_order_worked_example():
    # reading R14: heads in the top digit group, string 0 most significant inside a group
    assert fo.encode_tuple(["21", "02"], 3, 2, 2) == 2 * 27 + 0 * 9 + 1 * 3 + 2 == 59
    assert fo.decode_tuple(59, 3, 2, 2) == ["21", "02"]


@pytest.mark.parametrize("sigma,d,ell", [(2, 2, 3), (3, 2, 2), (2, 3, 2), (3, 3, 1), (4, 2, 2),
                                         (5, 2, 1), (2, 4, 2)])
def test_codec_roundtrip_and_c_codec(sigma, d, ell):
    import ctypes
    lib = fo._lib()
    n = fo.n_states(sigma, d, ell)
    for x in range(n):
        A = fo.decode_tuple(x, sigma, d, ell)
        assert fo.encode_tuple(A, sigma, d, ell) == x
        flat = (ctypes.c_int * (d * ell))(*[int(A[j][k]) for j in range(d) for k in range(ell)])
        assert lib.fo_encode(sigma, d, ell, flat) == x


def test_head_range_classes():
    # [0,2^(2l-2)) heads 00; then (0,1); then (1,0); then 11
    for ell in range(1, 6):
        L = 2 * ell
        for x in range(1 << L):
            a, b = fo.deinterleave_pair(x, ell)
            q = x >> (L - 2)
            assert (a[0], b[0]) == {0: ("0", "0"), 1: ("0", "1"), 2: ("1", "0"), 3: ("1", "1")}[q]


# ---------------------------------------------------------------- one sweep from zero

def _b_vector(sigma, d, ell):
    n = fo.n_states(sigma, d, ell)
    out = np.zeros(n)
    for x in range(n):
        A = fo.decode_tuple(x, sigma, d, ell)
        out[x] = 1.0 if len({s[0] for s in A}) == 1 else 0.0
    return out


@pytest.mark.parametrize("sigma,d,ell,form", [(2, 2, 3, "ks"), (2, 2, 3, "two_array"),
                                              (3, 2, 2, "ks"), (2, 3, 2, "ks"), (3, 3, 1, "ks"),
                                              (4, 2, 2, "ks")])
def test_first_sweep_is_b_vector(sigma, d, ell, form):
    # W_0 = 0; with zero inputs every F_z is 0, so F = b (Eq. ineq3).
    run = fo.Run(sigma, d, ell, form)
    run.sweep()
    b = _b_vector(sigma, d, ell)
    assert np.array_equal(run.newest, b)
    # sigma choices of the shared head times sigma^(l-1) tails per string
    assert int(b.sum()) == sigma ** (d * ell - d + 1)


def test_spec_fz_toy_value():
    # sigma=2,d=2,l=1, A=("0","1"): F_1 advances a and reads v_1 at ("0","1"), ("1","1");
    # F_0 advances b and reads v_1 at ("0","0"), ("0","1")  (Eqs. F1/F0)
    v1 = np.array([0.0, 0.5, 0.0, 0.7])
    v2 = np.zeros(4)
    out = fo.apply_F(2, 2, 1, [v1, v2])
    assert out[1] == pytest.approx(0.6, abs=0)  # max(0.25, 0.6)
    assert out[0] == 1.0 + 0.0 and out[3] == 1.0


# ---------------------------------------------------------------- exact small cases

def _ell1_binary_ks(sweeps):
    """Hand specialisation of Eqs. (F1), (F0) to l = 1, using the complement
    symmetry x = v[00] = v[11], y = v[01] = v[10] and m = (x + y)/2:
      x_n = 1 + m_{n-2}   (match, both heads equal, reads two sweeps back)
      y_n = m_{n-1}       (both single advances average to m, read one sweep back)
    so m_n = (1 + m_{n-1} + m_{n-2}) / 2 with m_0 = m_{-1} = 0."""
    m = {-1: Fraction(0), 0: Fraction(0)}
    xs, ys = [], []
    for n in range(1, sweeps + 1):
        x = 1 + m[n - 2]
        y = m[n - 1]
        m[n] = (x + y) / 2
        xs.append(x)
        ys.append(y)
    return xs, ys


def test_ell1_binary_ks_exact_rationals():
    xs, ys = _ell1_binary_ks(12)
    # first terms, by hand: x = 1, 1, 3/2, 7/4, ...; y = 0, 1/2, 3/4, 9/8, ...
    assert xs[:4] == [1, 1, Fraction(3, 2), Fraction(7, 4)]
    assert ys[:4] == [0, Fraction(1, 2), Fraction(3, 4), Fraction(9, 8)]
    run = fo.Run(2, 2, 1, "ks")
    for n in range(12):
        run.sweep()
        v = run.newest
        assert v[0] == float(xs[n]) and v[3] == float(xs[n])
        assert v[1] == float(ys[n]) and v[2] == float(ys[n])


def test_ell1_binary_two_array_exact():
    # two-array form: x' = 1 + m, y' = m  =>  x_k = (k+1)/2, y_k = (k-1)/2; R = 1/2, W = 0,
    # rho = 1/2, adjusted bound 2 rho / (1 + rho) = 2/3 (reading R10)
    run = fo.Run(2, 2, 1, "two_array")
    for k in range(1, 15):
        run.sweep()
        v = run.newest
        assert list(v) == [(k + 1) / 2, (k - 1) / 2, (k - 1) / 2, (k + 1) / 2]
    res = run.bound()
    assert res["R_max"] == 0.5 and res["R_min"] == 0.5
    assert res["E_at_Rmax"] == 0.0
    assert res["bound_at_Rmax"] == pytest.approx(2.0 / 3.0, abs=1e-15)


@pytest.mark.parametrize("sigma", range(2, 11))
def test_ell1_d2_closed_form(sigma):
    # l = 1, d = 2: x_n = 1 + m_{n-2}, y_n = m_{n-1}, m = (x + (sigma-1) y)/sigma gives growth
    # r = 1/(sigma+1) per character, i.e. gamma >= 2/(sigma+1) -- Appendix 3 row l=1, d=2
    # prints exactly these values.
    res = fo.feasible_triplet(sigma, 2, 1, 300, form="ks")
    assert res["bound_at_Rmax"] == pytest.approx(2.0 / (sigma + 1), abs=1e-10)
    assert res["bound_at_Rmin"] == pytest.approx(2.0 / (sigma + 1), abs=1e-10)


# ---------------------------------------------------------------- the paper's tables

def _table2():
    return {int(r[0]): (r[1], float(r[2])) for r in _load("table2.txt")}


@pytest.mark.parametrize("ell", range(1, 9))
@pytest.mark.parametrize("form", ["two_array", "ks"])
def test_table2_binary(ell, form):
    lueker, ours = _table2()[ell]
    res = fo.feasible_triplet(2, 2, ell, 250, form=form)
    assert fo.floor6(res["bound_at_Rmax"]) == ours           # PAPER.md:56-63 "ours"
    assert fo.floor6(res["bound_at_Rmax"]) == float(lueker)  # Lueker's column
    assert fo.floor6(res["bound_at_Rmin"]) == ours


@pytest.mark.slow
@pytest.mark.parametrize("ell", [9, 10])
def test_table2_binary_larger(ell):
    _, ours = _table2()[ell]
    res = fo.feasible_triplet(2, 2, ell, 200, form="two_array")
    assert fo.floor6(res["bound_at_Rmax"]) == ours


def _appendix_cells(max_cost=3e6):
    out = []
    for r in _load("appendix3.txt"):
        s, d, ell = int(r[0]), int(r[1]), int(r[2])
        cost = s ** (d * ell) * s ** (d + 1)
        if cost <= max_cost:
            out.append((s, d, ell, float(r[3]), int(r[4]), len(r) > 5))
    return out


@pytest.mark.parametrize("sigma,d,ell,printed,line,typo", _appendix_cells())
def test_appendix3_cell(sigma, d, ell, printed, line, typo):
    run = fo.Run(sigma, d, ell, "ks")
    value = None
    for k in range(1, 601):
        run.sweep()
        if k % 25 == 0:
            value = run.bound()["bound_at_Rmax"]
            if not typo and _in_band(value, printed):
                break
    if typo:
        # reading R9: (2,4,1), (2,5,1) give 8/13; (3,6,1) gives Table 3's 0.421436
        expect = {(2, 4, 1): 8 / 13, (2, 5, 1): 8 / 13, (3, 6, 1): 0.421436}[(sigma, d, ell)]
        assert _in_band(value, expect) or abs(value - expect) < 1e-9
    else:
        assert _in_band(value, printed), (value, printed, f"PAPER.md:{line}")


# ------------------------------------------ two-array form for d = 2, sigma > 2 (reading R20)

def _appendix_d2():
    return {(int(r[0]), int(r[2])): (float(r[3]), int(r[4]))
            for r in _load("appendix3.txt") if r[1] == "2" and len(r) == 5}


def _converge(run, printed, max_sweeps=600):
    value = None
    for k in range(1, max_sweeps + 1):
        run.sweep()
        if k % 25 == 0:
            value = run.bound()["bound_at_Rmax"]
            if _in_band(value, printed):
                break
    return value


@pytest.mark.parametrize("sigma,ell", [(3, 1), (3, 2), (3, 3), (3, 4), (4, 1), (4, 2), (4, 3),
                                       (5, 1), (5, 2), (5, 3), (7, 2)])
def test_two_array_d2_matches_appendix3(sigma, ell):
    # The two-array form with the drop-both option removed (every remaining option consumes
    # 1 + gain characters, so 2 rho / (1 + rho) is a certified bound, reading R20) converges to
    # the value Appendix 3 prints for the KS form.
    printed, line = _appendix_d2()[(sigma, ell)]
    value = _converge(fo.Run(sigma, 2, ell, "two_array"), printed)
    assert _in_band(value, printed), (value, printed, f"PAPER.md:{line}")


@pytest.mark.parametrize("sigma", range(2, 11))
def test_two_array_d2_ell1_closed_form(sigma):
    # l = 1: growth 1/(sigma+1) per character in both forms, gamma >= 2/(sigma+1)
    res = fo.feasible_triplet(sigma, 2, 1, 300, form="two_array")
    assert res["bound_at_Rmax"] == pytest.approx(2.0 / (sigma + 1), abs=1e-10)


def test_two_array_d2_drop_both_must_be_excluded():
    # Keeping the drop-both option in the two-array form (cost 1 step for 2 characters, gain 0)
    # breaks the tau = 1 + gain identity and overshoots the paper's value: sigma = 3, l = 2 reaches
    # 2/3 against the printed 0.620690.  The rule therefore has to be in the oracle.
    sigma, ell = 3, 2
    g = np.zeros(fo.n_states(sigma, 2, ell))
    for _ in range(200):
        prev, g = g, fo.apply_F(sigma, 2, ell, [g, g], two_array=False)
    R = float((g - prev).max())
    E = max(0.0, float(((g + R) - fo.apply_F(sigma, 2, ell, [g, g])).max()))
    rho = R - E
    assert 2 * rho / (1 + rho) > 0.620690 + 0.01
    res = fo.feasible_triplet(sigma, 2, ell, 200, form="two_array")
    assert _in_band(res["bound_at_Rmax"], 0.620690)


def test_two_array_rejects_d_above_2():
    with pytest.raises(ValueError):
        fo.Run(3, 3, 1, "two_array")
    with pytest.raises(ValueError):
        fo.apply_F(2, 3, 1, [np.zeros(8)] * 3, two_array=True)


# ---------------------------------------------------------------- brute force

@pytest.mark.parametrize("sigma,nmax", [(2, 6), (3, 3)])
def test_iterate_dominated_by_bruteforce_W(sigma, nmax):
    # v_n <= W_n: every option of F is a valid strategy for the expected LCS (Eqs. ineq1/ineq2)
    run = fo.Run(sigma, 2, 1, "ks")
    for n in range(1, nmax + 1):
        run.sweep()
        for x in range(sigma * sigma):
            a, b = fo.decode_tuple(x, sigma, 2, 1)
            W = brute.W_pair(n, a, b, sigma)
            assert run.newest[x] <= float(W) + 1e-12
    # and the first match step is tight: W_1(0,0) = 1 = v_1[00]
    assert float(brute.W_pair(1, "0", "0", sigma)) == 1.0


def test_expected_lcs_small():
    # E[X_{2,2,1}] = 1/2 (match probability), E[X_{3,2,1}] = 1/3
    assert brute.expected_lcs(2, 1) == Fraction(1, 2)
    assert brute.expected_lcs(3, 1) == Fraction(1, 3)


# ---------------------------------------------------------------- Lemma 1 hypotheses

@pytest.mark.parametrize("sigma,d,ell", [(2, 2, 3), (3, 2, 2), (2, 3, 2), (3, 3, 1), (4, 2, 2)])
def test_lemma1_monotone_and_translation_invariant(sigma, d, ell):
    rng = np.random.default_rng(20240710 + sigma * 100 + d * 10 + ell)
    n = fo.n_states(sigma, d, ell)
    for _ in range(3):
        v = [rng.random(n) for _ in range(d)]
        u = [x + rng.random(n) for x in v]
        Fv = fo.apply_F(sigma, d, ell, v)
        Fu = fo.apply_F(sigma, d, ell, u)
        assert np.all(Fu >= Fv)                                   # monotonicity
        c = float(rng.random() * 10)
        Fc = fo.apply_F(sigma, d, ell, [x + c for x in v])
        np.testing.assert_allclose(Fc, Fv + c, rtol=0, atol=1e-12)  # translation


# ---------------------------------------------------------------- invariants of the iterates

def test_binary_iterates_complement_and_swap_symmetric():
    ell = 4
    n = 1 << (2 * ell)
    for form in ("ks", "two_array"):
        run = fo.Run(2, 2, ell, form, dtype="f32")
        for _ in range(12):
            run.sweep()
            v = run.newest
            for x in range(n):
                a, b = fo.deinterleave_pair(x, ell)
                assert v[x] == v[fo.complement_index(x, ell)]
                assert v[x] == v[fo.interleave_pair(b, a)]          # W(a,b) = W(b,a)


def test_general_iterates_alphabet_and_string_permutation_invariant():
    sigma, d, ell = 3, 2, 2
    run = fo.Run(sigma, d, ell, "ks", dtype="f32")
    for _ in range(10):
        run.sweep()
    v = run.newest
    for x in range(fo.n_states(sigma, d, ell)):
        A = fo.decode_tuple(x, sigma, d, ell)
        for perm in permutations(range(sigma)):
            B = ["".join(str(perm[int(ch)]) for ch in s) for s in A]
            assert v[fo.encode_tuple(B, sigma, d, ell)] == v[x]
        assert v[fo.encode_tuple(A[::-1], sigma, d, ell)] == v[x]


def test_iterates_monotone_in_n():
    for sigma, d, ell in [(2, 2, 3), (3, 2, 2), (2, 3, 2)]:
        run = fo.Run(sigma, d, ell, "ks")
        prev = run.newest.copy()
        for _ in range(20):
            run.sweep()
            assert np.all(run.newest >= prev)
            prev = run.newest.copy()


def test_forms_agree_at_convergence():
    for ell in range(2, 7):
        a = fo.feasible_triplet(2, 2, ell, 300, form="ks")["bound_at_Rmax"]
        b = fo.feasible_triplet(2, 2, ell, 300, form="two_array")["bound_at_Rmax"]
        assert abs(a - b) < 1e-9


def test_bound_is_below_known_upper_bound():
    # Lueker's upper bound 0.82628 -- a certified lower bound must stay below it
    for ell in range(1, 9):
        res = fo.feasible_triplet(2, 2, ell, 100, form="two_array")
        assert 0 < res["bound_at_Rmax"] < 0.82628


# ---------------------------------------------------------------- sampled mode and f32 storage

@pytest.mark.parametrize("form", ["ks", "two_array"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_sampled_mode_equals_full_table(form, dtype):
    ell = 4
    run = fo.Run(2, 2, ell, form, dtype)
    idx = np.arange(1 << (2 * ell), dtype=np.uint64)
    for s in range(1, 4):
        run.sweep()
        samp = fo.sample_values(2, 2, ell, s, idx, form=form, dtype=dtype)
        assert np.array_equal(samp, run.newest)
    for f in ("ks", "two_array"):
        run = fo.Run(3, 2, 2, f, dtype)
        idx = np.arange(81, dtype=np.uint64)
        for s in range(1, 4):
            run.sweep()
            assert np.array_equal(fo.sample_values(3, 2, 2, s, idx, form=f, dtype=dtype),
                                  run.newest)


def test_f32_storage_drift_small():
    a = fo.feasible_triplet(2, 2, 6, 150, form="two_array", dtype="f64")["bound_at_Rmax"]
    b = fo.feasible_triplet(2, 2, 6, 150, form="two_array", dtype="f32")["bound_at_Rmax"]
    assert abs(a - b) / a < 2e-5
    assert math.isfinite(b)


# ---------------------------------------------------------------- best-so-far (Alg. 2 l.2, 8-10)
#
# Alg. 2 and Alg. 5 start from the triplet (v_0, 0, 0)
# (line 2 / line 4) and replace it whenever R - E >= r - eps (line 8 / line 11: ">=", so a
# tie replaces).  The oracle reports best as a bound: d * best (KS) or 2 best / (1 + best)
# (two-array, reading R10).

def _ell1_ks_exact_bounds(sweeps):
    """Exact (R, E) after every sweep of Alg. 2 at sigma = d = 2, l = 1, from the hand
    specialisation above (x = v[00] = v[11], y = v[01] = v[10], m = (x + y)/2).  Line 6 with
    d = 2, F(v + R, v): a same-head state takes the match (reads the 2nd argument, unshifted,
    through its 4-entry mean; the z = head option gives 0 <= m), a different-head state averages
    the 1st argument over its 2 appended characters:
      W[00] = x + 2R - (1 + m),   W[01] = y + 2R - (m + R)."""
    xs, ys = _ell1_binary_ks(sweeps)
    px, py = Fraction(0), Fraction(0)
    out = []
    for x, y in zip(xs, ys):
        m = (x + y) / 2
        rs = {"max": max(x - px, y - py), "min": min(x - px, y - py)}
        row = {}
        for mode, R in rs.items():
            E = max(Fraction(0), x + 2 * R - (1 + m), y + 2 * R - (m + R))
            row[mode] = (R, E)
        out.append(row)
        px, py = x, y
    return out


def test_best_ell1_ks_exact_every_sweep():
    """Every sweep's R, E and bound d(R - E) equal the exact rationals; best = d * (the largest
    R - E so far, or 0 from the initial triplet); best_sweep = the last sweep reaching it."""
    exact = _ell1_ks_exact_bounds(40)
    run = fo.Run(2, 2, 1, "ks")
    best = {"max": (Fraction(0), 0), "min": (Fraction(0), 0)}
    for n, row in enumerate(exact, start=1):
        run.sweep()
        res = run.bound()
        for mode in ("max", "min"):
            R, E = row[mode]
            assert res["R_" + mode] == float(R)
            assert res["E_at_R" + mode] == pytest.approx(float(E), abs=1e-15)
            assert res["bound_at_R" + mode] == pytest.approx(float(2 * (R - E)), abs=1e-15)
            if R - E >= best[mode][0]:
                best[mode] = (R - E, n)
            assert res["best_at_R" + mode] == pytest.approx(float(2 * best[mode][0]), abs=1e-15)
            assert run.best_sweep[mode] == best[mode][1]
    # converged: 2/(sigma+1) = 2/3 (closed form)
    assert res["best_at_Rmax"] == pytest.approx(2 / 3, abs=1e-9)


def test_best_starts_from_initial_triplet_ks_transient():
    """KS at l = 10: for the first 20 sweeps every evaluated bound is negative (A.3's
    "<= 0" transient), so best stays the initial triplet's 0 exactly -- not -inf, not the first
    evaluated bound -- and best_sweep stays 0."""
    run = fo.Run(2, 2, 10, "ks")
    seen = []
    for _ in range(20):
        run.sweep()
        res = run.bound()
        seen.append(res["bound_at_Rmax"])
        assert res["bound_at_Rmax"] < 0.0
        assert res["best_at_Rmax"] == 0.0
        assert run.best_sweep["max"] == 0
    assert seen[0] == -2.0          # sweep 1: R = 1 (the b-vector), E = 2


def test_best_ties_replace_two_array_ell1():
    """Two-array l = 1 (exact dyadics): from sweep 1 on R_max - E = 1/2 at every sweep, so
    the ">=" of Alg. 2 line 8 replaces the triplet every time: best_sweep = the latest sweep.
    R_min = 0 at sweep 1 gives rho = 0 (a tie with the initial triplet: best_sweep 1, bound 0)."""
    run = fo.Run(2, 2, 1, "two_array")
    run.sweep()
    res = run.bound()
    assert res["R_max"] == 1.0 and res["E_at_Rmax"] == 0.5
    assert res["R_min"] == 0.0 and res["E_at_Rmin"] == 0.0
    assert res["bound_at_Rmin"] == 0.0 and res["best_at_Rmin"] == 0.0
    assert run.best_sweep == {"max": 1, "min": 1}
    for k in range(2, 12):
        run.sweep()
        res = run.bound()
        for mode in ("max", "min"):
            assert res["bound_at_R" + mode] == pytest.approx(2 / 3, abs=1e-15)
            assert res["best_at_R" + mode] == pytest.approx(2 / 3, abs=1e-15)
        assert run.best_sweep == {"max": k, "min": k}


@pytest.mark.parametrize("form", ["two_array", "ks"])
def test_best_running_max_to_table2(form):
    """l = 4, bound after every one of 300 sweeps: best is non-decreasing, equals
    max(0, every bound so far), and floors to Table 2's 0.758576 for both R
    readings."""
    run = fo.Run(2, 2, 4, form)
    running = {"max": 0.0, "min": 0.0}
    last = {"max": 0.0, "min": 0.0}
    for _ in range(300):
        run.sweep()
        res = run.bound()
        for mode in ("max", "min"):
            b = res["best_at_R" + mode]
            running[mode] = max(running[mode], res["bound_at_R" + mode])
            assert b >= last[mode]
            assert b == pytest.approx(running[mode], abs=1e-15)
            last[mode] = b
    assert fo.floor6(last["max"]) == 0.758576
    assert fo.floor6(last["min"]) == 0.758576


# ---------------------------------------------------------------- integer offsets (C17 / R23)

@pytest.mark.parametrize("ell", [1, 3, 6, 8])
def test_offsets_fp64_equal_plain_run(ell):
    """Translation invariance (Lemma 1 (2)): the offset run's values s_n + o_n
    equal the plain iterate (fp64: to rounding, 1e-12 relative) and the bound is the same to
    1e-12 (Table 2's value at convergence)."""
    a = fo.Run(2, 2, ell, "two_array", "f64")
    b = fo.Run(2, 2, ell, "two_array", "f64", offsets=True)
    for k in range(1, 121):
        a.sweep()
        b.sweep()
        if k in (1, 2, 5, 40, 120):
            np.testing.assert_allclose(b.values(0), a.newest, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(b.values(1), a.prev, rtol=1e-12, atol=1e-12)
    ra, rb = a.bound(), b.bound()
    for key in ("R_max", "R_min", "bound_at_Rmax", "bound_at_Rmin"):
        assert rb[key] == pytest.approx(ra[key], abs=1e-12), key
    assert b.off > 0 and b.off == int(b.off)


def test_offsets_ell1_exact_and_bounded_storage():
    """l = 1 two-array with offsets, exact dyadics: values (k+1)/2, (k-1)/2 at sweep k as
    without offsets; c_n = floor(min s_n) is an integer and the stored minimum stays in [0, 1)
    after the subtraction."""
    run = fo.Run(2, 2, 1, "two_array", "f64", offsets=True)
    for k in range(1, 30):
        run.sweep()
        assert list(run.values(0)) == [(k + 1) / 2, (k - 1) / 2, (k - 1) / 2, (k + 1) / 2]
        assert run.off == int(run.off)
        assert 0.0 <= run.newest.min() < 1.0 + 0.5   # min(s_n) - c_{n-1} plus one sweep's growth
    res = run.bound()
    assert res["bound_at_Rmax"] == pytest.approx(2 / 3, abs=1e-15)


def test_offsets_cut_fp32_drift():
    """fp32 storage: the offset run's bound is closer to the fp64 bound than the plain fp32 run
    (C17: the stored magnitudes stay small); l = 8, 150 sweeps."""
    ref = fo.feasible_triplet(2, 2, 8, 150, form="two_array", dtype="f64")["bound_at_Rmax"]
    plain = fo.feasible_triplet(2, 2, 8, 150, form="two_array", dtype="f32")["bound_at_Rmax"]
    off = fo.feasible_triplet(2, 2, 8, 150, form="two_array", dtype="f32",
                              offsets=True)["bound_at_Rmax"]
    assert abs(off - ref) < abs(plain - ref)
    assert abs(off - ref) / ref < 2e-6


# KS form (reading R26): every generation keeps its own integer offset

def test_offsets_ks_ell1_exact_rationals():
    """l = 1 binary KS with offsets, fp64: the values s_n + o_n are the exact rationals of the
    hand recurrence (x = 1, 1, 3/2, 7/4, ...; y = 0, 1/2, 3/4, 9/8, ...) for 12 sweeps, every
    o is an integer, and each generation's o is the one it was stored with."""
    xs, ys = _ell1_binary_ks(12)
    run = fo.Run(2, 2, 1, "ks", "f64", offsets=True)
    for n in range(12):
        run.sweep()
        v = run.values(0)
        assert v[0] == float(xs[n]) and v[3] == float(xs[n])
        assert v[1] == float(ys[n]) and v[2] == float(ys[n])
        if n >= 1:
            p = run.values(1)
            assert p[0] == float(xs[n - 1]) and p[1] == float(ys[n - 1])
        assert all(o == int(o) for o in run.goff)
        assert run.goff[0] == run.off and run.goff[1] == run.off_prev
    assert run.off > 0


@pytest.mark.parametrize("sigma,d,ell", [(2, 2, 3), (2, 2, 5), (3, 2, 2), (2, 3, 2), (4, 2, 2),
                                         (2, 3, 1), (2, 4, 1), (2, 5, 1)])
def test_offsets_ks_fp64_equal_plain_run(sigma, d, ell):
    """Translation invariance (Lemma 1 (2)) for the KS form: with per-generation
    offsets the values equal the plain KS iterate (fp64, 1e-12) at every generation, and so do
    R and the bound (Alg. 2 lines 5-7).  (2,3,1), (2,4,1), (2,5,1): the |N| = 0 option must be
    the translated 0 (-o_n, reading R26); R3's literal 0 in stored terms wins there for d >= 3
    and moves the values by up to 0.42."""
    a = fo.Run(sigma, d, ell, "ks", "f64")
    b = fo.Run(sigma, d, ell, "ks", "f64", offsets=True)
    for k in range(1, 61):
        a.sweep()
        b.sweep()
        if k in (1, 2, 3, 17, 60):
            np.testing.assert_allclose(b.values(0), a.newest, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(b.values(1), a.prev, rtol=1e-12, atol=1e-12)
            for g, o, ga in zip(b.gens, b.goff, a.gens):
                np.testing.assert_allclose(g + o, ga, rtol=1e-12, atol=1e-12)
    ra, rb = a.bound(), b.bound()
    for key in ("R_max", "R_min", "bound_at_Rmax", "bound_at_Rmin"):
        assert rb[key] == pytest.approx(ra[key], abs=1e-12), key
    assert b.off > 0 and b.off == int(b.off)


def test_offsets_ks_cut_fp32_drift():
    """KS form, fp32 storage: per-generation offsets bring the bound closer to the fp64 bound
    (sigma = 4, d = 2, l = 4, 150 sweeps: 2.0e-5 -> 1.0e-6 relative)."""
    ref = fo.feasible_triplet(4, 2, 4, 150, form="ks", dtype="f64")["bound_at_Rmax"]
    plain = fo.feasible_triplet(4, 2, 4, 150, form="ks", dtype="f32")["bound_at_Rmax"]
    off = fo.feasible_triplet(4, 2, 4, 150, form="ks", dtype="f32",
                              offsets=True)["bound_at_Rmax"]
    assert abs(off - ref) < 0.2 * abs(plain - ref)
    assert abs(off - ref) / ref < 2e-6


@pytest.mark.parametrize("sigma,d,ell", [(2, 2, 4), (4, 2, 2), (2, 3, 2), (3, 3, 1)])
def test_offsets_ks_fp32_reaches_appendix3(sigma, d, ell):
    """fp32 storage with KS offsets converges to Appendix 3's printed cell."""
    cells = {(int(r[0]), int(r[1]), int(r[2])): (float(r[3]), int(r[4]))
             for r in _load("appendix3.txt") if len(r) == 5}
    printed, line = cells[(sigma, d, ell)]
    run = fo.Run(sigma, d, ell, "ks", "f32", offsets=True)
    value = _converge(run, printed)
    assert _in_band(value, printed), (value, printed, f"PAPER.md:{line}")


# ---------------------------------------------------------------- residual storage (R24)

@pytest.mark.parametrize("ell", [6, 8, 10])
def test_residual_storage_reaches_fp64_precision(ell):
    """fp32 with offsets for 100 sweeps, then a rebase (H := the stored table, e := 0) and 80
    residual sweeps: the bound is within 1e-7 relative of the fp64 run (fp32 + offsets alone:
    ~1e-6), the residual stays below one unit, and the fp64 residual run equals the plain fp64
    run (translation invariance and exact H + e)."""
    ref = fo.feasible_triplet(2, 2, ell, 180, form="two_array", dtype="f64")
    run = fo.Run(2, 2, ell, "two_array", "f32", offsets=True)
    for _ in range(100):
        run.sweep()
    run.rebase()
    with pytest.raises(RuntimeError):
        run.bound()                       # no previous generation right after a rebase
    for _ in range(80):
        run.sweep()
    b = run.bound()
    assert abs(b["bound_at_Rmax"] - ref["bound_at_Rmax"]) / ref["bound_at_Rmax"] < 1e-7
    assert np.abs(run.newest).max() < 1.0
    r64 = fo.Run(2, 2, ell, "two_array", "f64", offsets=True)
    for _ in range(100):
        r64.sweep()
    r64.rebase()
    for _ in range(80):
        r64.sweep()
    np.testing.assert_allclose(r64.values(0), ref["table"], rtol=1e-12, atol=1e-12)
    assert r64.bound()["bound_at_Rmax"] == pytest.approx(ref["bound_at_Rmax"], abs=1e-12)


def test_residual_refold_keeps_the_iterate():
    """A second rebase folds e into H (H := round32(H + e), e := the exact residual): the values
    H + e + o are unchanged bit for bit."""
    run = fo.Run(2, 2, 5, "two_array", "f32", offsets=True)
    run.sweep(20)
    run.rebase()
    run.sweep(10)
    before = run.values(0).copy()
    run.rebase()
    assert np.array_equal(run.values(0), before)
    assert np.abs(run.newest).max() <= np.abs(run.base).max() * 2.0 ** -24
