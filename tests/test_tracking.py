"""Tracking sweeps and the fused bound (round 2, reading R25; include/lcsb.h
lcsb_sweep_ex / lcsb_sweep_bound).  A tracking sweep v_k = F(v_{k-1}) of the quarter table also
reduces R of v_k (max / min of v_k - v_{k-1}, Alg. 5 line 7) and
D = min(F(v_{k-1}) - v_{k-1}) (Alg. 5 line 8 in the form of reading R21).  Checks: tracked sweeps
store exactly the plain sweeps' tables; lcsb_bound after a tracked sweep (the D-only pass) equals
the one-pass bound bit for bit; lcsb_sweep_bound(n) equals lcsb_sweep(n-1) + lcsb_bound +
lcsb_sweep(1) bit for bit and the oracle's bound of iterate N-1 within the parity bar."""
import numpy as np
import pytest

from tests.conftest import has_cuda
from paper_2407_10925_b200 import lcsb as L

BOUND_KEYS = ("R_max", "R_min", "E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin",
              "bound", "best_bound", "sweeps_done", "best_sweep")


def _same_bound(a, b):
    for k in BOUND_KEYS:
        assert getattr(a, k) == getattr(b, k), (k, getattr(a, k), getattr(b, k))


def _cmp_oracle(gb, rb, dtype):
    for key in ("R_max", "R_min"):
        g, r = getattr(gb, key), rb[key]
        if dtype == "f32":
            assert g == r, (key, g, r)
        else:
            assert abs(g - r) <= 1e-12 * max(1.0, abs(r)), (key, g, r)
    for key in ("E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin"):
        g, r = getattr(gb, key), rb[key]
        assert abs(g - r) <= 1e-12 * max(1.0, abs(r)), (key, g, r)


def test_sweep_ex_and_sweep_bound_are_exported():
    assert "lcsb_sweep_ex" in L.EXPORTS and "lcsb_sweep_bound" in L.EXPORTS
    assert (L.SWEEP_TRACK, L.SWEEP_TRACK2) == (1, 3)


CASES = [(3, 2, "f32"), (5, 3, "f64"), (6, 3, "f32"), (7, 6, "f32"), (8, 4, "f64"),
         (9, 5, "f32"), (10, 6, "f32"), (10, 6, "f64"), (12, 7, "f32"), (13, 6, "f64")]


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,K,dtype", CASES)
def test_tracked_sweeps_store_the_plain_tables_and_bound(ell, K, dtype):
    """tracked and plain sweeps write identical tables; the bound after a tracked sweep (R from the
    sweep, D-only pass) equals the one-pass bound bit for bit, at several iterates"""
    hp = L.Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
    ht = L.Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
    assert ht.kernel_in_use == "bin2q"
    for n in (1, 2, 7, 13):
        hp.sweep(n)
        ht.sweep_ex(n, L.SWEEP_TRACK if n % 2 else L.SWEEP_TRACK2)
        assert np.array_equal(hp.table(0), ht.table(0))
        assert np.array_equal(hp.table(1), ht.table(1))
        _same_bound(hp.bound(), ht.bound())
    hp.destroy()
    ht.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,K,dtype", CASES[:8])
def test_sweep_bound_equals_sweeps_bound_sweep_and_oracle(ell, K, dtype):
    """lcsb_sweep_bound(n): the bound of iterate N-1 (its W's F(u,u) is sweep N) equals
    sweep(n-1) + bound + sweep(1) bit for bit (values, best-so-far, sweep counts), and the
    oracle's bound of iterate N-1; the n = 1 call after a tracked sweep stays fused"""
    from oracle import ft_oracle as fo
    ha = L.Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
    hb = L.Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
    run = fo.Run(2, 2, ell, "two_array", dtype)
    done = 0
    for n in (2, 1, 5, 1, 9, 3):
        la = ha.launch_count
        ba = ha.sweep_bound(n)
        if n == 1:  # fused: one tracking sweep (reduction init + sweep), no bound pass
            assert ha.launch_count - la <= 2
        done += n
        assert ba.sweeps_done == done - 1 and ha.sweeps_done == done
        hb.sweep(n - 1)
        bb = hb.bound()
        hb.sweep(1)
        _same_bound(ba, bb)
        assert np.array_equal(ha.table(0), hb.table(0))
        assert np.array_equal(ha.table(1), hb.table(1))
        run.sweep(n - 1)
        _cmp_oracle(ba, run.bound(), dtype)
        run.sweep(1)
    ha.destroy()
    hb.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_sweep_bound_first_call_and_errors():
    h = L.Lcsb(2, 2, 6, dtype="f32", symmetry=2, block_log4=3)
    with pytest.raises(L.LcsbError):
        h.sweep_bound(1)  # the bounded iterate would be v_0
    with pytest.raises(L.LcsbError):
        h.sweep_bound(0)
    with pytest.raises(L.LcsbError):
        h.sweep_ex(1, 4)  # unknown flag
    b = h.sweep_bound(2)  # bound of v_1 (the b-vector)
    assert b.sweeps_done == 1 and h.sweeps_done == 2
    h2 = L.Lcsb(2, 2, 6, dtype="f32", symmetry=2, block_log4=3)
    h2.sweep(1)
    _same_bound(b, h2.bound())
    h.destroy()
    h2.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("kw", [dict(symmetry=1), dict(symmetry=0), dict(sigma=3, d=2, ell=3),
                                dict(offset_policy=1, symmetry=2, block_log4=4)])
def test_sweep_bound_without_tracking_layouts(kw):
    """half / full tables, the generic kernel and integer offsets have no tracking sweeps:
    lcsb_sweep_bound gives the same values by sweep(n-1) + bound + sweep(1); sweep_ex flags are
    accepted and ignored"""
    kw = dict(kw)
    sigma, d, ell = kw.pop("sigma", 2), kw.pop("d", 2), kw.pop("ell", 8)
    ha = L.Lcsb(sigma, d, ell, dtype="f64", form="two_array", **kw)
    hb = L.Lcsb(sigma, d, ell, dtype="f64", form="two_array", **kw)
    ha.sweep_ex(4, L.SWEEP_TRACK2)
    hb.sweep(4)
    assert np.array_equal(ha.table(0), hb.table(0))
    ba = ha.sweep_bound(6)
    hb.sweep(5)
    bb = hb.bound()
    hb.sweep(1)
    _same_bound(ba, bb)
    assert np.array_equal(ha.table(0), hb.table(0))
    ha.destroy()
    hb.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_tracking_after_graph_replay_small_table():
    """l = 8 replays captured graphs for most of a long call; the tracked sweeps run after them"""
    from oracle import ft_oracle as fo
    h = L.Lcsb(2, 2, 8, dtype="f64", symmetry=2, block_log4=4)
    run = fo.Run(2, 2, 8, "two_array", "f64")
    b = h.sweep_bound(70)
    run.sweep(69)
    _cmp_oracle(b, run.bound(), "f64")
    run.sweep(1)
    np.testing.assert_allclose(h.table(0), run.newest, rtol=1e-12, atol=0)
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_tracked_bound_config4_full_size():
    """config 4 (l = 17, fp32): 49 sweeps, sweep_bound(1) after a tracked sweep and the bound
    after a tracked sweep against the one-pass bound of a plain run, bit for bit"""
    from seeded_inputs import splitmix64_indices
    import torch
    idx = splitmix64_indices(0x240710925, 1 << 18, 1 << 34)
    h = L.Lcsb(2, 2, 17, dtype="f32", symmetry=2)
    h.sweep(48)
    h.sweep_ex(1, L.SWEEP_TRACK)         # v_49, R of v_49 tracked
    b49 = h.bound()                       # D-only pass
    bf = h.sweep_bound(1)                 # v_50; bound of v_49 from the tracking sets
    t50 = h.table_gather(idx)
    h.destroy()
    torch.cuda.empty_cache()
    h = L.Lcsb(2, 2, 17, dtype="f32", symmetry=2)
    h.sweep(49)
    p49 = h.bound()                       # one-pass bound
    h.sweep(1)
    assert np.array_equal(h.table_gather(idx), t50)
    h.destroy()
    for k in BOUND_KEYS:
        if k in ("best_bound", "best_sweep"):
            continue
        assert getattr(b49, k) == getattr(p49, k), k
        assert getattr(bf, k) == getattr(p49, k), k
