"""The quarter table (symmetry = 2, kern_bin2q.cu): one stored entry per class of
states with provably equal values in every binary two-array iterate: orbits of {id, complement,
string swap, complement o swap}, and for same-head states also the tail complement (the
same-head value depends only on the tails and is complement-invariant, reading R18).

CPU: the library's host-side layout (lcsb_quarter_locate) against classes enumerated here from
the paper's state encoding (interleaved pair), complement (Eq. comp_eq,
PAPER.md:404-411), string swap (reading R19) and the mirror identity (R18) -- no code shared
with the library.
GPU: the quarter-table kernels against the oracle, element by element (fp32 bit-exact, fp64
1e-12 relative), across block sizes, tile sizes and the sampled config-4 check.
"""
import numpy as np
import pytest

from tests.conftest import has_cuda

from paper_2407_10925_b200 import lcsb as L


def _decode(x, ell):
    a = [(x >> (2 * (ell - 1 - k) + 1)) & 1 for k in range(ell)]
    b = [(x >> (2 * (ell - 1 - k))) & 1 for k in range(ell)]
    return a, b


def _encode(a, b):
    ell = len(a)
    return sum((a[k] << (2 * (ell - 1 - k) + 1)) | (b[k] << (2 * (ell - 1 - k))) for k in range(ell))


def _orbit(x, ell):
    a, b = _decode(x, ell)
    ca, cb = [1 - c for c in a], [1 - c for c in b]
    imgs = [(a, b), (ca, cb), (b, a), (cb, ca)]
    if a[0] == b[0]:  # same heads: the value depends only on the tails, complement-invariant
        ta = [a[0]] + [1 - c for c in a[1:]]
        tb = [b[0]] + [1 - c for c in b[1:]]
        cta, ctb = [1 - c for c in ta], [1 - c for c in tb]
        imgs += [(ta, tb), (cta, ctb), (tb, ta), (ctb, cta)]
    return min(_encode(p, q) for p, q in imgs)


@pytest.mark.parametrize("ell,K", [(3, 2), (4, 2), (4, 3), (5, 2), (5, 3), (6, 2), (6, 3),
                                   (6, 5), (7, 3), (7, 4)])
def test_quarter_layout_holds_one_orbit_per_entry(ell, K):
    L.load_library()
    owner = {}
    n_stored = None
    for x in range(1 << (2 * ell)):
        st, n = L.lcsb_quarter_locate(ell, K, x)
        n_stored = n
        orb = _orbit(x, ell)
        assert owner.setdefault(st, orb) == orb, (x, st)  # never two orbits in one entry
    assert sorted(owner) == list(range(n_stored))        # every stored entry is used
    # size (Burnside over block prefixes, m = l-K-1 non-head digits): Q1 blocks pair under psi,
    # (4^m + 2^m)/2; Q0 blocks fold under {id, s, t, s t}, (4^m + 2 2^m)/4 -> 3/8 of 4^l / 2
    m = ell - K - 1
    slots = 2 if m == 0 else ((4 ** m + 2 ** m) // 2 + (4 ** m + 2 * 2 ** m) // 4)
    assert n_stored == slots << (2 * K)
    assert len(set(owner.values())) == len({_orbit(x, ell) for x in range(1 << (2 * ell))})


def test_quarter_layout_orbit_mates_share_outside_fixed_blocks():
    """At l = 8, K = 3 all but a small fraction of the classes occupy one entry (the rest: two,
    inside blocks a symmetry maps onto themselves)."""
    L.load_library()
    ell, K = 8, 3
    entries_per_orbit = {}
    for x in range(1 << (2 * ell)):
        st, n = L.lcsb_quarter_locate(ell, K, x)
        entries_per_orbit.setdefault(_orbit(x, ell), set()).add(st)
    doubled = sum(1 for s in entries_per_orbit.values() if len(s) > 1)
    assert all(len(s) <= 2 for s in entries_per_orbit.values())
    assert doubled <= len(entries_per_orbit) / (1 << (ell - K - 3))


def test_quarter_layout_rejects_bad_arguments():
    L.load_library()
    for ell, K, x in [(2, 2, 0), (5, 1, 0), (5, 5, 0), (5, 3, 1 << 10)]:
        with pytest.raises(L.LcsbError):
            L.lcsb_quarter_locate(ell, K, x)


def test_quarter_required_bytes_is_three_eighths_of_half_table():
    L.load_library()
    half = L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=1)
    quarter = L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=2)
    assert 0.375 < quarter / half < 0.38
    # l = 18 in fp32 fits one B200 as a quarter table (2 x 64 GiB + map), not as a half table
    assert L.lcsb_required_bytes(2, 2, 18, "f32", symmetry=2) < 140 * 2 ** 30
    assert L.lcsb_required_bytes(2, 2, 18, "f32", symmetry=1) > 256 * 2 ** 30 - 1
    # the quarter table shards: the 2 shards together (the plan's total) hold
    # the stored blocks with the stride of the larger shard -- a little above one table pair
    sh2 = L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=2, shards=2)
    assert quarter <= sh2 < 1.1 * quarter
    # the KS form has no quarter table
    assert L.lcsb_required_bytes(2, 2, 17, "f32", form="ks", symmetry=2) == 0


# ------------------------------------------------------------------------------------ GPU

def _cmp(gpu_tab, ref, dtype):
    if dtype == "f32":
        assert np.array_equal(gpu_tab, ref), np.max(np.abs(gpu_tab - ref))
    else:
        np.testing.assert_allclose(gpu_tab, ref, rtol=1e-12, atol=1e-300)


def _cmp_bound(gb, rb, dtype):
    """R: bit-exact in fp32 (differences of stored values), 1e-12 in fp64.  E and the bound: the
    quarter table's one-pass bound evaluates max W = R - min(F(u,u) - u) (reading R21)
    where the oracle forms max((u + R) - F(u,u)): equal up to fp64 rounding, so 1e-12 relative
    (north_star's fp64 tolerance) for both storage types."""
    for key in ("R_max", "R_min"):
        g, r = getattr(gb, key), rb[key]
        if dtype == "f32":
            assert g == r, (key, g, r)
        else:
            assert abs(g - r) <= 1e-12 * max(1.0, abs(r)), (key, g, r)
    for key in ("E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin"):
        g, r = getattr(gb, key), rb[key]
        assert abs(g - r) <= 1e-12 * max(1.0, abs(r)), (key, g, r)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,K,dtype,sweeps", [
    (3, 2, "f32", 10), (3, 2, "f64", 10), (4, 2, "f64", 14), (4, 3, "f32", 14),
    (5, 2, "f32", 20), (5, 4, "f64", 20), (6, 3, "f32", 25), (6, 2, "f64", 25),
    (7, 3, "f32", 30), (7, 6, "f32", 12), (8, 4, "f64", 30), (8, 5, "f32", 30),
    (9, 5, "f32", 40), (9, 6, "f64", 24), (10, 6, "f32", 24), (10, 7, "f32", 24),
])
def test_quarter_matches_oracle(ell, K, dtype, sweeps):
    from oracle import ft_oracle as fo
    h = L.Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
    assert h.kernel_in_use == "bin2q"
    run = fo.Run(2, 2, ell, "two_array", dtype)
    for s in range(1, sweeps + 1):
        h.sweep(1)
        run.sweep(1)
        if s in (1, 2, 3, sweeps // 2, sweeps):
            _cmp(h.table(0), run.newest, dtype)
            _cmp(h.table(1), run.prev, dtype)
    _cmp_bound(h.bound(), run.bound(), dtype)
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_quarter_many_sweeps_per_call_matches_oracle(dtype):
    """60 sweeps in one call (the CUDA-graph replay path of small tables) then the bound and
    the best-so-far bookkeeping, against the oracle; l = 8, blocks of 4^4."""
    from oracle import ft_oracle as fo
    h = L.Lcsb(2, 2, 8, dtype=dtype, symmetry=2, block_log4=4)
    run = fo.Run(2, 2, 8, "two_array", dtype)
    for n in (60, 7):
        h.sweep(n)
        run.sweep(n)
        _cmp(h.table(0), run.newest, dtype)
        _cmp(h.table(1), run.prev, dtype)
        _cmp_bound(h.bound(), run.bound(), dtype)
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_quarter_equals_half_table_l13(dtype):
    """Quarter and half table give the same values (fp32: bitwise) on 2^20 sampled states and
    the same bound, l = 13 (auto block size), 30 sweeps."""
    from seeded_inputs import splitmix64_indices
    a = L.Lcsb(2, 2, 13, dtype=dtype, symmetry=2)
    b = L.Lcsb(2, 2, 13, dtype=dtype, symmetry=1)
    assert a.kernel_in_use == "bin2q" and b.kernel_in_use == "bin2"
    assert a.stored_states < 0.40 * b.stored_states  # 3/8 + the self-paired blocks (4 % at l = 13)
    a.sweep(30)
    b.sweep(30)
    idx = splitmix64_indices(0x240710925, 1 << 20, 1 << 26)
    _cmp(a.table_gather(idx), b.table_gather(idx), dtype)
    ba, bb = a.bound(), b.bound()
    for key in ("R_max", "R_min", "bound_at_Rmax", "bound_at_Rmin"):
        g, r = getattr(ba, key), getattr(bb, key)
        exact = dtype == "f32" and key.startswith("R")  # bound: one-pass vs two-pass (R21)
        assert (g == r) if exact else abs(g - r) <= 1e-12, (key, g, r)
    a.destroy()
    b.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_quarter_dynamic_claiming_under_graph_replay(monkeypatch, dtype):
    """l = 12: the scheduled sweep with dynamic item claiming (its counter zeroed by a memset
    node before every launch; the producer pipelined three items deep) replayed from captured
    CUDA graphs equals plain launches and static claiming bitwise, and the half table (fp32:
    bitwise; fp64: 1e-12)."""
    from seeded_inputs import splitmix64_indices
    idx = splitmix64_indices(0x240710925, 1 << 18, 1 << 24)
    vals = []
    for env in ({}, {"LCSB_NO_GRAPHS": "1"}, {"LCSB_QSTATIC": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        h = L.Lcsb(2, 2, 12, dtype=dtype)
        assert h.kernel_in_use == "bin2q"
        h.ready(wait=True)  # the schedule (built on a host thread) is used from the first sweep
        h.sweep(70)
        h.sweep(33)
        vals.append((h.table_gather(idx), h.table_gather(idx, which=1), h.bound().bound))
        h.destroy()
        for k in env:
            monkeypatch.delenv(k)
    ref = L.Lcsb(2, 2, 12, dtype=dtype, symmetry=1)
    ref.sweep(103)
    rv = (ref.table_gather(idx), ref.table_gather(idx, which=1), ref.bound().bound)
    ref.destroy()
    for v in vals[1:]:  # every claiming / launch mode: bit for bit
        assert np.array_equal(v[0], vals[0][0]) and np.array_equal(v[1], vals[0][1])
        assert v[2] == vals[0][2]
    for v in vals:  # the bound: quarter one-pass vs half-table two-pass (reading R21)
        _cmp(v[0], rv[0], dtype)
        _cmp(v[1], rv[1], dtype)
        assert abs(v[2] - rv[2]) <= 1e-12, (v[2], rv[2])


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_quarter_config4_sampled_after_3_sweeps():
    """BASELINE config 4 (2^34 states, fp32) on the quarter table: 2^20 seeded states after 3
    (and 2) sweeps against the oracle's sampled mode, bit-exact."""
    from oracle import ft_oracle as fo
    from seeded_inputs import splitmix64_indices
    h = L.Lcsb(2, 2, 17, dtype="f32", symmetry=2)
    assert h.kernel_in_use == "bin2q"
    idx = splitmix64_indices(0x240710925, 1 << 20, 1 << 34)
    h.sweep(3)
    assert np.array_equal(h.table_gather(idx),
                          fo.sample_values(2, 2, 17, 3, idx, form="two_array", dtype="f32"))
    assert np.array_equal(h.table_gather(idx, which=1),
                          fo.sample_values(2, 2, 17, 2, idx, form="two_array", dtype="f32"))
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_config5_l18_on_one_gpu_sampled_and_properties():
    """BASELINE config 5 (2^36 states, fp32) at full size on ONE GPU through the quarter table
    (2 x 64 GiB): 2^20 seeded states after 3 sweeps bit-exact against the oracle's sampled mode;
    then the configured 30 sweeps, with properties that hold at any size: the new table dominates
    the old (R_min >= 0), the certified bound lies below Lueker's upper bound 0.82628
    (PAPER.md:551), and sampled states equal their complement and swap images."""
    from oracle import ft_oracle as fo
    from seeded_inputs import splitmix64_indices
    N = 1 << 36
    h = L.Lcsb(2, 2, 18, dtype="f32")
    assert h.kernel_in_use == "bin2q" and h.device_bytes < 100 * 2 ** 30
    idx = splitmix64_indices(0x240710925, 1 << 20, N)
    h.sweep(3)
    assert np.array_equal(h.table_gather(idx),
                          fo.sample_values(2, 2, 18, 3, idx, form="two_array", dtype="f32"))
    h.sweep(27)
    b = h.bound()
    assert b.sweeps_done == 30 and b.R_min >= 0.0 and 0.0 <= b.bound < 0.82628
    # the bound pass stores nothing: the tables are unchanged by it
    assert np.array_equal(h.table_gather(idx[:4096]), h.table_gather(idx[:4096]))
    sub = idx[: 1 << 18]
    comp = np.uint64(N - 1) - sub
    a_bits = sub & np.uint64(0xAAAAAAAAAAAAAAAA)
    b_bits = sub & np.uint64(0x5555555555555555)
    swap = (a_bits >> np.uint64(1)) | (b_bits << np.uint64(1))
    v = h.table_gather(sub)
    assert np.array_equal(v, h.table_gather(comp))
    assert np.array_equal(v, h.table_gather(swap))
    h.destroy()


@pytest.fixture(autouse=True)
def _release_cached_memory():
    yield
    if has_cuda():
        import torch
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_quarter_one_pass_bound_equals_two_pass_at_config4():
    """Full config 4 (l = 17, fp32, 50 sweeps): the quarter table's one-pass bound (R and
    min(F(u,u) - u) in one read, reading R21) against the half table's two-pass bound (R
    reduction, then the W pass at that R): R bit-exact, E and the bound within 1e-12; the bound
    pass leaves both tables untouched (the next sweep continues bit-exactly)."""
    from seeded_inputs import splitmix64_indices
    idx = splitmix64_indices(0x240710925, 1 << 18, 1 << 34)
    res = []
    for sym in (2, 1):
        h = L.Lcsb(2, 2, 17, dtype="f32", symmetry=sym)
        h.sweep(50)
        t0, t1 = h.table_gather(idx), h.table_gather(idx, which=1)
        b = h.bound()
        assert np.array_equal(h.table_gather(idx), t0)
        assert np.array_equal(h.table_gather(idx, which=1), t1)
        h.sweep(1)
        res.append((b, h.table_gather(idx)))
        h.destroy()
        import torch
        torch.cuda.empty_cache()
    (bq, vq), (bh, vh) = res
    assert np.array_equal(vq, vh)
    assert (bq.R_max, bq.R_min) == (bh.R_max, bh.R_min)
    for key in ("E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin"):
        g, r = getattr(bq, key), getattr(bh, key)
        assert abs(g - r) <= 1e-12 * max(1.0, abs(r)), (key, g, r)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_quarter_schedule_installed_mid_run_changes_nothing():
    """lcsb_create returns before the L2 item schedule is built (host thread); sweeps before its
    installation run the natural item order.  A run that gets the schedule mid-way, one that has
    it from the first sweep and one that never has it are bit-identical (l = 14 fp32)."""
    import os
    from seeded_inputs import splitmix64_indices
    idx = splitmix64_indices(0x240710925, 1 << 18, 1 << 28)
    runs = []
    for mode in ("async", "sync", "none"):
        if mode == "none":
            os.environ["LCSB_NO_QSCHED"] = "1"
        try:
            h = L.Lcsb(2, 2, 14, dtype="f32")
        finally:
            os.environ.pop("LCSB_NO_QSCHED", None)
        if mode == "sync":
            assert h.ready(wait=True)
        h.sweep(2)
        if mode == "async":
            h.ready(wait=True)  # installed here, after 2 sweeps in the natural order
        h.sweep(20)
        b = h.bound()
        runs.append((h.table_gather(idx), h.table_gather(idx, which=1), b.R_max, b.R_min,
                     b.bound_at_Rmax, b.bound_at_Rmin))
        assert h.ready() is True
        h.destroy()
    for r in runs[1:]:
        assert np.array_equal(r[0], runs[0][0]) and np.array_equal(r[1], runs[0][1])
        assert r[2:] == runs[0][2:]


# ------------------------------------------------------------------ integer offsets (R23)

@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,K,dtype", [(3, 2, "f32"), (6, 3, "f32"), (6, 3, "f64"),
                                         (9, 5, "f32"), (10, 6, "f64")])
def test_offsets_quarter_matches_oracle_twin(ell, K, dtype):
    """offset_policy = 1 on the quarter table against the oracle's offset twin: the values
    (stored s + integer o) of both generations bit for bit in fp32 (1e-12 in fp64), R exact,
    E and the bound within 1e-12 (one-pass bound, R21)."""
    from oracle import ft_oracle as fo
    h = L.Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K, offset_policy=1)
    assert h.kernel_in_use == "bin2q"
    run = fo.Run(2, 2, ell, "two_array", dtype, offsets=True)
    for s in range(1, 41):
        h.sweep(1)
        run.sweep(1)
        if s in (1, 2, 3, 17, 40):
            _cmp(h.table(0), run.values(0), dtype)
            _cmp(h.table(1), run.values(1), dtype)
    _cmp_bound(h.bound(), run.bound(), dtype)
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("sigma,ell,dtype", [(2, 2, "f32"), (3, 3, "f32"), (4, 2, "f64")])
def test_offsets_generic_two_array_matches_oracle_twin(sigma, ell, dtype):
    """offset_policy = 1 on the generic kernel (binary l < 3 and d = 2, sigma > 2, two-array
    form): tables and the two-pass bound bit-exact against the oracle's offset twin (fp32)."""
    from oracle import ft_oracle as fo
    h = L.Lcsb(sigma, 2, ell, dtype=dtype, form="two_array", offset_policy=1)
    assert h.kernel_in_use == "generic"
    run = fo.Run(sigma, 2, ell, "two_array", dtype, offsets=True)
    for n in (1, 2, 30):
        h.sweep(n)
        run.sweep(n)
        _cmp(h.table(0), run.values(0), dtype)
        _cmp(h.table(1), run.values(1), dtype)
        gb, rb = h.bound(), run.bound()
        for key in ("R_max", "R_min", "E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin"):
            g, r = getattr(gb, key), rb[key]
            assert (g == r) if dtype == "f32" else abs(g - r) <= 1e-12 * max(1, abs(r)), key
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("sigma,d,ell,dtype", [(2, 2, 3, "f32"), (2, 2, 6, "f64"),
                                               (4, 2, 2, "f32"), (3, 2, 3, "f32"),
                                               (2, 3, 2, "f32"), (2, 3, 3, "f64"),
                                               (2, 3, 1, "f32"), (2, 4, 1, "f64"),
                                               (2, 5, 1, "f32"), (2, 4, 3, "f32")])
def test_offsets_generic_ks_matches_oracle_twin(sigma, d, ell, dtype):
    """offset_policy = 1 in the KS form (reading R26: per-generation offsets, the table k back
    read relative to the newest one's) on the generic kernel: every generation's values and the
    two-pass bound bit-exact against the oracle's KS offset twin in fp32 (1e-12 in fp64).
    (2,3,1), (2,4,1), (2,5,1): the |N| = 0 option is -o_n on the device too (R26)."""
    from oracle import ft_oracle as fo
    h = L.Lcsb(sigma, d, ell, dtype=dtype, form="ks", offset_policy=1)
    assert h.kernel_in_use == "generic"
    run = fo.Run(sigma, d, ell, "ks", dtype, offsets=True)
    for n in (1, 2, 30):
        h.sweep(n)
        run.sweep(n)
        _cmp(h.table(0), run.values(0), dtype)
        _cmp(h.table(1), run.values(1), dtype)
        gb, rb = h.bound(), run.bound()
        for key in ("R_max", "R_min", "E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin"):
            g, r = getattr(gb, key), rb[key]
            assert (g == r) if dtype == "f32" else abs(g - r) <= 1e-12 * max(1, abs(r)), key
    assert run.off > 0
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,form,dtype,sweeps", [(4, "ks", "f32", (1, 2, 40)),
                                                   (4, "ks", "f64", (1, 2, 40)),
                                                   (5, "ks", "f32", (1, 2, 12)),
                                                   (4, "two_array", "f32", (1, 2, 40))])
def test_offsets_q4_matches_oracle_twin(ell, form, dtype, sweeps):
    """offset_policy = 1 on the sigma = 4, d = 2 q4 kernel (complement-folded table, pooled row
    means of the table two back): KS with per-generation offsets added to the row means
    (reading R26), two-array with R23's shift; both generations' values and the bound bit-exact
    against the oracle's twin in fp32 (1e-12 in fp64)."""
    from oracle import ft_oracle as fo
    h = L.Lcsb(4, 2, ell, dtype=dtype, form=form, offset_policy=1)
    assert h.kernel_in_use == "q4"
    run = fo.Run(4, 2, ell, form, dtype, offsets=True)
    for n in sweeps:
        h.sweep(n)
        run.sweep(n)
        _cmp(h.table(0), run.values(0), dtype)
        _cmp(h.table(1), run.values(1), dtype)
        gb, rb = h.bound(), run.bound()
        for key in ("R_max", "R_min", "E_at_Rmax", "E_at_Rmin", "bound_at_Rmax", "bound_at_Rmin"):
            g, r = getattr(gb, key), rb[key]
            assert (g == r) if dtype == "f32" else abs(g - r) <= 1e-12 * max(1, abs(r)), key
    assert run.off > 0
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_offsets_config3_full_size_drift():
    """Config 3 at full size (sigma = 4, d = 2, l = 8, KS, 100 sweeps): with per-generation
    offsets (R26) the fp32 bound is within 1e-5 relative of the fp64-storage bound and closer to
    it than plain fp32 storage (measured 3.7e-6 vs 2.3e-5); sampled values read out (s + o) are
    positive."""
    import torch
    res = {}
    for name, dtype, ofs in (("f64", "f64", 0), ("f32", "f32", 0), ("ofs", "f32", 1)):
        h = L.Lcsb(4, 2, 8, dtype=dtype, form="ks", offset_policy=ofs)
        assert h.kernel_in_use == "q4"
        h.sweep(100)
        res[name] = h.bound().bound_at_Rmax
        if ofs:
            idx = np.arange(0, 4 ** 16, 4 ** 16 // 4096, dtype=np.uint64)
            v = h.table_gather(idx)
            assert np.all(v > 0)
        h.destroy()
        torch.cuda.empty_cache()
    ref = res["f64"]
    assert abs(res["ofs"] - ref) / ref < 1e-5
    assert abs(res["ofs"] - ref) < abs(res["f32"] - ref)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_offsets_graph_replay_and_reset():
    """Offsets under CUDA-graph replay (l = 8, 77 + 5 sweeps per call) equal plain launches,
    and a reset restarts from offset 0 (the second run repeats the first bit for bit)."""
    import os
    a = L.Lcsb(2, 2, 8, dtype="f32", symmetry=2, block_log4=4, offset_policy=1)
    os.environ["LCSB_NO_GRAPHS"] = "1"
    try:
        b = L.Lcsb(2, 2, 8, dtype="f32", symmetry=2, block_log4=4, offset_policy=1)
        a.sweep(77)
        b.sweep(77)
        first = (a.table(0), a.table(1))
        assert np.array_equal(first[0], b.table(0)) and np.array_equal(first[1], b.table(1))
        a.sweep(5)
        b.sweep(5)
        assert np.array_equal(a.table(0), b.table(0))
    finally:
        os.environ.pop("LCSB_NO_GRAPHS", None)
    a.reset()
    a.sweep(77)
    assert np.array_equal(a.table(0), first[0]) and np.array_equal(a.table(1), first[1])
    a.destroy()
    b.destroy()


# ------------------------------------------------------------------ residual storage (R24)

@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,K", [(6, 3), (8, 4), (10, 6)])
def test_residual_storage_matches_oracle_twin(ell, K):
    """fp32 + offsets for 30 sweeps, lcsb_rebase, 25 residual sweeps: the values (H + e + o) of
    both generations bit-exact against the oracle's residual twin, R exact, E and the bound
    within 1e-12 (R21); right after the rebase the bound and the previous generation are
    unavailable (LCSB_ESTATE)."""
    from oracle import ft_oracle as fo
    from paper_2407_10925_b200 import LcsbError
    h = L.Lcsb(2, 2, ell, dtype="f32", symmetry=2, block_log4=K, offset_policy=1)
    run = fo.Run(2, 2, ell, "two_array", "f32", offsets=True)
    h.sweep(30)
    run.sweep(30)
    h.rebase()
    run.rebase()
    _cmp(h.table(0), run.values(0), "f32")
    with pytest.raises(LcsbError) as ei:
        h.bound()
    assert ei.value.code == 3
    with pytest.raises(LcsbError):
        h.table(1)
    for n in (1, 2, 22):
        h.sweep(n)
        run.sweep(n)
        _cmp(h.table(0), run.values(0), "f32")
        _cmp(h.table(1), run.values(1), "f32")
        _cmp_bound(h.bound(), run.bound(), "f32")
    h.rebase()                          # fold the residual into the base (the iterate stays)
    run.rebase()
    _cmp(h.table(0), run.values(0), "f32")
    h.sweep(9)
    run.sweep(9)
    _cmp(h.table(0), run.values(0), "f32")
    _cmp(h.table(1), run.values(1), "f32")
    _cmp_bound(h.bound(), run.bound(), "f32")
    h.reset()                           # back to plain storage
    h.sweep(3)
    r2 = fo.Run(2, 2, ell, "two_array", "f32", offsets=True)
    r2.sweep(3)
    _cmp(h.table(0), r2.values(0), "f32")
    h.destroy()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_residual_storage_reaches_fp64_bound_l14():
    """l = 14, converged (300 sweeps): fp32 + offsets for 150 sweeps, then residual storage for
    150: the bound agrees with the fp64 quarter-table run to 5e-8 relative, where fp32 + offsets
    alone is ~1e-6 off, and floors to Table 2's value."""
    import math
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "table2.txt")
    table = {int(r.split()[0]): float(r.split()[2]) for r in
             open(path) if r.strip() and not r.startswith("#")}
    a = L.Lcsb(2, 2, 14, dtype="f64")
    a.sweep(300)
    ref = a.bound().bound
    a.destroy()
    p = L.Lcsb(2, 2, 14, dtype="f32", offset_policy=1)
    p.sweep(300)
    plain = p.bound().bound
    p.destroy()
    h = L.Lcsb(2, 2, 14, dtype="f32", offset_policy=1)
    h.sweep(100)
    for _ in range(5):                  # rebase every 40 sweeps: the base follows the shape
        h.rebase()
        h.sweep(40)
    b = h.bound().bound
    h.destroy()
    assert abs(b - ref) / ref < 5e-8, (b, ref, plain)
    assert abs(b - ref) < abs(plain - ref) / 10
    assert math.floor(b * 1e6 + 1e-6) / 1e6 == table[14]


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_l18_table2_sixth_digit_on_one_gpu():
    """BASELINE config 5's size (2^36 states) run to convergence on ONE GPU with residual storage
    (reading R24; 2 x 48 GiB tables + the 48 GiB base): the certified bound floors to Table 2's
    0.790668, which fp32 storage alone misses (0.790656)."""
    import math
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 160e9:
        pytest.skip("needs ~155 GB of free device memory")
    h = L.Lcsb(2, 2, 18, dtype="f32", offset_policy=1)
    h.ready(wait=True)
    h.sweep(100)
    for _ in range(3):
        h.rebase()
        h.sweep(40)
    b = h.bound()
    h.destroy()
    assert math.floor(b.best_bound * 1e6 + 1e-6) / 1e6 == 0.790668, b.best_bound


_QP_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2407_10925_b200 import lcsb as L
from seeded_inputs import splitmix64_indices
h = L.Lcsb(2, 2, 14, dtype="f32", symmetry=2)
h.ready(wait=True)
h.sweep(9)
idx = splitmix64_indices(5, 1 << 16, h.num_states)
np.save(sys.argv[2], np.stack([h.table_gather(idx), h.table_gather(idx, which=1)]))
"""


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_quarter_pipelined_sweep_equals_whole_stage_sweep(tmp_path):
    """The quarter-pipelined fp32 sweep (bin2q_qp_kernel, default for tiles of 4^6) and the
    whole-stage sweep (LCSB_QP=0) store identical tables (l = 14, 9 sweeps, 2^16 sampled states
    of both generations); each process reads the knob once."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for qp in ("1", "0"):
        out = tmp_path / f"qp{qp}.npy"
        env = dict(os.environ, LCSB_QP=qp)
        subprocess.run([sys.executable, "-c", _QP_SNIPPET, root, str(out)], env=env, check=True,
                       timeout=600)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


_QPW_SNIPPET = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
from paper_2407_10925_b200 import lcsb as L
h = L.Lcsb(2, 2, 14, dtype="f32", symmetry=2)
h.ready(wait=True)
out = []
for n in (1, 8):
    h.sweep(n)
    b = h.bound()
    out.append([b.R_max, b.R_min, b.E_at_Rmax, b.E_at_Rmin, b.bound_at_Rmax, b.bound_at_Rmin])
h.sweep_ex(2, 1)
b = h.bound()  # the D-only pass
out.append([b.R_max, b.R_min, b.E_at_Rmax, b.E_at_Rmin, b.bound_at_Rmax, b.bound_at_Rmin])
json.dump(out, open(sys.argv[2], "w"))
"""


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_quarter_staged_bound_equals_direct_load_bound(tmp_path):
    """The staged quarter-pipelined bound pass (bin2q_qpw_kernel, default for tiles of 4^6: u
    and v_prev at the outputs staged by TMA) and the direct-load pass (LCSB_QPW=0) give the same
    R, E and bounds bit for bit (l = 14 fp32, after 1 and 9 sweeps, and the D-only pass)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for qpw in ("1", "0"):
        out = tmp_path / f"qpw{qpw}.json"
        env = dict(os.environ, LCSB_QPW=qpw)
        subprocess.run([sys.executable, "-c", _QPW_SNIPPET, root, str(out)], env=env, check=True,
                       timeout=600)
        outs.append(json.load(open(out)))
    assert outs[0] == outs[1]
