"""The sharded binary half table (config 5): host-side plan checks on CPU, a
world-size-2 gloo test of the multi-process plumbing, and (GPU) virtual shards on one device
bitwise equal to the unsharded run.

The item / window / run geometry is re-derived here in plain Python from the paper's index
arithmetic (Alg. 3/4; comp_eq PAPER.md:404-411), independently of the CUDA
code, and checked against the library's host-side shard map (lcsb_shard_locate)."""
import os
import socket

import numpy as np
import pytest

from tests.conftest import has_cuda

from paper_2407_10925_b200 import lcsb as L


def _pairswap(v):
    return ((v & 0xAAAAAAAAAAAAAAAA) >> 1) | ((v & 0x5555555555555555) << 1)


def _items(ell, M):
    """Every tile pair {t, psi(t)} of the bin2 sweep: (tile, partner, windows, output runs)."""
    Lb = 2 * ell
    lmask = (1 << Lb) - 1
    q1 = 1 << (Lb - 2)
    A = 0xAAAAAAAAAAAAAAAA & lmask
    B = 0x5555555555555555 & lmask
    T = 1 << (2 * M)
    out = []
    for tau in range(1 << (Lb - 2 - 2 * M)):
        x0 = q1 + tau * T
        p0 = _pairswap(~x0 & lmask) & ~(T - 1)
        taup = (p0 - q1) // T
        if taup < tau:
            continue
        wb = (x0 & A) | ((x0 & B & ~q1) << 2)
        wp = (p0 & A) | ((p0 & B & ~q1) << 2)
        windows = [(wb, 2 * T), (wp, 2 * T)]
        runs = [(x0, T), (wb >> 2, T // 2), (q1 - (wb >> 2) - T // 2, T // 2)]
        if taup != tau:
            runs += [(p0, T), (wp >> 2, T // 2), (q1 - (wp >> 2) - T // 2, T // 2)]
        out.append((tau, taup, windows, runs))
    return out


@pytest.mark.parametrize("ell,shards", [(6, 2), (6, 4), (7, 8), (8, 2), (8, 8)])
def test_shard_map_is_a_balanced_bijection(ell, shards):
    H = 1 << (2 * ell - 1)
    seen = np.zeros((shards, H // shards), dtype=np.int8)
    for s in range(H):
        k, loc = L.lcsb_shard_locate(ell, shards, s)
        assert 0 <= k < shards and 0 <= loc < H // shards
        seen[k, loc] += 1
        # the complemented logical state lives in the same place
        assert L.lcsb_shard_locate(ell, shards, (1 << (2 * ell)) - 1 - s) == (k, loc)
    assert np.all(seen == 1)


@pytest.mark.parametrize("ell,M,shards", [(8, 4, 2), (8, 4, 4), (9, 4, 8), (10, 5, 8)])
def test_items_read_one_shard_and_write_contiguous_runs(ell, M, shards):
    """Both windows of an item lie in ONE shard (so the sweep reads only local memory), the
    item's owner is the key of its tile's leading characters, items partition the stored
    table, and every output run is contiguous inside one shard."""
    p = shards.bit_length() - 1
    assert p < ell - 1 - M
    H = 1 << (2 * ell - 1)
    covered = np.zeros(H, dtype=np.int8)
    written = np.zeros(H, dtype=np.int8)
    per_shard = [0] * shards
    h = ell - 1 - M
    for tau, taup, windows, runs in _items(ell, M):
        owners = set()
        for base, n in windows:
            locs = [L.lcsb_shard_locate(ell, shards, base + i) for i in (0, n // 2, n - 1)]
            owners |= {k for k, _ in locs}
            assert locs[-1][1] - locs[0][1] == n - 1  # contiguous in the shard
        assert len(owners) == 1
        owner = owners.pop()
        # owner from the tile's first p character pairs: kappa_i = a_i ^ b_i ^ 1
        key = 0
        for i in range(1, p + 1):
            a_i = (tau >> (2 * (h - i) + 1)) & 1
            b_i = (tau >> (2 * (h - i))) & 1
            key = (key << 1) | (a_i ^ b_i ^ 1)
        assert key == owner
        per_shard[owner] += 1
        for base, n in windows if taup != tau else windows[:1]:
            covered[base:base + n] += 1
        for base, n in runs:
            k0, l0 = L.lcsb_shard_locate(ell, shards, base)
            k1, l1 = L.lcsb_shard_locate(ell, shards, base + n - 1)
            assert k0 == k1 and l1 - l0 == n - 1
            written[base:base + n] += 1
    assert np.all(covered == 1)   # every stored entry is read by exactly one item
    assert np.all(written == 1)   # and written by exactly one item
    assert max(per_shard) - min(per_shard) <= max(per_shard) // 4 + 2  # balanced


# ------------------------------------------------------------------ world size 2 on CPU (gloo)

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, ell, M, result_dir):
    import torch.distributed as dist
    from paper_2407_10925_b200 import dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # 1. the ncclUniqueId broadcast used by create_sharded (bytes from rank 0 on every rank)
    fake = bytes(range(128)) if rank == 0 else None
    got = pdist.broadcast_id(fake)
    # 2. each rank's owned items (the kernel's enumeration, re-derived), gathered everywhere
    p = world.bit_length() - 1
    h = ell - 1 - M
    mine = []
    for tau, taup, windows, runs in _items(ell, M):
        k, _ = L.lcsb_shard_locate(ell, world, windows[0][0])
        if k == rank:
            mine.append(tau)
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    np.save(os.path.join(result_dir, f"r{rank}.npy"),
            np.array([got == bytes(range(128)), len(mine)] + sorted(sum(allv, []))))
    dist.destroy_process_group()
    del p, h


def test_world_size_2_gloo_plumbing(tmp_path):
    import torch.multiprocessing as mp
    ell, M, world = 8, 4, 2
    port = _free_port()
    mp.spawn(_gloo_worker, args=(world, port, ell, M, str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "r0.npy")
    r1 = np.load(tmp_path / "r1.npy")
    assert r0[0] == 1 and r1[0] == 1                      # id arrived intact on both ranks
    all_items = sorted(t for t, *_ in _items(ell, M))
    assert list(r0[2:]) == all_items == list(r1[2:])      # the ranks' items partition them
    assert r0[1] + r1[1] == len(all_items) and r0[1] > 0 and r1[1] > 0


# ------------------------------------------------------------------ GPU: virtual shards

@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,shards,dtype", [(8, 2, "f32"), (8, 4, "f32"), (9, 8, "f32"),
                                              (8, 2, "f64"), (9, 4, "f64"), (12, 2, "f32"),
                                              (12, 8, "f32")])
def test_virtual_shards_bitwise_equal_unsharded(ell, shards, dtype):
    import torch
    from paper_2407_10925_b200 import Lcsb
    from oracle import ft_oracle as fo
    a = Lcsb(2, 2, ell, dtype=dtype)
    b = Lcsb(2, 2, ell, dtype=dtype, shards=shards, virtual_shards=True)
    assert b.num_shards == shards
    for k in (1, 2, 9):
        a.sweep(k)
        b.sweep(k)
        assert np.array_equal(a.table(0), b.table(0))
        assert np.array_equal(a.table(1), b.table(1))
        ba, bb = a.bound(), b.bound()
        assert (ba.R_max, ba.R_min, ba.E_at_Rmax, ba.E_at_Rmin) == \
               (bb.R_max, bb.R_min, bb.E_at_Rmax, bb.E_at_Rmin)
    # tracking sweeps (reading R25) on the shards: the fused bound and the D-only pass
    a.reset()
    b.reset()
    for h in (a, b):
        h.sweep(5)
        h.bound()
        h.sweep(1)
    fa, fb = a.sweep_bound(4), b.sweep_bound(4)
    a.sweep_ex(3, 1)
    b.sweep_ex(3, 1)
    da, db = a.bound(), b.bound()
    for x, y in ((fa, fb), (da, db)):
        assert (x.R_max, x.R_min, x.E_at_Rmax, x.E_at_Rmin, x.best_bound, x.sweeps_done) == \
               (y.R_max, y.R_min, y.E_at_Rmax, y.E_at_Rmin, y.best_bound, y.sweeps_done)
    assert np.array_equal(a.table(0), b.table(0))
    a.reset()
    b.reset()
    a.sweep(12)
    b.sweep(12)
    if ell <= 9:
        ref = fo.feasible_triplet(2, 2, ell, 12, form="two_array", dtype=dtype)
        tab = b.table(0)
        if dtype == "f32":
            assert np.array_equal(tab, ref["table"])
        else:
            np.testing.assert_allclose(tab, ref["table"], rtol=1e-12)
    a.destroy()
    b.destroy()
    torch.cuda.empty_cache()


def _pm_worker(rank, world, port, out_dir):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2407_10925_b200 import Lcsb
    from paper_2407_10925_b200.dist import create_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    h = create_sharded(10, dtype="f32")   # process mode: own NCCL comm, IPC exchange, barriers
    ref = Lcsb(2, 2, 10, dtype="f32")
    h.sweep(23)
    ref.sweep(23)
    same = np.array_equal(h.table(0), ref.table(0)) and np.array_equal(h.table(1), ref.table(1))
    bh, br = h.bound(), ref.bound()
    h.reset()
    h.sweep(5)
    ref.reset()
    ref.sweep(5)
    same2 = np.array_equal(h.table(0), ref.table(0))
    np.save(os.path.join(out_dir, "pm.npy"), np.array([same, bh.bound == br.bound,
                                                       bh.R_min == br.R_min, same2]))
    h.destroy()
    ref.destroy()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_process_mode_single_rank_equals_single_gpu(tmp_path):
    """The NCCL process mode with one rank (communicator, IPC handle all-gather, per-sweep
    barrier all-reduce, bound all-reduces, collective reset/destroy) gives the single-GPU
    results bit for bit.  Runs in a spawned process (own CUDA context / process group)."""
    import torch.multiprocessing as mp
    mp.spawn(_pm_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    assert np.load(tmp_path / "pm.npy").all()


# ------------------------------------------------------------------ comm hooks (host transport)

def _hooks_worker(rank, world, port, result_dir):
    """Calls the lcsb_comm_hooks callbacks through their C function pointers, as the library
    does, over a world-size-`world` gloo group (CPU only)."""
    import ctypes
    import torch.distributed as dist
    from paper_2407_10925_b200 import dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hk = pdist.comm_hooks()
    # allgather: 64 rank-specific bytes (a cudaIpcMemHandle_t is 64 bytes)
    mine = bytes((rank * 37 + i) % 256 for i in range(64))
    allb = ctypes.create_string_buffer(64 * world)
    rc1 = hk.allgather(ctypes.c_char_p(mine), allb, 64, None)
    # allreduce_max_u64, with values whose order depends on the top bit (and a complemented min)
    top = (1 << 64) - 1
    vals = (ctypes.c_uint64 * 3)(top - rank, rank, top ^ (1000 + rank))
    rc2 = hk.allreduce_max_u64(vals, 3, None)
    rc3 = hk.barrier(None)
    np.save(os.path.join(result_dir, f"h{rank}.npy"),
            np.array([rc1, rc2, rc3] + list(allb.raw) + [int(v) for v in vals], dtype=object))
    dist.destroy_process_group()


def test_comm_hooks_over_gloo_world_size_2(tmp_path):
    """The host-transport hooks (paper_2407_10925_b200/dist.py) on CPU: allgather returns every
    rank's bytes in rank order, allreduce_max_u64 is an unsigned max (also across the top bit;
    a min passes as the max of complements, as the library encodes R_min), barrier returns 0."""
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_hooks_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    top = (1 << 64) - 1
    want = b"".join(bytes((r * 37 + i) % 256 for i in range(64)) for r in range(world))
    for r in range(world):
        res = list(np.load(tmp_path / f"h{r}.npy", allow_pickle=True))
        assert res[:3] == [0, 0, 0]
        assert bytes(res[3:3 + 64 * world]) == want
        v = res[3 + 64 * world:]
        assert v[0] == top and v[1] == world - 1
        assert top ^ v[2] == 1000  # max of complements = complement of the min


def _pm_host_worker(rank, world, port, out_dir, ell, dtype):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2407_10925_b200 import Lcsb
    from paper_2407_10925_b200.dist import create_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # every rank on the one GPU: the host transport never spins
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = create_sharded(ell, dtype=dtype, transport="host")
    assert h.num_shards == world
    out = {}
    for n in (1, 2, 20):
        h.sweep(n)
        b = h.bound()
        if rank == 0:  # any rank reads any shard (the peers' tables are IPC-mapped)
            out[n] = (h.table(0), h.table(1), b)
    h.reset()
    h.sweep(3)
    if rank == 0:
        out["reset"] = (h.table(0),)
    dist.barrier()
    h.destroy()  # collective
    if rank == 0:
        ok = []
        ref = Lcsb(2, 2, ell, dtype=dtype, symmetry=1)
        for n in (1, 2, 20):
            ref.sweep(n)
            rb = ref.bound()
            t0, t1, b = out[n]
            ok += [np.array_equal(t0, ref.table(0)), np.array_equal(t1, ref.table(1)),
                   (b.R_max, b.R_min, b.E_at_Rmax, b.E_at_Rmin, b.best_bound) ==
                   (rb.R_max, rb.R_min, rb.E_at_Rmax, rb.E_at_Rmin, rb.best_bound)]
        ref.reset()
        ref.sweep(3)
        ok.append(np.array_equal(out["reset"][0], ref.table(0)))
        if ell <= 9:  # and the oracle, element by element (23 sweeps in total before the reset)
            from oracle import ft_oracle as fo
            r = fo.feasible_triplet(2, 2, ell, 23, form="two_array", dtype=dtype)
            t = out[20][0]
            ok.append(np.array_equal(t, r["table"]) if dtype == "f32" else
                      bool(np.allclose(t, r["table"], rtol=1e-12, atol=0)))
        ref.destroy()
        np.save(os.path.join(out_dir, "pmh.npy"), np.array(ok))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("world,ell,dtype", [(2, 9, "f32"), (2, 10, "f64"), (4, 9, "f64"),
                                             (4, 11, "f32")])
def test_process_mode_multi_rank_on_one_gpu(tmp_path, world, ell, dtype):
    """2 and 4 PROCESSES, one shard each, all on cuda:0, through the host comm hooks (gloo):
    CUDA-IPC handle exchange, outputs pushed into the other processes' tables, the per-sweep
    barrier (stream synchronise + host barrier: no kernel waits on another process, so sharing
    one GPU is safe), the bound's cross-rank reductions, collective reset and destroy.  Tables
    (both generations) and bounds equal the unsharded single-process run bit for bit, and the
    oracle at l <= 9."""
    import torch.multiprocessing as mp
    mp.spawn(_pm_host_worker, args=(world, _free_port(), str(tmp_path), ell, dtype),
             nprocs=world, join=True)
    res = np.load(tmp_path / "pmh.npy")
    assert res.all(), res


# ------------------------------------------------------------------ sigma = 4 shard map (q4)

def _q4_decode(x, ell):
    """Logical sigma = 4, d = 2 index -> (a, b) digit lists (reading R14: char-position-major,
    string 0 in the more significant digit of each group)."""
    a = [(x >> (4 * (ell - 1 - k) + 2)) & 3 for k in range(ell)]
    b = [(x >> (4 * (ell - 1 - k))) & 3 for k in range(ell)]
    return a, b


def _q4_encode(a, b):
    ell = len(a)
    return sum((a[k] << (4 * (ell - 1 - k) + 2)) | (b[k] << (4 * (ell - 1 - k)))
               for k in range(ell))


@pytest.mark.parametrize("ell,shards", [(4, 2), (4, 4), (5, 8), (5, 2)])
def test_sigma4_shard_map_is_a_balanced_bijection(ell, shards):
    """lcsb_shard_locate_sigma4: complement images share a location (the fold, d -> 3 - d), the
    stored half (a_0 < 2) maps one-to-one onto P shards of N / (2P) entries."""
    L.load_library()
    N = 4 ** (2 * ell)
    seen = set()
    for x in range(N):
        k, loc = L.lcsb_shard_locate_sigma4(ell, shards, x)
        a, b = _q4_decode(x, ell)
        comp = _q4_encode([3 - c for c in a], [3 - c for c in b])
        assert L.lcsb_shard_locate_sigma4(ell, shards, comp) == (k, loc)
        if a[0] < 2:
            assert 0 <= k < shards and 0 <= loc < N // (2 * shards)
            seen.add((k, loc))
    assert len(seen) == N // 2


@pytest.mark.parametrize("ell,shards", [(4, 2), (4, 4), (5, 8)])
def test_sigma4_shard_map_keeps_every_sweep_read_local(ell, shards):
    """For every stored state x = (a, b) (a_0 < 2), the entries the q4 sweep reads for it -- the
    advance-b row (a, b[1:] c) (|N| = 1 for string b) and, through the string-swap
    symmetry W(a, b) = W(b, a) (reading R19), the advance-b row of (b, a) in place of the
    advance-a row -- all lie on ONE shard, and so do those of its swap and complement images
    (the q4 item group): a sweep reads only its own shard."""
    L.load_library()

    def home(a, b):  # shard of the advance-b row of (a, b), every appended c
        ks = {L.lcsb_shard_locate_sigma4(ell, shards, _q4_encode(a, b[1:] + [c]))[0]
              for c in range(4)}
        assert len(ks) == 1
        return ks.pop()

    rng = np.random.default_rng(7)
    xs = rng.integers(0, 4 ** (2 * ell), size=3000)
    for x in xs:
        a, b = _q4_decode(int(x), ell)
        if a[0] >= 2:
            continue
        k = home(a, b)
        assert home(b, a) == k                                   # adv_a via the swap
        ca, cb = [3 - c for c in a], [3 - c for c in b]
        assert home(ca, cb) == k and home(cb, ca) == k           # complement images


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,shards,dtype,form", [
    (4, 2, "f32", "ks"), (4, 4, "f64", "ks"), (5, 8, "f32", "ks"), (5, 4, "f32", "two_array"),
    (6, 2, "f64", "two_array"), (6, 8, "f64", "ks")])
def test_sigma4_virtual_shards_bitwise_equal_unsharded(ell, shards, dtype, form):
    """sigma = 4 (q4) on P virtual shards of one GPU: both table generations and the bound equal
    the unsharded run bit for bit after 1, 2, 3 and 12 sweeps, and the oracle at l <= 5."""
    import torch
    from paper_2407_10925_b200 import Lcsb
    from oracle import ft_oracle as fo
    a = Lcsb(4, 2, ell, dtype=dtype, form=form)
    b = Lcsb(4, 2, ell, dtype=dtype, form=form, shards=shards, virtual_shards=True)
    assert a.kernel_in_use == "q4" and b.kernel_in_use == "q4" and b.num_shards == shards
    for k in (1, 1, 1, 9):
        a.sweep(k)
        b.sweep(k)
        assert np.array_equal(a.table(0), b.table(0))
        assert np.array_equal(a.table(1), b.table(1))
        ba, bb = a.bound(), b.bound()
        assert (ba.R_max, ba.R_min, ba.E_at_Rmax, ba.E_at_Rmin) == \
               (bb.R_max, bb.R_min, bb.E_at_Rmax, bb.E_at_Rmin)
    if ell <= 5:
        ref = fo.feasible_triplet(4, 2, ell, 12, form=form, dtype=dtype)
        tab = b.table(0)
        if dtype == "f32":
            assert np.array_equal(tab, ref["table"])
        else:
            np.testing.assert_allclose(tab, ref["table"], rtol=1e-12)
    a.destroy()
    b.destroy()
    torch.cuda.empty_cache()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_sigma4_config3_virtual_shards_sampled():
    """BASELINE config 3 at full size (4^16 states, fp32, KS) on 2 virtual shards: 2^20 seeded
    states after 3 sweeps against the oracle's sampled mode, bit-exact (config 3 is the sigma = 4
    workload BASELINE runs at 1/2/4/8 GPUs)."""
    import torch
    from paper_2407_10925_b200 import Lcsb
    from oracle import ft_oracle as fo
    from seeded_inputs import splitmix64_indices
    h = Lcsb(4, 2, 8, dtype="f32", shards=2, virtual_shards=True)
    idx = splitmix64_indices(0x240710925, 1 << 20, 4 ** 16)
    h.sweep(3)
    assert np.array_equal(h.table_gather(idx),
                          fo.sample_values(4, 2, 8, 3, idx, form="ks", dtype="f32"))
    b = h.bound()  # KS after 3 sweeps: a negative (transient) bound; best stays the initial 0
    assert b.R_min >= 0.0 and b.bound < 1.0 and b.best_bound == 0.0
    h.destroy()
    torch.cuda.empty_cache()


def _pm_sigma4_worker(rank, world, port, out_dir, ell, dtype, form):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2407_10925_b200 import Lcsb
    from paper_2407_10925_b200.dist import create_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = create_sharded(ell, dtype=dtype, transport="host", sigma=4, form=form)
    out = {}
    for n in (1, 2, 10):
        h.sweep(n)
        b = h.bound()
        if rank == 0:
            out[n] = (h.table(0), h.table(1), b)
    dist.barrier()
    h.destroy()
    if rank == 0:
        ok = []
        ref = Lcsb(4, 2, ell, dtype=dtype, form=form)
        for n in (1, 2, 10):
            ref.sweep(n)
            rb = ref.bound()
            t0, t1, b = out[n]
            ok += [np.array_equal(t0, ref.table(0)), np.array_equal(t1, ref.table(1)),
                   (b.R_max, b.R_min, b.E_at_Rmax, b.E_at_Rmin) ==
                   (rb.R_max, rb.R_min, rb.E_at_Rmax, rb.E_at_Rmin)]
        ref.destroy()
        np.save(os.path.join(out_dir, "pm4.npy"), np.array(ok))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("world,ell,dtype,form", [(2, 5, "f32", "ks"), (4, 5, "f64", "two_array")])
def test_sigma4_process_mode_multi_rank_on_one_gpu(tmp_path, world, ell, dtype, form):
    """sigma = 4 over 2 and 4 PROCESSES sharing cuda:0 (host comm hooks): the row means and the
    outputs pushed into the other processes' tables; tables and bounds equal the unsharded run."""
    import torch.multiprocessing as mp
    mp.spawn(_pm_sigma4_worker, args=(world, _free_port(), str(tmp_path), ell, dtype, form),
             nprocs=world, join=True)
    assert np.load(tmp_path / "pm4.npy").all()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_comm_hook_failures_fail_loudly():
    """A process-mode handle whose comm hook reports failure does not come up: lcsb_create
    returns LCSB_ENCCL (5) with the hook named in the message; hooks missing a function are
    rejected as LCSB_EINVAL (1).  One rank (P = 1) on the GPU, no torch process group needed."""
    import ctypes
    from paper_2407_10925_b200 import Lcsb, LcsbError
    from paper_2407_10925_b200.lcsb import (ALLGATHER_FN, ALLREDUCE_FN, BARRIER_FN,
                                            LcsbCommHooks)

    def hooks(fail_allgather):
        h = LcsbCommHooks()
        h.allgather = ALLGATHER_FN(
            lambda mine, all_, n, ctx: 1 if fail_allgather else (ctypes.memmove(all_, mine, n), 0)[1])
        h.barrier = BARRIER_FN(lambda ctx: 0)
        h.allreduce_max_u64 = ALLREDUCE_FN(lambda v, n, ctx: 0)
        return h

    with pytest.raises(LcsbError) as ei:
        Lcsb(2, 2, 10, dtype="f32", shards=1, shard=0, comm_hooks=hooks(True),
             torch_allocator=False)
    assert ei.value.code == 5 and "allgather" in str(ei.value)
    bad = hooks(False)
    bad.barrier = BARRIER_FN()  # NULL function pointer
    with pytest.raises(LcsbError) as ei:
        Lcsb(2, 2, 10, dtype="f32", shards=1, shard=0, comm_hooks=bad, torch_allocator=False)
    assert ei.value.code == 1
    # and a working single-rank hook set gives the unsharded result
    ok = Lcsb(2, 2, 10, dtype="f32", shards=1, shard=0, comm_hooks=hooks(False),
              torch_allocator=False)
    ref = Lcsb(2, 2, 10, dtype="f32")
    ok.sweep(7)
    ref.sweep(7)
    assert np.array_equal(ok.table(0), ref.table(0))
    assert ok.bound().bound == ref.bound().bound
    ok.destroy()
    ref.destroy()


# ------------------------------------------------------------------ sharded quarter table (§9c)

@pytest.mark.parametrize("ell,K,shards", [(8, 4, 2), (9, 4, 4), (10, 5, 8)])
def test_quarter_shard_plan_sizes(ell, K, shards):
    """The sharded quarter table's plan (CPU): every shard gets the stride of the largest shard,
    and the shards together hold every stored block (balance within 40 % of the mean)."""
    L.load_library()
    one = L.lcsb_required_bytes(2, 2, ell, "f32", symmetry=2, block_log4=K, shards=1)
    sh = L.lcsb_required_bytes(2, 2, ell, "f32", symmetry=2, block_log4=K, shards=shards)
    map_bytes = 4 << (2 * (ell - K) - 1)
    tables_one = one - 256 - map_bytes
    tables_sh = sh - 256 - map_bytes
    assert tables_sh >= tables_one and tables_sh <= 1.4 * tables_one
    # too few prefix pairs for the key: rejected
    assert L.lcsb_required_bytes(2, 2, ell, "f32", symmetry=2, block_log4=ell - 1,
                                 shards=shards) == 0


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("ell,K,shards,dtype", [(8, 4, 2, "f32"), (9, 4, 4, "f64"),
                                                (10, 5, 8, "f32"), (12, 6, 2, "f32"),
                                                (12, 5, 4, "f64"), (13, 7, 8, "f32")])
def test_quarter_virtual_shards_bitwise_equal_unsharded(ell, K, shards, dtype):
    """The sharded quarter table (§9c) on P virtual shards of one GPU -- one virtual address
    range per table over P physical allocations, per-shard item lists, reads of other shards'
    windows and stores of their outputs -- equals the unsharded quarter table bit for bit: both
    generations and the one-pass bound after 1, 2, 3 and 12 sweeps; the oracle at l <= 9."""
    import torch
    from paper_2407_10925_b200 import Lcsb
    from oracle import ft_oracle as fo
    a = Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
    b = Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K, shards=shards,
             virtual_shards=True)
    assert b.kernel_in_use == "bin2q" and b.num_shards == shards
    a.ready(wait=True)
    for k in (1, 1, 1, 9):
        a.sweep(k)
        b.sweep(k)
        assert np.array_equal(a.table(0), b.table(0))
        assert np.array_equal(a.table(1), b.table(1))
        ba, bb = a.bound(), b.bound()
        assert (ba.R_max, ba.R_min, ba.E_at_Rmax, ba.E_at_Rmin) == \
               (bb.R_max, bb.R_min, bb.E_at_Rmax, bb.E_at_Rmin)
    if ell <= 9:
        ref = fo.feasible_triplet(2, 2, ell, 12, form="two_array", dtype=dtype)
        tab = b.table(0)
        if dtype == "f32":
            assert np.array_equal(tab, ref["table"])
        else:
            np.testing.assert_allclose(tab, ref["table"], rtol=1e-12)
    a.destroy()
    b.destroy()
    torch.cuda.empty_cache()


def _pm_quarter_worker(rank, world, port, out_dir, ell, K, dtype):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2407_10925_b200 import Lcsb
    from paper_2407_10925_b200.dist import create_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = create_sharded(ell, dtype=dtype, transport="host", symmetry=2, block_log4=K)
    assert h.kernel_in_use == "bin2q"
    out = {}
    for n in (1, 2, 15):
        h.sweep(n)
        b = h.bound()
        if rank == 0:
            out[n] = (h.table(0), h.table(1), b)
    h.reset()
    h.sweep(2)
    if rank == 0:
        out["reset"] = h.table(0)
    # tracking sweeps across processes (reading R25): the tracking sets are reduced over ranks
    h.reset()
    fb = h.sweep_bound(5)
    h.sweep_ex(3, 1)
    db = h.bound()
    if rank == 0:
        out["trk"] = (fb, db, h.table(0))
    dist.barrier()
    h.destroy()
    if rank == 0:
        ok = []
        ref = Lcsb(2, 2, ell, dtype=dtype, symmetry=2, block_log4=K)
        for n in (1, 2, 15):
            ref.sweep(n)
            rb = ref.bound()
            t0, t1, b = out[n]
            ok += [np.array_equal(t0, ref.table(0)), np.array_equal(t1, ref.table(1)),
                   (b.R_max, b.R_min, b.E_at_Rmax, b.E_at_Rmin, b.best_bound) ==
                   (rb.R_max, rb.R_min, rb.E_at_Rmax, rb.E_at_Rmin, rb.best_bound)]
        ref.reset()
        ref.sweep(2)
        ok.append(np.array_equal(out["reset"], ref.table(0)))
        ref.reset()
        ref.sweep(4)
        r4 = ref.bound()
        ref.sweep(4)
        r8 = ref.bound()
        fb, db, t8 = out["trk"]
        for x, y in ((fb, r4), (db, r8)):
            ok.append((x.R_max, x.R_min, x.E_at_Rmax, x.E_at_Rmin, x.best_bound, x.sweeps_done) ==
                      (y.R_max, y.R_min, y.E_at_Rmax, y.E_at_Rmin, y.best_bound, y.sweeps_done))
        ok.append(np.array_equal(t8, ref.table(0)))
        ref.destroy()
        np.save(os.path.join(out_dir, "pmq.npy"), np.array(ok))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("world,ell,K,dtype", [(2, 10, 5, "f32"), (4, 12, 6, "f64"),
                                                (2, 12, 7, "f32")])
def test_quarter_process_mode_multi_rank_on_one_gpu(tmp_path, world, ell, K, dtype):
    """The sharded quarter table over 2 and 4 PROCESSES on cuda:0: each process maps the peers'
    shard allocations into its table's address range (POSIX fds over Unix sockets), reads the
    peers' windows and stores into their memory; tables and bounds equal the unsharded run."""
    import torch.multiprocessing as mp
    mp.spawn(_pm_quarter_worker, args=(world, _free_port(), str(tmp_path), ell, K, dtype),
             nprocs=world, join=True)
    assert np.load(tmp_path / "pmq.npy").all()


@pytest.mark.parametrize("ell,shards", [(12, 2), (12, 4), (13, 8)])
def test_quarter_shard_plan_partitions_items_and_search_cuts_nvlink(ell, shards):
    """Host-only plan of the sharded quarter table (§9c, `lcsb_quarter_shard_plan`): the shards'
    item lists partition the tile pairs (each pair {t, psi t} run once), stay balanced, and the
    placement search moves fewer entries over NVLink than the plain xor key -- both at most the
    entries the items touch."""
    L.load_library()
    items, rd, wr = L.lcsb_quarter_shard_plan(ell, "f32", shards, 24)
    items0, rd0, wr0 = L.lcsb_quarter_shard_plan(ell, "f32", shards, 0)
    # tile pairs: the tiles of 4^M Q1 outputs (M = K - 1, K = min(7, l - 5)), paired by psi
    K = min(7, ell - 5)
    M = min(K - 1, 6)
    ntiles = 4 ** (ell - 1 - M)
    npairs = sum(1 for t in range(ntiles) if _psi_tile(ell, M, t) >= t)
    assert int(items.sum()) == npairs == int(items0.sum())
    # balance: few blocks per shard at these sizes (1.2-1.35 under either owner rule; ell = 18:
    # 1.03 / 1.09 / 1.05 at 2 / 4 / 8 shards)
    assert items.max() <= 1.4 * items.mean()
    assert (rd + wr).sum() < 0.8 * (rd0 + wr0).sum()
    T = 4 ** M
    assert (rd + wr).sum() <= npairs * (4 * T + 2 * T + 4 * (T // 2))
    with pytest.raises(L.LcsbError):
        L.lcsb_quarter_shard_plan(ell, "f32", 3, 24)


def _psi_tile(ell, M, t):
    """Tile index of psi(t) (complement o swap of the first output of Q1 tile t)."""
    L2 = 2 * ell
    lmask = (1 << L2) - 1
    q1 = 1 << (L2 - 2)
    x0 = q1 + (t << (2 * M))
    v = ~x0 & lmask
    ps = ((v & 0xAAAAAAAAAAAAAAAA) >> 1) | ((v & 0x5555555555555555) << 1)
    p0 = ps & ~((1 << (2 * M)) - 1)
    return (p0 - q1) >> (2 * M)


# ------------------------------------------------- integer offsets on the sharded layouts (R23/R26)

@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("sigma,ell,shards,dtype,form,K", [
    (2, 10, 2, "f32", "two_array", 5), (2, 12, 4, "f64", "two_array", 6),
    (2, 13, 8, "f32", "two_array", 7), (4, 5, 2, "f32", "ks", 0), (4, 5, 8, "f64", "ks", 0),
    (4, 6, 4, "f32", "two_array", 0)])
def test_offsets_virtual_shards_bitwise_equal_unsharded(sigma, ell, shards, dtype, form, K):
    """offset_policy = 1 on P virtual shards (the quarter table, sigma = 4): every shard's launch
    reduces its outputs' min into the one offset state, so the offsets, both generations' values
    and the bound equal the unsharded offset run bit for bit (and the oracle's twin at small l)."""
    import torch
    from paper_2407_10925_b200 import Lcsb
    from oracle import ft_oracle as fo
    kw = dict(symmetry=2, block_log4=K) if sigma == 2 else {}
    a = Lcsb(sigma, 2, ell, dtype=dtype, form=form, offset_policy=1, **kw)
    b = Lcsb(sigma, 2, ell, dtype=dtype, form=form, offset_policy=1, shards=shards,
             virtual_shards=True, **kw)
    assert b.num_shards == shards and a.kernel_in_use == b.kernel_in_use
    a.ready(wait=True)
    for k in (1, 1, 1, 27):
        a.sweep(k)
        b.sweep(k)
        assert np.array_equal(a.table(0), b.table(0))
        assert np.array_equal(a.table(1), b.table(1))
        ba, bb = a.bound(), b.bound()
        assert (ba.R_max, ba.R_min, ba.E_at_Rmax, ba.E_at_Rmin) == \
               (bb.R_max, bb.R_min, bb.E_at_Rmax, bb.E_at_Rmin)
    if sigma ** (2 * ell) <= 1 << 20:
        run = fo.Run(sigma, 2, ell, form, dtype, offsets=True)
        run.sweep(30)
        assert run.off > 0
        tab = b.table(0)
        if dtype == "f32":
            assert np.array_equal(tab, run.values(0))
        else:
            np.testing.assert_allclose(tab, run.values(0), rtol=1e-12)
    a.destroy()
    b.destroy()
    torch.cuda.empty_cache()


def _pm_offsets_worker(rank, world, port, out_dir, sigma, ell, dtype, form, K):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2407_10925_b200 import Lcsb
    from paper_2407_10925_b200.dist import create_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kw = dict(symmetry=2, block_log4=K) if sigma == 2 else {}
    h = create_sharded(ell, dtype=dtype, transport="host", sigma=sigma, form=form,
                       offset_policy=1, **kw)
    out = {}
    for n in (1, 2, 27):
        h.sweep(n)
        b = h.bound()
        if rank == 0:
            out[n] = (h.table(0), h.table(1), b)
    dist.barrier()
    h.destroy()
    if rank == 0:
        ok = []
        ref = Lcsb(sigma, 2, ell, dtype=dtype, form=form, offset_policy=1, **kw)
        for n in (1, 2, 27):
            ref.sweep(n)
            rb = ref.bound()
            t0, t1, b = out[n]
            ok += [np.array_equal(t0, ref.table(0)), np.array_equal(t1, ref.table(1)),
                   (b.R_max, b.R_min, b.E_at_Rmax, b.E_at_Rmin) ==
                   (rb.R_max, rb.R_min, rb.E_at_Rmax, rb.E_at_Rmin)]
        ref.destroy()
        np.save(os.path.join(out_dir, "pmo.npy"), np.array(ok))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("world,sigma,ell,dtype,form,K", [(2, 2, 10, "f32", "two_array", 5),
                                                          (4, 4, 5, "f32", "ks", 0)])
def test_offsets_process_mode_multi_rank_on_one_gpu(tmp_path, world, sigma, ell, dtype, form, K):
    """Integer offsets over 2 and 4 PROCESSES sharing cuda:0 (host comm hooks): each rank reduces
    the min of the outputs it computed, the ranks all-reduce it before every sweep's prep, and
    tables and bounds equal the unsharded offset run bit for bit."""
    import torch.multiprocessing as mp
    mp.spawn(_pm_offsets_worker, args=(world, _free_port(), str(tmp_path), sigma, ell, dtype,
                                       form, K), nprocs=world, join=True)
    assert np.load(tmp_path / "pmo.npy").all()
