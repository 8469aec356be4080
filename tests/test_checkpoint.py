"""Checkpoint / resume (lcsb_save / lcsb_load, include/lcsb.h): a run saved after k
sweeps and resumed in a fresh handle continues bit-identically to the uninterrupted run --
tables of every generation the next sweep reads, the bound and the best-so-far triplet
(Alg. 2 lines 8-10)."""
import numpy as np
import pytest

from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


@pytest.mark.parametrize("sigma,d,ell,dtype,kw", [
    (2, 2, 12, "f32", {}),                                  # quarter table (bin2q), schedule
    (2, 2, 8, "f64", {"symmetry": 1}),                      # half table (bin2)
    (4, 2, 5, "f32", {}),                                   # q4: KS ring + row-mean ring
    (3, 3, 3, "f64", {}),                                   # small, pooled KS means
    (3, 2, 3, "f32", {"form": "two_array", "offset_policy": 1}),  # generic + offsets
    (2, 2, 9, "f32", {"offset_policy": 1}),                 # quarter table + offsets
    (4, 2, 5, "f32", {"form": "ks", "offset_policy": 1}),   # q4 + KS per-generation offsets
    (2, 3, 3, "f64", {"offset_policy": 1}),                 # generic KS (d = 3) + offsets
])
def test_resume_equals_uninterrupted(tmp_path, sigma, d, ell, dtype, kw):
    from paper_2407_10925_b200 import Lcsb
    path = str(tmp_path / "run.ckpt")
    a = Lcsb(sigma, d, ell, dtype=dtype, **kw)
    a.sweep(11)
    b1 = a.bound()                      # the best-so-far triplet is part of the state
    a.save(path)
    a.sweep(9)
    ta = [a.table(k) for k in range(2)]
    ba = a.bound()
    b = Lcsb(sigma, d, ell, dtype=dtype, **kw)
    b.load(path)
    assert b.sweeps_done == 11
    b.sweep(9)
    tb = [b.table(k) for k in range(2)]
    bb = b.bound()
    for x, y in zip(ta, tb):
        assert np.array_equal(x, y)
    for key in ("R_max", "R_min", "E_at_Rmax", "E_at_Rmin", "bound", "best_bound",
                "sweeps_done", "best_sweep"):
        assert getattr(ba, key) == getattr(bb, key), key
    assert b1.sweeps_done == 11
    a.destroy()
    b.destroy()


def test_load_rejects_other_config_and_truncated_file(tmp_path):
    from paper_2407_10925_b200 import Lcsb, LcsbError
    path = str(tmp_path / "run.ckpt")
    a = Lcsb(2, 2, 8, dtype="f32", symmetry=2, block_log4=4)
    a.sweep(5)
    a.save(path)
    for other in (dict(dtype="f64", symmetry=2, block_log4=4), dict(dtype="f32", symmetry=1),
                  dict(dtype="f32", symmetry=2, block_log4=3)):
        h = Lcsb(2, 2, 8, **other)
        with pytest.raises(LcsbError) as ei:
            h.load(path)
        assert ei.value.code == 1
        h.destroy()
    data = open(path, "rb").read()
    with open(path, "wb") as f:
        f.write(data[: len(data) // 2])
    h = Lcsb(2, 2, 8, dtype="f32", symmetry=2, block_log4=4)
    with pytest.raises(LcsbError) as ei:
        h.load(path)
    assert ei.value.code == 1 and "truncated" in str(ei.value)
    with pytest.raises(LcsbError):
        h.load(str(tmp_path / "missing.ckpt"))
    h.destroy()
    a.destroy()


def test_resume_a_rebased_run(tmp_path):
    """A checkpoint of a residual-storage run (R24) resumes in a fresh handle rebased first."""
    from paper_2407_10925_b200 import Lcsb
    path = str(tmp_path / "res.ckpt")
    a = Lcsb(2, 2, 10, dtype="f32", offset_policy=1)
    a.sweep(20)
    a.rebase()
    a.sweep(5)
    a.save(path)
    a.sweep(6)
    ta, ba = a.table(0), a.bound()
    b = Lcsb(2, 2, 10, dtype="f32", offset_policy=1)
    b.rebase()                          # allocates the base; the load overwrites it
    b.load(path)
    b.sweep(6)
    assert np.array_equal(ta, b.table(0))
    assert (ba.R_max, ba.bound, ba.best_bound) == (b.bound().R_max, b.bound().bound,
                                                    b.bound().best_bound)
    a.destroy()
    b.destroy()
