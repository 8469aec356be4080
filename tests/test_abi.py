"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/lcsb.h
declares, and validates configurations on the host (no compute without a GPU)."""
import ctypes
import os
import re

import pytest

from tests.conftest import ROOT, has_cuda

import paper_2407_10925_b200 as pkg
from paper_2407_10925_b200 import lcsb as L


def _header_functions():
    src = open(os.path.join(ROOT, "include", "lcsb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lcsb_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = pkg.load_library()
    declared = _header_functions()
    assert "lcsb_create" in declared and "lcsb_sweep" in declared
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(L.EXPORTS) == declared


def test_library_is_sm100a():
    # the product .so carries sm_100a SASS (built by __graft_entry__.build())
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.SO_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_required_bytes_and_validation():
    lib = pkg.load_library()
    # config 4: two-array half table, 2 x 2^33 fp32 entries = 64 GiB (+ scratch)
    assert L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=1) == 2 * (1 << 33) * 4 + 256
    # default (auto) for l >= 12: the quarter table, 2 x ((4^9 + 2^9)/2 + (4^9 + 2^10)/4) blocks
    # of 4^7 fp32 + the block map (2^19 uint32)
    assert L.lcsb_required_bytes(2, 2, 17, "f32") == \
        2 * (131328 + 65792) * (1 << 14) * 4 + 256 + (1 << 19) * 4
    # full table when symmetry is off
    assert L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=0) == 2 * (1 << 34) * 4 + 256
    # config 3: complement-folded pooled-history KS (kern_q4.cu): 2 half tables of 4^16 / 2 fp32
    # + 3 row-mean arrays of 4^16 / 32 fp64 (the generic kernel keeps the d+1 = 3 full tables)
    assert L.lcsb_required_bytes(4, 2, 8, "f32") == 2 * (1 << 31) * 4 + 256 + 3 * (1 << 27) * 8
    assert L.lcsb_required_bytes(4, 2, 8, "f32", kernel="generic") == 3 * (1 << 32) * 4 + 256
    # config 2: 4 tables of 3^12 fp64 + the pooled means of every ring slot (kern_small.cu):
    # per row of 27, 9 means for |N| = 2 and 1 for |N| = 3
    assert L.lcsb_required_bytes(3, 3, 4, "f64") == 4 * 3 ** 12 * 8 + 256 + 4 * 3 ** 9 * 10 * 8
    # two-array for d = 2, sigma > 2 (reading R20): 2 full tables
    assert L.lcsb_required_bytes(3, 2, 2, "f32", form="two_array") == 2 * 81 * 4 + 256
    # sigma = 4 two-array runs on q4 too: the same folded tables + row-mean ring as KS
    assert L.lcsb_required_bytes(4, 2, 8, "f32", form="two_array") == \
        2 * (1 << 31) * 4 + 256 + 3 * (1 << 27) * 8
    # invalid: two-array for d > 2, d > 16, sigma^(d l) too large, symmetry without binary
    assert L.lcsb_required_bytes(2, 3, 2, "f32", form="two_array") == 0
    assert L.lcsb_required_bytes(3, 2, 2, "f32", form="two_array", symmetry=1) == 0
    assert L.lcsb_required_bytes(2, 17, 1, "f32") == 0
    assert L.lcsb_required_bytes(2, 2, 40, "f32") == 0
    assert L.lcsb_required_bytes(3, 2, 2, "f32", symmetry=1) == 0
    assert L.lcsb_required_bytes(2, 2, 1, "f32", symmetry=1) == 0
    # quarter table: the item schedule packs tile indices in 28 bits, so tiles of 4^(K-1) must
    # number <= 2^28: l = 17 with block_log4 = 2 (4^15 tiles) is rejected, while
    # block_log4 = 3 (4^14 tiles) and the auto block_log4 = 7 are accepted
    assert L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=2, block_log4=2) == 0
    assert L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=2, block_log4=3) > 0
    assert L.lcsb_required_bytes(2, 2, 17, "f32", symmetry=2, block_log4=7) > 0
    assert L.lcsb_required_bytes(2, 2, 18, "f32", symmetry=2, block_log4=3) == 0
    # integer offsets (readings R23, R26): not the half table, not sharded; + 512 B.  KS form:
    # sigma = 4, d = 2 keeps the q4 layout; otherwise the generic kernel over d + 1 full tables
    # (never the quarter table or the small kernels)
    q8 = L.lcsb_required_bytes(2, 2, 8, "f32", symmetry=2)
    assert L.lcsb_required_bytes(2, 2, 8, "f32", offset_policy=1) == q8 + 512
    assert L.lcsb_required_bytes(2, 2, 8, "f32", form="ks", offset_policy=1) == \
        3 * 4 ** 8 * 4 + 256 + 512
    assert L.lcsb_required_bytes(4, 2, 4, "f32", form="ks", offset_policy=1) == \
        L.lcsb_required_bytes(4, 2, 4, "f32", form="ks") + 512
    assert L.lcsb_required_bytes(4, 2, 5, "f32", form="two_array", offset_policy=1) == \
        L.lcsb_required_bytes(4, 2, 5, "f32", form="two_array") + 512
    assert L.lcsb_required_bytes(2, 3, 3, "f64", offset_policy=1) == 4 * 2 ** 9 * 8 + 256 + 512
    assert L.lcsb_required_bytes(2, 2, 8, "f32", form="ks", symmetry=2, offset_policy=1) == 0
    assert L.lcsb_required_bytes(2, 2, 8, "f32", symmetry=1, offset_policy=1) == 0
    # sharded: the quarter table and sigma = 4 carry offsets (the min crosses the ranks), the
    # half table does not
    assert L.lcsb_required_bytes(2, 2, 12, "f32", shards=2, symmetry=1, offset_policy=1) == 0
    assert L.lcsb_required_bytes(2, 2, 12, "f32", shards=2, symmetry=2, offset_policy=1) == \
        L.lcsb_required_bytes(2, 2, 12, "f32", shards=2, symmetry=2) + 512
    assert L.lcsb_required_bytes(4, 2, 5, "f32", form="ks", shards=2, offset_policy=1) == \
        L.lcsb_required_bytes(4, 2, 5, "f32", form="ks", shards=2) + 512
    assert L.lcsb_required_bytes(2, 2, 8, "f32", offset_policy=2) == 0
    assert L.lcsb_required_bytes(3, 2, 3, "f32", form="two_array", offset_policy=1) == \
        2 * 3 ** 6 * 4 + 256 + 512


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure path")
def test_create_fails_loudly_without_gpu():
    lib = pkg.load_library()
    cfg = L.make_config(2, 2, 4, "f32")
    h = ctypes.c_void_p()
    rc = lib.lcsb_create_ex(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == 4  # LCSB_ECUDA: there is no CPU fallback
    assert b"CUDA" in lib.lcsb_last_error(None)
    with pytest.raises(pkg.LcsbError):
        pkg.Lcsb(2, 2, 4)
