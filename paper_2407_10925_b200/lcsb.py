"""Thin ctypes binding of liblcsb.so (include/lcsb.h).  Argument marshalling only: every step of
the sweep and the bound runs in the library's CUDA kernels.  PyTorch provides the device, the
stream and (through the allocation hooks) the caching allocator.

There is no fallback: if liblcsb.so is missing or no CUDA device is present, every call raises.
"""
from __future__ import annotations

import atexit
import ctypes
import os
import weakref
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# LCSB_SO: an alternative build of the same library (A/B of compile-time variants only)
SO_PATH = os.environ.get("LCSB_SO") or os.path.join(_PKG, "liblcsb.so")

LCSB_F64, LCSB_F32 = 0, 1
LCSB_FORM_AUTO, LCSB_FORM_KS, LCSB_FORM_TWO_ARRAY = 0, 1, 2
LCSB_R_MAX, LCSB_R_MIN = 0, 1
LCSB_KERNEL_AUTO, LCSB_KERNEL_GENERIC = 0, 1
STATUS = {0: "LCSB_OK", 1: "LCSB_EINVAL", 2: "LCSB_ECAPACITY", 3: "LCSB_ESTATE", 4: "LCSB_ECUDA",
          5: "LCSB_ENCCL"}

_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                            ctypes.c_void_p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_void_p)
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int32,
                                ctypes.c_void_p)


class LcsbCommHooks(ctypes.Structure):
    """lcsb_comm_hooks (include/lcsb.h): host collectives of the process-sharded mode."""
    _fields_ = [("allgather", ALLGATHER_FN), ("barrier", BARRIER_FN),
                ("allreduce_max_u64", ALLREDUCE_FN), ("ctx", ctypes.c_void_p)]


class LcsbConfig(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_int32), ("d", ctypes.c_int32), ("ell", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("form", ctypes.c_int32), ("rmode", ctypes.c_int32),
                ("symmetry", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("alloc", _ALLOC_FN), ("free_", _FREE_FN),
                ("alloc_ctx", ctypes.c_void_p), ("shards", ctypes.c_int32),
                ("shard", ctypes.c_int32), ("virtual_shards", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("block_log4", ctypes.c_int32),
                ("comm", ctypes.POINTER(LcsbCommHooks)), ("offset_policy", ctypes.c_int32)]


# lcsb_sweep_ex flags (include/lcsb.h)
SWEEP_TRACK, SWEEP_TRACK2 = 1, 3


class LcsbBound(ctypes.Structure):
    _fields_ = [("R_max", ctypes.c_double), ("R_min", ctypes.c_double),
                ("E_at_Rmax", ctypes.c_double), ("E_at_Rmin", ctypes.c_double),
                ("bound_at_Rmax", ctypes.c_double), ("bound_at_Rmin", ctypes.c_double),
                ("bound", ctypes.c_double), ("best_bound", ctypes.c_double),
                ("sweeps_done", ctypes.c_int64), ("best_sweep", ctypes.c_int64)]


# every symbol include/lcsb.h declares (checked by tests/test_abi.py)
EXPORTS = ["lcsb_config_init", "lcsb_required_bytes", "lcsb_create", "lcsb_create_ex",
           "lcsb_reset", "lcsb_sweep", "lcsb_sweep_ex", "lcsb_bound", "lcsb_sweep_bound", "lcsb_table", "lcsb_table_gather",
           "lcsb_nccl_unique_id", "lcsb_shard_locate", "lcsb_shard_locate_sigma4",
           "lcsb_quarter_locate", "lcsb_quarter_shard_plan", "lcsb_ready", "lcsb_rebase", "lcsb_save", "lcsb_load",
           "lcsb_sweeps_done",
           "lcsb_num_shards",
           "lcsb_num_states", "lcsb_stored_states", "lcsb_device_bytes", "lcsb_kernel_in_use",
           "lcsb_shard_traffic",
           "lcsb_launch_count", "lcsb_last_error", "lcsb_destroy"]
NCCL_ID_BYTES = 128

_LIB = None


class LcsbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def load_library():
    """Load liblcsb.so (raises if it was not built: run __graft_entry__.build())."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing; build it with `python -c 'import __graft_entry__ "
                          "as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(SO_PATH)
    P = ctypes.c_void_p
    lib.lcsb_config_init.argtypes = [ctypes.POINTER(LcsbConfig)]
    lib.lcsb_config_init.restype = None
    lib.lcsb_required_bytes.argtypes = [ctypes.POINTER(LcsbConfig)]
    lib.lcsb_required_bytes.restype = ctypes.c_uint64
    lib.lcsb_create.argtypes = [ctypes.c_int32] * 4 + [ctypes.POINTER(P)]
    lib.lcsb_create.restype = ctypes.c_int
    lib.lcsb_create_ex.argtypes = [ctypes.POINTER(LcsbConfig), ctypes.POINTER(P)]
    lib.lcsb_create_ex.restype = ctypes.c_int
    lib.lcsb_reset.argtypes = [P]
    lib.lcsb_reset.restype = ctypes.c_int
    lib.lcsb_sweep.argtypes = [P, ctypes.c_int64]
    lib.lcsb_sweep.restype = ctypes.c_int
    lib.lcsb_bound.argtypes = [P, ctypes.POINTER(LcsbBound)]
    lib.lcsb_bound.restype = ctypes.c_int
    lib.lcsb_sweep_ex.argtypes = [P, ctypes.c_int64, ctypes.c_uint32]
    lib.lcsb_sweep_ex.restype = ctypes.c_int
    lib.lcsb_sweep_bound.argtypes = [P, ctypes.c_int64, ctypes.POINTER(LcsbBound)]
    lib.lcsb_sweep_bound.restype = ctypes.c_int
    lib.lcsb_table.argtypes = [P, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64, P]
    lib.lcsb_table.restype = ctypes.c_int
    lib.lcsb_table_gather.argtypes = [P, ctypes.c_int32, P, ctypes.c_uint64, P]
    lib.lcsb_table_gather.restype = ctypes.c_int
    lib.lcsb_nccl_unique_id.argtypes = [P, ctypes.c_size_t]
    lib.lcsb_nccl_unique_id.restype = ctypes.c_int
    lib.lcsb_shard_locate.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.POINTER(ctypes.c_int32),
                                      ctypes.POINTER(ctypes.c_uint64)]
    lib.lcsb_shard_locate.restype = ctypes.c_int
    lib.lcsb_shard_locate_sigma4.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                             ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_uint64)]
    lib.lcsb_shard_locate_sigma4.restype = ctypes.c_int
    lib.lcsb_quarter_locate.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(ctypes.c_uint64)]
    lib.lcsb_quarter_locate.restype = ctypes.c_int
    lib.lcsb_quarter_shard_plan.argtypes = [ctypes.c_int32] * 4 + [ctypes.POINTER(ctypes.c_uint64)] * 3
    lib.lcsb_quarter_shard_plan.restype = ctypes.c_int
    for name, rt in [("lcsb_sweeps_done", ctypes.c_int64), ("lcsb_num_states", ctypes.c_uint64),
                     ("lcsb_num_shards", ctypes.c_int32),
                     ("lcsb_stored_states", ctypes.c_uint64),
                     ("lcsb_device_bytes", ctypes.c_uint64),
                     ("lcsb_kernel_in_use", ctypes.c_int32),
                     ("lcsb_launch_count", ctypes.c_int64)]:
        getattr(lib, name).argtypes = [P]
        getattr(lib, name).restype = rt
    lib.lcsb_rebase.argtypes = [P]
    lib.lcsb_rebase.restype = ctypes.c_int
    lib.lcsb_save.argtypes = [P, ctypes.c_char_p]
    lib.lcsb_save.restype = ctypes.c_int
    lib.lcsb_load.argtypes = [P, ctypes.c_char_p]
    lib.lcsb_load.restype = ctypes.c_int
    lib.lcsb_ready.argtypes = [P, ctypes.c_int32]
    lib.lcsb_ready.restype = ctypes.c_int32
    lib.lcsb_shard_traffic.argtypes = [P] + [ctypes.POINTER(ctypes.c_uint64)] * 3
    lib.lcsb_shard_traffic.restype = ctypes.c_int
    lib.lcsb_last_error.argtypes = [P]
    lib.lcsb_last_error.restype = ctypes.c_char_p
    lib.lcsb_destroy.argtypes = [P]
    lib.lcsb_destroy.restype = None
    _LIB = lib
    return lib


def _check(rc: int, h=None):
    if rc != 0:
        msg = load_library().lcsb_last_error(h).decode(errors="replace")
        raise LcsbError(rc, msg)


def _dtype_code(dtype) -> int:
    return {"f32": LCSB_F32, "f64": LCSB_F64, LCSB_F32: LCSB_F32, LCSB_F64: LCSB_F64}[dtype]


def _form_code(form) -> int:
    return {"auto": 0, "ks": 1, "two_array": 2, 0: 0, 1: 1, 2: 2}[form]


class _TorchAllocator:
    """Routes the library's device allocations through torch's caching allocator."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = device
        self.alloc_cb = _ALLOC_FN(self._alloc)
        self.free_cb = _FREE_FN(self._free)

    def _alloc(self, nbytes, stream, ctx):
        try:
            return self.torch.cuda.caching_allocator_alloc(int(nbytes), self.device,
                                                           int(stream or 0))
        except Exception:  # out of memory -> NULL -> LCSB_ECAPACITY
            return None

    def _free(self, ptr, nbytes, stream, ctx):
        try:
            self.torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:  # noqa: BLE001 -- interpreter shutdown: torch is gone, so is the memory
            pass


def make_config(sigma, d, ell, dtype="f32", form="auto", rmode="max", symmetry=-1,
                kernel="auto", shards=1, shard=0, virtual_shards=False,
                block_log4=0, offset_policy=0) -> LcsbConfig:
    cfg = LcsbConfig()
    load_library().lcsb_config_init(ctypes.byref(cfg))
    cfg.sigma, cfg.d, cfg.ell = sigma, d, ell
    cfg.dtype = _dtype_code(dtype)
    cfg.form = _form_code(form)
    cfg.rmode = {"max": LCSB_R_MAX, "min": LCSB_R_MIN}[rmode]
    cfg.symmetry = symmetry
    cfg.kernel = {"auto": LCSB_KERNEL_AUTO, "generic": LCSB_KERNEL_GENERIC}[kernel]
    cfg.shards = int(shards)
    cfg.shard = int(shard)
    cfg.virtual_shards = 1 if virtual_shards else 0
    cfg.block_log4 = int(block_log4)
    cfg.offset_policy = int(offset_policy)
    return cfg


def lcsb_required_bytes(sigma, d, ell, dtype="f32", form="auto", symmetry=-1,
                        kernel="auto", shards=1, virtual_shards=True, block_log4=0,
                        offset_policy=0) -> int:
    cfg = make_config(sigma, d, ell, dtype, form, "max", symmetry, kernel, shards, 0,
                      virtual_shards, block_log4, offset_policy)
    return int(load_library().lcsb_required_bytes(ctypes.byref(cfg)))


@dataclass
class BoundResult:
    R_max: float
    R_min: float
    E_at_Rmax: float
    E_at_Rmin: float
    bound_at_Rmax: float
    bound_at_Rmin: float
    bound: float
    best_bound: float
    sweeps_done: int
    best_sweep: int


_LIVE: "weakref.WeakSet[Lcsb]" = weakref.WeakSet()


@atexit.register
def _destroy_live_handles():
    """Handles still alive at exit are released before torch is torn down (their device
    memory came from torch's allocator).  Process-mode handles are only dropped: destroying
    them is collective, and the peers may be gone."""
    for h in list(_LIVE):
        try:
            if h._process_mode:
                h._h = ctypes.c_void_p()
            else:
                h.destroy()
        except Exception:  # noqa: BLE001
            pass


class Lcsb:
    """One handle: the device tables of one (sigma, d, l) run."""

    def __init__(self, sigma, d, ell, dtype="f32", form="auto", rmode="max", symmetry=-1,
                 kernel="auto", stream=None, torch_allocator=True, shards=1, shard=0,
                 virtual_shards=False, nccl_id: bytes | None = None, block_log4: int = 0,
                 comm_hooks: "LcsbCommHooks | None" = None, offset_policy: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise LcsbError(4, "no CUDA device (the library has no CPU path)")
        lib = load_library()
        self._lib = lib
        self.device = torch.cuda.current_device()
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        cfg = make_config(sigma, d, ell, dtype, form, rmode, symmetry, kernel, shards, shard,
                          virtual_shards, block_log4, offset_policy)
        cfg.stream = ctypes.c_void_p(self.stream.cuda_stream)
        self._nccl_id = None
        if nccl_id is not None:
            if len(nccl_id) != NCCL_ID_BYTES:
                raise ValueError("nccl_id must be 128 bytes")
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
            cfg.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        self._comm_hooks = comm_hooks  # kept alive with the handle (the library calls into it)
        if comm_hooks is not None:
            cfg.comm = ctypes.pointer(comm_hooks)
        self._alloc = _TorchAllocator(self.device) if torch_allocator else None
        if self._alloc is not None:
            cfg.alloc = self._alloc.alloc_cb
            cfg.free_ = self._alloc.free_cb
        self._cfg = cfg
        h = ctypes.c_void_p()
        _check(lib.lcsb_create_ex(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.sigma, self.d, self.ell = sigma, d, ell
        self._process_mode = int(shards) > 1 and not virtual_shards
        _LIVE.add(self)

    # --- the C-ABI calls -------------------------------------------------------------------
    def reset(self):
        _check(self._lib.lcsb_reset(self._h), self._h)

    def sweep(self, n: int = 1):
        _check(self._lib.lcsb_sweep(self._h, int(n)), self._h)

    def bound(self) -> BoundResult:
        out = LcsbBound()
        _check(self._lib.lcsb_bound(self._h, ctypes.byref(out)), self._h)
        return BoundResult(**{f: getattr(out, f) for f, _ in LcsbBound._fields_})

    def sweep_ex(self, n: int = 1, flags: int = SWEEP_TRACK):
        """lcsb_sweep_ex: n sweeps, the last one (SWEEP_TRACK) or two (SWEEP_TRACK2) tracking"""
        _check(self._lib.lcsb_sweep_ex(self._h, int(n), int(flags)), self._h)

    def sweep_bound(self, n: int) -> BoundResult:
        """lcsb_sweep_bound: n sweeps and the bound of the iterate before the last of them"""
        out = LcsbBound()
        _check(self._lib.lcsb_sweep_bound(self._h, int(n), ctypes.byref(out)), self._h)
        return BoundResult(**{f: getattr(out, f) for f, _ in LcsbBound._fields_})

    def table(self, which: int = 0, first: int = 0, count: int | None = None) -> np.ndarray:
        if count is None:
            count = self.num_states - first
        out = np.empty(int(count), dtype=np.float64)
        _check(self._lib.lcsb_table(self._h, int(which), int(first), int(count),
                                    out.ctypes.data_as(ctypes.c_void_p)), self._h)
        return out

    def table_gather(self, idx, which: int = 0, out=None) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        if out is None:
            out = np.empty(idx.shape[0], dtype=np.float64)
        _check(self._lib.lcsb_table_gather(self._h, int(which),
                                           idx.ctypes.data_as(ctypes.c_void_p), idx.shape[0],
                                           out.ctypes.data_as(ctypes.c_void_p)), self._h)
        return out

    def rebase(self):
        """lcsb_rebase: residual storage against the newest table (reading R24)."""
        _check(self._lib.lcsb_rebase(self._h), self._h)

    def save(self, path: str):
        """lcsb_save: checkpoint the run (tables, rings, offsets, best-so-far) to `path`."""
        _check(self._lib.lcsb_save(self._h, os.fsencode(path)), self._h)

    def load(self, path: str):
        """lcsb_load: resume a checkpoint written by a handle of the same config."""
        _check(self._lib.lcsb_load(self._h, os.fsencode(path)), self._h)

    def ready(self, wait: bool = False) -> bool:
        """lcsb_ready: the speed-only host preparations (quarter-table item schedule) are in
        place; wait=True blocks until they are."""
        rc = int(self._lib.lcsb_ready(self._h, 1 if wait else 0))
        if rc < 0:
            _check(4, self._h)
        return rc == 1

    @property
    def sweeps_done(self) -> int:
        return int(self._lib.lcsb_sweeps_done(self._h))

    @property
    def num_shards(self) -> int:
        return int(self._lib.lcsb_num_shards(self._h))

    @property
    def num_states(self) -> int:
        return int(self._lib.lcsb_num_states(self._h))

    @property
    def stored_states(self) -> int:
        return int(self._lib.lcsb_stored_states(self._h))

    @property
    def device_bytes(self) -> int:
        return int(self._lib.lcsb_device_bytes(self._h))

    @property
    def kernel_in_use(self) -> str:
        return {1: "generic", 2: "bin2", 3: "q4", 4: "small", 5: "bin2q"}.get(
            int(self._lib.lcsb_kernel_in_use(self._h)), "?")

    def shard_traffic(self):
        """lcsb_shard_traffic: (peer-read, peer-written, requested) bytes per sweep of this
        handle's shards (sharded quarter table), or None for other layouts."""
        r, w, a = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        if self._lib.lcsb_shard_traffic(self._h, ctypes.byref(r), ctypes.byref(w),
                                        ctypes.byref(a)) != 0:
            return None
        return int(r.value), int(w.value), int(a.value)

    @property
    def launch_count(self) -> int:
        return int(self._lib.lcsb_launch_count(self._h))

    def destroy(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.lcsb_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def lcsb_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(load_library().lcsb_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p), NCCL_ID_BYTES))
    return buf.raw


def lcsb_shard_locate(ell: int, shards: int, logical: int):
    """(shard, local index) holding logical binary state `logical` (host-only plan)."""
    sh = ctypes.c_int32()
    loc = ctypes.c_uint64()
    _check(load_library().lcsb_shard_locate(int(ell), int(shards), int(logical), ctypes.byref(sh),
                                            ctypes.byref(loc)))
    return int(sh.value), int(loc.value)


def lcsb_shard_locate_sigma4(ell: int, shards: int, logical: int):
    """(shard, local index) holding logical sigma = 4, d = 2 state `logical` (host-only plan)."""
    sh = ctypes.c_int32()
    loc = ctypes.c_uint64()
    _check(load_library().lcsb_shard_locate_sigma4(int(ell), int(shards), int(logical),
                                                   ctypes.byref(sh), ctypes.byref(loc)))
    return int(sh.value), int(loc.value)


# module-level names mirroring the C-ABI
def lcsb_create(sigma, d, ell, dtype="f32", **kw) -> Lcsb:
    return Lcsb(sigma, d, ell, dtype, **kw)


def lcsb_reset(h: Lcsb):
    h.reset()


def lcsb_sweep(h: Lcsb, n: int = 1):
    h.sweep(n)


def lcsb_bound(h: Lcsb) -> BoundResult:
    return h.bound()


def lcsb_sweep_ex(h: Lcsb, n: int = 1, flags: int = 1):
    h.sweep_ex(n, flags)


def lcsb_sweep_bound(h: Lcsb, n: int) -> BoundResult:
    return h.sweep_bound(n)


def lcsb_table(h: Lcsb, which=0, first=0, count=None) -> np.ndarray:
    return h.table(which, first, count)


def lcsb_table_gather(h: Lcsb, idx, which=0) -> np.ndarray:
    return h.table_gather(idx, which)


def lcsb_destroy(h: Lcsb):
    h.destroy()


def lcsb_quarter_shard_plan(ell: int, dtype: str = "f32", shards: int = 2, passes: int = 24):
    """Host-only plan of the sharded quarter table: per shard, the items it runs
    and the table entries one sweep reads from / stores into other shards (numpy uint64 arrays)."""
    n = int(shards)
    items, rd, wr = (np.zeros(n, dtype=np.uint64) for _ in range(3))
    P = ctypes.POINTER(ctypes.c_uint64)
    _check(load_library().lcsb_quarter_shard_plan(int(ell), _dtype_code(dtype), n, int(passes),
                                                  items.ctypes.data_as(P), rd.ctypes.data_as(P),
                                                  wr.ctypes.data_as(P)))
    return items, rd, wr


def lcsb_quarter_locate(ell: int, block_log4: int, logical: int):
    """(stored index, stored entries) of a logical binary state in the quarter table (host-only)."""
    st = ctypes.c_uint64()
    n = ctypes.c_uint64()
    _check(load_library().lcsb_quarter_locate(int(ell), int(block_log4), int(logical),
                                              ctypes.byref(st), ctypes.byref(n)))
    return int(st.value), int(n.value)
