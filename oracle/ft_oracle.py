"""CPU ORACLE driver for the Feasible Triplet method of arXiv 2407.10925.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(``paper_2407_10925_b200``) never imports it and shares no code with it.

This module drives the literal C transcription of Alg. 1 / Eq. (ineq3) in ``ft_oracle.c``
through the iteration and bound bookkeeping of

* Alg. 2 "The Feasible Triplet Algorithm"
* Alg. 5 "The Binary Feasible Triplet Algorithm"
* Lueker's two-array form for sigma=2, d=2 ("storing only two arrays ... with the bound
  calculation adjusted appropriately")               PAPER.md:400   (reading R10 in DESIGN.md),
  extended to d = 2 and any sigma with the drop-both option removed (reading R20)

Everything is fp64 over the FULL logical table.  ``dtype='f32'`` emulates fp32 storage: the
result of every sweep is rounded to fp32 (round-to-nearest-even) and widened back, exactly what
storing it in an fp32 table does; all arithmetic stays fp64 (BASELINE.json: "fp32 storage with
fp64 accumulation").

Bound bookkeeping (both R readings are computed, reading R5 in DESIGN.md):
  R_max = max(v_new - v_prev), R_min = min(v_new - v_prev)            Alg. 2 line 5 / PAPER.md:694
  KS:        W = (v_new + d*R) - F(v_new + (d-1)R, ..., v_new + 0R)    Alg. 2 line 6
             E = max(0, max W);  bound = d (R - E)                     Alg. 2 line 7, Eq. (lwrbound)
  two-array: W = (v_new + R) - F(v_new, v_new);  E = max(0, max W)
             rho = R - E;  bound = 2 rho / (1 + rho) if rho > 0 else 0 (reading R10)
  best: the largest R - E over the evaluations so far, starting from the triplet (v_0, 0, 0)
        (Alg. 2 lines 2, 8-10), reported as a bound.

Integer offsets (``offsets=True``, readings R23, R26): by
translation invariance, F(v + c 1) = F(v) + c 1 (Lemma 1 (2)), so the
table may hold s_n = v_n - o_n with an integer o_n: each sweep subtracts c_n = floor(min s_n),
  s_{n+1} = round_storage(F(s_n, s_n) - c_n),   o_{n+1} = o_n + c_n,   o_0 = 0,
which keeps the stored magnitudes (and so the fp32 rounding) small.  The bound in stored terms:
R = max(s_n - s_{n-1}) + c_{n-1} (min likewise), W = (s_n + R) - F(s_n, s_n).
KS form (R26): every generation keeps its own o; F reads the table k sweeps back relative to the
newest one's offset, F(v_n, ..., v_{n-d+1}) - o_n = F(s_n, s_{n-1} + (o_{n-1} - o_n), ...), with
p_k = o_{n+1-k} - o_n added to each option's mean over the table k back (the mean of s + p is
the mean of s plus p; added after the mean, as kernels that keep pooled row means can), and the
|N| = 0 option's 0 (R3) written in stored terms, -o_n (the 0 is a constant, not an iterate
value, so translating the tables translates it too; it never wins: every iterate is >= 0), so
  s_{n+1} = round_storage(F_p(s_n, ..., s_{n-d+1}) - c_n),  o_{n+1} = o_n + c_n,
and W (Alg. 2 line 6) reads only the newest table: W = (s_n + dR) - F(s_n + (d-1)R, ..., s_n).

Residual storage (``Run.rebase()``, offsets on; reading R24): the table is split into
a fixed base H (the stored table at the rebase, fp32) and a stored residual e, v = H + e + o.
H + e is exact in fp64, each sweep subtracts c_n = floor(64 min(H + e_n)) / 64 (a dyadic, exact)
and stores round_storage((F(H + e, H + e) - c_n) - H): the residual's magnitude stays below one
sweep's growth, so fp32 residuals carry ~64x the precision of fp32 values.

Parity pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ft_oracle.c")
_SO = os.path.join(_HERE, "libftoracle.so")
_LOCK = threading.Lock()
_LIB = None

FORM_KS = 1
FORM_TWO_ARRAY = 2


def build(force: bool = False) -> str:
    """Compile ft_oracle.c with gcc (plain C, -O2, OpenMP).  Returns the .so path."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            lib = ctypes.CDLL(build())
            dpp = ctypes.POINTER(ctypes.c_void_p)
            lib.fo_apply_F.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dpp,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                       ctypes.c_int]
            lib.fo_apply_F.restype = ctypes.c_int
            lib.fo_apply_F_post.argtypes = lib.fo_apply_F.argtypes
            lib.fo_apply_F_post.restype = ctypes.c_int
            lib.fo_apply_F_at.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dpp,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p]
            lib.fo_apply_F_at.restype = ctypes.c_int
            lib.fo_sample.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p, ctypes.c_int64,
                                                           ctypes.c_void_p, ctypes.c_int]
            lib.fo_sample.restype = ctypes.c_int
            lib.fo_encode.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
            lib.fo_encode.restype = ctypes.c_uint64
            lib.fo_num_threads.restype = ctypes.c_int
            _LIB = lib
        return _LIB


def num_threads() -> int:
    return int(_lib().fo_num_threads())


# --------------------------------------------------------------------------------------------
# State codec (reading R14).  Pure Python, independent of ft_oracle.c's codec and of the GPU's.
# --------------------------------------------------------------------------------------------

def n_states(sigma: int, d: int, ell: int) -> int:
    """sigma^(d*ell): the number of d-tuples of length-ell strings."""
    return sigma ** (d * ell)


def encode_tuple(A, sigma: int, d: int, ell: int) -> int:
    """idx = sum_k sum_j A_j[k] * sigma^(d(ell-1-k) + (d-1-j))  (reading R14)."""
    if len(A) != d:
        raise ValueError("need d strings")
    x = 0
    for s in A:
        if len(s) != ell or any(not (0 <= int(ch) < sigma) for ch in s):
            raise ValueError("bad string")
    for k in range(ell):
        for j in range(d):
            x += int(A[j][k]) * sigma ** (d * (ell - 1 - k) + (d - 1 - j))
    return x


def decode_tuple(x: int, sigma: int, d: int, ell: int):
    if not (0 <= x < n_states(sigma, d, ell)):
        raise ValueError("index out of range")
    A = [[0] * ell for _ in range(d)]
    for k in range(ell):
        for j in range(d):
            p = d * (ell - 1 - k) + (d - 1 - j)
            A[j][k] = (x // sigma ** p) % sigma
    return ["".join(str(c) for c in s) for s in A]


def interleave_pair(a: str, b: str) -> int:
    """The paper's interleaved string pair: "interleaving their bits starting with a"
    (PAPER.md:393-394), a's character in the more significant bit of each pair."""
    if len(a) != len(b):
        raise ValueError("length mismatch")
    bits = "".join(x + y for x, y in zip(a, b))
    return int(bits, 2) if bits else 0


def deinterleave_pair(x: int, ell: int):
    bits = format(x, f"0{2 * ell}b")
    return bits[0::2], bits[1::2]


def complement_index(i: int, ell: int) -> int:
    """j = 2^(2 ell) - 1 - i."""
    return (1 << (2 * ell)) - 1 - i


# --------------------------------------------------------------------------------------------
# F and the iteration.
# --------------------------------------------------------------------------------------------

def _as_f64(v) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return v


def apply_F(sigma: int, d: int, ell: int, src, shift=None, threads: int = 0,
            two_array: bool = False, post=None) -> np.ndarray:
    """F(src[0], ..., src[d-1]): src[k-1] is read when |N| = k (reading R1).  ``shift[k-1]`` is
    added to every value read from src[k-1] (used for Alg. 2 line 6).  ``two_array`` (d = 2):
    the drop-both option (both heads differ, |N| = 2) is not offered (reading R20).  ``post[k-1]``
    (instead of ``shift``; d + 1 entries) is added to each option's mean with |N| = k >= 1, and
    ``post[0]`` replaces the |N| = 0 option's 0 (KS offsets, reading R26)."""
    n = n_states(sigma, d, ell)
    if len(src) != d:
        raise ValueError("need d source vectors")
    arrs = [_as_f64(s) for s in src]
    for a in arrs:
        if a.shape != (n,):
            raise ValueError("bad vector length")
    ptrs = (ctypes.c_void_p * d)(*[a.ctypes.data for a in arrs])
    out = np.empty(n, dtype=np.float64)
    if post is not None:
        if shift is not None:
            raise ValueError("shift and post are exclusive")
        po = np.ascontiguousarray(post, np.float64)
        if po.shape != (d + 1,):
            raise ValueError("post needs d + 1 entries")
        rc = _lib().fo_apply_F_post(sigma, d, ell, ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)),
                                    po.ctypes.data, out.ctypes.data, int(threads),
                                    int(bool(two_array)))
        if rc:
            raise ValueError("fo_apply_F_post rejected the parameters")
        return out
    sh = np.zeros(d, dtype=np.float64) if shift is None else np.ascontiguousarray(shift, np.float64)
    rc = _lib().fo_apply_F(sigma, d, ell, ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)),
                           sh.ctypes.data, out.ctypes.data, int(threads), int(bool(two_array)))
    if rc:
        raise ValueError("fo_apply_F rejected the parameters")
    return out


def apply_F_at(sigma, d, ell, src, idx, shift=None, two_array: bool = False) -> np.ndarray:
    arrs = [_as_f64(s) for s in src]
    ptrs = (ctypes.c_void_p * d)(*[a.ctypes.data for a in arrs])
    sh = np.zeros(d, dtype=np.float64) if shift is None else np.ascontiguousarray(shift, np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(idx.shape[0], dtype=np.float64)
    rc = _lib().fo_apply_F_at(sigma, d, ell, ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)),
                              sh.ctypes.data, idx.ctypes.data, idx.shape[0], out.ctypes.data,
                              int(bool(two_array)))
    if rc:
        raise ValueError("fo_apply_F_at rejected the parameters")
    return out


def round_storage(v: np.ndarray, dtype: str) -> np.ndarray:
    """Storage rounding: f32 = round-to-nearest-even to fp32 and back (numpy casts are RNE)."""
    if dtype == "f32":
        return v.astype(np.float32).astype(np.float64)
    if dtype == "f64":
        return v
    raise ValueError(dtype)


def resolve_form(sigma: int, d: int, form: str) -> int:
    if form == "auto":
        return FORM_TWO_ARRAY if (sigma, d) == (2, 2) else FORM_KS
    if form == "ks":
        return FORM_KS
    if form == "two_array":
        # PAPER.md:400 states it for sigma = d = 2; reading R20 extends it to d = 2, any sigma
        if d != 2:
            raise ValueError("two-array form is defined for d = 2 only (PAPER.md:400, reading R20)")
        return FORM_TWO_ARRAY
    raise ValueError(form)


class Run:
    """State of Alg. 2 (KS form) or Lueker's two-array form, over the full logical table.

    KS: ``gens[k-1]`` is the table k sweeps back (k = 1..d), all zero at the start
    (Alg. 2 line 2: a (d+1) x sigma^(d l) zero matrix).  One sweep computes
    v_new = F(gens[0], ..., gens[d-1]) and shifts the rows (Alg. 2 lines 4, 11).
    Two-array: one table g; v_new = F(g, g); the previous table is kept for R.
    """

    def __init__(self, sigma: int, d: int, ell: int, form: str = "auto", dtype: str = "f64",
                 threads: int = 0, offsets: bool = False):
        if sigma < 2 or d < 2 or ell < 1:
            raise ValueError("need sigma >= 2, d >= 2, ell >= 1")
        self.sigma, self.d, self.ell = sigma, d, ell
        self.form = resolve_form(sigma, d, form)
        self.dtype = dtype
        self.threads = threads
        self.n = n_states(sigma, d, ell)
        depth = d if self.form == FORM_KS else 1
        self.gens = [np.zeros(self.n) for _ in range(depth)]
        self.prev = np.zeros(self.n)
        self.sweeps_done = 0
        self.best = {"max": 0.0, "min": 0.0}     # best r - eps per R reading (Alg. 2 line 3)
        self.best_sweep = {"max": 0, "min": 0}
        self.offsets = bool(offsets)
        self.off = 0.0        # o_n of the newest table (an integer, exact in fp64)
        self.off_prev = 0.0   # o_{n-1}
        self.goff = [0.0] * depth  # KS (R26): o of gens[k-1], the table k sweeps back
        self.base = None      # residual storage: the fixed base H (rebase), else None
        self.quantum = 1.0    # offset granularity: 1 (integer offsets), 1/64 after a rebase
        self.rebase_sweep = -1

    def rebase(self):
        """Residual storage (reading R24): H := the newest stored table, e := 0; on a rebased
        run H := round32(H + e) and e := (H + e) - H (the iterate is unchanged)."""
        if not self.offsets or self.form != FORM_TWO_ARRAY:
            raise ValueError("rebase needs the two-array form with offsets")
        if self.base is None:
            self.base = self.gens[0].copy()
            self.gens = [np.zeros(self.n)]
        else:
            full = self.base + self.gens[0]
            self.base = round_storage(full, self.dtype)
            self.gens = [full - self.base]
        self.prev = np.full(self.n, np.nan)   # the previous generation is not representable
        self.quantum = 1.0 / 64.0
        self.rebase_sweep = self.sweeps_done

    def _full(self, t):
        """H + e (exact in fp64: both are storage-rounded values of similar or smaller scale)."""
        return t if self.base is None else self.base + t

    # -- one application of F (Alg. 2 line 4 / Alg. 5 line 6) --
    def sweep(self, count: int = 1):
        for _ in range(count):
            if self.form == FORM_KS:
                post = None
                c = 0.0
                if self.offsets:  # read every generation relative to o_n (R26)
                    # the |N| = 0 option's 0 (R3) in stored terms is -o_n; |N| = k: o_{n+1-k} - o_n
                    post = [-self.goff[0]] + [o - self.goff[0] for o in self.goff]
                    c = float(math.floor(float(self.gens[0].min())))
                new = apply_F(self.sigma, self.d, self.ell, self.gens, threads=self.threads,
                              post=post)
                if self.offsets:
                    new = new - c
                new = round_storage(new, self.dtype)
                self.prev = self.gens[0]
                self.gens = [new] + self.gens[:-1]          # shift the rows (line 11)
                self.goff = [self.goff[0] + c] + self.goff[:-1]
                self.off_prev, self.off = self.off, self.goff[0]
            else:
                g = self.gens[0]
                full = self._full(g)
                new = apply_F(self.sigma, self.d, self.ell, [full] * self.d, threads=self.threads,
                              two_array=True)
                c = 0.0
                if self.offsets:  # s_{n+1} = F(s_n) - floor(min s_n)  (translation invariance)
                    q = self.quantum
                    c = float(math.floor(float(full.min()) / q)) * q
                    new = new - c
                if self.base is not None:  # the residual against the fixed base (R24)
                    new = new - self.base
                new = round_storage(new, self.dtype)
                self.prev = g
                self.gens = [new]
                self.off_prev, self.off = self.off, self.off + c
            self.sweeps_done += 1

    @property
    def newest(self) -> np.ndarray:
        """The newest table as stored (with offsets: s_n; the values are s_n + o_n)."""
        return self.gens[0]

    def values(self, which: int = 0) -> np.ndarray:
        """The iterate's values: stored + integer offset (o_n, or o_{n-1} for which = 1)."""
        t = self._full(self.gens[0] if which == 0 else self.prev)
        return t + (self.off if which == 0 else self.off_prev)

    def _W(self, R: float) -> np.ndarray:
        v = self._full(self.gens[0])
        d = self.d
        if self.form == FORM_KS:
            shift = np.array([float(d - k) * R for k in range(1, d + 1)])
            Fv = apply_F(self.sigma, d, self.ell, [v] * d, shift=shift, threads=self.threads)
            return (v + float(d) * R) - Fv
        Fv = apply_F(self.sigma, d, self.ell, [v] * d, threads=self.threads, two_array=True)
        return (v + R) - Fv

    def bound_from(self, R: float, E: float) -> float:
        rho = R - E
        if self.form == FORM_KS:
            return float(self.d) * rho
        return 2.0 * rho / (1.0 + rho) if rho > 0.0 else 0.0

    def bound(self) -> dict:
        """Alg. 2 lines 5-10 for both R readings; updates best-so-far."""
        if self.sweeps_done < 1:
            raise RuntimeError("bound needs at least one sweep")
        if self.base is not None and self.sweeps_done <= self.rebase_sweep:
            raise RuntimeError("bound needs a sweep after a rebase")
        diff = self._full(self.gens[0]) - self._full(self.prev)
        c = self.off - self.off_prev  # offsets: v_n - v_{n-1} = s_n - s_{n-1} + c_{n-1}
        out = {"R_max": float(diff.max()) + c, "R_min": float(diff.min()) + c}
        for mode in ("max", "min"):
            R = out["R_" + mode]
            W = self._W(R)
            E = max(0.0, float(W.max()))
            out["E_at_R" + mode] = E
            out["bound_at_R" + mode] = self.bound_from(R, E)
            if R - E >= self.best[mode]:                     # Alg. 2 line 8
                self.best[mode] = R - E
                self.best_sweep[mode] = self.sweeps_done
            out["best_at_R" + mode] = self.bound_from(self.best[mode], 0.0)
        out["sweeps_done"] = self.sweeps_done
        return out


def feasible_triplet(sigma: int, d: int, ell: int, sweeps: int, form: str = "auto",
                     dtype: str = "f64", bound_every: bool = False, threads: int = 0,
                     offsets: bool = False) -> dict:
    """Run `sweeps` sweeps from the zero start; evaluate the bound after every sweep
    (``bound_every``, as Alg. 2/5 do) or only after the last one (as BASELINE.json's configs).
    ``table`` / ``prev`` are the stored tables (with offsets: ``values`` holds s + o)."""
    run = Run(sigma, d, ell, form, dtype, threads, offsets)
    res = None
    for _ in range(sweeps):
        run.sweep(1)
        if bound_every:
            res = run.bound()
    if not bound_every:
        res = run.bound()
    res["table"] = run.newest
    res["prev"] = run.prev
    res["values"] = run.values(0)
    res["offset"] = run.off
    return res


def sample_values(sigma: int, d: int, ell: int, sweeps: int, idx, form: str = "auto",
                  dtype: str = "f64", threads: int = 0) -> np.ndarray:
    """Sampled mode: the table after ``sweeps`` sweeps at the given logical indices, by top-down
    recursion from the zero start (for l >= 17 where no full table fits in host RAM)."""
    f = resolve_form(sigma, d, form)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(idx.shape[0], dtype=np.float64)
    rc = _lib().fo_sample(sigma, d, ell, f, 1 if dtype == "f32" else 0, int(sweeps),
                          idx.ctypes.data, idx.shape[0], out.ctypes.data, int(threads))
    if rc:
        raise ValueError("fo_sample rejected the parameters")
    return out


def floor6(x: float) -> float:
    """The paper's printing rule: "rounded down to their 6th decimal place"."""
    return math.floor(x * 1e6 + 1e-6) / 1e6
