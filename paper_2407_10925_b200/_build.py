"""Build liblcsb.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "liblcsb.so")
SOURCES = ["lcsb_api.cu", "quarter_host.cu", "kern_generic.cu", "kern_bin2.cu", "kern_bin2_tma.cu",
           "kern_bin2q.cu", "kern_bin2q_bound.cu", "kern_bin2q_ext.cu", "kern_bin2q_diff.cu", "kern_q4.cu",
           "kern_small.cu", "kern_reduce.cu", "vmm.cu"]
NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # no FMA contraction: every fp64 op rounds exactly as written (parity with the oracle)
    "-fmad=false",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "lcsb.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(src: str, obj: str, inc: list) -> subprocess.CompletedProcess:
    return subprocess.run([nvcc(), *NVCC_FLAGS, *inc, "-c", src, "-o", obj],
                          capture_output=True, text=True)


def _compile_d(src: str, obj: str, inc: list, defines) -> subprocess.CompletedProcess:
    return subprocess.run([nvcc(), *NVCC_FLAGS, *defines, *inc, "-c", src, "-o", obj],
                          capture_output=True, text=True)


OBJDIR = os.path.join(ROOT, "build", "obj")  # git-ignored object cache of the default build


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
        [os.path.join(ROOT, "include", "lcsb.h"), os.path.abspath(__file__)]


def build(force: bool = False, verbose: bool = False, out: str = SO, defines=()) -> str:
    """One nvcc -c per source (in parallel), then one shared-library link.  The default build keeps
    its objects in build/obj and recompiles only sources newer than their object (any header
    change recompiles everything).  ``out`` / ``defines`` (A/B builds only, e.g.
    build/liblcsb_spin.so with -DLCSB_MBAR_SPIN; loaded through LCSB_SO) always compile afresh."""
    default = out == SO and not defines
    if default and not force and not stale():
        return SO
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor
    tag = f".tmp{os.getpid()}"
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    if default:
        os.makedirs(OBJDIR, exist_ok=True)
        objs = [os.path.join(OBJDIR, s[:-3] + ".o") for s in SOURCES]
        hdr_t = max(os.path.getmtime(h) for h in _headers())
        todo = [i for i, (s, o) in enumerate(zip(SOURCES, objs))
                if force or not os.path.exists(o) or
                os.path.getmtime(o) < max(hdr_t, os.path.getmtime(os.path.join(CSRC, s)))]
        outs = [objs[i] + tag for i in todo]
    else:
        objs = [os.path.join(CSRC, s[:-3] + tag + ".o") for s in SOURCES]
        todo = list(range(len(SOURCES)))
        outs = list(objs)
    try:
        with ThreadPoolExecutor(max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
            results = list(ex.map(lambda io: _compile_d(os.path.join(CSRC, SOURCES[io[0]]), io[1],
                                                        inc, list(defines)),
                                  zip(todo, outs)))
        for i, res in zip(todo, results):
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed compiling {SOURCES[i]}")
            if verbose:
                sys.stderr.write(res.stderr)
        if default:
            for i, o in zip(todo, outs):
                os.replace(o, objs[i])
        tmp = out + tag
        res = subprocess.run([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                              *objs, "-o", tmp, "-lcudart", "-lnccl", "-Xlinker", "-export-dynamic"],
                             capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking liblcsb.so")
        os.replace(tmp, out)
    finally:
        for o in (outs if default else objs):
            if os.path.exists(o):
                os.remove(o)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
