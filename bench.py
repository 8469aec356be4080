#!/usr/bin/env python
"""bench.py -- the Feasible Triplet hot path on B200 (BASELINE.json config 4 by default).

A "step" is one whole run of the workload through the C-ABI: lcsb_reset (W_0 = 0) +
lcsb_sweep(S) + lcsb_bound.  metric = logical state-updates per second (sigma^(d l) x S per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config4] [--impl ours|reference]

Prints ONE JSON line on rank 0.  N = 1 runs config 4 (l = 17, the largest single-GPU config);
under torchrun (N > 1) the ranks run config 5 (l = 18) with the symmetry-folded table sharded
over the N GPUs (one virtual address range per table over the shards' memory,
peer reads and stores over NVLink, NCCL or host collectives), timed as the max over ranks, or `--workload config3` (sigma = 4, the q4 table sharded, §9b; strong scaling of
the same workload as its N = 1 line).  For config 5 rank 0 also times the same sharded-path
kernel on one GPU at l = 17 (`config.u1_same_kernel`), so U_P / (P U_1) is
computable from the line.  `--impl reference` times the CPU oracle (oracle/, the reference arm
of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (sigma, d, ell, dtype, form, sweeps, bound resource)
    "config1": dict(sigma=2, d=2, ell=8, dtype="f64", form="two_array", sweeps=500),
    "config2": dict(sigma=3, d=3, ell=4, dtype="f64", form="ks", sweeps=300),
    "config3": dict(sigma=4, d=2, ell=8, dtype="f32", form="ks", sweeps=100),
    # config 3's shape in the two-array form (d = 2, any sigma: DESIGN.md reading R20)
    "config3ta": dict(sigma=4, d=2, ell=8, dtype="f32", form="two_array", sweeps=100),
    "config4": dict(sigma=2, d=2, ell=17, dtype="f32", form="two_array", sweeps=50),
    # l = 18: 2 x 128 GiB fp32 half tables, sharded over the ranks (needs >= 2 GPUs)
    "config5": dict(sigma=2, d=2, ell=18, dtype="f32", form="two_array", sweeps=30),
}
METRIC = "state-updates/sec per sweep (1/2/4/8 B200) and % of HBM roofline"
SAMPLE_SEED = 0x240710925


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LCSB_BENCH_DEVICE=k (tests only): every rank on device k -- exercises the N > 1 code path
    # on a one-GPU box with --transport host (no kernel waits on another rank); its timings
    # are not scaling numbers
    if os.environ.get("LCSB_BENCH_DEVICE") is not None:
        local = int(os.environ["LCSB_BENCH_DEVICE"])
    return ws, rank, local


def algorithmic_bytes_per_sweep(w: dict, stored: int) -> int:
    """Compulsory bytes of one sweep: every input generation read once and the
    new table written once, for the stored layout.  two-array: 2 tables; KS: (d + 1) tables."""
    esize = 4 if w["dtype"] == "f32" else 8
    tables = 2 if w["form"] == "two_array" else w["d"] + 1
    return tables * stored * esize


def algorithmic_bytes_for_kernel(w: dict, stored: int, kernel: str) -> int:
    """The compulsory bytes of the stored representation the kernel sweeps: the pooled-history
    KS sweep (q4) keeps v_{n-2} only as its row means (fp64, one per 16 states), so it must read
    v_{n-1} and the means of v_{n-2} and write v_n and its means."""
    if kernel == "q4":
        esize = 4 if w["dtype"] == "f32" else 8
        return 2 * stored * esize + 2 * (stored // 16) * 8
    return algorithmic_bytes_per_sweep(w, stored)


def requested_bytes_per_sweep(w: dict, stored: int, kernel: str) -> int:
    """Bytes the sweep kernel requests from the memory system: equal to the
    compulsory bytes except for the quarter table, which loads every logical window of the half
    table once (2^(2l-1) entries: each stored block once per logical image, 2.67 x stored at
    l = 17) and writes every stored entry once; its L2 item schedule serves part of the repeated
    reads from L2, so DRAM sees fewer (roofline.traffic, ncu: 1.6 x stored read)."""
    esize = 4 if w["dtype"] == "f32" else 8
    if kernel == "bin2q":
        return (1 << (2 * w["ell"] - 1)) * esize + stored * esize
    return algorithmic_bytes_for_kernel(w, stored, kernel)


def workload_name(args, w) -> str:
    """The `config.workload` string (identical in both arms)."""
    return (f"{args.workload}: sigma={w['sigma']}, d={w['d']}, l={w['ell']}, {w['form']} form, "
            f"{w['dtype']} storage, {w['sweeps']} sweeps + 1 bound per step")


def same_kernel_1gpu(w, stream, sweeps=8):
    """State-updates/s of the sharded path's kernel (the quarter table, bin2q -- sharded as in
    DESIGN.md §9c) on ONE GPU at l = 17 (config 4's size): the U_1 of SURVEY §8(e)'s efficiency
    U_P / (P U_1) for config 5."""
    import torch
    from paper_2407_10925_b200 import Lcsb
    h = Lcsb(2, 2, 17, dtype=w["dtype"], form="two_array", stream=stream)
    h.ready(wait=True)
    h.sweep(3)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    h.sweep(sweeps)
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / sweeps
    kernel = h.kernel_in_use
    h.destroy()
    torch.cuda.empty_cache()
    return {"value": (1 << 34) / (ms / 1e3), "unit": "state-updates/s", "ms_per_sweep": ms,
            "kernel": kernel, "what": "l = 17 (config 4 size), fp32, the quarter table (bin2q: the "
            "kernel of the sharded run), one GPU, sweeps only"}


def run_ours(args, w, ws, rank, local):
    import torch
    from paper_2407_10925_b200 import Lcsb
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sharded = ws > 1 or args.force_sharded

    u1 = None
    if sharded and w["sigma"] == 2 and not args.no_u1:
        if rank == 0:
            u1 = same_kernel_1gpu(w, stream)
        torch.distributed.barrier()

    def make():
        if sharded:
            from paper_2407_10925_b200.dist import create_sharded
            return create_sharded(w["ell"], dtype=w["dtype"], stream=stream,
                                  transport=args.transport, sigma=w["sigma"], form=w["form"])
        return Lcsb(w["sigma"], w["d"], w["ell"], dtype=w["dtype"], form=w["form"],
                    symmetry=args.symmetry)

    tc = time.perf_counter()
    h = make()  # the first create of the process: cold (host map; schedule thread started)
    cold_create_ms = (time.perf_counter() - tc) * 1e3
    h.ready(wait=True)  # the L2 item schedule (host thread) is in place before warm-up
    ready_ms = (time.perf_counter() - tc) * 1e3
    S = w["sweeps"]
    n_logical = h.num_states
    stored = h.stored_states
    kernel_name = h.kernel_in_use

    def step(ev=None):
        h.reset()
        if ev is not None:
            ev[0].record(stream)
        h.sweep(S)
        if ev is not None:
            ev[1].record(stream)
        out = h.bound()
        if ev is not None:
            ev[2].record(stream)
        return out

    for _ in range(args.warmup):
        b = step()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sweep_evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
                 for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = h.launch_count
    t0.record(stream)
    for i in range(args.steps):
        b = step(sweep_evs[i])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = h.launch_count - launches0
    clk = clocks.stop()
    if ws > 1:
        torch.distributed.barrier()
    ms_total = t0.elapsed_time(t1)
    sweep_ms = [s.elapsed_time(e) for s, e, _ in sweep_evs]
    bound_ms = statistics.mean(e.elapsed_time(f) for _, e, f in sweep_evs)
    if ws > 1:
        t = torch.tensor([ms_total], device=dev if args.transport == "nccl" else "cpu",
                         dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_per_step = ms_total / args.steps
    value = n_logical * S / (ms_per_step / 1e3)  # all ranks together (sharded: one table)
    # dominant kernel: the sweep; one launch per sweep on `stream`
    launch_ms = statistics.mean(sweep_ms) / S
    alg_bytes = algorithmic_bytes_for_kernel(w, stored // ws, kernel_name)  # per GPU (its shard)
    peak, peak_kind = _peaks()
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    requested_bytes = requested_bytes_per_sweep(w, stored // ws, kernel_name)
    traffic = None
    # ncu DRAM bytes per launch of this workload's sweep kernel (tools/summarize_ncu.py)
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}_{kernel_name}.json")
    if os.path.exists(tpath) and ws == 1:  # the committed profiles are single-GPU captures
        try:
            with open(tpath) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    tr = h.shard_traffic() if ws > 1 else None
    if tr is not None:
        nvlink_bytes = int(tr[0] + tr[1])
    else:
        nvlink_bytes = int(((stored // ws) * (4 if w["dtype"] == "f32" else 8) +
                            (stored // ws // 16 * 8 if kernel_name == "q4" else 0)) * (1 - 1 / ws))

    # ---- end-to-end through the public API with host buffers (create .. gather to host)
    import numpy as np
    from seeded_inputs import splitmix64_indices  # the seeded index generator (no method math)
    idx = splitmix64_indices(SAMPLE_SEED, 1 << 20, n_logical)
    idx_pinned = torch.from_numpy(idx.view(np.int64)).pin_memory()
    out_pinned = torch.empty(1 << 20, dtype=torch.float64).pin_memory()
    h.destroy()
    torch.cuda.synchronize()
    e2e_times, phases = [], []
    for rep in range(3):
        torch.cuda.synchronize()
        te = time.perf_counter()
        h2 = make()
        t1 = time.perf_counter()
        h2.sweep(S)
        be = h2.bound()  # synchronises the stream
        t2 = time.perf_counter()
        if rank == 0:
            h2.table_gather(idx_pinned.numpy().view(np.uint64), out=out_pinned.numpy())
        t3 = time.perf_counter()
        h2.destroy()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        e2e_times.append(t4 - te)
        phases.append({"create_ms": (t1 - te) * 1e3, "sweeps_bound_ms": (t2 - t1) * 1e3,
                       "gather_ms": (t3 - t2) * 1e3, "destroy_ms": (t4 - t3) * 1e3})
    best = min(range(1, len(e2e_times)), key=lambda i: e2e_times[i])
    e2e_s = e2e_times[best]
    if ws > 1:
        t = torch.tensor([e2e_s], device=dev if args.transport == "nccl" else "cpu",
                         dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = n_logical * S / e2e_s

    res = {
        "metric": METRIC,
        "value": value,
        "unit": "state-updates/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        # config 4 / 5 (binary): per-GPU logical work roughly fixed as N grows (2^34 at N = 1,
        # 2^36 / N at N > 1); config 3 and the others: the same workload at every N
        "scaling": "weak" if w["sigma"] == 2 and w["ell"] >= 17 else "strong",
        "vs_baseline": None,
        "dtype": "f64" if w["dtype"] == "f64" else "f32-storage/f64-arith",
        "data": "synthetic (the method's only input is (sigma, d, l) and W_0 = 0)",
        "config": {
            "workload": workload_name(args, w),
            "states": n_logical, "stored_states": stored, "sweeps_per_step": S,
            "kernel": kernel_name,
            "parallelism": (f"sharded over {ws} GPUs ({args.transport} collectives; "
                            + ("one mapped address range per table: peer reads + stores"
                               if kernel_name == "bin2q" else "CUDA-IPC peer stores") + ")")
                           if ws > 1
                           else ("process-sharded mode, 1 rank" if args.force_sharded
                                 else "single-gpu"),
            "scaling_definition": ("U_P / (P U_1) with U_1 = u1_same_kernel (SURVEY 8(e))"
                                   if u1 else "value_N / (N value_1), same workload"),
            "u1_same_kernel": u1,
            "cold_create_ms": cold_create_ms,
            "create_to_schedule_ready_ms": ready_ms,
            "l2_flush": "inputs larger than L2 (each table %.1f GiB vs 126 MB L2)"
                        % (stored * (4 if w["dtype"] == "f32" else 8) / 2**30)
            if stored * 4 > 2**27 else "working set L2-resident (latency-bound config)",
            "sweep_ms_per_launch": launch_ms,
            "bound_ms_per_step": bound_ms,  # lcsb_bound: R reduction + W pass + E
            # ncu DRAM bytes of one sweep launch per LOGICAL state update, and per STORED entry
            # (the table holds 3/16 of the logical states for the quarter table)
            "dram_bytes_per_state_update": (traffic / (n_logical / ws)) if traffic else None,
            "dram_bytes_per_stored_state": (traffic / (stored / ws)) if traffic else None,
            "algorithmic_bytes_per_stored_state": alg_bytes / (stored / ws),
            "bound": b.bound, "bound_at_Rmin": b.bound_at_Rmin,
            "sweeps_per_s": S / (ms_per_step / 1e3),
            "sweep_only_state_updates_per_s": n_logical / (launch_ms / 1e3),
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "requested_bytes_per_launch": requested_bytes,
                     # per GPU per sweep: sharded quarter table -- the exact peer reads and
                     # stores of its items (lcsb_shard_traffic, §9c); otherwise the outputs (and,
                     # q4, the row means) whose owner is another shard, (1 - 1/P) of the shard's
                     "nvlink_bytes_per_launch": nvlink_bytes,
                     # SURVEY 8(d) number (1): the DRAM bytes the kernel really moves (ncu,
                     # `traffic`) per launch time, against the same peak -- how close the kernel
                     # runs to the copy bandwidth for the bytes it moves (frac: for the
                     # compulsory bytes)
                     "dram_achieved": (traffic / (launch_ms / 1e3) / 1e9) if traffic else None,
                     "dram_frac": (traffic / (launch_ms / 1e3) / 1e9 / peak) if traffic else None,
                     "kernel": kernel_name + " sweep kernel"},
        "e2e": {"value": e2e_value, "unit": "state-updates/s",
                "h2d_bytes_per_step": int(idx.nbytes),
                "d2h_bytes_per_step": int(out_pinned.numel() * 8 + 32),
                "what": "lcsb_create + lcsb_sweep(S) + lcsb_bound + lcsb_table_gather of 2^20 "
                        "seeded states to pinned host memory + lcsb_destroy, wall clock, best of "
                        "2 after one untimed",
                "phases": phases[best],
                # the first create of this process (host block map, schedule thread started) and
                # the time until the L2 item schedule was in place
                "cold_create_ms": cold_create_ms,
                "cold_schedule_ready_ms": ready_ms,
                "bound": be.bound},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    return res


def _host_info():
    model, ram = None, None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    ram = round(int(line.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    return model, ram


def cpu_baseline(w, budget_s=15.0, single_s=4.0):
    """The oracle as it stands, timed on this host, on a bounded sample of the same workload:
    one sweep of F (oracle/ft_oracle.c fo_apply_F_at, all OpenMP threads) over a contiguous
    slice of the workload's logical states (the paper's thread-slice unit),
    reading a full-size logical input table (np.zeros: W_0, sweep 1 of the run)."""
    import numpy as np
    from oracle import ft_oracle as fo
    w = dict(w)
    n = fo.n_states(w["sigma"], w["d"], w["ell"])
    try:
        src = np.zeros(n, dtype=np.float64)
        table_note = "full-size fp64 logical input table"
    except MemoryError:  # host too small for the logical table: same recurrence at l - 3
        w["ell"] -= 3
        n = fo.n_states(w["sigma"], w["d"], w["ell"])
        src = np.zeros(n, dtype=np.float64)
        table_note = (f"host RAM too small for the full table; l reduced to {w['ell']} "
                      "(per-state cost of the same recurrence)")
    d = w["d"]
    count = 1 << 16
    cores = fo.num_threads()
    x0 = n // 3
    spent, done = 0.0, 0
    # calibrate, then run ~budget_s of work
    while spent < budget_s:
        idx = np.arange(x0 + done, x0 + done + count, dtype=np.uint64) % np.uint64(n)
        t = time.perf_counter()
        _parallel_apply_at(fo, w, [src] * d, idx, cores)
        dt = time.perf_counter() - t
        spent += dt
        done += count
        if dt < budget_s / 20:
            count *= 2
    # the same on ONE thread (single-thread and all-core numbers)
    spent1, done1, c1 = 0.0, 0, 1 << 12
    while spent1 < single_s:
        idx = np.arange(x0 + done1, x0 + done1 + c1, dtype=np.uint64) % np.uint64(n)
        t = time.perf_counter()
        _parallel_apply_at(fo, w, [src] * d, idx, 1)
        dt = time.perf_counter() - t
        spent1 += dt
        done1 += c1
        if dt < single_s / 20:
            c1 *= 2
    model, ram = _host_info()
    return {"value": done / spent, "unit": "state-updates/s", "cores": cores, "kind": "oracle",
            "sample": f"{done} consecutive logical states of one sweep of {w['sigma']},{w['d']},"
                      f"{w['ell']} ({table_note}), {spent:.1f} s",
            "single_thread_value": done1 / spent1,
            "single_thread_sample": f"{done1} states, {spent1:.1f} s",
            "cpu_model": model, "ram_gib": ram}


def _parallel_apply_at(fo, w, src, idx, cores):
    from concurrent.futures import ThreadPoolExecutor
    parts = [idx[i::cores] for i in range(cores)]
    with ThreadPoolExecutor(cores) as ex:  # ctypes releases the GIL during the C call
        two = (w["form"] == "two_array")  # d = 2: no drop-both option (reading R20)
        list(ex.map(lambda p: fo.apply_F_at(w["sigma"], w["d"], w["ell"], src, p,
                                            two_array=two), parts))


class _JsonOnlyStdout:
    """Library chatter written to file descriptor 1 by C code (e.g. NCCL's version banner) goes
    to stderr while the bench runs; only the JSON line is printed to the real stdout."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def emit(self, line: str):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        print(line, flush=True)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def main():
    with _JsonOnlyStdout() as out:
        _main(out)


def _main(out):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: config4 at N=1, config5 (sharded l=18) at N>1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--symmetry", type=int, default=-1,
                    help="table layout: -1 auto, 1 half table, 2 quarter table (binary)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the process-sharded path even at N = 1 (tests the N > 1 code)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="sharded collectives: NCCL on the stream (default) or host hooks (gloo)")
    ap.add_argument("--ell", type=int, default=None,
                    help="override the workload's l (tests of the code path only; the line's "
                         "workload then names the changed l)")
    ap.add_argument("--no-u1", action="store_true",
                    help="config 5 at N > 1: skip timing the same kernel on one GPU at l = 17")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    ws, rank, local = _dist()
    if args.workload is None:
        args.workload = "config4" if ws == 1 else "config5"
    w = dict(WORKLOADS[args.workload])
    if args.ell:
        w["ell"] = args.ell
    if ws > 1 and args.workload not in ("config5", "config3", "config3ta"):
        raise SystemExit("N > 1 runs a sharded workload: config5 (binary) or config3/config3ta "
                         "(sigma = 4)")

    if args.impl == "reference":
        if rank != 0:
            return
        base = cpu_baseline(w, budget_s=max(5.0, 3.0 * args.steps))
        res = {"impl": "reference", "metric": METRIC, "value": base["value"],
               "unit": "state-updates/s", "n_gpus": ws, "steps": args.steps,
               "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": workload_name(args, w),
                          "states": w["sigma"] ** (w["d"] * w["ell"]),
                          "sweeps_per_step": w["sweeps"]},
               "cpu_baseline": base,
               "e2e": {"value": base["value"], "unit": "state-updates/s",
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        out.emit(json.dumps(res))
        return

    import torch
    if ws > 1 or args.force_sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(ws))
        if args.transport == "host":
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = run_ours(args, w, ws, rank, local)
    if rank == 0:
        if not args.no_cpu_baseline and ws == 1:
            res["cpu_baseline"] = cpu_baseline(w)
        out.emit(json.dumps(res))
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
