"""Power / clock behaviour of the config-4 sweep against a plain device copy (round 2): samples
nvidia-smi (power, SM and memory clocks, sw_power_cap) every 50 ms while (a) torch copies a 6 GiB
buffer back and forth for ~3 s and (b) the quarter-table sweep runs back to back for ~3 s; prints
per phase the median power / clocks, the fraction of samples under sw_power_cap, the achieved
GB/s (copy) and the per-sweep times over the run (first 10 vs last 100)."""
import json, os, statistics, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

FIELDS = "power.draw,clocks.sm,clocks.mem,clocks_event_reasons.sw_power_cap"


class Sampler:
    def __init__(self):
        self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={FIELDS}", "--format=csv,noheader,nounits",
                                   "-lms", "50"], stdout=subprocess.PIPE, text=True)
        self.rows = []
        self.tag = "idle"
        threading.Thread(target=self._r, daemon=True).start()

    def _r(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((self.tag, float(parts[0]), float(parts[1]), float(parts[2]),
                                  parts[3].lower() == "active"))
            except (ValueError, IndexError):
                pass

    def summary(self, tag):
        r = [x for x in self.rows if x[0] == tag]
        if not r:
            return {}
        return {"samples": len(r), "power_w": statistics.median(x[1] for x in r),
                "power_max_w": max(x[1] for x in r), "sm_mhz": statistics.median(x[2] for x in r),
                "mem_mhz": statistics.median(x[3] for x in r),
                "power_cap_frac": sum(x[4] for x in r) / len(r)}


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-copy", action="store_true")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    from paper_2407_10925_b200 import Lcsb
    s = Sampler()
    time.sleep(1.0)
    out = {"tag": args.tag, "so": os.environ.get("LCSB_SO", "default")}
    if not args.skip_copy:
        copy_phase(s, out)
    run_sweeps(s, out, Lcsb)


def copy_phase(s, out):
    a = torch.empty(3 << 30, dtype=torch.float16, device="cuda")
    b = torch.empty_like(a)
    torch.cuda.synchronize()
    s.tag = "copy"
    t0 = time.time(); n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 3.0:
        for _ in range(20):
            b.copy_(a); a.copy_(b); n += 2
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    out["copy_gbs"] = n * 2 * a.numel() * 2 / (e0.elapsed_time(e1) / 1e3) / 1e9
    s.tag = "gap"
    del a, b
    torch.cuda.empty_cache()
    time.sleep(1.0)


def run_sweeps(s, out, Lcsb):
    h = Lcsb(2, 2, 17, dtype="f32")
    h.ready(wait=True)
    h.sweep(2)
    torch.cuda.synchronize()
    time.sleep(1.0)
    s.tag = "sweep"
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(601)]
    evs[0].record()
    for k in range(600):
        h.sweep(1)
        evs[k + 1].record()
    torch.cuda.synchronize()
    s.tag = "end"
    ts = [evs[k].elapsed_time(evs[k + 1]) for k in range(600)]
    out["sweep_ms_first10"] = statistics.median(ts[:10])
    out["sweep_ms_last100"] = statistics.median(ts[-100:])
    out["sweep_ms_series_every50"] = [round(statistics.median(ts[i:i + 50]), 3) for i in range(0, 600, 50)]
    time.sleep(0.3)
    s.p.terminate()
    for tag in ("idle", "copy", "sweep"):
        out[tag] = s.summary(tag)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
