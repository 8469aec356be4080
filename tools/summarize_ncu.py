"""Summarise ncu outputs into profiles/ (run here, no GPU):
  python tools/summarize_ncu.py <round> <workload> [<kernel tag>]
reads gpurun_out/launches_<wl>.csv and gpurun_out/prof_<wl>.ncu-rep, writes
profiles/<round>_<wl>_launches.csv (per-kernel totals and shares), profiles/<round>_<wl>_ncu.json
(key --set full metrics of the captured launch) and profiles/traffic_<wl>.json (the DRAM bytes
per launch bench.py reports as roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def main():
    rnd, wl = sys.argv[1], sys.argv[2]
    tag = sys.argv[3] if len(sys.argv) > 3 else ""  # kernel short name (bench: kernel_in_use)
    base = f"{rnd}_{wl}_{tag}" if tag else f"{rnd}_{wl}"
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    txt = open(os.path.join(ROOT, "gpurun_out", f"launches_{wl}.csv")).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        agg[r["Kernel Name"]][0] += 1
        agg[r["Kernel Name"]][1] += float(r["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(out, f"{base}_launches.csv"), "w") as f:
        f.write("kernel,launches,total_ms,avg_ms,share_pct\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f'"{k}",{n},{t / 1e6:.3f},{t / n / 1e6:.4f},{100 * t / tot:.2f}\n')
    raw = subprocess.run(["ncu", "-i", os.path.join(ROOT, "gpurun_out", f"prof_{wl}.ncu-rep"),
                          "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rr[0], rr[1], rr[2]
    m = {h: (vals[i], units[i]) for i, h in enumerate(hdr) if h in WANT or h == "Kernel Name"}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    def num(key):
        v, u = m[key]
        return float(v.replace(",", "")) * scale.get(u, 1)
    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    summary = {"round": rnd, "workload": wl, "kernel": m.get("Kernel Name", ("?", ""))[0],
               "metrics": {k: f"{v} {u}".strip() for k, (v, u) in m.items() if k != "Kernel Name"},
               "dram_bytes_per_launch": dram}
    json.dump(summary, open(os.path.join(out, f"{base}_ncu.json"), "w"), indent=1)
    json.dump({"workload": wl, "round": rnd, "kernel": summary["kernel"],
               "dram_bytes_per_launch": dram, "source": f"profiles/{base}_ncu.json"},
              open(os.path.join(out, f"traffic_{wl}_{tag}.json" if tag else f"traffic_{wl}.json"), "w"),
              indent=1)
    print(json.dumps(summary, indent=1))
    print(open(os.path.join(out, f"{base}_launches.csv")).read())


if __name__ == "__main__":
    main()
