"""Per-source-line and per-opcode instruction counts of one kernel in an .ncu-rep (run here).

  python tools/ncu_lines.py gpurun_out/prof_config3.ncu-rep [--kernel-index 0] [--top 30]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--launch", type=int, default=None, help="ncu --print-kernel-base / launch filter")
    args = ap.parse_args()
    cmd = ["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if args.launch is not None:
        cmd += ["--launch-skip", str(args.launch), "--launch-count", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    heads = [i for i, r in enumerate(rows) if "Instructions Executed" in r]
    for n, hi in enumerate(heads):
        h = rows[hi]
        iE = h.index("Instructions Executed")
        iS2 = len(h) - 1 - h[::-1].index("Source")  # the SASS text column
        end = heads[n + 1] if n + 1 < len(heads) else len(rows)
        fn = [r for r in rows[max(0, hi - 3):hi] if r and r[0] == "Function Name"]
        print("==", fn[0][1] if fn else "?")
        lines, ops = collections.Counter(), collections.Counter()
        cur = None
        for r in rows[hi + 1:end]:
            if len(r) <= iE:
                continue
            if r[0]:
                cur = (r[0], r[1].strip()[:90])
            try:
                c = int(r[iE])
            except ValueError:
                continue
            if not r[0]:  # SASS rows carry the per-instruction counts
                lines[cur] += c
                t = r[iS2].split()
                if t:
                    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
                    ops[op.split(".")[0]] += c
        tot = sum(lines.values()) or 1
        print("warp instructions", tot)
        for (ln, src), c in lines.most_common(args.top):
            print(f"{c:>12} {100 * c / tot:5.1f}%  {ln:>5}  {src}")
        print("-- opcodes")
        for op, c in ops.most_common(15):
            print(f"{c:>12} {100 * c / tot:5.1f}%  {op}")


if __name__ == "__main__":
    main()
