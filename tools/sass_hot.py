"""Summarise an ncu report's SASS page for one kernel: instructions executed and stall samples per
instruction, the hottest instructions, and totals per basic-block-like region (split at branch
targets). Diagnostic tool: python tools/sass_hot.py report.ncu-rep [kernel-substring] [--top N]"""
import argparse
import csv
import io
import subprocess
import sys


def load(rep, kname):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = {"name": line.split(",", 1)[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(line)
    for b in blocks:
        if kname in b["name"]:
            r = list(csv.reader(io.StringIO("\n".join(b["rows"]))))
            h = r[0]
            return b["name"], [dict(zip(h, x)) for x in r[1:] if len(x) == len(h)]
    sys.exit(f"kernel {kname!r} not in {[b['name'] for b in blocks]}")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel", nargs="?", default="k_raster<")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--regions", action="store_true")
    a = ap.parse_args()
    name, rows = load(a.rep, a.kernel)
    tot_i = sum(num(r["Instructions Executed"]) for r in rows)
    tot_s = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rows)
    print(f"{name}\n  instructions {tot_i:.4g}  samples {tot_s:.4g}  sass lines {len(rows)}")
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(num(r[c]) for r in rows) for c in stall_cols}
    print("  stalls:", ", ".join(f"{c[6:]} {v / tot_s:.1%}" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    top = sorted(range(len(rows)), key=lambda i: -num(rows[i]["Warp Stall Sampling (All Samples)"]))[: a.top]
    print(f"\n  top {a.top} by stall samples (idx: samples% inst threads | sass | top stalls)")
    for i in sorted(top):
        r = rows[i]
        s = num(r["Warp Stall Sampling (All Samples)"])
        st = sorted(((c[6:], num(r[c])) for c in stall_cols), key=lambda x: -x[1])[:2]
        print(f"  {i:5d}: {s / tot_s:6.2%} {num(r['Instructions Executed']):10.3g} {num(r['Avg. Threads Executed']):5.1f} | "
              f"{r['Source'].strip()[:60]:60s} | {st[0][0]} {st[1][0]}")
    if a.regions:
        # regions: split where the executed count changes
        print("\n  regions (start-end: inst% samples% | first sass)")
        start = 0
        for i in range(1, len(rows) + 1):
            if i == len(rows) or rows[i]["Instructions Executed"] != rows[start]["Instructions Executed"]:
                ins = sum(num(rows[k]["Instructions Executed"]) for k in range(start, i))
                smp = sum(num(rows[k]["Warp Stall Sampling (All Samples)"]) for k in range(start, i))
                if ins / tot_i > 0.005 or smp / tot_s > 0.005:
                    print(f"  {start:5d}-{i - 1:5d}: {ins / tot_i:6.2%} {smp / tot_s:6.2%} | {rows[start]['Source'].strip()[:70]}")
                start = i


if __name__ == "__main__":
    main()
