"""Per-CUDA-source-line totals (instructions executed, stall samples) of one kernel from an ncu
report (needs -lineinfo). Diagnostic tool:
    python tools/src_hot.py report.ncu-rep k_raster< [--top 40]"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    rows, fpath, func, hdr = [], None, None, None
    for line in out.splitlines():
        if line.startswith('"File Path"'):
            fpath = line.split(",", 1)[1].strip('"')
            continue
        if line.startswith('"Function Name"'):
            func = line.split(",", 1)[1]
            continue
        if line.startswith('"Line No"'):
            hdr = next(csv.reader(io.StringIO(line)))
            continue
        if hdr is None or a.kernel not in (func or ""):
            continue
        r = next(csv.reader(io.StringIO(line)))
        if r and r[0] not in ("", "..."):
            d = dict(zip(hdr, r))
            def num(k):
                try:
                    return float(d[k])
                except (KeyError, ValueError):
                    return 0.0
            rows.append((fpath.split("/")[-1], int(r[0]), r[1].strip(), num("Instructions Executed"),
                         num("Warp Stall Sampling (All Samples)")))
    ti = sum(x[3] for x in rows) or 1
    ts = sum(x[4] for x in rows) or 1
    print(f"{a.kernel}: {ti:.4g} instructions, {ts:.4g} samples over {len(rows)} source lines")
    for f, ln, src, i, s in sorted(rows, key=lambda x: -x[4])[: a.top]:
        print(f"{f}:{ln:4d} inst {i / ti:6.2%} samp {s / ts:6.2%} | {src[:90]}")


if __name__ == "__main__":
    main()
