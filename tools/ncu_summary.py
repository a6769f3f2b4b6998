"""Turn a round's ncu outputs (tools/profile_round.sh) into the committed profiles/ summaries:
  profiles/<R>_launches.md   per-kernel launch counts, mean duration and share of one view
                             (from the gpu__time_duration.sum launch list of the bench command)
  profiles/<R>_full.md       key --set full metrics of every kernel of one view
  profiles/ncu_traffic.json  DRAM bytes (read + write) per launch of each bench stage, read by
                             bench.py for roofline.traffic
usage: python tools/ncu_summary.py r01"""
import csv
import json
import re
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

# bench.py stage -> kernels of that stage
STAGE_KERNELS = {
    "preprocess": ["k_preprocess"],
    "scan": ["k_scan"],
    "cull_emit": ["k_cull_emit"],
    "sort": ["k_sort_hist", "k_sort_hist_scan", "k_onesweep"],
    "ranges": ["k_ranges"],
    "raster": ["k_tile_order", "k_raster", "k_raster_spill"],
}

FULL_METRICS = [
    ("gpu__time_duration.sum", "time (ms)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / instruction"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__inst_executed_pipe_fma.sum", "FMA-pipe warp instr"),
    ("sm__inst_executed_pipe_alu.sum", "ALU-pipe warp instr"),
    ("sm__inst_executed_pipe_xu.sum", "XU (MUFU) warp instr"),
    ("sm__inst_executed_pipe_lsu.sum", "LSU warp instr"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct", "stall long scoreboard %"),
    ("smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct", "stall short scoreboard %"),
    ("smsp__warps_issue_stalled_wait_per_warp_active.pct", "stall wait %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem / CTA (B)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def base(name):
    n = re.sub(r"\(.*", "", name).replace("void ", "").strip()
    n = re.sub(r"^aaa::", "", n)
    return re.sub(r"<.*", "", n)


def main():
    r = sys.argv[1] if len(sys.argv) > 1 else "r01"
    PROF.mkdir(exist_ok=True)
    # ---- launch list
    rows = [x for x in csv.reader(open(OUT / f"launches_{r}.csv")) if len(x) > 10]
    h, rows = rows[0], rows[1:]
    agg = OrderedDict()
    load = OrderedDict()  # scene load (validation, pack, Morton order): every launch before the first K1
    seen_k1 = False
    for x in rows:
        d = dict(zip(h, x))
        k = base(d["Kernel Name"])
        seen_k1 = seen_k1 or k == "k_preprocess"
        (agg if seen_k1 else load).setdefault(k, []).append(float(d["Metric Value"]) / 1e3)  # us
    n_views = len(agg.get("k_preprocess", [1]))
    per_view = {k: sum(v) / n_views for k, v in agg.items()}
    tot = sum(per_view.values())
    lines = [f"# {r}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Command: `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 "
             "--warmup 3 --scaling weak --views-per-rank 4 --no-cpu-baseline --no-e2e` (c3: 3M Gaussians, 1920x1080). "
             "Per-launch times are cold-cache and serialised; compare the SHARE of a view with bench.py's "
             "`stages`.", "",
             f"{len(rows)} launches ({sum(len(v) for v in load.values())} at scene load), {n_views} views.", "",
             "| kernel | launches | mean us/launch | us per view | share of view |", "|---|---|---|---|---|"]
    for k, v in load.items():
        lines.append(f"| {k} (scene load) | {len(v)} | {sum(v) / len(v):.1f} | (load, once) | |")
    for k, v in agg.items():
        pv = per_view[k]
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {pv:.1f} | {pv / tot:.1%} |")
    lines += ["", f"Sum per view: {tot / 1e3:.3f} ms."]
    (PROF / f"{r}_launches.md").write_text("\n".join(lines) + "\n")
    # ---- full capture
    raw = list(csv.reader(open(OUT / f"full_{r}_raw.csv")))
    hh, units, data = raw[0], raw[1], raw[2:]
    kern = []
    for x in data:
        d = dict(zip(hh, x))
        kern.append((base(d["Kernel Name"]), d))
    # one view's kernels: stop where the first captured kernel comes round again (the capture
    # window may run into the next view)
    for i in range(1, len(kern)):
        if kern[i][0] == kern[0][0]:
            kern = kern[:i]
            break
    lines = [f"# {r}: ncu --set full of one c3 view (every kernel, 2nd rendered view)", "",
             "Command: `ncu --set full --clock-control none --import-source on -k regex:^k_ -s 15 -c 15 "
             "python bench.py --steps 1 --warmup 3 --scaling weak --views-per-rank 1 --no-cpu-baseline --no-e2e` (plus the pipe / bank-conflict metrics). "
             "ncu flushes caches before each replay (cold L2).", "",
             "| metric | " + " | ".join(k for k, _ in kern) + " |", "|---|" + "---|" * len(kern)]
    for m, label in FULL_METRICS:
        if m not in hh:
            continue
        vals = []
        for _, d in kern:
            v = d.get(m, "")
            try:
                f = float(v.replace(",", ""))
                vals.append(f"{f:.4g}")
            except ValueError:
                vals.append(v)
        lines.append(f"| {label} | " + " | ".join(vals) + " |")
    (PROF / f"{r}_full.md").write_text("\n".join(lines) + "\n")
    # ---- traffic per stage (bytes per launch of the stage's kernels, summed over one view)
    unit_r = units[hh.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit_r]
    assert units[hh.index("dram__bytes_write.sum")] == unit_r
    traffic = {}
    for st, ks in STAGE_KERNELS.items():
        b = 0.0
        for k, d in kern:
            if k in ks:
                b += (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * scale
        traffic[st] = b
    traffic["raster_k6"] = sum((float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * scale
                               for k, d in kern if k == "k_raster")
    # K6's issue-slot utilisation and lane efficiency (it is latency-bound: the FP32 roofline
    # fraction alone does not say how busy the SM is)
    for k, d in kern:
        if k == "k_raster":
            traffic["raster_k6_issue_active"] = float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]) / 100.0
            traffic["raster_k6_threads_per_inst"] = float(d["smsp__thread_inst_executed_per_inst_executed.ratio"])
            traffic["raster_k6_warps_active"] = float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]) / 100.0
    traffic["_source"] = f"profiles/{r}_full.md (dram__bytes_read.sum + dram__bytes_write.sum, one c3 view)"
    (PROF / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print((PROF / f"{r}_launches.md").read_text())
    print((PROF / f"{r}_full.md").read_text())
    print(traffic)


if __name__ == "__main__":
    main()
