#!/bin/bash
# Table 5 analogue on c3: the same kernels with each ablation switch; one JSON line each
R=${1:-r02}
for a in none no_cull no_hier no_3d 3dgs; do
  timeout 900 python bench.py --steps 3 --warmup 3 --scaling weak --views-per-rank 10 --no-cpu-baseline --no-e2e --ablation $a \
    >> gpurun_out/ablations_${R}.jsonl 2> gpurun_out/ablation_${a}.err || tail -3 gpurun_out/ablation_${a}.err
done
python - <<PY
import json
for l in open("gpurun_out/ablations_${R}.jsonl"):
    d = json.loads(l)
    print(d["config"]["ablation"], round(d["value"], 1), "FPS", round(d["ms_per_step"] / d["config"]["views_per_rank_per_step"], 3), "ms/view",
          {k: round(v["ms_per_view"], 3) for k, v in d["stages"].items()}, "pairs", d["counters_per_view"]["pairs"])
PY
