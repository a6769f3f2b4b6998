#!/bin/bash
# A/B timing of compile-time variants, each bounded: tools/ab.sh OUT "" "-DFOO" ...
# (c2 window/spill diagnostic vs the oracle + a short c3 bench per variant; one line per variant in OUT)
out=$1; shift
for v in "$@"; do
  AAA_NVCC_FLAGS="$v" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)" || exit 1
  timeout 200 python tools/diag_spill.py c2 0 2>&1 | grep "^K32" >> "$out"
  timeout 300 python bench.py --steps 3 --warmup 2 --views-per-rank 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err || { echo "variant [$v] FAILED" >> "$out"; tail -3 gpurun_out/bench_v.err >> "$out"; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print('variant [$v] FPS', round(d['value'],1), {k: round(v['ms_per_view'],3) for k,v in d['stages'].items()}, 'spilled', d['counters_per_view']['spilled_pixels'])" >> "$out"
done
python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
