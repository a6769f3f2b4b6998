#!/bin/bash
# Round-end measurement pass (run under gpurun from the repo root). Outputs in gpurun_out/; the
# committed summaries are written here from them (profiles/r02_*).
set -u
R=${1:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gputest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 python bench.py --gpus 2 --views 16 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final_bench_g2.json 2> gpurun_out/final_bench_g2.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err
timeout 900 python bench.py --config c5 --gpus 2 --steps 2 --warmup 1 > gpurun_out/final_bench_c5_g2.json 2> gpurun_out/final_bench_c5_g2.err
timeout 900 python tools/bench_configs.py gpurun_out/final_configs.jsonl > gpurun_out/final_configs.log 2>&1
: > gpurun_out/ablations_${R}.jsonl
timeout 1500 bash tools/ablations.sh ${R} > gpurun_out/final_ablations.log 2>&1
timeout 2400 bash tools/profile_round.sh ${R} > gpurun_out/final_profile.log 2>&1
echo done
