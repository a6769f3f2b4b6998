#!/bin/bash
# GPU call F (checkpoint): build, full GPU tests, smoke, bench, per-config bench, full-frame parity, profile
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/F_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/F_gputest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/F_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/F_bench.json 2> gpurun_out/F_bench.err
timeout 900 python tools/bench_configs.py gpurun_out/F_configs.jsonl > gpurun_out/F_configs.log 2>&1
timeout 2400 python tools/full_frame_parity.py r02 > gpurun_out/F_fullframe.log 2>&1
cp profiles/r02_full_frame_parity.jsonl gpurun_out/F_full_frame_parity.jsonl 2>/dev/null
echo done
