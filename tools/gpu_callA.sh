#!/bin/bash
# GPU call A (round 2): build, FFMA peak, GPU tests, compute-sanitizer memcheck/racecheck/synccheck
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/A_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma tools/ffma_peak.cu && /tmp/ffma > gpurun_out/A_ffma.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/A_gputest.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/A_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py small > gpurun_out/A_racecheck.log 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py small > gpurun_out/A_synccheck.log 2>&1
echo done
