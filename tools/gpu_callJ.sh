#!/bin/bash
# GPU call J: full GPU tests + smoke after the host-sync removal, bench, memcheck
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/J_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/J_gputest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/J_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/J_bench.json 2> gpurun_out/J_bench.err
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/J_memcheck.log 2>&1
timeout 600 python tools/quick_cfg.py c4zoomout 25 3 > gpurun_out/J_zoom.json 2>&1
echo done
