#!/bin/bash
# Checkpoint under gpurun: build, full GPU tests, smoke, default bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/chk_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/chk_gputest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/chk_smoke.log
timeout 900 python bench.py > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err
echo done
