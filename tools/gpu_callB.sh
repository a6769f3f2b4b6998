#!/bin/bash
# GPU call B (round 2): c4inside view 48 diagnosis, new bench modes, band render test, round profile
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/B_build.log 2>&1
timeout 600 python tools/dump_view.py --config c4inside --view 48 --out /tmp/dump48.npz > gpurun_out/B_dump.log 2>&1
timeout 900 python tools/analyze_dump.py /tmp/dump48.npz --config c4inside --view 48 --show 8 > gpurun_out/B_analyze48.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "band" -p no:cacheprovider > gpurun_out/B_bandtest.log 2>&1
timeout 900 python bench.py > gpurun_out/B_bench.json 2> gpurun_out/B_bench.err
timeout 900 python bench.py --gpus 2 --views 16 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/B_bench_g2.json 2> gpurun_out/B_bench_g2.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/B_bench_c5.json 2> gpurun_out/B_bench_c5.err
timeout 900 python bench.py --config c5 --gpus 2 --steps 2 --warmup 1 > gpurun_out/B_bench_c5_g2.json 2> gpurun_out/B_bench_c5_g2.err
timeout 2400 bash tools/profile_round.sh r02 > gpurun_out/B_profile.log 2>&1
echo done
