#!/bin/bash
# GPU call M: K1/K2-beside-K6 overlap A/B (AAA_OVERLAP_K1), sort items 24; then GPU tests
python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
out=gpurun_out/M_ab.jsonl; : > $out
for ov in 0 1; do
  for cfg in "c3 40" "c4wide 25" "c4zoomout 25" "c2 100"; do
    echo "{\"variant\": \"overlap=$ov\"}" >> $out
    AAA_OVERLAP_K1=$ov timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/M_err.log
  done
done
AAA_OVERLAP_K1=0 timeout 600 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/M_bench_ov0.json 2>> gpurun_out/M_err.log
AAA_OVERLAP_K1=1 timeout 600 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/M_bench_ov1.json 2>> gpurun_out/M_err.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/M_gputest.log 2>&1
echo done
