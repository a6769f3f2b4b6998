#!/bin/bash
# GPU call C: K6 lazy-settle A/B, giant-list threshold sweep, parity subset
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/C_ab.jsonl; : > $out
for v in "-DAAA_K6_LAZY=0" "-DAAA_K6_LAZY=1"; do
  B "$v" || exit 1
  for cfg in "c3 40" "c2 100" "c4wide 25" "c4zoomout 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/C_err.log
  done
done
for thr in 32768 16384 8192 4096 2048 1024; do
  for cfg in "c4zoomout 25" "c3 40"; do
    echo "{\"variant\": \"LAZY=1 giant=$thr\"}" >> $out
    AAA_GIANT_LIST=$thr timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/C_err.log
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -q -p no:cacheprovider -k "determinism or giant or c2_full or targeted or c4inside or band" > gpurun_out/C_tests.log 2>&1
echo done
