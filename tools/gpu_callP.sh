#!/bin/bash
# GPU call P: K6 chunk sort network + back-merge (AAA_K6_MERGE) A/B, then the GPU tests on it
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/P_ab.jsonl; : > $out
for v in "-DAAA_K6_MERGE=0" "-DAAA_K6_MERGE=1"; do
  B "$v" || { echo "{\"variant\": \"$v FAILED\"}" >> $out; continue; }
  for cfg in "c3 40" "c4wide 25" "c4zoomout 25" "c4inside 25" "c2 50"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/P_err.log
  done
done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/P_tests.log 2>&1
echo done
