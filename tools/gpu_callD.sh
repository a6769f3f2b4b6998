#!/bin/bash
# GPU call D: K3 dense emission x K1 colour split A/B (automatic giant-list threshold), full GPU tests
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/D_ab.jsonl; : > $out
for v in "-DAAA_K3_DENSE=0 -DAAA_K1_SPLIT=0" "-DAAA_K3_DENSE=1 -DAAA_K1_SPLIT=0" "-DAAA_K3_DENSE=0 -DAAA_K1_SPLIT=1" "-DAAA_K3_DENSE=1 -DAAA_K1_SPLIT=1"; do
  B "$v" || exit 1
  for cfg in "c3 40" "c2 100" "c4wide 25" "c4zoomout 25" "c4inside 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/D_err.log
  done
done
B ""
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/D_gputest.log 2>&1
echo done
