#!/bin/bash
# GPU call L: K3 items/occupancy and K6 staging/pop retune A/B on c3 (+ c4wide)
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/L_ab.jsonl; : > $out
for v in "" "-DAAA_K3_ITEMS=4" "-DAAA_K3_ITEMS=16" "-DAAA_K3_MINB=4" "-DAAA_K6_CH=8" "-DAAA_K6_CH=12" "-DAAA_K6_POP=3" "-DAAA_SORT_ITEMS=12" "-DAAA_SORT_ITEMS=20"; do
  B "$v" || { echo "{\"variant\": \"$v FAILED\"}" >> $out; continue; }
  for cfg in "c3 40" "c4wide 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/L_err.log
  done
done
B ""
echo done
