#!/bin/bash
# K1/K2 of the next view beside K6 (AAA_OVERLAP_K1) with 64-thread K1 CTAs
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/OV_ab.jsonl; : > $out
for v in "" "-DAAA_K1_THREADS=64"; do
  B "$v"
  for ov in 0 1; do
    for cfg in "c3 40" "c4wide 25"; do
      echo "{\"variant\": \"$v overlap=$ov\"}" >> $out
      AAA_OVERLAP_K1=$ov timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/OV_err.log
    done
  done
done
B ""
