#!/bin/bash
# GPU call R: K6 merge v2 A/B (float keys + tie fallback, rolled per-entry fallback), CH 8 / 10,
# and bit identity of the images against the insertion-sort build
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/R_ab.jsonl; : > $out
for v in "-DAAA_K6_MERGE=0" "-DAAA_K6_MERGE=1" "-DAAA_K6_MERGE=1 -DAAA_K6_CH=8"; do
  B "$v" || { echo "{\"variant\": \"$v FAILED\"}" >> $out; continue; }
  if [ "$v" = "-DAAA_K6_MERGE=0" ]; then timeout 600 python tools/ab_images.py save /tmp/ab_ref.npz 2>> gpurun_out/R_err.log;
  else echo "{\"variant\": \"$v\", \"images\": 1}" >> $out; timeout 600 python tools/ab_images.py cmp /tmp/ab_ref.npz >> $out 2>> gpurun_out/R_err.log; fi
  for cfg in "c3 40" "c4wide 25" "c4zoomout 25" "c4inside 25" "c2 50"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/R_err.log
  done
done
B ""
echo done
