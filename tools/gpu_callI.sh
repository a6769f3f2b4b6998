#!/bin/bash
# GPU call I: 24-bit keys (3 radix passes) A/B; c5 full-frame comparator with the tie band
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/I_ab.jsonl; : > $out
for v in "" "-DAAA_KEY_BITS=24 -DAAA_KEY_LOG_RANGE=16.0"; do
  B "$v" || exit 1
  for cfg in "c3 40" "c4wide 25" "c4zoomout 25" "c4inside 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/I_err.log
  done
done
B ""
rm -f profiles/r02_full_frame_parity.jsonl
timeout 3000 python tools/full_frame_parity.py r02 c5:0 > gpurun_out/I_fullframe.log 2>&1
cp profiles/r02_full_frame_parity.jsonl gpurun_out/I_full_frame_parity.jsonl 2>/dev/null
echo done
