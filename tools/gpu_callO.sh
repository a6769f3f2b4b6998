#!/bin/bash
# GPU call O: compact K6s A/B + bit-identity tests
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/O_ab.jsonl; : > $out
for v in "-DAAA_K6S_COMPACT=0 -DAAA_K1_SPHERE=0" "-DAAA_K1_SPHERE=0" "-DAAA_K6S_COMPACT=0" ""; do
  B "$v" || { echo "{\"variant\": \"$v FAILED\"}" >> $out; continue; }
  for cfg in "c4zoomout 25" "c4wide 25" "c3 40" "c4inside 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/O_err.log
  done
done
B ""
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -q -p no:cacheprovider -k "determinism or giant or c2_full or c1_full or random_scene or spill or band or overflow or k1_records or full_size" > gpurun_out/O_tests.log 2>&1
echo done
