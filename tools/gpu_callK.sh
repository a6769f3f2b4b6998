#!/bin/bash
# GPU call K: K3 persistent-grid A/B; c2 full-image parity with the two-pass comparator
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/K_ab.jsonl; : > $out
for v in "-DAAA_K3_PERSIST=0" "-DAAA_K3_PERSIST=1"; do
  B "$v" || exit 1
  for cfg in "c3 40" "c4zoomout 25" "c2 100"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/K_err.log
  done
done
B ""
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "c2_full or overflow or batch or band or giant" > gpurun_out/K_tests.log 2>&1
echo done
