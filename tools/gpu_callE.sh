#!/bin/bash
# GPU call E: K6 pooled-g A/B (giant FRAC 1.0, K3 dense, K1 inline), giant fixed sweep on c4wide
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/E_ab.jsonl; : > $out
for v in "-DAAA_K6_GPOOL=0" "-DAAA_K6_GPOOL=1" "-DAAA_K6_GPOOL=0 -DAAA_K1_MINB=4"; do
  B "$v" || exit 1
  for cfg in "c3 40" "c2 100" "c4wide 25" "c4zoomout 25" "c4inside 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/E_err.log
  done
done
B "-DAAA_K6_GPOOL=1"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "determinism or giant or c2_full or c1_full or random_scene or full_size" > gpurun_out/E_tests_gpool.log 2>&1
B ""
for thr in 8192 16384; do
  for cfg in "c4wide 25" "c4zoomout 25"; do
    echo "{\"variant\": \"giant=$thr\"}" >> $out
    AAA_GIANT_LIST=$thr timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/E_err.log
  done
done
echo done
