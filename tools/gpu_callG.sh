#!/bin/bash
# GPU call G: K1 prefetch A/B, Table 5 ablations (incl. the 3DGS-style baseline), 3DGS test,
# full-frame comparator reports for c4 x 3 and c5
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
out=gpurun_out/G_ab.jsonl; : > $out
for v in "-DAAA_K1_ITEMS=1" "-DAAA_K1_ITEMS=2" "-DAAA_K1_ITEMS=4"; do
  B "$v" || exit 1
  for cfg in "c3 40" "c4inside 25"; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py $cfg 3 >> $out 2>> gpurun_out/G_err.log
  done
done
B ""
timeout 600 python -m pytest tests/test_gpu_ablations.py -q -p no:cacheprovider > gpurun_out/G_ablation_tests.log 2>&1
: > gpurun_out/ablations_r02.jsonl
timeout 1500 bash tools/ablations.sh r02 > gpurun_out/G_ablations.log 2>&1
rm -f profiles/r02_full_frame_parity.jsonl
timeout 3600 python tools/full_frame_parity.py r02 c4wide:3 c4zoomout:10 c4inside:48 c5:0 > gpurun_out/G_fullframe.log 2>&1
cp profiles/r02_full_frame_parity.jsonl gpurun_out/G_full_frame_parity.jsonl 2>/dev/null
echo done
