#!/bin/bash
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
for v in "" "-DAAA_BAND_APPROX=1"; do
  B "$v"; echo "{\"variant\": \"$v\"}" >> gpurun_out/band_ab.jsonl
  timeout 600 python tools/band_ab.py 8 >> gpurun_out/band_ab.jsonl 2>> gpurun_out/band_ab.err
  timeout 600 python tools/band_ab.py 4 >> gpurun_out/band_ab.jsonl 2>> gpurun_out/band_ab.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "band or host_pointer" > gpurun_out/band_tests.log 2>&1
B ""
