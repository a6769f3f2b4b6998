#!/bin/bash
# GPU call Q: ncu source-level capture of K6 (one c3 view) for the insertion (MERGE=0) and merge (MERGE=1) variants
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
for v in 0 1; do
  B "-DAAA_K6_MERGE=$v"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:'^k_raster$' -s 1 -c 1 \
     -o gpurun_out/k6_merge$v -f python tools/prof_view.py c3 2 > gpurun_out/Q_ncu$v.log 2>&1
  ncu -i gpurun_out/k6_merge$v.ncu-rep --page raw --csv > gpurun_out/k6_merge${v}_raw.csv 2>/dev/null
  ncu -i gpurun_out/k6_merge$v.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/k6_merge${v}_src.csv 2>/dev/null
done
B ""
echo done
