#!/bin/bash
# GPU call S: ncu source-level capture of the default K6 (one c3 view)
python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'^k_raster$' -s 1 -c 1 \
   -o gpurun_out/k6_S -f python tools/prof_view.py c3 2 > gpurun_out/S_ncu.log 2>&1
ncu -i gpurun_out/k6_S.ncu-rep --page raw --csv > gpurun_out/k6_S_raw.csv 2>/dev/null
ncu -i gpurun_out/k6_S.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/k6_S_src.csv 2>/dev/null
echo done
