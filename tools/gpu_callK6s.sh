#!/bin/bash
# ncu capture of K6s on a c4 zoom-out view (giant tiles)
python -c "from paper_2504_12811_b200 import _build; _build.build()"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'^k_raster_spill' -s 2 -c 1 \
   -o gpurun_out/k6s_zo -f python tools/prof_view.py c4zoomout 2 > gpurun_out/k6s_ncu.log 2>&1
ncu -i gpurun_out/k6s_zo.ncu-rep --page raw --csv > gpurun_out/k6s_zo_raw.csv 2>/dev/null
ncu -i gpurun_out/k6s_zo.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/k6s_zo_src.csv 2>/dev/null
