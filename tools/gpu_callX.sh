#!/bin/bash
# GPU call X: ncu source-level captures of K1, K3 and one onesweep pass (one c3 view)
python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
for k in k_preprocess k_cull_emit k_onesweep; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$k" -s 1 -c 1 \
     -o gpurun_out/X_$k -f python tools/prof_view.py c3 2 > gpurun_out/X_ncu_$k.log 2>&1
  ncu -i gpurun_out/X_$k.ncu-rep --page raw --csv > gpurun_out/X_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/X_$k.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/X_${k}_src.csv 2>/dev/null
done
echo done
