#!/bin/bash
# A/B of compile-time variants under gpurun: tools/ab_variants.sh OUT "CFGS" "flags A" "flags B" ...
# The first variant is the reference: its images are saved and every other variant's images are
# compared bit for bit (tools/ab_images.py); then tools/quick_cfg.py times each config in CFGS
# (e.g. "c3:40 c4wide:25"). One JSON line per measurement in OUT; the default build is restored.
out=$1; cfgs=$2; shift 2
: > $out
B() { AAA_NVCC_FLAGS="$1" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"; }
first=1
for v in "$@"; do
  B "$v" || { echo "{\"variant\": \"$v\", \"build\": \"FAILED\"}" >> $out; continue; }
  if [ $first = 1 ]; then timeout 600 python tools/ab_images.py save /tmp/ab_ref.npz 2>> ${out%.jsonl}.err; first=0;
  else echo "{\"variant\": \"$v\", \"images\": 1}" >> $out; timeout 600 python tools/ab_images.py cmp /tmp/ab_ref.npz >> $out 2>> ${out%.jsonl}.err; fi
  for c in $cfgs; do
    echo "{\"variant\": \"$v\"}" >> $out
    timeout 300 python tools/quick_cfg.py ${c%:*} ${c#*:} 3 >> $out 2>> ${out%.jsonl}.err
  done
done
B ""
