#!/bin/bash
# GPU call N: full-frame comparator reports for the rest of SURVEY 8(d)'s checked subset
# (c3: every 20th view; c4: 5 views per sub-batch)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/N_build.log 2>&1
rm -f profiles/r02_full_frame_parity.jsonl
timeout 6600 python tools/full_frame_parity.py r02 c3:20 c3:40 c3:60 c3:80 c3:120 c3:140 c3:160 c3:180 \
    c4wide:13 c4wide:23 c4wide:33 c4wide:43 c4zoomout:0 c4zoomout:20 c4zoomout:30 c4zoomout:40 \
    c4inside:9 c4inside:19 c4inside:29 c4inside:49 > gpurun_out/N_fullframe.log 2>&1
cp profiles/r02_full_frame_parity.jsonl gpurun_out/N_full_frame_parity.jsonl 2>/dev/null
echo done
