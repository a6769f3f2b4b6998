#!/bin/bash
# merge-path statistics (AAA_K6_FBSTATS): chunks, full-window and exact-tie fallbacks, lanes over capacity, staged entries
AAA_NVCC_FLAGS="-DAAA_K6_STATS -DAAA_K6_FBSTATS -DAAA_DEBUG_STATS" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
python - <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2504_12811_b200 as pkg
from synth import scenes as S
R = pkg.Renderer(0)
for cfg, views in (("c3", [0, 100]), ("c4wide", [0]), ("c4inside", [30])):
    scene, cams = S.make_config(cfg)
    R.load(scene)
    for v in views:
        R.render(cams[v], with_T=False); torch.cuda.synchronize()
        print(cfg, v, flush=True)
        R.stats()
PY
python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
