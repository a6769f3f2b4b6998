AAA_NVCC_FLAGS="-DAAA_K6_STATS -DAAA_DEBUG_STATS" python -c "from paper_2504_12811_b200 import _build; _build.build(force=True)"
python - <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2504_12811_b200 as pkg
from synth import scenes as S
R = pkg.Renderer(0)
for cfg, views in (("c3", [0, 50, 100, 150]), ("c4wide", [0, 20]), ("c4zoomout", [0, 20]), ("c4inside", [10, 30, 49]), ("c2", [0, 30])):
    scene, cams = S.make_config(cfg)
    R.load(scene)
    for v in views:
        if v >= len(cams): continue
        R.render(cams[v], with_T=False); torch.cuda.synchronize()
        st = R.stats()
        print(cfg, v, "spilled", st["spilled_pixels"], "unresolved", st["unresolved_pixels"], flush=True)
PY
