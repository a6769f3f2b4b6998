"""Summarise an ab_variants.sh output: python tools/ab_show.py OUT.jsonl"""
import json
import sys

v = None
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "variant" in d:
        v = d["variant"]
        continue
    if "case" in d:
        if not d["bit_identical"]:
            print(f"    IMAGE DIFF {v}: {d}")
        continue
    s = d["stages"]
    print(f"{v:44s} {d['config']:10s} fps {d['fps']:7.1f} K1 {s['preprocess']:.3f} K3 {s['cull_emit']:.3f} "
          f"sort {s['sort']:.3f} K6 {s['raster']:.3f} K6s {s['raster_spill']:.3f} spilled {d['counters']['spilled_pixels']:.0f}")
