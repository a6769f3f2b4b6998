"""The C-ABI library loads on a CPU box and exports every symbol include/aaa.h declares;
the ctypes mirrors match the header's struct layouts (compiled with gcc). No compute calls."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def built():
    from paper_2504_12811_b200 import _build
    return _build.build()


def test_library_exports_every_declared_symbol(built):
    import paper_2504_12811_b200 as pkg
    header = (ROOT / "include" / "aaa.h").read_text()
    declared = set(re.findall(r"\b(aaa_[a-z_]+)\s*\(", header))
    L = pkg.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(pkg.EXPORTED_SYMBOLS) == declared
    assert L.aaa_version() == 1
    nm = subprocess.run(["nm", "-D", str(built)], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf" T {name}$", nm, re.M), name


def test_ctypes_layout_matches_header(tmp_path):
    import paper_2504_12811_b200 as pkg
    src = tmp_path / "sz.c"
    src.write_text('#include "aaa.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(aaa_camera), sizeof(aaa_config), sizeof(aaa_gaussians), sizeof(aaa_stats),'
                   'offsetof(aaa_stats, ms), offsetof(aaa_gaussians, n));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    want = [C.sizeof(pkg.Camera), C.sizeof(pkg.Config), C.sizeof(pkg.Gaussians), C.sizeof(pkg.Stats),
            pkg.Stats.ms.offset, pkg.Gaussians.n.offset]
    assert got == want


def test_default_config_without_gpu(built):
    """aaa_default_config is pure host code: callable on a CPU box."""
    import paper_2504_12811_b200 as pkg
    cfg = pkg.Config()
    assert pkg.lib().aaa_default_config(C.byref(cfg)) == 0
    assert abs(cfg.k - 0.3) < 1e-7 and abs(cfg.alpha_max - 0.99) < 1e-7 and cfg.window_k == 32


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (and has no CPU render path)."""
    pkg_dir = ROOT / "paper_2504_12811_b200"
    for f in pkg_dir.rglob("*.py"):
        txt = f.read_text()
        assert "import oracle" not in txt and "from oracle" not in txt, f
    for f in (pkg_dir / "csrc").glob("*"):
        assert "oracle" not in f.read_text(), f
