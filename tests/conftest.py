import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
# the unmodified reference, installed by `pip install --target baseline/_ref`
# (travels to the GPU box with the repo snapshot); the /root/reference source
# tree is used only in the build container
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if p.exists() and str(p) not in sys.path:
        sys.path.append(str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


def golden(name: str) -> dict:
    return json.loads((GOLDEN / f"{name}.json").read_text())


SMALL_APPS = ["four_loops", "nest2d", "stencil", "triple_nest", "matmul", "three_loops_fft",
              "himeno_xs_inline", "himeno_xs_temps", "matmul_48", "nasmg_18", "himeno_17x9x33"]


def has_reference() -> bool:
    try:
        import gpuoffload  # noqa: F401
        return True
    except ImportError:
        return False
