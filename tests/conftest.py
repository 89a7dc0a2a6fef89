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


_FINAL: dict = {}


def oracle_final(doc: dict, spec: dict) -> dict:
    """Final state of a program by the reference's own C emission
    (oracle/_ref, prebuilt by __graft_entry__.build() and travelling with the
    snapshot), falling back to the C restatement oracle/cgen.py (pinned to
    the emission bit for bit by tests/test_refc.py) when no object was
    prebuilt for this document.  Cached per (document, precision, inputs)."""
    import hashlib

    from oracle.externals import make_binder
    from oracle.refc import reference_state
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    # the spec's inputs matter: fuzz programs share documents and differ by seeds
    key = hashlib.sha256((json.dumps(doc, sort_keys=True) + spec.get("precision", "fp32")
                          + json.dumps(spec.get("inputs", {}), sort_keys=True)).encode()).hexdigest()
    if key not in _FINAL:
        st = appspec.initial_state(Program(doc), spec)
        _FINAL[key] = reference_state(doc, spec, st, make_binder(doc, spec))[0]
    return _FINAL[key]
