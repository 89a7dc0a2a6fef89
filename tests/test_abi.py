"""The C-ABI library loads without a GPU and exports every entry point
declared in include/b2o.h; ctypes struct layouts equal the C layouts."""

import ctypes
import os
import sys
import re
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT
from paper_2011_03602_b200 import runtime

HEADER = ROOT / "include" / "b2o.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(b2o_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = runtime.lib()
    names = declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_abi_version_matches_header():
    m = re.search(r"#define B2O_ABI_VERSION (\d+)", HEADER.read_text())
    assert runtime.lib().b2o_abi_version() == int(m.group(1))


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        f'#include <stdio.h>\n#include <stddef.h>\n#include "{HEADER}"\n'
        "int main(void) { printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(b2o_directive), sizeof(b2o_pattern),"
        " sizeof(b2o_result), offsetof(b2o_result, diag), offsetof(b2o_pattern, priority)); return 0; }\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    want = [ctypes.sizeof(runtime.Directive), ctypes.sizeof(runtime.Pattern), ctypes.sizeof(runtime.Result),
            runtime.Result.diag.offset, runtime.Pattern.priority.offset]
    assert got == want


def test_module_abi_matches(tmp_path):
    m = re.search(r"#define B2O_MODULE_ABI (\d+)", (ROOT / "paper_2011_03602_b200" / "csrc" / "b2o_module.h").read_text())
    assert int(m.group(1)) >= 4


@pytest.mark.skipif(Path("/dev/nvidia0").exists(), reason="GPU present")
def test_init_without_gpu_fails_loudly():
    with pytest.raises(runtime.B2OError):
        runtime.Runtime([0])


def _build_c_consumer():
    import shutil
    import subprocess

    if shutil.which("gcc") is None or not (ROOT / "paper_2011_03602_b200" / "libb2o.so").exists():
        pytest.skip("gcc or libb2o.so missing")
    subprocess.run(["make", "-s", "-B", "-C", str(ROOT / "tests" / "c")], check=True, capture_output=True, text=True)
    return ROOT / "tests" / "c" / "abi_ops"


def test_c_consumer_builds_against_the_header():
    """A plain-C program (tests/c/abi_ops.c) compiles against include/b2o.h
    and links libb2o.so: the boundary needs neither Python nor torch."""
    assert _build_c_consumer().exists()


@pytest.mark.gpu
def test_c_consumer_runs():
    import subprocess

    exe = _build_c_consumer()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
    assert "bit-exact" in r.stdout and "histogram: exact" in r.stdout


@pytest.mark.gpu
def test_c_consumer_loads_and_measures(tmp_path):
    """The whole boundary from plain C (tests/c/abi_app.c): b2o_app_load
    from the IR document + app spec JSON (SURVEY.md §8(b) app_load), every
    Himeno 17x9x33 genome through b2o_submit / b2o_wait, each valid with
    directive executions == the plan's multiplicities, and each final state
    bit-identical to the reference's own C emission (oracle/_ref)."""
    import json
    import subprocess

    from conftest import golden, oracle_final
    from paper_2011_03602_b200.ir import Program

    exe = _build_c_consumer().with_name("abi_app")
    g = golden("himeno_17x9x33")
    (tmp_path / "doc.json").write_text(json.dumps(g["doc"]))
    (tmp_path / "spec.json").write_text(json.dumps(g["spec"]))
    lines = []
    for genome in sorted(g["patterns"]):
        p = g["patterns"][genome]
        lines.append(f"pattern {genome} {len(p['gpu_roots'])} {' '.join(map(str, p['gpu_roots']))} "
                     f"{len(p['directives'])}")
        for d in p["directives"]:
            lines.append(f"{d['var']} {0 if d['dir'] == 'h2d' else 1} {d['anchor_loop']} "
                         f"{0 if d['side'] == 'before' else 1} {d['multiplicity']} {d['batch']}")
    (tmp_path / "patterns.txt").write_text("\n".join(lines) + "\n")
    want = oracle_final(g["doc"], g["spec"])
    prog = Program(g["doc"])
    exp = []
    for name in g["spec"]["outputs"]:
        arr = want[prog.var_by_name[name].id]
        f = tmp_path / f"expect_{name}.bin"
        arr.tofile(f)
        exp.append(f"{name} {arr.nbytes} {f}")
    (tmp_path / "expect.txt").write_text("\n".join(exp) + "\n")
    env = dict(os.environ, B2O_PYTHON=sys.executable)
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr[-3000:]
    assert "malformed document refused" in r.stdout


def test_compile_service_manifest(tmp_path):
    """compile_cli (the build step behind b2o_app_load) writes the host
    module, the cubin and every variable's initial value; a program the
    compiler cannot take exits 2 with the reason."""
    import json

    import numpy as np

    from conftest import golden
    from paper_2011_03602_b200 import appspec, compile_cli
    from paper_2011_03602_b200.ir import Program

    g = golden("matmul_48")
    (tmp_path / "doc.json").write_text(json.dumps(g["doc"]))
    (tmp_path / "spec.json").write_text(json.dumps(g["spec"]))
    assert compile_cli.main([str(tmp_path / "doc.json"), str(tmp_path / "spec.json"), str(tmp_path / "out")]) == 0
    man = (tmp_path / "out" / "manifest.txt").read_text().split("\n")
    assert man[0].startswith("host ") and Path(man[0][5:]).exists()
    assert man[1].startswith("cubin ") and Path(man[1][6:]).exists()
    st = appspec.initial_state(Program(g["doc"]), g["spec"])
    for ln in man[3:]:
        if not ln:
            continue
        _, vid, nbytes, path, name = ln.split()
        got = np.fromfile(path, dtype=st[int(vid)].dtype)
        assert got.nbytes == int(nbytes) and np.array_equal(got, st[int(vid)]), name
    (tmp_path / "bad.json").write_text(json.dumps({"not": "a program"}))
    assert compile_cli.main([str(tmp_path / "bad.json"), str(tmp_path / "spec.json"), str(tmp_path / "o2")]) == 2
