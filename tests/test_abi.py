"""The C-ABI library loads without a GPU and exports every entry point
declared in include/b2o.h; ctypes struct layouts equal the C layouts."""

import ctypes
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
