"""The bench's reference arm (``bench.py --impl reference``) keeps the driver
contract on CPU: one JSON line with the metric, a value, the CPU baseline it
measured (the reference's own C emission of the headline pattern) and an e2e
object without copies; under a 2-rank torchrun-style environment only rank 0
prints."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_reference

pytestmark = pytest.mark.skipif(not has_reference(), reason="reference not importable (needed to emit the C)")


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    return [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]


def test_reference_arm_line():
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == len(os.sched_getaffinity(0))
    assert "emit_annotated" in cb["sample"] and d["config"]["workload"].startswith("himeno_M")


def test_reference_arm_two_ranks_rank0_prints_once():
    """torchrun-style world of 2 (gloo rendezvous on 127.0.0.1): rank 0 runs
    the reference program on every host core and prints the line, rank 1
    exits without work."""
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    procs = []
    for rank in (0, 1):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(rank), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                                       "--steps", "1", "--warmup", "0"], stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True, env=env, cwd=ROOT))
    outs = [p.communicate(timeout=600) for p in procs]
    assert [p.returncode for p in procs] == [0, 0], [o[1][-1000:] for o in outs]
    lines = [[ln for ln in o[0].splitlines() if ln.startswith("{")] for o in outs]
    assert len(lines[0]) == 1 and lines[1] == []
    d = json.loads(lines[0][0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    # torchrun's OMP_NUM_THREADS=1 is overridden: the reference arm uses every core
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
