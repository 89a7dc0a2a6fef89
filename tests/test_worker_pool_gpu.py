"""The in-process worker pool (one worker thread + stream per device, LPT job
queue): several workers (here sharing the box's GPU) return every result in
request order, identical in validity and accounting to a single worker."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


def run(devices):
    out = subprocess.run([sys.executable, str(HERE / "_worker_pool.py"), "himeno_xs_inline", json.dumps(devices)],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def test_four_workers_match_one():
    one = run([0])
    four = run([0, 0, 0, 0])
    assert one["workers"] == 1 and four["workers"] == 4
    assert len(four["results"]) == 64
    assert {r[2] for r in four["results"]} == {0, 1, 2, 3}   # every worker took jobs
    for a, b in zip(one["results"], four["results"]):
        assert a[0] == b[0] and a[1] == b[1] == "valid" and a[3] == b[3] and a[4] == b[4]
