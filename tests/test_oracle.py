"""The CPU oracle pinned: the C restatement (oracle/cgen.py) equals the
pure-Python interpreter (oracle/interp.py) bit for bit on every small app,
and both agree with closed forms (numpy matmul; a numpy Himeno written with
the same float32 operation order)."""

import numpy as np
import pytest

from conftest import SMALL_APPS, golden
from oracle.cgen import CProgram
from oracle.externals import fft2d, gemm, make_binder
from oracle.interp import run_program
from paper_2011_03602_b200 import appspec
from paper_2011_03602_b200.ir import Program


def _state(g):
    return appspec.initial_state(Program(g["doc"]), g["spec"])


@pytest.mark.parametrize("name", SMALL_APPS)
def test_c_restatement_equals_interpreter(name):
    g = golden(name)
    st = _state(g)
    binder = make_binder(g["doc"], g["spec"])
    a = run_program(g["doc"], st, externals=binder)
    b = CProgram(g["doc"]).run(st, binder)
    for k in a:
        assert np.array_equal(a[k], b[k]), (name, k)


@pytest.mark.parametrize("name", ["himeno_xs_inline", "nasmg_18", "matmul_48", "four_loops"])
def test_openmp_restatement_equals_sequential(name):
    g = golden(name)
    st = _state(g)
    a = CProgram(g["doc"]).run(st)
    b = CProgram(g["doc"], openmp=True).run(st)
    for k in a:
        assert np.array_equal(a[k], b[k]), (name, k)


def test_matmul_oracle_matches_numpy():
    g = golden("matmul_48")
    prog = Program(g["doc"])
    st = _state(g)
    out = CProgram(g["doc"]).run(st)
    n = 48
    ma = st[prog.var_by_name["ma"].id].reshape(n, n).astype(np.float64)
    mb = st[prog.var_by_name["mb"].id].reshape(n, n).astype(np.float64)
    mc = out[prog.var_by_name["mc"].id].reshape(n, n)
    np.testing.assert_allclose(mc, ma @ mb, rtol=2e-6)


def _himeno_numpy(st, prog, dims, nn):
    """Direct float32 restatement of the inline Himeno app, same op order."""
    I, J, K = dims
    f = {n: st[prog.var_by_name[n].id].reshape(I, J, K).copy() for n in
         ("p", "a0", "a1", "a2", "a3", "b0", "b1", "b2", "c0", "c1", "c2", "bnd", "wrk1", "wrk2", "gs")}
    omega = np.float32(0.8)
    s = (slice(1, I - 1), slice(1, J - 1), slice(1, K - 1))

    def P(di, dj, dk):
        return f["p"][1 + di:I - 1 + di, 1 + dj:J - 1 + dj, 1 + dk:K - 1 + dk]

    gosa = np.float32(0)
    for _ in range(nn):
        gosa = np.float32(0.0)
        s0 = (f["a0"][s] * P(1, 0, 0) + f["a1"][s] * P(0, 1, 0) + f["a2"][s] * P(0, 0, 1)
              + f["b0"][s] * (P(1, 1, 0) - P(1, -1, 0) - P(-1, 1, 0) + P(-1, -1, 0))
              + f["b1"][s] * (P(0, 1, 1) - P(0, -1, 1) - P(0, 1, -1) + P(0, -1, -1))
              + f["b2"][s] * (P(1, 0, 1) - P(-1, 0, 1) - P(1, 0, -1) + P(-1, 0, -1))
              + f["c0"][s] * P(-1, 0, 0) + f["c1"][s] * P(0, -1, 0) + f["c2"][s] * P(0, 0, -1)
              + f["wrk1"][s])
        ss = (s0 * f["a3"][s] - f["p"][s]) * f["bnd"][s]
        f["gs"][s] = ss * ss
        f["wrk2"][s] = f["p"][s] + omega * ss
        for v in f["gs"][s].reshape(-1):
            gosa = np.float32(gosa + v)
        f["p"][s] = f["wrk2"][s]
    return f, gosa


def test_himeno_oracle_matches_direct_formula():
    g = golden("himeno_17x9x33")
    prog = Program(g["doc"])
    st = _state(g)
    out = CProgram(g["doc"]).run(st)
    f, gosa = _himeno_numpy(st, prog, (17, 9, 33), nn=2)
    assert np.array_equal(out[prog.var_by_name["p"].id].reshape(17, 9, 33), f["p"])
    assert np.array_equal(out[prog.var_by_name["gs"].id].reshape(17, 9, 33), f["gs"])
    assert out[prog.var_by_name["gosa"].id][0] == gosa


def test_external_semantics():
    rng = np.random.default_rng(3)
    a = rng.random(6 * 4).astype(np.float32)
    b = rng.random(4 * 5).astype(np.float32)
    np.testing.assert_allclose(gemm(a, b, 6, 5, 4, np.float32).reshape(6, 5),
                               a.reshape(6, 4) @ b.reshape(4, 5), rtol=1e-6)
    x = rng.random(2 * 8 * 8).astype(np.float32)
    z = x.reshape(8, 8, 2)
    want = np.fft.fft2(z[..., 0].astype(np.float64) + 1j * z[..., 1].astype(np.float64))
    y = fft2d(x, 8, np.float64).reshape(8, 8, 2)
    np.testing.assert_allclose(y[..., 0] + 1j * y[..., 1], want, rtol=1e-12, atol=1e-12)
