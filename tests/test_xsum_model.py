"""CPU check of the exact in-order sum's arithmetic (tests/_xsum_model.py, a
plain-Python model of csrc/b2o_xsum.cu): applying run summaries -- units per
binade, the round-half-even parity rule, two-variant summaries, merges, the
mirrored negative case -- reproduces the sequential fp32 / fp64 loop bit for
bit, and the summaries really carry the walk (ties included)."""

import numpy as np
import pytest

from _xsum_model import exact_sum, merge, summarise


def seq(xs, s0, dtype):
    s = dtype(s0)
    for x in xs:
        s = dtype(s + x)
    return s


def _data(kind, n, dtype, seed):
    r = np.random.default_rng(seed)
    if kind == "uniform":
        return r.random(n).astype(dtype)
    if kind == "mixed":
        return r.standard_normal(n).astype(dtype)
    if kind == "dyadic":  # quantised: ties at every coarse binade
        return (r.integers(0, 64, n) * 2.0 ** -10).astype(dtype)
    if kind == "constant":
        return np.full(n, 0.1, dtype)
    if kind == "wide":
        return (r.random(n) * 10.0 ** r.integers(-8, 8, n)).astype(dtype)
    raise ValueError(kind)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("kind,s0", [("uniform", 0.0), ("mixed", 5.0), ("dyadic", 1024.0), ("constant", 0.0),
                                     ("wide", -3.0)])
def test_model_walk_is_the_sequential_sum(dtype, kind, s0):
    xs = _data(kind, 3000, dtype, 7)
    stats = {}
    got = exact_sum(xs, s0, dtype, stats=stats)
    want = seq(xs, s0, dtype)
    assert np.asarray(got, dtype).tobytes() == np.asarray(want, dtype).tobytes(), (kind, got, want)
    if kind in ("uniform", "dyadic", "constant"):
        assert stats["fast"] > stats["slow"], stats  # the summaries carry the walk


def test_merge_is_associative_and_matches_the_whole_run():
    xs = _data("dyadic", 96, np.float32, 3)
    e = 10  # s in [1024, 2048)
    a, b, c = summarise(xs[:32], e, np.float32), summarise(xs[32:64], e, np.float32), summarise(xs[64:], e, np.float32)
    whole = summarise(xs, e, np.float32)
    assert merge(merge(a, b), c) == merge(a, merge(b, c)) == whole


def test_tie_depends_on_parity():
    # u = 2^(10-23) at s in [1024, 2048): x = 1.5 u is a tie -> +1 or +2
    u = 2.0 ** -13
    x = np.float32(1.5 * u)
    summ = summarise(np.array([x], np.float32), 10, np.float32)
    assert summ[0][0] == 2 and summ[1][0] == 1  # even start rounds up to even, odd start down
    for s0 in (np.float32(1024.0), np.float32(1024.0) + np.float32(u)):
        assert exact_sum(np.array([x], np.float32), s0, np.float32) == np.float32(s0 + x)
