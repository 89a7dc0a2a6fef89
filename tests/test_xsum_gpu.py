"""The exact sequential fp32 sum on the GPU (csrc/b2o_xsum.cu) against the
sequential loop itself (numpy's add.accumulate in float32 is the loop
``s = s + x[i]`` with one fp32 rounding per step): bit-identical on every
input family the binade-segmented scan has a special case for."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def seq_sum(x: np.ndarray, s0: float) -> np.float32:
    acc = np.add.accumulate(np.concatenate([np.array([s0], np.float32), x.astype(np.float32)]), dtype=np.float32)
    return acc[-1]


def gpu_sum(x: np.ndarray, s0: float) -> np.float32:
    from paper_2011_03602_b200.runtime import lib

    dx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib().b2o_exact_sum_f32(dx.data_ptr(), dx.numel(), float(np.float32(s0)), out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    return out.cpu().numpy()[0]


def same(a, b) -> bool:
    return np.float32(a).tobytes() == np.float32(b).tobytes() or (np.isnan(a) and np.isnan(b))


def cases():
    r = np.random.default_rng(20201106)
    yield "uniform_pos_4M", r.random(4_112_895, dtype=np.float32), 0.0
    yield "squares_like_gs", (r.standard_normal(1 << 20, dtype=np.float32) * 1e-3) ** 2, 0.0
    yield "mixed_sign", r.standard_normal(1 << 20, dtype=np.float32), 0.0
    yield "mixed_sign_s0", r.standard_normal(300_001, dtype=np.float32), -1234.5
    yield "negative", -r.random(1 << 20, dtype=np.float32), 0.0
    yield "ties_dyadic", (r.integers(0, 64, 1 << 20) * np.float32(2.0 ** -10)).astype(np.float32), 1024.0
    yield "wide_range", (r.random(1 << 19, dtype=np.float32) * 10.0 ** r.integers(-30, 30, 1 << 19)).astype(np.float32), 0.0
    yield "zeros", np.zeros(100_000, np.float32), 0.0
    yield "subnormal", np.full(70_000, np.float32(1e-40)), 0.0
    yield "cancel", np.tile(np.array([1e8, 1.0, -1e8, 3.0], np.float32), 50_000), 0.5
    yield "small_n", r.random(37, dtype=np.float32), 2.0
    yield "one", np.array([3.25], np.float32), 1.0
    yield "ragged", r.random(256 * 32 * 3 + 17, dtype=np.float32), 0.0
    x = r.random(200_000, dtype=np.float32)
    x[123_456] = np.inf
    yield "inf", x, 0.0
    x = r.random(200_000, dtype=np.float32)
    x[77] = np.nan
    yield "nan", x, 0.0


@pytest.mark.parametrize("name,x,s0", list(cases()), ids=[c[0] for c in cases()])
def test_exact_sum_matches_sequential_loop(name, x, s0):
    want = seq_sum(x, s0)
    got = gpu_sum(x, s0)
    assert same(got, want), (name, got, want)


def test_exact_sum_empty():
    assert same(gpu_sum(np.zeros(0, np.float32), 5.0), np.float32(5.0))


def test_exact_sum_differs_from_pairwise():
    """The point of the kernel: the sequential fp32 loop and a reassociated
    (pairwise / double) sum differ at this size, the kernel returns the loop."""
    x = np.random.default_rng(1).random(4_112_895, dtype=np.float32)
    want = seq_sum(x, 0.0)
    assert want != np.float32(np.sum(x, dtype=np.float64))
    assert same(gpu_sum(x, 0.0), want)


def seq_sum64(x: np.ndarray, s0: float) -> np.float64:
    return np.add.accumulate(np.concatenate([np.array([s0], np.float64), x.astype(np.float64)]),
                             dtype=np.float64)[-1]


def gpu_sum64(x: np.ndarray, s0: float) -> np.float64:
    from paper_2011_03602_b200.runtime import lib

    dx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib().b2o_exact_sum_f64(dx.data_ptr(), dx.numel(), float(s0), out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    return out.cpu().numpy()[0]


def cases64():
    r = np.random.default_rng(1106)
    yield "uniform64", r.random(2_000_003), 0.0
    yield "squares64", r.standard_normal(1 << 20) ** 2 * 1e-6, 0.0
    yield "mixed64", r.standard_normal(1 << 19), 3.0
    yield "ties64", r.integers(0, 64, 1 << 20) * 2.0 ** -10, 1024.0
    yield "wide64", r.random(1 << 18) * 10.0 ** r.integers(-200, 200, 1 << 18), 0.0
    yield "subnormal64", np.full(70_000, 1e-310), 0.0
    yield "ragged64", r.random(256 * 32 * 3 + 17), -5.0
    yield "small64", r.random(37), 2.0


@pytest.mark.parametrize("name,x,s0", list(cases64()), ids=[c[0] for c in cases64()])
def test_exact_sum_f64_matches_sequential_loop(name, x, s0):
    want = seq_sum64(x, s0)
    got = gpu_sum64(x, s0)
    assert np.float64(got).tobytes() == np.float64(want).tobytes(), (name, got, want)
