"""Hand-written block kernels vs numpy float64: the tcgen05 3xTF32 GEMM that
replaces cublas_gemm and the shared-memory radix-2 FFT that replaces
cufft_exec (reference fixtures/sample_db.json:6,15).  Called through the C
ABI on device buffers (PyTorch only hands over the memory)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available()
    return torch


def _gemm(torch, m, n, k, seed=0, lo=0.0):
    from paper_2011_03602_b200.runtime import lib

    g = torch.Generator(device="cpu").manual_seed(seed)
    a = (torch.rand(m, k, generator=g) * (1 - lo) + lo).cuda()
    b = (torch.rand(k, n, generator=g) * (1 - lo) + lo).cuda()
    c = torch.empty(m, n, device="cuda")
    rc = lib().b2o_gemm_f32(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                            torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    ref = a.double().cpu().numpy() @ b.double().cpu().numpy()
    return c.double().cpu().numpy(), ref


@pytest.mark.parametrize("m,n,k", [(128, 256, 32), (256, 512, 96), (1024, 1024, 1024), (2560, 2560, 512),
                                   (3072, 4096, 1024), (4096, 4096, 4096)])
def test_tcgen05_gemm_matches_float64(torch_cuda, m, n, k):
    from paper_2011_03602_b200.runtime import lib

    assert lib().b2o_gemm_impl() == 1
    c, ref = _gemm(torch_cuda, m, n, k)
    normwise = np.linalg.norm(c - ref) / np.linalg.norm(ref)
    elem = np.max(np.abs(c - ref) / np.abs(ref))
    # 3xTF32 with chunked TMEM accumulation: ~1e-6 norm-wise independent of
    # K (a single TMEM accumulator reached 1e-5 at K=1024; plain TF32 ~1e-4)
    assert normwise < 3e-6, normwise
    assert elem < 1e-5, elem  # the reference's element-wise rule at fp32 (U[0,1) inputs)


def test_tcgen05_gemm_signed_inputs(torch_cuda):
    c, ref = _gemm(torch_cuda, 512, 512, 512, seed=3, lo=-1.0)
    assert np.linalg.norm(c - ref) / np.linalg.norm(ref) < 3e-6


def test_simt_fallback_for_odd_shapes(torch_cuda):
    c, ref = _gemm(torch_cuda, 48, 40, 24)
    assert np.linalg.norm(c - ref) / np.linalg.norm(ref) < 1e-6


@pytest.mark.parametrize("n", [8, 64, 256, 1024, 4096])
def test_fft2d_matches_numpy(torch_cuda, n):
    from paper_2011_03602_b200.runtime import lib

    torch = torch_cuda
    rng = np.random.default_rng(n)
    x = (rng.random(2 * n * n) * 2 - 1).astype(np.float32)
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    assert lib().b2o_fft2d_c64(dx.data_ptr(), dy.data_ptr(), n, torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    z = x.astype(np.float64).reshape(n, n, 2)
    want = np.fft.fft2(z[..., 0] + 1j * z[..., 1])
    y = dy.cpu().numpy().astype(np.float64).reshape(n, n, 2)
    got = y[..., 0] + 1j * y[..., 1]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5


def test_gemm_deterministic_with_split_tail(torch_cuda):
    """The K-split tail tiles add their two halves into a zeroed C: 0 + a + b
    equals 0 + b + a in IEEE arithmetic, so repeated runs are bit-identical."""
    from paper_2011_03602_b200.runtime import lib

    torch = torch_cuda
    g = torch.Generator(device="cpu").manual_seed(11)
    a = torch.rand(2560, 512, generator=g).cuda()
    b = torch.rand(512, 2560, generator=g).cuda()
    outs = []
    for _ in range(3):
        c = torch.full((2560, 2560), float("nan"), device="cuda")
        assert lib().b2o_gemm_f32(a.data_ptr(), b.data_ptr(), c.data_ptr(), 2560, 2560, 512,
                                  torch.cuda.current_stream().cuda_stream) == 0
        outs.append(c.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
