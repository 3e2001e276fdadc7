"""GPU parity of the sm_100a building blocks (run under gpurun).

* tcgen05 GEMM (all four operand-major combinations, ragged M/N/K, several
  UMMA N) vs a torch fp32 matmul of the same bf16 inputs; tolerance
  |d| <= 1e-3 * sqrt(K) * max|ref| (fp32 accumulation-order noise only).
* synthetic data generator vs oracle/rng.py: bit-exact pixels and labels.
"""

import numpy as np
import pytest
import torch

from oracle import rng
from paper_2410_22254_b200 import runtime as rt

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_tcgen05_gemm_matches_torch(a_mn, b_mn, bn):
    torch.manual_seed(1234 + bn + 2 * a_mn + b_mn)
    batch, M, N, K = 2, 200, 192, 136
    A = torch.randn(batch, M, K, device="cuda").bfloat16()
    B = torch.randn(batch, N, K, device="cuda").bfloat16()
    a_arg = A.transpose(1, 2).contiguous() if a_mn else A.contiguous()
    b_arg = B.transpose(1, 2).contiguous() if b_mn else B.contiguous()
    C = torch.full((batch, M, N), float("nan"), device="cuda")
    rt.selftest_gemm(a_mn, b_mn, bn, a_arg, b_arg, C, batch, M, N, K)
    torch.cuda.synchronize()
    ref = torch.bmm(A.float(), B.float().transpose(1, 2))
    err = (C - ref).abs().max().item()
    assert err <= 1e-3 * K**0.5 * ref.abs().max().item(), err


def test_tcgen05_gemm_large_k():
    torch.manual_seed(7)
    batch, M, N, K = 3, 384, 128, 2048
    A = torch.randn(batch, M, K, device="cuda").bfloat16()
    B = torch.randn(batch, N, K, device="cuda").bfloat16()
    C = torch.zeros(batch, M, N, device="cuda")
    rt.selftest_gemm(False, False, 128, A, B, C, batch, M, N, K)
    torch.cuda.synchronize()
    ref = torch.bmm(A.float(), B.float().transpose(1, 2))
    assert (C - ref).abs().max().item() <= 1e-3 * K**0.5 * ref.abs().max().item()


@pytest.mark.parametrize("seed,step", [(0, 0), (3, 17), (2**40 + 5, 123456)])
def test_datagen_bit_exact(seed, step):
    batch = 64
    px = torch.zeros(batch, 784, dtype=torch.uint8, device="cuda")
    lb = torch.zeros(batch, dtype=torch.int32, device="cuda")
    rt.selftest_datagen(seed, step, batch, px, lb)
    torch.cuda.synchronize()
    ref_px, ref_lb = rng.batch(seed, step, batch)
    assert np.array_equal(px.cpu().numpy(), ref_px)
    assert np.array_equal(lb.cpu().numpy(), ref_lb)


@pytest.mark.parametrize("kind", [rt.OPT_ADAM, rt.OPT_ADAMW, rt.OPT_SGD])
def test_optimizer_fastpath_is_bit_identical_to_library_sqrt_div(kind):
    """The straight-line sqrt / div of the packed optimizer reproduce the
    library __fsqrt_rn / __fdiv_rn update bit for bit on 2^28 random states
    (exponents over the whole float range, zeros, denormals, both signs)."""
    assert rt.selftest_optimizer(kind, 20251017 + kind, 1 << 28) == 0
