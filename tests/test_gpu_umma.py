"""tcgen05 building blocks (umma.cuh) against torch: descriptor / instruction
encodings, TMEM allocation and loads.  kind::tf32 keeps 10 mantissa bits of
each operand (truncated), so the bar is |D - A B^T| <= 2^-9 * sum|a||b|."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [8, 16, 64, 256])
def test_umma_tf32_matches_torch(cuda, K):
    torch = cuda
    from paper_1702_08159_b200 import _native as nat
    g = torch.Generator(device="cuda").manual_seed(K)
    A = torch.randn((128, K), generator=g, device="cuda")
    B = torch.randn((16, K), generator=g, device="cuda")
    D = torch.full((128, 16), float("nan"), device="cuda")
    nat.call("mck_diag_umma_tf32", A.data_ptr(), B.data_ptr(), D.data_ptr(), K,
             nat.stream_handle(D.device))
    want = A.double() @ B.double().T
    bound = 2.0 ** -9 * (A.abs().double() @ B.abs().double().T)
    assert torch.isfinite(D).all()
    assert bool(((D.double() - want).abs() <= bound + 1e-6).all())
