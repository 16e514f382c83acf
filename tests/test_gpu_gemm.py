"""tcgen05 GEMM (csrc/gemm_tc.cu) against a float64 reference: every operand
layout the dense-layer GEMMs use, partial tiles, accumulate mode.
Tolerance: 3xTF32 max |err| <= 2e-5 * sum_k |a||b| (fp32-level); 1xTF32 <= 2e-3."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2602_19699_b200 import _lib  # noqa: E402


def run(M, N, K, a_kmajor, b_kmajor, passes, accumulate=False, alpha=1.0, seed=0):
    # TMA needs 16-byte row strides: K-major operands need K % 4 == 0, MN-major M/N % 4 == 0
    g = torch.Generator(device="cpu").manual_seed(seed)
    A = torch.randn(M, K, generator=g, dtype=torch.float64)
    B = torch.randn(N, K, generator=g, dtype=torch.float64)
    D0 = torch.randn(M, N, generator=g, dtype=torch.float64)
    Ad = (A if a_kmajor else A.t().contiguous()).float().cuda()
    Bd = (B if b_kmajor else B.t().contiguous()).float().cuda()
    sam, sak = (K, 1) if a_kmajor else (1, M)
    sbn, sbk = (K, 1) if b_kmajor else (1, N)
    D = D0.float().cuda()
    wsb = _lib.load().cacto_gemm_workspace_bytes(M, N, K)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    _lib.call("cacto_gemm_tf32", M, N, K, Ad.data_ptr(), sam, sak, Bd.data_ptr(), sbn, sbk, D.data_ptr(), N,
              int(accumulate), float(alpha), passes, ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    Af, Bf = A.float().double(), B.float().double()
    ref = alpha * Af @ Bf.t() + (D0.float().double() if accumulate else 0.0)
    scale = alpha * (Af.abs() @ Bf.abs().t()) + 1e-30
    return float(((D.double().cpu() - ref).abs() / scale).max())


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 128, 64), (300, 200, 100), (64, 64, 512),
                                   (1000, 512, 512), (128, 8, 64), (5, 300, 36), (512, 512, 20000),
                                   (300, 96, 4000),
                                   # 96-wide tiles (65..96 columns), incl. the critic's K = 2B reduction
                                   # shape with split-K over every SM; 256-wide tiles (N >= 512)
                                   (64, 68, 131072), (200, 72, 3000), (130, 768, 96)])
@pytest.mark.parametrize("a_k,b_k", [(True, True), (False, True), (True, False), (False, False)])
def test_gemm_3xtf32(M, N, K, a_k, b_k):
    if (not a_k and M % 4) or (not b_k and N % 4):
        pytest.skip("MN-major operand needs a 16-byte row stride")
    assert run(M, N, K, a_k, b_k, 3) < 2e-5


@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (300, 200, 100)])
def test_gemm_1xtf32(M, N, K):
    assert run(M, N, K, True, True, 1) < 2e-3


def test_gemm_accumulate_alpha():
    assert run(200, 132, 68, True, False, 3, accumulate=True, alpha=-0.5) < 2e-5
