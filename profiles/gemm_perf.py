"""Throughput of cacto_gemm_tf32 (3xTF32 / 1xTF32) vs torch.matmul (cuBLAS fp32 / TF32)
on the dense-layer GEMM shapes of the H=512 critic at B=65536."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2602_19699_b200 import _lib

st = torch.cuda.current_stream().cuda_stream


def time_it(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for (M, N, K, name) in [(65536, 512, 512, "z = a W^T"), (512, 512, 65536, "gW = g^T a"), (65536, 128, 128, "H=128")]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    if name.startswith("gW"):  # weight gradient: both operands MN-major (g [B][H], a [B][H])
        At, Bt = torch.randn(K, M, device="cuda"), torch.randn(K, N, device="cuda")
        fl = 2.0 * M * N * K
        D = torch.empty(M, N, device="cuda")
        wsb = _lib.load().cacto_gemm_workspace_bytes(M, N, K)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        for passes in (3, 1):
            ms = time_it(lambda: _lib.call("cacto_gemm_tf32", M, N, K, At.data_ptr(), 1, M, Bt.data_ptr(), 1, N,
                                           D.data_ptr(), N, 0, 1.0, passes, ws.data_ptr(), wsb, st))
            print(f"{name:12s} {M}x{N}x{K} (MN-major) cacto {passes}xTF32: {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s")
        torch.backends.cuda.matmul.allow_tf32 = False
        ms = time_it(lambda: torch.matmul(At.t(), Bt, out=D))
        print(f"{name:12s} torch fp32 (cuBLAS): {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s")
        continue
    D = torch.empty(M, N, device="cuda")
    wsb = _lib.load().cacto_gemm_workspace_bytes(M, N, K)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    fl = 2.0 * M * N * K
    for passes in (3, 1):
        ms = time_it(lambda: _lib.call("cacto_gemm_tf32", M, N, K, A.data_ptr(), K, 1, B.data_ptr(), K, 1,
                                       D.data_ptr(), N, 0, 1.0, passes, ws.data_ptr(), wsb, st))
        print(f"{name:12s} {M}x{N}x{K} cacto {passes}xTF32: {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s")
    torch.backends.cuda.matmul.allow_tf32 = False
    ms = time_it(lambda: torch.matmul(A, B.t(), out=D))
    print(f"{name:12s} torch fp32 (cuBLAS): {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s")
    torch.backends.cuda.matmul.allow_tf32 = True
    ms = time_it(lambda: torch.matmul(A, B.t(), out=D))
    print(f"{name:12s} torch tf32 (cuBLAS): {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s")
