import torch, sys
sys.path.insert(0, '.')
from paper_2602_19699_b200 import _lib
st = torch.cuda.current_stream().cuda_stream
M, N, K = 128, 64, 32
# A(m,k) one-hot: 1 if k == m % 32; stored MN-major as At[k][m]
A = torch.zeros(M, K)
for m in range(M): A[m, m % K] = 1.0
B = torch.zeros(N, K)
for n in range(N):
    for k in range(K): B[n, k] = k * 1000 + n
At = A.t().contiguous().cuda(); Bd = B.cuda()
D = torch.zeros(M, N, device='cuda')
ws = torch.empty(16, dtype=torch.uint8, device='cuda')
_lib.call("cacto_gemm_tf32", M, N, K, At.data_ptr(), 1, M, Bd.data_ptr(), K, 1, D.data_ptr(), N, 0, 1.0, 1, ws.data_ptr(), 0, st)
torch.cuda.synchronize()
Dc = D.cpu()
# expected D[m][n] = (m%32)*1000 + n ; infer which k the hardware used for row m (col 0)
got_k = (Dc[:, 0] / 1000).round().int().tolist()
print("row->k (expect m%32):", got_k[:40])
print("row 0 cols:", Dc[0, :8].tolist())
# B MN-major probe: A K-major one-hot, B stored Bt[k][n]
Ak = A.cuda()
Bt = B.t().contiguous().cuda()
D.zero_()
_lib.call("cacto_gemm_tf32", M, N, K, Ak.data_ptr(), K, 1, Bt.data_ptr(), 1, N, D.data_ptr(), N, 0, 1.0, 1, ws.data_ptr(), 0, st)
torch.cuda.synchronize()
Dc = D.cpu()
print("Bmn row1:", Dc[1, :12].tolist())
print("Bmn row5:", Dc[5, :12].tolist())
