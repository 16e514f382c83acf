import torch, sys
sys.path.insert(0, '.')
from paper_2602_19699_b200 import _lib
out = torch.empty(148*8, device='cuda')
st = torch.cuda.current_stream().cuda_stream
for mode in (0, 1, 2):
    blocks, iters = 148*8, 4096
    flops = 2*16*8*iters*blocks*256
    for _ in range(2): _lib.call("cacto_fma_peak_mode", mode, blocks, iters, out.data_ptr(), st)
    best = 0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); _lib.call("cacto_fma_peak_mode", mode, blocks, iters, out.data_ptr(), st); b.record(); b.synchronize()
        best = max(best, flops/(a.elapsed_time(b)*1e-3)/1e12)
    print("mode", mode, "TFLOP/s", round(best, 2))
