#!/usr/bin/env python
"""Sobolev critic training sweep (batch 4k-1M x hidden
64-512): one critic update = fused gather + target forward + Sobolev loss with
double backprop + fold + Adam + Polyak, timed with CUDA events on the launching
stream.  Hidden 64 runs the fused SIMT kernel; > 64 the layer-wise tcgen05 path.

Beside it: the same update written with PyTorch autograd (create_graph double
backprop, fp32, cuBLAS) on the same GPU -- the library baseline a user would
otherwise write.  Prints one JSON line per cell.

  python profiles/critic_sweep.py [--hidden 64,128,256,512] [--batch 4096,65536,262144,1048576]
"""

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2602_19699_b200 import _lib, specs  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets  # noqa: E402
from paper_2602_19699_b200.buffer import ReplayBuffer, SampleBatch  # noqa: E402
from paper_2602_19699_b200.device import DeviceNet, set_precision  # noqa: E402


def flops_per_sample(H, d, nh=3):
    # 7 passes over every dense layer (target fwd, fwd, sweep, rbar, g^T u, zbar^T a, abar)
    hh = (nh - 1) * H * H
    return 2 * (7 * hh + 6 * d * H) + 2 * 8 * H


def timed(fn, K, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(K):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / K


def torch_critic_step(Ws, bs, opt, xa, xk, vbar, vbarx, center, half, k_s, tgt):
    def fwd(params, x):
        h = (x - center) / half
        for i, (W, b) in enumerate(params):
            h = h @ W.t() + b
            if i < len(params) - 1:
                h = torch.nn.functional.elu(h)
        return h[:, 0]

    opt.zero_grad(set_to_none=True)
    with torch.no_grad():
        vn = fwd(tgt, xk)
    x = xa.detach().requires_grad_(True)
    v = fwd(list(zip(Ws, bs)), x)
    (g,) = torch.autograd.grad(v.sum(), x, create_graph=True)
    n = vbarx.shape[1]
    y = vbar + vn
    loss = ((y - v) ** 2).mean() + k_s * ((vbarx - g[:, :n]) ** 2).sum(1).mean()
    loss.backward()
    opt.step()
    with torch.no_grad():
        for (tw, tb), w, b in zip(tgt, Ws, bs):
            tw.lerp_(w, 0.005)
            tb.lerp_(b, 0.005)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hidden", default="64,128,256,512")
    ap.add_argument("--batch", default="4096,65536,262144,1048576")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--no-torch", action="store_true")
    ap.add_argument("--timeline", action="store_true",
                    help="print the per-layer clock64 timeline of the last update (CACTO_CTC_TIMELINE=1 build)")
    args = ap.parse_args()
    set_precision("fp32")
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    spec, _ = specs.config("manipulator3")
    d = spec.n + 1
    c, h = specs.normalisation(spec)
    rng = np.random.default_rng(0)
    rows = 1 << 20
    lo, hi = specs.region_box(spec)
    xa = np.concatenate([rng.uniform(size=(rows, spec.n)) * (hi - lo) + lo, rng.integers(0, spec.t_max, (rows, 1))], 1)
    xk = np.concatenate([rng.uniform(size=(rows, spec.n)) * (hi - lo) + lo,
                         rng.integers(1, spec.t_max + 1, (rows, 1))], 1)
    buf = ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=rows)
    buf.push_many(SampleBatch(xa, rng.normal(size=(rows, spec.m)), rng.normal(size=rows),
                              rng.normal(size=(rows, spec.n)), xk, spec.t_max))
    L = _lib.load()
    for H in [int(x) for x in args.hidden.split(",")]:
        critic = B_nets.init_mlp([d, H, H, H, 1], rng, in_center=c, in_half=h)
        net, tgt = DeviceNet(critic), DeviceNet(critic)
        m, v = torch.zeros_like(net.params), torch.zeros_like(net.params)
        for B in [int(x) for x in args.batch.split(",")]:
            idx = torch.as_tensor(rng.integers(0, rows, B), device=dev)
            desc = buf.ring_desc(idx, rows=B)
            nbytes = L.cacto_loss_workspace_bytes(net.desc, B)
            ws = torch.empty(nbytes, device=dev, dtype=torch.uint8)
            npart = ctypes.c_int32(0)
            step = [0]

            def one():
                _lib.call("cacto_critic_loss", net.desc, tgt.desc, desc, 1.0, 1, ws.data_ptr(), nbytes, npart, stream)
                _lib.call("cacto_reduce_adam", net.desc.dtype, ws.data_ptr(), npart.value, net.count,
                          net.params.data_ptr(), m.data_ptr(), v.data_ptr(), step[0], 1e-3, 0.9, 0.999, 1e-8,
                          tgt.params.data_ptr(), 0.005, None, None, stream)
                step[0] += 1

            ms = timed(one, args.steps, torch.cuda.current_stream())
            f = flops_per_sample(H, d)
            line = {"hidden": H, "batch": B,
                    "path": "tcgen05 layer-wise" if H > 64 else ("tcgen05 fused (critic_tc)" if B >= 8192 else "simt fused"),
                    "ms_per_update": ms, "samples_per_s": B / (ms * 1e-3),
                    "tflops": f * B / (ms * 1e-3) / 1e12, "flops_per_sample": f,
                    "workspace_mb": nbytes / 2 ** 20}
            del ws
            if not args.no_torch:
                g = torch.Generator(device="cpu").manual_seed(1)
                sizes = [d, H, H, H, 1]
                Ws = [torch.randn(sizes[i + 1], sizes[i], generator=g).mul_(0.1).to(dev).requires_grad_()
                      for i in range(4)]
                bs = [torch.zeros(sizes[i + 1], device=dev, requires_grad=True) for i in range(4)]
                tg = [(W.detach().clone(), b.detach().clone()) for W, b in zip(Ws, bs)]
                opt = torch.optim.Adam(Ws + bs, lr=1e-3)
                ii = idx
                tx = torch.as_tensor(xa[:1], device=dev, dtype=torch.float32)  # noqa: F841
                cols = buf.cols
                xa_d, xk_d = cols[0][ii].float(), cols[4][ii].float()
                vb, vbx = cols[2][ii].float(), cols[3][ii].float()
                cc = torch.as_tensor(c, device=dev, dtype=torch.float32)
                hh = torch.as_tensor(h, device=dev, dtype=torch.float32)
                torch.backends.cuda.matmul.allow_tf32 = False
                try:
                    tms = timed(lambda: torch_critic_step(Ws, bs, opt, xa_d, xk_d, vb, vbx, cc, hh, 1.0, tg),
                                args.steps, torch.cuda.current_stream())
                    line["torch_autograd_ms"] = tms
                    line["speedup_vs_torch"] = tms / ms
                except torch.OutOfMemoryError:
                    line["torch_autograd_ms"] = None
                del Ws, bs, tg, opt, xa_d, xk_d, vb, vbx
                torch.cuda.empty_cache()
            print(json.dumps(line), flush=True)
    if args.timeline:
        buf = (ctypes.c_ulonglong * 48)()
        assert _lib.load().cacto_debug_ctc_timeline(buf) == 0
        t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(12, 4)
        t = t - t[0, 0]
        # per critic-chain layer: hand-off seen by the MMA warp, MMAs issued, completion
        # seen by epilogue warp 0, next hand-off by warp 0
        rows = [dict(layer=i, mma_seen=int(t[i, 0]), issued=int(t[i, 1] - t[i, 0]),
                     done_after_issue=int(t[i, 2] - t[i, 1]),
                     epilogue=int(t[i + 1, 3] - t[i, 2]) if i + 1 < 12 else None,
                     handoff_to_mma=int(t[i + 1, 0] - t[i + 1, 3]) if i + 1 < 12 else None) for i in range(12)]
        print(json.dumps({"critic_tc_timeline_cycles": rows, "tile_cycles": int(t[11, 2] - t[0, 0])}), flush=True)


if __name__ == "__main__":
    main()
