"""NumPy stand-in for the device phases of the distributed select (test
scaffolding for the CPU gloo tests; the real phases are csrc/select.cu
cacto_dselect_*, checked on the GPU by tests/test_gpu_multiproc.py).  Same key
map (ascending key = descending score, NaN last, -0.0 == +0.0), digits, counts
and element encoding (fp32: key << 32 | global index in one int64)."""

from __future__ import annotations

import numpy as np
import torch


def keys32(s):
    s = np.asarray(s, np.float32).copy()
    s[s == 0] = 0.0
    b = s.view(np.uint32).astype(np.uint64)
    u = np.where(b & 0x80000000, ~b & 0xFFFFFFFF, b | 0x80000000)
    k = (~u) & 0xFFFFFFFF
    return np.where(np.isnan(s), np.uint64(0xFFFFFFFE), k).astype(np.uint64)


class NumpyDselect:
    passes = 4
    words = 1
    device = torch.device("cpu")

    def __init__(self, N, keep):
        self.N, self.keep = N, keep

    def begin(self):
        self.prefix, self.mask, self.need, self.lt = 0, 0, self.keep, 0

    def _keys(self, scores):
        return keys32(scores.numpy())

    def hist(self, scores, p, out):
        k = self._keys(scores)
        shift = 32 - 8 * (p + 1)
        sel = (k & np.uint64(self.mask)) == np.uint64(self.prefix)
        h = np.bincount(((k[sel] >> np.uint64(shift)) & np.uint64(255)).astype(np.int64), minlength=256)
        self.loc_hist = h
        out.copy_(torch.as_tensor(h, dtype=torch.int64))

    def digit(self, p, hist_global, counts):
        g = hist_global.numpy()
        cg, cl = np.cumsum(g), np.cumsum(self.loc_hist)
        d = int(np.searchsorted(cg, self.need))     # first digit with cumulative >= need
        before = int(cg[d - 1]) if d else 0
        self.need -= before
        shift = 32 - 8 * (p + 1)
        self.prefix |= d << shift
        self.mask |= 255 << shift
        self.lt += int(cl[d - 1]) if d else 0
        if p == self.passes - 1:
            counts.copy_(torch.tensor([self.lt, int(self.loc_hist[d]), self.need], dtype=torch.int64))

    def local(self, scores, base, n_cand, n_take, off, elems, local_sel):
        k = self._keys(scores)
        idx = np.nonzero(k <= np.uint64(self.prefix))[0]
        assert idx.size == n_cand
        e = (k[idx] << np.uint64(32)) | (idx + base).astype(np.uint64)
        e = np.sort(e)[:n_take]
        elems[off:off + n_take, 0] = torch.as_tensor(e.view(np.int64))
        local_sel[:n_take] = torch.as_tensor((e & np.uint64(0xFFFFFFFF)).astype(np.int64) - base)

    def finish(self, elems, order, top):
        e = np.sort(elems[:, 0].numpy().view(np.uint64))
        order.copy_(torch.as_tensor((e & np.uint64(0xFFFFFFFF)).astype(np.int64)))
