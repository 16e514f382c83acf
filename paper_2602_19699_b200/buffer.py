"""Device-resident replay ring (reference `trajrl.buffer`, buffer.py:85-168).

Columns live in HBM in the compute precision; `push_many` appends with FIFO
eviction (buffer.py:108-130) through `cacto_ring_push`, `sample_minibatch`
draws indices from the caller's NumPy Generator -- the exact reference stream
(buffer.py:136) -- and gathers rows on device (`cacto_gather`).

The replay producer `push_kstep(results, K)` turns a batch of iLQR solutions
into their k-step training rows on the device and appends them in one launch
(`cacto_kstep_push`): the drop-in for the trainer's
`for res in results: buffer.push_many(kstep_targets(res, K))` (trainer.py:200-201,
ilqr.py:358-407).  `dump` / `restore` read and write the reference's TRLB
binary format (buffer.py:17-18, 142-168).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _lib
from .device import abi_dtype, device, to_device, torch_dtype

_MAGIC = b"TRLB"
_HEADER = struct.Struct("<4s16sIIIQ")  # magic, model name, n, m, K, count (buffer.py:17-18)


class SampleBatch:
    """Columnar batch (buffer.py:39-82).  Arrays are float64 NumPy on the host
    view; `device_cols` optionally keeps the device tensors."""

    def __init__(self, xa, u, v_bar, v_bar_x, xa_plus_k, t_max: int, device_cols=None):
        self.xa = np.asarray(xa, dtype=float)
        self.u = np.asarray(u, dtype=float)
        self.v_bar = np.asarray(v_bar, dtype=float)
        self.v_bar_x = np.asarray(v_bar_x, dtype=float)
        self.xa_plus_k = np.asarray(xa_plus_k, dtype=float)
        self.t_max = int(t_max)
        self.device_cols = device_cols

    def __len__(self):
        return self.xa.shape[0]

    @property
    def n(self):
        return self.xa.shape[1] - 1


def _columns(samples, t_max):
    if hasattr(samples, "xa") and hasattr(samples, "v_bar"):
        return (np.asarray(samples.xa, float), np.asarray(samples.u, float), np.asarray(samples.v_bar, float),
                np.asarray(samples.v_bar_x, float), np.asarray(samples.xa_plus_k, float))
    samples = list(samples)
    if not samples:
        return None
    return (np.stack([s.state.augmented for s in samples]), np.stack([np.asarray(s.u, float) for s in samples]),
            np.array([float(s.v_bar) for s in samples]), np.stack([np.asarray(s.v_bar_x, float) for s in samples]),
            np.stack([s.state_plus_k.augmented for s in samples]))


class ReplayBuffer:
    """FIFO ring with uniform with-replacement sampling, resident in HBM."""

    def __init__(self, n: int, m: int, t_max: int, capacity: int = 2 ** 20, model_name: str = "",
                 k_lookahead: int = 0, precision=None):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.n, self.m, self.t_max = n, m, t_max
        self.capacity = capacity
        self.model_name = model_name
        self.k_lookahead = k_lookahead
        self.precision = precision
        dev = device()
        dt = torch_dtype(precision)
        self.cols = [torch.zeros((capacity, n + 1), device=dev, dtype=dt),
                     torch.zeros((capacity, m), device=dev, dtype=dt),
                     torch.zeros((capacity,), device=dev, dtype=dt),
                     torch.zeros((capacity, n), device=dev, dtype=dt),
                     torch.zeros((capacity, n + 1), device=dev, dtype=dt)]
        self._size = 0
        self._cursor = 0

    def __len__(self):
        return self._size

    def _desc(self, cols, rows, idx=None):
        d = _lib.CactoBatch()
        d.dtype = abi_dtype(self.precision)
        d.n, d.m, d.t_max = self.n, self.m, self.t_max
        d.rows = int(rows)
        d.denom = 0
        d.idx = None if idx is None else idx.data_ptr()
        d.xa, d.u, d.v_bar, d.v_bar_x, d.xa_plus_k = [c.data_ptr() for c in cols]
        return d

    def ring_desc(self, idx=None, rows=None):
        """cacto_batch_t over the ring columns (fused-gather view for the losses)."""
        return self._desc(self.cols, self._size if rows is None else rows, idx)

    def push_many(self, samples) -> int:
        """buffer.py:108-130."""
        cols = _columns(samples, self.t_max)
        if cols is None:
            return 0
        count = cols[0].shape[0]
        if count == 0:
            return 0
        first = max(0, count - self.capacity)
        kept = count - first
        src = [to_device(c[first:], self.precision) for c in cols]
        stream = torch.cuda.current_stream().cuda_stream
        _lib.call("cacto_ring_push", self._desc(src, kept), *[c.data_ptr() for c in self.cols],
                  self.capacity, self._cursor, stream)
        self._cursor = int((self._cursor + kept) % self.capacity)
        self._size = min(self._size + kept, self.capacity)
        return kept

    def push_kstep(self, results, K: int) -> int:
        """`for res in results: self.push_many(kstep_targets(res, K))` (trainer.py:200-201)
        as one H2D copy of the solutions and one `cacto_kstep_push` launch.  Rows are
        bit-identical to the reference's (fp64 ring) or to their fp32 rounding.
        Raises ValueError like the reference for K < 1 and for a non-finite v_bar
        (TOSample, buffer.py:33-35).  On the latter the size / cursor do not move,
        but the slots this push targeted have been overwritten (the reference
        raises part-way through the batch, after pushing the earlier solutions)."""
        if K < 1:
            raise ValueError("K must be >= 1")
        sols = _solutions_host(results)
        if sols is None:
            return 0
        offsets, t0, X, U, sc, vb, vbx = sols
        rows = int(offsets[-1])
        first = max(0, rows - self.capacity)
        kept = rows - first
        dev = self.cols[0].device
        # one pinned staging block -> one H2D copy
        parts = [offsets.astype(np.int64).view(np.float64), X.ravel(), U.ravel(), sc, vb, vbx.ravel()]
        host = torch.from_numpy(np.concatenate(parts)).pin_memory()
        flat = host.to(dev, non_blocking=True)
        t0_d = torch.as_tensor(t0, dtype=torch.int32).to(dev)
        views, o = [], 0
        for p in parts:
            views.append(flat[o:o + p.size])
            o += p.size
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        d = _lib.CactoSolutions()
        d.n, d.m, d.count, d.rows = X.shape[1], U.shape[1], len(t0), rows
        d.offsets, d.t0 = views[0].data_ptr(), t0_d.data_ptr()
        d.X, d.U, d.step_costs, d.v_bar, d.v_bar_x = [v.data_ptr() for v in views[1:]]
        if d.n != self.n or d.m != self.m:
            raise ValueError("solution dimensions do not match the buffer")
        stream = torch.cuda.current_stream().cuda_stream
        _lib.call("cacto_kstep_push", d, int(K), abi_dtype(self.precision), *[c.data_ptr() for c in self.cols],
                  self.capacity, self._cursor, first, bad.data_ptr(), stream)
        if int(bad.item()):
            raise ValueError("v_bar must be finite")
        self._cursor = int((self._cursor + kept) % self.capacity)
        self._size = min(self._size + kept, self.capacity)
        return kept

    def dump(self, path):
        """TRLB dump, oldest first (buffer.py:142-152): fixed-width little-endian float64 records."""
        order = (torch.arange(self._size, device=self.cols[0].device) + (self._cursor - self._size)) % self.capacity
        rec = torch.cat([self.cols[0][order], self.cols[1][order], self.cols[2][order, None], self.cols[3][order],
                         self.cols[4][order]], dim=1).to("cpu", torch.float64).numpy()
        name = self.model_name.encode()[:16].ljust(16, b"\0")
        with open(path, "wb") as fh:
            fh.write(_HEADER.pack(_MAGIC, name, self.n, self.m, self.k_lookahead, self._size))
            fh.write(np.ascontiguousarray(rec, dtype="<f8").tobytes())

    @classmethod
    def restore(cls, path, capacity: int = 2 ** 20, t_max: int = 0, precision=None) -> "ReplayBuffer":
        """buffer.py:153-168."""
        with open(path, "rb") as fh:
            head = fh.read(_HEADER.size)
            if len(head) < _HEADER.size or head[:4] != _MAGIC:
                raise ValueError(f"not a buffer dump: {path}")
            _, name, n, m, k, count = _HEADER.unpack(head)
            width = (n + 1) + m + 1 + n + (n + 1)
            data = np.frombuffer(fh.read(count * width * 8), dtype="<f8")
        rec = data.reshape(count, width).astype(float)
        buf = cls(n, m, t_max=t_max, capacity=capacity, model_name=name.rstrip(b"\0").decode(), k_lookahead=k,
                  precision=precision)
        cols = np.split(rec, np.cumsum([n + 1, m, 1, n]), axis=1)
        buf.push_many(SampleBatch(cols[0], cols[1], cols[2][:, 0], cols[3], cols[4], t_max))
        return buf

    def draw_indices(self, batch_size: int, rng: np.random.Generator) -> np.ndarray:
        """buffer.py:134-136 -- the reference's own index stream."""
        if self._size == 0:
            raise ValueError("cannot sample from an empty buffer")
        return rng.integers(0, self._size, size=batch_size)

    def gather_device(self, idx: torch.Tensor):
        """K4: coalesced indexed row gather -> 5 device columns."""
        B = idx.shape[0]
        dev = idx.device
        dt = self.cols[0].dtype
        out = [torch.empty((B, self.n + 1), device=dev, dtype=dt), torch.empty((B, self.m), device=dev, dtype=dt),
               torch.empty((B,), device=dev, dtype=dt), torch.empty((B, self.n), device=dev, dtype=dt),
               torch.empty((B, self.n + 1), device=dev, dtype=dt)]
        stream = torch.cuda.current_stream().cuda_stream
        _lib.call("cacto_gather", self._desc(self.cols, B, idx), *[o.data_ptr() for o in out], stream)
        return out

    def sample_minibatch(self, batch_size: int, rng: np.random.Generator) -> SampleBatch:
        """buffer.py:132-138."""
        idx = self.draw_indices(batch_size, rng)
        out = self.gather_device(torch.as_tensor(idx, dtype=torch.int64).to(device()))
        host = [o.to("cpu", torch.float64).numpy() for o in out]
        return SampleBatch(*host, self.t_max, device_cols=out)


def _solutions_host(results):
    """Concatenate solutions (reference `SolveResult`: .traj.X/.U/.step_costs/.t0,
    .V_bar, .V_bar_x, ilqr.py:59-94) row-wise; U gets one padding row each."""
    results = list(results)
    if not results:
        return None
    offs = np.zeros(len(results) + 1, dtype=np.int64)
    Xs, Us, SCs, VBs, VBXs, t0 = [], [], [], [], [], []
    for i, r in enumerate(results):
        tr = r.traj
        X = np.asarray(tr.X, float)
        U = np.asarray(tr.U, float)
        T = U.shape[0]
        offs[i + 1] = offs[i] + T + 1
        Xs.append(X)
        Us.append(np.concatenate([U, np.zeros((1, U.shape[1]))]))
        SCs.append(np.asarray(tr.step_costs, float))
        VBs.append(np.asarray(r.V_bar, float))
        VBXs.append(np.asarray(r.V_bar_x, float).reshape(T + 1, X.shape[1]))
        t0.append(int(tr.t0))
    return (offs, np.array(t0, dtype=np.int32), np.concatenate(Xs), np.concatenate(Us), np.concatenate(SCs),
            np.concatenate(VBs), np.concatenate(VBXs))


def kstep_targets(result, K: int, critic_eval=None) -> SampleBatch:
    """`ilqr.kstep_targets` (ilqr.py:358-407) for one solution, computed on the
    device, returned as a SampleBatch (accepted by `push_many` wherever the
    reference's list[TOSample] is).  The critic-hook variant (ilqr.py:375-401)
    is not on the trainer's path (trainer.py:201 passes none) and is rejected."""
    if critic_eval is not None:
        raise NotImplementedError("kstep_targets with a critic hook stays on the reference's CPU solver")
    if K < 1:
        raise ValueError("K must be >= 1")
    T = np.asarray(result.traj.U).shape[0]
    X = np.asarray(result.traj.X)
    tmp = ReplayBuffer(X.shape[1], np.asarray(result.traj.U).shape[1], 0, capacity=T + 1, precision="fp64")
    tmp.push_kstep([result], K)
    host = [c.to("cpu", torch.float64).numpy() for c in tmp.cols]
    return SampleBatch(*host, 0, device_cols=tmp.cols)
