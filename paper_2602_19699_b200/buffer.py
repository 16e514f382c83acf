"""Device-resident replay ring (reference `trajrl.buffer`, buffer.py:85-168).

Columns live in HBM in the compute precision; `push_many` appends with FIFO
eviction (buffer.py:108-130) through `cacto_ring_push`, `sample_minibatch`
draws indices from the caller's NumPy Generator -- the exact reference stream
(buffer.py:136) -- and gathers rows on device (`cacto_gather`).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import abi_dtype, device, to_device, torch_dtype


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
