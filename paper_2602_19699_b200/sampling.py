"""Device replay of the reference's candidate sampling (envs/__init__.py:112-122).

`sample_initial_states(model, count, rng_seed)` draws
`default_rng(rng_seed).uniform(size=(count, n)) * (hi - lo) + lo`; candidate i
uses raw PCG64 outputs [i*n, i*n + n) of that stream.  `cacto_sample_states`
(K9, csrc/gather.cu) replays the same 128-bit LCG + XSL-RR output on device with
a jump-ahead per row, so candidates are generated in HBM bit-exactly, shard by
shard (first_row), and never cross PCIe.  The seed handling stays on the host:
`np.random.default_rng(seed).bit_generator.state` gives the 128-bit state and
increment (SeedSequence expansion exactly as NumPy does it).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, specs
from .device import device

_M64 = (1 << 64) - 1


def pcg64_state(rng_seed):
    """(state, inc) 128-bit integers of np.random.default_rng(rng_seed)."""
    st = np.random.default_rng(rng_seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def sample_initial_states_device(model, count: int, rng_seed, region=specs.Region.WORKSPACE, first_row: int = 0,
                                 rows: int = None, out: torch.Tensor = None) -> torch.Tensor:
    """Rows [first_row, first_row + rows) of sample_initial_states(model, count, rng_seed, region)
    as a float64 [rows, n] device tensor (bit-identical to the host draw)."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    rows = count - first_row if rows is None else int(rows)
    if first_row < 0 or rows < 0 or first_row + rows > count:
        raise ValueError("rows outside [0, count)")
    lo, hi = specs.region_box(model, region)
    dev = device()
    lo_d = torch.as_tensor(lo, dtype=torch.float64).to(dev)
    hi_d = torch.as_tensor(hi, dtype=torch.float64).to(dev)
    x = out if out is not None else torch.empty((rows, int(model.n)), device=dev, dtype=torch.float64)
    s, inc = pcg64_state(rng_seed)
    if rows:
        _lib.call("cacto_sample_states", s >> 64, s & _M64, inc >> 64, inc & _M64, first_row, rows, int(model.n),
                  lo_d.data_ptr(), hi_d.data_ptr(), x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return x
