"""Oracle: FIFO replay ring and uniform minibatch gather (float64 columns).

Restates `ReplayBuffer.push_many` (buffer.py:108-130) and `sample_minibatch`
(buffer.py:132-138).  Test infrastructure only.
"""

from __future__ import annotations

import numpy as np

COLUMNS = ("xa", "u", "v_bar", "v_bar_x", "xa_plus_k")


class Ring:
    def __init__(self, n, m, capacity):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.n, self.m, self.capacity = n, m, capacity
        self.cols = {
            "xa": np.zeros((capacity, n + 1)), "u": np.zeros((capacity, m)),
            "v_bar": np.zeros(capacity), "v_bar_x": np.zeros((capacity, n)),
            "xa_plus_k": np.zeros((capacity, n + 1)),
        }
        self.size = 0
        self.cursor = 0

    def push_many(self, rows: dict) -> int:
        """Append in order; when more rows than capacity arrive keep the newest
        (buffer.py:118-130)."""
        count = len(rows["v_bar"])
        if count == 0:
            return 0
        first = max(0, count - self.capacity)
        kept = count - first
        slots = (self.cursor + np.arange(kept)) % self.capacity
        for name in COLUMNS:
            self.cols[name][slots] = np.asarray(rows[name])[first:]
        self.cursor = int((self.cursor + kept) % self.capacity)
        self.size = min(self.size + kept, self.capacity)
        return kept

    def draw_indices(self, batch_size, rng):
        """buffer.py:134-136: uniform with replacement from the generator."""
        if self.size == 0:
            raise ValueError("cannot sample from an empty buffer")
        return rng.integers(0, self.size, size=batch_size)

    def gather(self, idx):
        """buffer.py:137-138."""
        return {name: self.cols[name][idx] for name in COLUMNS}
