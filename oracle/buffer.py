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


# -- replay producer ---------------------------------------------

def kstep_rows(X, U, step_costs, t0, V_bar, V_bar_x, K):
    """`kstep_targets(result, K)` without a critic hook (ilqr.py:358-407), as
    columns.  Row k of a horizon-T solution (k = 0..T): window end
    j = k + min(K, T - k); v_bar = V_bar[k] when the window reaches the horizon,
    else the NumPy sum of step_costs[k:j] (ilqr.py:386-390); v_bar_x = V_bar_x[k]
    (ilqr.py:391-392); u = U[k], zeros at k = T (ilqr.py:403); states carry the
    absolute time t0 + k / t0 + j (Trajectory.state_at, ilqr.py:80-81)."""
    if K < 1:
        raise ValueError("K must be >= 1")
    X, U, sc = np.asarray(X, float), np.asarray(U, float), np.asarray(step_costs, float)
    T = U.shape[0]
    n, m = X.shape[1], U.shape[1]
    rows = {"xa": np.empty((T + 1, n + 1)), "u": np.zeros((T + 1, m)), "v_bar": np.empty(T + 1),
            "v_bar_x": np.array(V_bar_x, float).reshape(T + 1, n).copy(), "xa_plus_k": np.empty((T + 1, n + 1))}
    for k in range(T + 1):
        j = k + min(K, T - k)
        v = float(V_bar[k]) if j == T else float(sc[k:j].sum())
        if not np.isfinite(v):
            raise ValueError("v_bar must be finite")      # TOSample.__post_init__ (buffer.py:33-35)
        rows["v_bar"][k] = v
        rows["xa"][k, :n], rows["xa"][k, n] = X[k], t0 + k
        rows["xa_plus_k"][k, :n], rows["xa_plus_k"][k, n] = X[j], t0 + j
        if k < T:
            rows["u"][k] = U[k]
    return rows


def concat_rows(parts):
    return {name: np.concatenate([p[name] for p in parts]) for name in COLUMNS}


# TRLB dump: header <4s16sIIIQ> (magic, model name, n, m, K, count) then
# fixed-width little-endian float64 records [xa | u | v_bar | v_bar_x | xa_plus_k],
# oldest first (buffer.py:17-18, 142-152)
TRLB_HEADER = "<4s16sIIIQ"


def dump_bytes(ring: Ring, model_name: str, k_lookahead: int) -> bytes:
    import struct
    order = (np.arange(ring.size) + (ring.cursor - ring.size)) % ring.capacity
    rec = np.hstack([ring.cols["xa"][order], ring.cols["u"][order], ring.cols["v_bar"][order, None],
                     ring.cols["v_bar_x"][order], ring.cols["xa_plus_k"][order]])
    head = struct.pack(TRLB_HEADER, b"TRLB", model_name.encode()[:16].ljust(16, b"\0"), ring.n, ring.m,
                       k_lookahead, ring.size)
    return head + np.ascontiguousarray(rec, dtype="<f8").tobytes()


def parse_dump(blob: bytes):
    """(model_name, n, m, K, rows dict) of a TRLB dump (buffer.py:153-168)."""
    import struct
    hs = struct.calcsize(TRLB_HEADER)
    if len(blob) < hs or blob[:4] != b"TRLB":
        raise ValueError("not a buffer dump")
    _, name, n, m, k, count = struct.unpack(TRLB_HEADER, blob[:hs])
    width = (n + 1) + m + 1 + n + (n + 1)
    rec = np.frombuffer(blob[hs:hs + count * width * 8], dtype="<f8").reshape(count, width)
    cols = np.split(rec, np.cumsum([n + 1, m, 1, n]), axis=1)
    rows = {"xa": cols[0], "u": cols[1], "v_bar": cols[2][:, 0], "v_bar_x": cols[3], "xa_plus_k": cols[4]}
    return name.rstrip(b"\0").decode(), n, m, k, rows
