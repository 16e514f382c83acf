"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

Rollouts and scoring shard by candidate index (contiguous ranges, no data-path
collective).  The global stable top-k (`np.argsort(-scores, kind="stable")[:keep]`
over the union of the shards, trainer.py:152) is found by a DISTRIBUTED radix
threshold (`DistributedSelect`, csrc/select.cu `cacto_dselect_*`): per 8-bit
digit one all-reduce of a 256-bin histogram (2 KB), then one all-gather of two
counts per rank and one all-reduce of the keep_global winners (each rank fills
its own disjoint segment of a zeroed buffer).  Traffic per rank is O(keep_global),
not O(world * keep_global), and each rank keeps only its OWN winners' warm starts
(no start states or controls cross ranks).
Training is data parallel (engine.UpdateEngine(dp_group=...)): the global minibatch
index stream is identical on all ranks; rank r takes its slice and the flat
gradient is all-reduced.
The older all-gather-and-merge path (`sharded_select`, `cacto_select_merge`) is
kept as an independent check of the distributed select in the tests.
"""

from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) candidate range of `rank` (sizes differ by <= 1)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_winners(scores: torch.Tensor, order: torch.Tensor, x0: torch.Tensor, keep: int,
                   group=None):
    """All-gather every rank's local winners (padded to `keep` rows).

    scores [k] (sorted desc, ties by index), order [k] global candidate indices,
    x0 [k, n] their start states, k <= keep.  Returns the concatenated runs
    (R*keep scores / indices / states) and the valid-count per run; padding rows
    carry NaN scores so they sort last (NaN-last semantics of the select).
    """
    world = dist.get_world_size(group)
    k = scores.shape[0]
    n = x0.shape[1]
    dev = scores.device
    ps = torch.full((keep,), float("nan"), device=dev, dtype=scores.dtype)
    po = torch.full((keep,), -1, device=dev, dtype=torch.int64)
    px = torch.zeros((keep, n), device=dev, dtype=x0.dtype)
    ps[:k], po[:k], px[:k] = scores, order, x0
    all_s = [torch.empty_like(ps) for _ in range(world)]
    all_o = [torch.empty_like(po) for _ in range(world)]
    all_x = [torch.empty_like(px) for _ in range(world)]
    dist.all_gather(all_s, ps, group=group)
    dist.all_gather(all_o, po, group=group)
    dist.all_gather(all_x, px, group=group)
    return torch.cat(all_s), torch.cat(all_o), torch.cat(all_x)


def merge_positions(run_scores: torch.Tensor, run_order: torch.Tensor, keep: int, merge_fn: Callable):
    """Positions (into the concatenated runs) of the global top-`keep`.

    Runs are contiguous shards in rank order and each run is sorted by
    (score desc, index asc), so ordering equal scores by run POSITION is the
    same as ordering them by global candidate index: the merge may carry
    positions instead of indices (see cacto_select_merge).  Padding rows
    (run_order < 0) carry -1 and sort after every real candidate, NaN included.
    """
    R = run_scores.shape[0] // keep
    pos = torch.arange(R * keep, device=run_scores.device, dtype=torch.int64)
    pos = torch.where(run_order < 0, torch.full_like(pos, -1), pos)
    return merge_fn(run_scores, pos, R, keep)


def device_merge(run_scores: torch.Tensor, run_index: torch.Tensor, R: int, keep: int):
    """The product merge: cacto_select_merge on device."""
    from . import _lib
    M = R * keep
    ws_bytes = 2 * (((M * 16) + 255) // 256) * 256
    ws = torch.empty(ws_bytes, device=run_scores.device, dtype=torch.uint8)
    order = torch.empty(keep, device=run_scores.device, dtype=torch.int64)
    top = torch.empty(keep, device=run_scores.device, dtype=run_scores.dtype)
    dt = _lib.F32 if run_scores.dtype == torch.float32 else _lib.F64
    _lib.call("cacto_select_merge", dt, run_scores.data_ptr(), run_index.data_ptr(), R, keep,
              order.data_ptr(), top.data_ptr(), ws.data_ptr(), ws_bytes,
              torch.cuda.current_stream().cuda_stream)
    return order


def sharded_select(local_scores: torch.Tensor, local_x0: torch.Tensor, base_index: int, keep: int,
                   local_topk: Callable, merge_fn: Optional[Callable] = None, group=None):
    """Global stable top-`keep` over all ranks' candidates.

    local_topk(scores, k, base_index) -> (order [k] global idx, top scores [k]).
    Returns (global order [keep], kept start states [keep, n]) identical on every rank.
    """
    merge_fn = merge_fn or device_merge
    k = min(keep, local_scores.shape[0])
    order, top = local_topk(local_scores, k, base_index)
    x_sel = local_x0.index_select(0, order - base_index)
    rs, ro, rx = gather_winners(top, order, x_sel, keep, group)
    pos = merge_positions(rs, ro, keep, merge_fn)
    return ro.index_select(0, pos), rx.index_select(0, pos)


def allreduce_grads(flat: torch.Tensor, group=None):
    """DP gradient sum over ranks (losses already divide by the GLOBAL batch)."""
    return all_reduce_sum(flat, group)


# ---- collectives (gloo cannot reduce CUDA tensors on every build: stage via host) ----

def _backend(group):
    return dist.get_backend(group)


def all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM over ranks (NCCL on device; gloo through a host copy)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    if t.is_cuda and _backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def all_gather_cat(t: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenation over ranks (rank order) of equally shaped tensors."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t.clone()
    world = dist.get_world_size(group)
    if t.is_cuda and _backend(group) != "nccl":
        h = t.cpu()
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h, group=group)
        return torch.cat(parts).to(t.device)
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), device=t.device, dtype=t.dtype)
    dist.all_gather_into_tensor(out, t, group=group)
    return out


class _DselectKernels:
    """The device phases of the distributed select (csrc/select.cu cacto_dselect_*)."""

    def __init__(self, N_local, keep, dtype, device):
        from . import _lib
        self.L = _lib
        self.N, self.keep, self.dtype = N_local, keep, dtype
        self.abi = _lib.F32 if dtype == torch.float32 else _lib.F64
        self.passes = 4 if dtype == torch.float32 else 8
        self.words = 1 if dtype == torch.float32 else 2
        self.device = device
        self.ws_bytes = _lib.load().cacto_dselect_workspace_bytes(self.abi, self.N, self.keep)
        self.ws = torch.empty(self.ws_bytes, device=device, dtype=torch.uint8)
        self.scratch = torch.empty((max(keep, 1), self.words), device=device, dtype=torch.int64)

    @staticmethod
    def _st():
        return torch.cuda.current_stream().cuda_stream

    def begin(self):
        self.L.call("cacto_dselect_begin", self.abi, self.N, self.keep, self.keep, self.ws.data_ptr(), self.ws_bytes,
                    self._st())

    def hist(self, scores, p, out):
        self.L.call("cacto_dselect_pass", self.abi, scores.data_ptr(), self.N, self.keep, p, self.ws.data_ptr(),
                    out.data_ptr(), self._st())

    def digit(self, p, hist_global, counts):
        self.L.call("cacto_dselect_digit", self.abi, self.N, self.keep, p, hist_global.data_ptr(), self.ws.data_ptr(),
                    counts.data_ptr(), self._st())

    def local(self, scores, base, n_cand, n_take, off, elems, local_sel):
        self.L.call("cacto_dselect_local", self.abi, scores.data_ptr(), self.N, self.keep, base, n_cand, n_take, off,
                    self.ws.data_ptr(), elems.data_ptr(), local_sel.data_ptr(), self._st())

    def finish(self, elems, order, top):
        self.L.call("cacto_dselect_finish", self.abi, elems.data_ptr(), self.keep, order.data_ptr(), top.data_ptr(),
                    self.scratch.data_ptr(), self.scratch.numel() * 8, self._st())


class DistributedSelect:
    """Exact global stable top-`keep_global` over contiguous candidate shards.

    Every rank calls `run(local_scores, base_index)` with its shard (global
    indices base_index .. base_index + N_local - 1, shards in rank order).
    Returns (order [keep_global] global indices, scores [keep_global]) identical on
    every rank, plus this rank's own winners: `local_sel` [c_r] (local indices,
    in global order) -- the rows whose warm starts this rank hands to its TO.
    Phases and collectives: see include/cacto_b200.h `cacto_dselect_*`; the
    host side here owns only the collectives and the tie split between ranks.
    `kernels` (tests only) swaps the device phases for a stand-in.
    """

    def __init__(self, N_local: int, keep_global: int, dtype=torch.float32, group=None, device=None, kernels=None):
        self.group = group
        self.N, self.keep = int(N_local), int(keep_global)
        self.dtype = dtype
        if kernels is None:
            dev = device or torch.device("cuda", torch.cuda.current_device())
            kernels = _DselectKernels(self.N, self.keep, dtype, dev)
        self.k = kernels
        self.passes = self.k.passes
        dev = self.k.device
        self.hist = torch.empty(256, device=dev, dtype=torch.int64)
        self.counts = torch.zeros(3, device=dev, dtype=torch.int64)
        self.elems = torch.empty((max(self.keep, 1), self.k.words), device=dev, dtype=torch.int64)
        self.order = torch.empty(self.keep, device=dev, dtype=torch.int64)
        self.top = torch.empty(self.keep, device=dev, dtype=dtype)
        self.local_sel = torch.empty(max(self.keep, 1), device=dev, dtype=torch.int64)
        self.collectives = 0

    @staticmethod
    def split(lt, eq, need, rank, keep):
        """Tie split between ranks (host): rank r takes its first
        take_r = clamp(need - sum_{q<r} eq_q, 0, eq_r) keys equal to the threshold
        (lower ranks hold lower global indices), so c_r = lt_r + take_r winners at
        offset sum_{q<r} c_q of the concatenated winner buffer."""
        lt, eq = np.asarray(lt, np.int64), np.asarray(eq, np.int64)
        before = np.concatenate([[0], np.cumsum(eq)[:-1]])
        take = np.clip(need - before, 0, eq)
        c = lt + take
        if int(c.sum()) != keep:
            raise RuntimeError(f"distributed select: {int(c.sum())} winners for keep={keep}")
        return int(c[:rank].sum()), int(c[rank])

    def run(self, scores: torch.Tensor, base_index: int):
        if scores.shape[0] != self.N or scores.dtype != self.dtype:
            raise ValueError("DistributedSelect: scores do not match the shard size / dtype")
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        if self.keep == 0:
            return self.order, self.top, self.local_sel[:0], 0
        self.k.begin()
        for p in range(self.passes):
            self.k.hist(scores, p, self.hist)
            all_reduce_sum(self.hist, self.group)
            self.k.digit(p, self.hist, self.counts)
        allc = all_gather_cat(self.counts[:2].contiguous(), self.group).view(world, 2).cpu().numpy()
        need = int(self.counts[2].item())
        self.collectives = self.passes + 2
        off, cr = self.split(allc[:, 0], allc[:, 1], need, rank, self.keep)
        self.elems.zero_()
        self.k.local(scores, base_index, int(allc[rank, 0] + allc[rank, 1]), cr, off, self.elems, self.local_sel)
        all_reduce_sum(self.elems, self.group)
        self.k.finish(self.elems, self.order, self.top)
        return self.order, self.top, self.local_sel[:cr], off
