"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

Rollouts and scoring shard by candidate index (contiguous ranges, no data-path
collective); the only exchange is ONE all-gather of each shard's stable
top-k winners (score, candidate index, start state), after which every rank
merges identically (`cacto_select_merge`) and reproduces the single-device
`np.argsort(-scores, kind="stable")[:keep]` exactly.
Training is data parallel: the global minibatch index stream is identical on
all ranks; rank r takes its slice and the flat gradient is all-reduced.
"""

from __future__ import annotations

from typing import Callable, Optional

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
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat
