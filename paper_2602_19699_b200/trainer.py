"""BIC selection and the rollout+BIC pipeline on the B200 (reference
`trajrl.trainer`, trainer.py:141-153, 181-193, 258-273).

`select_initial_states_bic` is the drop-in (same signature / order / errors).
`BicPipeline` is the device-resident form used by the benchmark and the
multi-GPU shard path: candidates -> [rollout cost-to-go] -> score -> stable
top-k -> warm-start rollouts of the kept starts, with no host round trip until
the kept indices / warm starts are read back.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib, specs
from .device import DeviceNet, abi_dtype, device, device_net, to_device, torch_dtype
from .nets import actor_rollout_batch


import os

# layout of the cost rollout's kept controls: time-major [T, m, N] (K1's per-step
# writes coalesced; the warm-start take reads one 4-byte value per 32-byte sector)
# or start-major [N, T, m] (take = one coalesced row copy per kept start, but
# K1's 12-byte strided writes cost more than the take saves: measured manipulator3
# step 4.12 -> 4.19 ms, dubins 0.83 -> 0.90 ms, profiles/README.md).
# Layout of every candidate's controls in the cost rollout (CACTO_WARM_LAYOUT):
# "step" [T, N, m] (kept warm starts = a step take), "time" [T, m, N] (a column take),
# "start" [N, T, m] (a row take; A/B only).
_LAYOUT = os.environ.get("CACTO_WARM_LAYOUT", "step")
# host warm-start output: the take kernel writes the pinned host buffer directly
# (zero-copy, "1") or runs in chunks whose device-to-host copies on a side stream
# overlap the next chunk's take ("0", default; measured faster)
_WARM_ZC = os.environ.get("CACTO_WARM_ZEROCOPY", "0") == "1"
_WARM_CHUNKS = int(os.environ.get("CACTO_WARM_CHUNKS", "4"))


def _dev(x0: torch.Tensor) -> torch.device:
    """Where the step's buffers live: x0's device, or the current GPU when x0 is a
    pinned host tensor (read zero-copy by the rollout kernel over PCIe/UVA)."""
    return torch.device("cuda", torch.cuda.current_device()) if x0.device.type == "cpu" else x0.device


def _stream():
    return torch.cuda.current_stream().cuda_stream


class SelectWorkspace:
    """Reusable scratch for cacto_select_topk."""

    def __init__(self):
        self.buf = None

    def get(self, dtype, N, keep):
        need = int(_lib.load().cacto_select_workspace_bytes(dtype, N, keep))
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.empty(max(need, 1), device=device(), dtype=torch.uint8)
        return self.buf, need


_WS = SelectWorkspace()


def select_topk_device(scores: torch.Tensor, keep: int, base_index: int = 0, ws: SelectWorkspace = _WS):
    """Stable descending top-k of a device score vector: (order int64 [keep], scores [keep]).
    Exactly np.argsort(-scores, kind='stable')[:keep] (trainer.py:152)."""
    N = scores.shape[0]
    if keep > N:
        raise ValueError(f"keep={keep} exceeds {N} candidates")
    dt = _lib.F32 if scores.dtype == torch.float32 else _lib.F64
    order = torch.empty(keep, device=scores.device, dtype=torch.int64)
    top = torch.empty(keep, device=scores.device, dtype=scores.dtype)
    if keep == 0:
        return order, top
    buf, need = ws.get(dt, N, keep)
    _lib.call("cacto_select_topk", dt, scores.data_ptr(), N, keep, base_index, order.data_ptr(),
              top.data_ptr(), buf.data_ptr(), need, _stream())
    return order, top


def score_device(mode: str, xa: torch.Tensor, std_net: Optional[DeviceNet] = None,
                 critic: Optional[DeviceNet] = None, rollout_cost: Optional[torch.Tensor] = None):
    """K2: std sigma(x0) / gap |V(x0) - J(x0)| / std*gap scores of augmented starts."""
    N = xa.shape[0]
    scores = torch.empty(N, device=xa.device, dtype=xa.dtype)
    _lib.call("cacto_score", _lib.SCORE[mode], std_net.desc if std_net else None,
              critic.desc if critic else None, xa.data_ptr(),
              rollout_cost.data_ptr() if rollout_cost is not None else None, N, scores.data_ptr(), _stream())
    return scores


def select_initial_states_bic(candidates, std_net, keep: int):
    """trainer.py:141-153: keep the candidates with the largest std-critic output,
    descending, ties by candidate index."""
    if keep > len(candidates):
        raise ValueError(f"keep={keep} exceeds {len(candidates)} candidates")
    xa = np.stack([c.augmented for c in candidates])
    sn = device_net(std_net)
    scores = score_device("std", to_device(xa, sn.precision), std_net=sn)
    order, _ = select_topk_device(scores, keep)
    return [candidates[i] for i in order.cpu().numpy()]


def sample_select_bic(model, count: int, rng_seed, std_net, keep: int, region=specs.Region.WORKSPACE):
    """`select_initial_states_bic(sample_initial_states(model, count, rng_seed, region),
    std_net, keep)` (trainer.py:183-186) with the candidates generated, scored and
    selected on the device: the count x n candidate block is the bit-exact device
    replay of the reference's PCG64 stream (sampling.py), so only the kept rows
    cross PCIe.  Returns (kept states [keep, n] float64 NumPy, kept candidate
    indices) in the reference's order."""
    from .sampling import sample_initial_states_device
    if keep > count:
        raise ValueError(f"keep={keep} exceeds {count} candidates")
    x = sample_initial_states_device(model, count, rng_seed, region)
    sn = device_net(std_net)
    xa = torch.zeros((count, int(model.n) + 1), device=x.device, dtype=torch_dtype(sn.precision))
    xa[:, :-1] = x
    scores = score_device("std", xa, std_net=sn)
    order, _ = select_topk_device(scores, keep)
    return x.index_select(0, order).cpu().numpy(), order.cpu().numpy()


class BicPipeline:
    """Rollout + BIC scoring + stable selection + warm starts, device resident.

    One `run(x0)` processes N candidate starts (float64 [N, n] device tensor):
      gap modes  K1 rollout (cost only) of every candidate -> J(x0)
      K2 score   sigma(x0) and/or |V(x0) - J(x0)|
      K3 select  stable top-keep (ties -> lower index)
      K1 rollout of the kept starts emitting U (TO warm starts, trainer.py:192-193)
    """

    def __init__(self, model, field, actor, critic=None, std_net=None, mode: str = "gap",
                 precision=None, base_index: int = 0):
        if mode not in _lib.SCORE:
            raise ValueError(f"unknown score mode {mode!r}")
        if mode != "std" and critic is None:
            raise ValueError("gap scores need a critic")
        if mode != "gap" and std_net is None:
            raise ValueError("std scores need a std net")
        self.model, self.field, self.mode = model, field, mode
        self.actor = actor if isinstance(actor, DeviceNet) else DeviceNet(actor, precision)
        self.critic = None if critic is None else (critic if isinstance(critic, DeviceNet) else DeviceNet(critic, precision))
        self.std = None if std_net is None else (std_net if isinstance(std_net, DeviceNet) else DeviceNet(std_net, precision))
        self.precision = self.actor.precision
        self.sysd = specs.system_struct(model)
        self.costd = specs.cost_struct(model, field)
        self.base_index = base_index
        self.ws = SelectWorkspace()
        self._copy_stream = None  # side stream of the chunked warm-start copies
        self.kernel_launches = 0

    def _u_all(self, N, T, dt, dev):
        """(pointer, flags) of the buffer the cost rollout writes every candidate's
        controls into (step-major [T, N, m], time-major [T, m, N] or start-major [N, T, m],
        _LAYOUT)."""
        m = self.model.m
        shape = {"step": (T, N, m), "time": (T, m, N)}.get(_LAYOUT, (N, T, m))
        if getattr(self, "u_all", None) is None or tuple(self.u_all.shape) != shape or self.u_all.dtype != dt:
            self.u_all = torch.empty(shape, device=dev, dtype=dt)
        flags = {"step": _lib.ROLLOUT_U_STEP_MAJOR, "time": _lib.ROLLOUT_U_TIME_MAJOR}.get(_LAYOUT, 0)
        return self.u_all.data_ptr(), flags

    def _take(self, sel_ptr: int, K: int, dst_ptr: int, N: int, T: int, stream):
        """The kept starts' controls out of self.u_all into dst [K, T, m] (one launch)."""
        m = self.model.m
        if _LAYOUT == "step":
            _lib.call("cacto_take_steps", abi_dtype(self.precision), self.u_all.data_ptr(), T, N, m, sel_ptr, K,
                      dst_ptr, stream)
        elif _LAYOUT == "time":
            _lib.call("cacto_take_columns", abi_dtype(self.precision), self.u_all.data_ptr(), T * m, N, sel_ptr, K,
                      dst_ptr, stream)
        else:
            _lib.call("cacto_take_rows", abi_dtype(self.precision), self.u_all.data_ptr(), T * m, sel_ptr, K,
                      dst_ptr, stream)

    def rollout_costs(self, x0: torch.Tensor, t0: int = 0, keep_controls: bool = False) -> torch.Tensor:
        """K1 cost-to-go of every candidate; with keep_controls the same launch
        also writes every candidate's controls into self.u_all, from which the
        kept warm starts are taken (no second rollout)."""
        N = x0.shape[0]
        dt = torch_dtype(self.precision)
        cost = torch.empty(N, device=_dev(x0), dtype=dt)
        T = self.model.t_max - t0
        U, flags = None, 0
        if keep_controls:
            U, flags = self._u_all(N, T, dt, _dev(x0))
        _lib.call("cacto_rollout_ex", self.sysd, self.costd, self.actor.desc, x0.data_ptr(), None, t0, N, T, flags,
                  U, None, None, cost.data_ptr(), _stream())
        return cost

    def _fused(self, x0: torch.Tensor, t0: int, keep_controls: bool):
        """K1 + K2 in one launch (cacto_rollout_score); (None, None) when the
        library reports the nets are not fusable."""
        N = x0.shape[0]
        dt = torch_dtype(self.precision)
        cost = torch.empty(N, device=_dev(x0), dtype=dt)
        scores = torch.empty(N, device=_dev(x0), dtype=dt)
        T = self.model.t_max - t0
        U, flags = None, 0
        if keep_controls:
            U, flags = self._u_all(N, T, dt, _dev(x0))
        rc = _lib.load().cacto_rollout_score(
            self.sysd, self.costd, self.actor.desc, _lib.SCORE[self.mode], self.std.desc if self.std else None,
            self.critic.desc if self.critic else None, x0.data_ptr(), t0, N, T, flags, U, cost.data_ptr(),
            scores.data_ptr(), _stream())
        if rc == _lib.EUNSUPPORTED:
            return None, None
        _lib.check(rc, "cacto_rollout_score")
        return scores, cost

    def _scores(self, x0: torch.Tensor, t0: int, reuse: bool):
        """(scores [N], cost [N] or None, launches): K1 + K2 fused when possible."""
        N, n = x0.shape
        dt = torch_dtype(self.precision)
        launches = 0
        cost = None
        scores = None
        if self.mode != "std":
            scores, cost = self._fused(x0, t0, reuse)
            launches += 1
            if scores is None:  # not fusable (fp64 / SIMT path / differing net shapes)
                cost = self.rollout_costs(x0, t0, keep_controls=reuse)
        if scores is None:
            xa = torch.empty((N, n + 1), device=_dev(x0), dtype=dt)
            xa[:, :n] = x0
            xa[:, n] = float(t0)
            launches += 3  # torch copy + fill of the augmented view, K2 score
            scores = score_device(self.mode, xa, self.std, self.critic, cost)
        return scores, cost, launches

    def _warm(self, x0: torch.Tensor, sel: torch.Tensor, t0: int, reuse: bool, out=None):
        """Warm starts U [K, T, m] of the candidates `sel` (local indices).  `out`
        (pinned host [>= K, T, m]) makes the take write them straight into host memory
        (zero-copy over PCIe/UVA: the gather and the transfer overlap)."""
        N = x0.shape[0]
        K = sel.shape[0]
        T = self.model.t_max - t0
        dt = torch_dtype(self.precision)
        if out is not None and reuse:
            if out[:K].dtype != dt or tuple(out.shape[1:]) != (T, self.model.m) or not out.is_contiguous():
                raise ValueError("warm-start output buffer does not match [K, T, m] / dtype")
        if out is not None and reuse and _WARM_ZC:
            U = out[:K]
        else:
            U = torch.empty((K, T, self.model.m), device=_dev(x0), dtype=dt)
        if K == 0:
            return (out[:0] if out is not None else U), 0
        if reuse and out is not None and not _WARM_ZC and not out.is_cuda:
            # chunked take; chunk c's copy to the pinned host buffer (side stream, copy
            # engine) overlaps chunk c + 1's take; the caller's stream waits for the
            # last copy, so the returned host rows are complete in stream order
            main = torch.cuda.current_stream()
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(device=_dev(x0))
            cs = self._copy_stream
            row = T * self.model.m
            es = U.element_size()
            nch = max(1, min(_WARM_CHUNKS, K))
            bounds = [K * c // nch for c in range(nch + 1)]
            for c in range(nch):
                c0, c1 = bounds[c], bounds[c + 1]
                if c1 == c0:
                    continue
                self._take(sel.data_ptr() + c0 * sel.element_size(), c1 - c0, U.data_ptr() + c0 * row * es, N, T,
                           main.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(main)
                cs.wait_event(ev)
                with torch.cuda.stream(cs):
                    out[c0:c1].copy_(U[c0:c1], non_blocking=True)
            done = torch.cuda.Event()
            done.record(cs)
            main.wait_event(done)
            U.record_stream(cs)
            return out[:K], nch
        if reuse:
            # the kept starts' controls from the cost rollout (same actor, start and t0:
            # the trajectories trainer.py:192-193 would roll out again)
            self._take(sel.data_ptr(), K, U.data_ptr(), N, T, _stream())
            if out is not None and U.is_cuda and not out.is_cuda:
                out[:K].copy_(U, non_blocking=True)
                U = out[:K]
            return U, 1
        kept = x0.to(_dev(x0)).index_select(0, sel)
        _lib.call("cacto_rollout", self.sysd, None, self.actor.desc, kept.data_ptr(), None, t0, K, T,
                  U.data_ptr(), None, None, None, _stream())
        if out is not None:
            out[:K].copy_(U, non_blocking=True)
            U = out[:K]
        return U, 2

    def run(self, x0: torch.Tensor, keep: int, t0: int = 0, warm_starts: bool = True, u_out=None):
        """x0 float64 [N, n] on device -> dict(order, scores, U, cost).

        x0 may also be a PINNED HOST tensor: the rollout kernel then reads each start
        zero-copy (over PCIe / UVA, overlapped with the other CTAs' compute) instead of
        a separate host-to-device copy; `u_out` (pinned host [>= keep, T, m]) receives
        the warm starts straight from the take kernel (trainer.py:192-193 hand-off)."""
        N, n = x0.shape
        reuse = warm_starts and keep > 0 and self.mode != "std"
        scores, cost, launches = self._scores(x0, t0, reuse)
        order, top = select_topk_device(scores, keep, 0, self.ws)
        if N <= 2048:
            launches += 1  # single-CTA select (csrc/select.cu small_select_kernel)
        else:
            launches += 4 + max(0, int(np.ceil(np.log2(max(keep, 1) / 2048.0))))  # memset, select, sort, merges, emit
        out = {"order": order, "scores": top, "cost": cost}
        if warm_starts and keep > 0:
            out["U"], nl = self._warm(x0, order, t0, reuse, out=u_out)
            launches += nl
        if self.base_index:
            out["order"] = order + self.base_index
        self.kernel_launches = launches
        return out

    def run_sharded(self, x0: torch.Tensor, keep_global: int, base_index: int, dsel=None, group=None,
                    t0: int = 0, warm_starts: bool = True, u_out=None):
        """This rank's share of the multi-GPU rollout+BIC step.

        x0 [N_local, n] are global candidates base_index .. base_index + N_local - 1
        (contiguous shards in rank order).  Scores are local; the global stable
        top-keep_global is found by the distributed radix threshold
        (`parallel.DistributedSelect`).  Returns dict(order [keep_global] global
        indices and scores, identical on every rank; local [c_r] this rank's own
        winners as local indices in global order; U [c_r, T, m] their warm starts,
        taken from this rank's cost rollout -- no states or controls cross ranks)."""
        from .parallel import DistributedSelect
        N = x0.shape[0]
        reuse = warm_starts and keep_global > 0 and self.mode != "std"
        scores, cost, launches = self._scores(x0, t0, reuse)
        if dsel is None:
            dsel = DistributedSelect(N, keep_global, scores.dtype, group, _dev(x0))
        order, top, local, _ = dsel.run(scores, base_index)
        # hist + digit per pass; compact, chunk sort, merges, emit; final chunk sort, merges, emit
        launches += 2 * dsel.passes + 5 + 2 * max(0, int(np.ceil(np.log2(max(keep_global, 1) / 2048.0))))
        out = {"order": order, "scores": top, "cost": cost, "local": local}
        if warm_starts:
            out["U"], nl = self._warm(x0, local, t0, reuse, out=u_out)
            launches += nl
        self.kernel_launches = launches
        return out


def evaluate_policy_costs(actor, model, fld, eval_starts, use_to: bool = False, **kwargs):
    """trainer.py:258-273 rollout leg (batched on device); the optional TO
    refinement stays on the reference CPU solver and is not provided here."""
    if not eval_starts:
        raise ValueError("eval_starts must be non-empty")
    if use_to:
        raise NotImplementedError("TO refinement runs on the reference CPU solver (out of scope)")
    x0 = np.stack([s.x for s in eval_starts])
    t0 = np.array([s.t for s in eval_starts])
    r = actor_rollout_batch(actor, model, x0, t0, None, fld, emit=("cost",))
    return r["cost"]
