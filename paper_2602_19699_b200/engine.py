"""Device-resident network-update loop (reference trainer.py:208-234).

Per iteration the reference runs M cycles of
    minibatch -> critic_loss -> adam -> polyak(target) -> actor_loss(updated critic) -> adam
and then M std-critic cycles, every minibatch drawn from one NumPy Generator
(`rng_batches`, trainer.py:123) over a replay buffer that does not change
during the loop.  `UpdateEngine` keeps the four networks, their Adam moments
and the replay ring in HBM, draws the SAME 2*M index lists from the
reference's generator up front (one H2D copy), and replays two captured CUDA
graphs -- one critic+actor cycle (9 kernels) and one std cycle (4 kernels) --
M times each.  Every per-cycle quantity (index list, Adam step, loss slot) is
read from device counters, so the graphs are captured once and reused for
every iteration.

Data parallel (`dp_group`): every rank draws the same global index lists from
the same generator (the reference stream), takes its contiguous slice
[lo, hi) of each list (`parallel.shard_range`), and its losses divide by the
GLOBAL minibatch (the actor's by the global live-row count, counted over the
whole list), so the sum over ranks of the local gradients is the reference
gradient.  Each update folds its partials into one [P + 1] vector (gradient +
loss), sums it over ranks with one all-reduce, and applies the replicated
fused Adam (+ Polyak) -- critic, then the actor on the UPDATED critic, then
std, the dependency order of trainer.py:211-233.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

from . import _lib, parallel, specs
from .buffer import ReplayBuffer
from .device import DeviceNet, abi_dtype, device, torch_dtype


def _stream():
    return torch.cuda.current_stream().cuda_stream


class _Net:
    """A trained network: parameters + Adam moments + step, all on device."""

    def __init__(self, mlp, precision, lr, adam=None):
        self.dn = DeviceNet(mlp, precision)
        self.m = torch.zeros_like(self.dn.params)
        self.v = torch.zeros_like(self.dn.params)
        self.step = 0
        self.lr = float(lr)
        self.beta1, self.beta2, self.eps = 0.9, 0.999, 1e-8
        if adam is not None:  # reference AdamState (nets.py:358-372)
            self.m.copy_(torch.as_tensor(self.dn.pack(adam.m)))
            self.v.copy_(torch.as_tensor(self.dn.pack(adam.v)))
            self.step = int(adam.step)
            self.lr, self.beta1, self.beta2, self.eps = adam.lr, adam.beta1, adam.beta2, adam.eps_adam
        self.base = torch.zeros(1, device=self.m.device, dtype=torch.int64)


class UpdateEngine:
    """Device-resident M-cycle critic / actor / std-critic updates."""

    def __init__(self, model, field, actor, critic, critic_target, std_net, buffer: ReplayBuffer, *,
                 minibatch: int, k_s: float = 1.0, bootstrap: bool = True, tau: float = 0.005,
                 lr_actor: float = 5e-4, lr_critic: float = 1e-3, lr_std: float = 1e-3,
                 adam_states=None, precision: Optional[str] = None, use_graphs: bool = True,
                 max_steps: int = 1 << 17, dp_group=None):
        self.model, self.field = model, field
        self.precision = precision or buffer.precision
        self.buffer = buffer
        self.B = int(minibatch)
        self.k_s, self.bootstrap, self.tau = float(k_s), bool(bootstrap), float(tau)
        ad = adam_states or (None, None, None)
        self.actor = _Net(actor, self.precision, lr_actor, ad[0])
        self.critic = _Net(critic, self.precision, lr_critic, ad[1])
        self.std = _Net(std_net, self.precision, lr_std, ad[2])
        self.target = DeviceNet(critic_target, self.precision)
        self.sysd = specs.system_struct(model)
        self.costd = specs.cost_struct(model, field)
        dev = device()
        L = _lib.load()
        # data parallel: this rank's slice [lo, hi) of every global minibatch
        self.dp_group = dp_group
        self.world, self.rank = 1, 0
        if dp_group is not None:
            import torch.distributed as dist
            grp = None if dp_group == "world" else dp_group
            self.dp_group = grp
            self.world, self.rank = dist.get_world_size(grp), dist.get_rank(grp)
        self.lo, self.hi = parallel.shard_range(self.B, self.rank, self.world)
        if self.hi <= self.lo:
            raise ValueError(f"minibatch {self.B} too small for {self.world} data-parallel ranks")
        B = self.hi - self.lo
        self.ws_c = torch.empty(L.cacto_loss_workspace_bytes(self.critic.dn.desc, B), device=dev, dtype=torch.uint8)
        self.ws_a = torch.empty(L.cacto_loss_workspace_bytes(self.actor.dn.desc, B)
                                + L.cacto_loss_workspace_bytes(self.critic.dn.desc, B), device=dev, dtype=torch.uint8)
        self.ws_s = torch.empty(L.cacto_loss_workspace_bytes(self.std.dn.desc, B), device=dev, dtype=torch.uint8)
        self.live = torch.zeros(1, device=dev, dtype=torch.int64)
        if self.world > 1:  # folded gradient + loss of each net, the all-reduced vectors
            dt = torch_dtype(self.precision)
            self.g = {id(n): torch.zeros(n.dn.count + 1, device=dev, dtype=dt)
                      for n in (self.actor, self.critic, self.std)}
            import torch.distributed as dist
            if use_graphs and dist.get_backend(self.dp_group) != "nccl":
                use_graphs = False  # only NCCL collectives can be captured in a CUDA graph
        # cycle counters: [critic (and, unpipelined, actor), std, actor (pipelined)]
        self.cnt = torch.zeros(3, device=dev, dtype=torch.int64)
        # bias-correction tables bc[t] = 1 - beta**t in Python double precision
        # (nets.py:380-381), grown on demand (_ensure_bc) so any run length works
        self.bc = {}
        self.max_steps = 0
        self._ensure_bc(max(int(max_steps), 1 + max(n.step for n in (self.actor, self.critic, self.std))))
        self.use_graphs = use_graphs
        self.K = 16          # cycles per captured chunk (pipelined schedule)
        # ring of RC chunks of per-cycle critics: the critic chain may run RC - 1 chunks
        # ahead of the actor chain (the std chain starts when the critic chain ends)
        self.RC = int(os.environ.get("CACTO_RING_CHUNKS", "8"))
        self.cview = None
        self._graphs = None
        self._cap_M = 0
        self.idx = None
        self.closs = None
        self.sloss = None
        self.aloss = None

    def _ensure_bc(self, need: int):
        """Make the device tables cover Adam steps t <= need + 1 (doubling), so a
        restored or long run never hits a fixed cap; growing them re-captures the
        graphs (the table pointers are baked into the captured launches)."""
        if need + 2 <= self.max_steps:
            return
        cap = max(1 << 17, self.max_steps)
        while cap < need + 2:
            cap *= 2
        t = np.arange(cap, dtype=np.float64)
        dev = device()
        self.bc = {}
        for net in (self.actor, self.critic, self.std):
            key = (net.beta1, net.beta2)
            if key not in self.bc:
                self.bc[key] = (torch.as_tensor(np.array([1.0 - net.beta1 ** k for k in t])).to(dev),
                                torch.as_tensor(np.array([1.0 - net.beta2 ** k for k in t])).to(dev))
        self.max_steps = cap
        self._graphs = None

    # -- one cycle, as kernel launches on the current stream -----------------------
    def _batch(self, slot, whole=False, cptr=None):
        """Batch descriptor of index list `slot` at the cycle held by the device
        counter `cptr` (default: cnt[slot]): this rank's slice of the global list (or
        the whole list), losses averaged over the global minibatch."""
        lo, hi = (0, self.B) if whole else (self.lo, self.hi)
        d = self.buffer.ring_desc(self.idx[slot, :, lo:], rows=hi - lo)
        d.cycle = self.cnt[slot:slot + 1].data_ptr() if cptr is None else cptr
        d.idx_stride = self.B
        d.denom = self.B if self.world > 1 else 0
        return d

    def _adam(self, net: _Net, ws, npart, slot, target=None, loss=None, cptr=None, ring=None):
        bc1, bc2 = self.bc[(net.beta1, net.beta2)]
        if self.world > 1:
            # fold -> [grad | loss] -> sum over ranks -> replicated Adam (+ Polyak)
            g = self.g[id(net)]
            _lib.call("cacto_reduce_grads", net.dn.desc.dtype, ws.data_ptr(), npart, net.dn.count, g.data_ptr(),
                      g[net.dn.count:].data_ptr(), _stream())
            parallel.allreduce_grads(g, self.dp_group)
            ws, npart = g, 1
        counter = self.cnt[slot:slot + 1].data_ptr() if cptr is None else cptr
        args = (net.dn.desc.dtype, ws.data_ptr(), npart, net.dn.count, net.dn.params.data_ptr(), net.m.data_ptr(),
                net.v.data_ptr(), counter, net.base.data_ptr(), bc1.data_ptr(), bc2.data_ptr(), net.lr, net.beta1,
                net.beta2, net.eps, None if target is None else target.params.data_ptr(), self.tau,
                None if loss is None else loss.data_ptr())
        if ring is None:
            _lib.call("cacto_reduce_adam_graph", *args, _stream())
        else:  # the updated parameters also into ring slot (*counter % ring rows)
            _lib.call("cacto_reduce_adam_graph_ring", *args, ring.data_ptr(), ring.shape[0], ring.shape[1], _stream())

    def _cycle_critic_actor(self):
        st = _stream()
        bd = self._batch(0)
        npart = ctypes.c_int32(0)
        tgt = self.target if self.bootstrap else None
        _lib.call("cacto_critic_loss", self.critic.dn.desc, tgt.desc if tgt else None, bd, self.k_s,
                  int(self.bootstrap), self.ws_c.data_ptr(), self.ws_c.numel(), npart, st)
        self._adam(self.critic, self.ws_c, npart.value, 0, target=self.target, loss=self.closs)  # trainer.py:216-220
        npa = ctypes.c_int32(0)
        # live rows (nets.py:310-312): counted inside the actor-loss launch (live_rows =
        # NULL), or over the whole global list when the batch is split over ranks
        live = None
        if self.world > 1:
            _lib.call("cacto_count_live", self._batch(0, whole=True), self.live.data_ptr(), st)
            live = self.live.data_ptr()
        _lib.call("cacto_actor_loss", self.actor.dn.desc, self.critic.dn.desc, self.sysd, self.costd, bd,
                  live, self.ws_a.data_ptr(), self.ws_a.numel(), npa, st)
        self._adam(self.actor, self.ws_a, npa.value, 0, loss=self.aloss)                        # trainer.py:223-225
        _lib.call("cacto_counter_tick", self.cnt[0:1].data_ptr(), st)

    # -- the pipelined schedule (one rank, graphs): the actor update of cycle i needs
    #    only the critic AFTER update i, so the critic chain runs ahead and keeps each
    #    cycle's critic in a ring slot (2K slots, written by cycle counter); the actor
    #    chain reads the slot of its own cycle through a static descriptor (even / odd
    #    chunks capture their own graphs).  The std phase uses the final critic for all
    #    M cycles, so its errors v_bar - V(xa) come from ONE batched critic forward.
    #    Inside a captured chunk cycle i reads counter span[i] (one launch per chunk
    #    sets span = base + 0..K-1) instead of ticking a counter every cycle.  Same
    #    kernels on the same inputs: bit-identical to the sequential loop. -----------
    def _cycle_critic(self, cptr=None):
        st = _stream()
        c = self.cnt[0:1].data_ptr() if cptr is None else cptr
        bd = self._batch(0, cptr=c)
        npart = ctypes.c_int32(0)
        tgt = self.target if self.bootstrap else None
        _lib.call("cacto_critic_loss", self.critic.dn.desc, tgt.desc if tgt else None, bd, self.k_s,
                  int(self.bootstrap), self.ws_c.data_ptr(), self.ws_c.numel(), npart, st)
        # Adam + Polyak + this cycle's critic into the ring (ring_copy fused into the update)
        self._adam(self.critic, self.ws_c, npart.value, 0, target=self.target, loss=self.closs, cptr=c,
                   ring=self.cring)
        if cptr is None:
            _lib.call("cacto_counter_tick", c, st)

    def _cycle_actor(self, cptr=None, slot_desc=None):
        st = _stream()
        c = self.cnt[2:3].data_ptr() if cptr is None else cptr
        bd = self._batch(0, cptr=c)
        if slot_desc is None:  # eager: copy the cycle's critic out of the ring
            _lib.call("cacto_ring_copy", self.critic.dn.desc.dtype, self.cring.data_ptr(), c,
                      self.cring.shape[0], self.cring.shape[1], self.critic.dn.count, self.cview.params.data_ptr(),
                      0, st)
            slot_desc = self.cview.desc
        npa = ctypes.c_int32(0)
        _lib.call("cacto_actor_loss", self.actor.dn.desc, slot_desc, self.sysd, self.costd, bd,
                  None, self.ws_a.data_ptr(), self.ws_a.numel(), npa, st)
        self._adam(self.actor, self.ws_a, npa.value, 2, loss=self.aloss, cptr=c)             # trainer.py:223-225
        if cptr is None:
            _lib.call("cacto_counter_tick", c, st)

    def _cycle_std_err(self, cptr=None):
        st = _stream()
        c = self.cnt[1:2].data_ptr() if cptr is None else cptr
        bd = self._batch(1, cptr=c)
        npart = ctypes.c_int32(0)
        _lib.call("cacto_std_loss_err", self.std.dn.desc, self.serr.data_ptr(), bd, self.ws_s.data_ptr(),
                  self.ws_s.numel(), npart, st)
        self._adam(self.std, self.ws_s, npart.value, 1, loss=self.sloss, cptr=c)                # trainer.py:229-232
        if cptr is None:
            _lib.call("cacto_counter_tick", c, st)

    def _std_errors(self, M):
        """e = v_bar - V_critic(xa) of every std-phase minibatch (nets.py:343), one launch."""
        d = self.buffer.ring_desc(self.idx[1, :M, self.lo:], rows=(self.hi - self.lo))
        d.rows = M * self.B
        _lib.call("cacto_value_errors", self.critic.dn.desc, d, self.serr.data_ptr(), _stream())

    def _cycle_std(self):
        st = _stream()
        bd = self._batch(1)
        npart = ctypes.c_int32(0)
        _lib.call("cacto_std_loss", self.std.dn.desc, self.critic.dn.desc, bd, self.ws_s.data_ptr(),
                  self.ws_s.numel(), npart, st)
        self._adam(self.std, self.ws_s, npart.value, 1, loss=self.sloss)                         # trainer.py:229-232
        _lib.call("cacto_counter_tick", self.cnt[1:2].data_ptr(), st)

    # -- buffers / graphs ---------------------------------------------------------------
    def _alloc(self, M):
        dev = device()
        dt = torch_dtype(self.precision)
        # index lists: [0] critic/actor cycles, [1] std cycles
        self.idx = torch.zeros((2, M, self.B), device=dev, dtype=torch.int64)
        self.closs = torch.zeros(M, device=dev, dtype=dt)
        self.aloss = torch.zeros(M, device=dev, dtype=dt)
        self.sloss = torch.zeros(M, device=dev, dtype=dt)
        self.serr = torch.zeros(M * self.B, device=dev, dtype=dt)   # std-phase errors [M][B]
        self._cap_M = M
        self._graphs = None

    def _pipelined(self):
        """The pipelined chunk schedule: one rank, graphs on, narrow nets (the std
        phase's precomputed-error loss is built for hidden width <= 64)."""
        return self.use_graphs and self.world == 1 and self.std.dn.desc.hp <= 64 and self.critic.dn.desc.hp <= 64

    def _capture(self):
        """Capture the cycle graphs (chunks of K cycles for the pipelined schedule,
        single cycles otherwise).  A first eager pass (on snapshots) performs every
        lazy runtime set-up outside the capture."""
        pipe = self._pipelined()
        dev = device()
        if pipe and self.cview is None:
            self.cview = DeviceNet(self.critic.dn.to_mlp(), self.precision)
            ld = (self.critic.dn.count + 63) // 64 * 64   # 256/512-byte aligned ring slots
            self.cring = torch.zeros((self.RC * self.K, ld), device=dev, dtype=torch_dtype(self.precision))
            # static descriptors of the ring slots (the actor chain's critic of cycle i)
            self.slot_desc = []
            for r in range(self.RC * self.K):
                d = type(self.cview.desc).from_buffer_copy(self.cview.desc)
                d.params = self.cring[r].data_ptr()
                self.slot_desc.append(d)
            self.span = torch.zeros((3, self.K), device=dev, dtype=torch.int64)
        tensors = [self.actor.dn.params, self.actor.m, self.actor.v, self.critic.dn.params, self.critic.m,
                   self.critic.v, self.std.dn.params, self.std.m, self.std.v, self.target.params, self.cnt]
        saved = [t.clone() for t in tensors]
        self.cnt.zero_()
        if pipe:
            self._cycle_critic()
            self._cycle_actor()
            self._std_errors(1)
            self._cycle_std_err()
        else:
            self._cycle_critic_actor()
        self._cycle_std()
        torch.cuda.synchronize()
        for t, sv in zip(tensors, saved):
            t.copy_(sv)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graphs = {}

        def chunk(fn, which, descs=None):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                _lib.call("cacto_counter_span", self.cnt[which:which + 1].data_ptr(), self.span[which].data_ptr(),
                          self.K, _stream())
                for i in range(self.K):
                    cp = self.span[which, i:i + 1].data_ptr()
                    if descs is None:
                        fn(cptr=cp)
                    else:
                        fn(cptr=cp, slot_desc=descs[i])
            return g

        with torch.cuda.stream(side):
            if pipe:
                graphs["c"] = chunk(self._cycle_critic, 0)
                for q in range(self.RC):  # actor chunk j reads ring chunk j % RC
                    graphs["a%d" % q] = chunk(self._cycle_actor, 2, self.slot_desc[q * self.K:(q + 1) * self.K])
                graphs["s"] = chunk(self._cycle_std_err, 1)
            else:
                for name, fn in (("ca", self._cycle_critic_actor), ("s", self._cycle_std)):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=side):
                        fn()
                    graphs[name] = g
        torch.cuda.current_stream().wait_stream(side)
        self._graphs = graphs

    def _run_pipelined(self, M):
        """critic chain | actor chain (behind it) | std chain (after the last critic
        chunk), on three streams; the ring holds RC chunks of K cycles' critics, so
        critic chunk j + RC waits for actor chunk j.  A partial last chunk runs eager."""
        g = self._graphs
        K = self.K
        main = torch.cuda.current_stream()
        if getattr(self, "_streams", None) is None:
            self._streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
        sc, sa, ss = self._streams
        for st in self._streams:
            st.wait_stream(main)
        nch = (M + K - 1) // K
        ev_c = [torch.cuda.Event() for _ in range(nch)]
        ev_a = [torch.cuda.Event() for _ in range(nch)]
        for j in range(nch):
            n = min(K, M - j * K)
            with torch.cuda.stream(sc):
                if j >= self.RC:
                    sc.wait_event(ev_a[j - self.RC])
                if n == K:
                    g["c"].replay()
                else:
                    for _ in range(n):
                        self._cycle_critic()
                ev_c[j].record(sc)
            with torch.cuda.stream(sa):
                sa.wait_event(ev_c[j])
                if n == K:
                    g["a%d" % (j % self.RC)].replay()
                else:
                    for _ in range(n):
                        self._cycle_actor()
                ev_a[j].record(sa)
        with torch.cuda.stream(ss):
            ss.wait_event(ev_c[nch - 1])
            self._std_errors(M)
            for j in range(nch):
                n = min(K, M - j * K)
                if n == K:
                    g["s"].replay()
                else:
                    for _ in range(n):
                        self._cycle_std_err()
        main.wait_stream(sa)
        main.wait_stream(ss)

    # -- the update loop ----------------------------------------------------------------
    def run(self, m_updates: int, rng: np.random.Generator):
        """M critic+actor cycles then M std cycles (trainer.py:209-233).  Returns
        (critic_losses [M], std_losses [M]) as float64 NumPy arrays."""
        M = int(m_updates)
        if M < 1:
            raise ValueError("m_updates must be >= 1")
        if self._cap_M < M:
            self._alloc(M)
        self._ensure_bc(max(n.step for n in (self.actor, self.critic, self.std)) + M)
        # the reference's minibatch stream: M lists for critic/actor, then M for std
        lists = np.stack([self.buffer.draw_indices(self.B, rng) for _ in range(2 * M)])
        stage = torch.zeros((2, self._cap_M, self.B), dtype=torch.int64)
        stage[0, :M] = torch.as_tensor(lists[:M])
        stage[1, :M] = torch.as_tensor(lists[M:])
        self.idx.copy_(stage.pin_memory(), non_blocking=True)
        for net in (self.actor, self.critic, self.std):
            net.base.fill_(net.step)
        if self.use_graphs and self._graphs is None:
            self._capture()
        self.cnt.zero_()
        if self._pipelined():
            self._run_pipelined(M)
        elif self.use_graphs:
            for _ in range(M):
                self._graphs["ca"].replay()
            for _ in range(M):
                self._graphs["s"].replay()
        else:
            for _ in range(M):
                self._cycle_critic_actor()
            for _ in range(M):
                self._cycle_std()
        for net in (self.actor, self.critic, self.std):
            net.step += M
        closs = self.closs[:M].to("cpu", torch.float64).numpy()
        sloss = self.sloss[:M].to("cpu", torch.float64).numpy()
        return closs, sloss

    # -- host views ------------------------------------------------------------------------
    def networks(self):
        """(actor, critic, critic_target, std) as reference-style networks."""
        return (self.actor.dn.to_mlp(), self.critic.dn.to_mlp(), self.target.to_mlp(), self.std.dn.to_mlp())

    def adam_host(self, net: _Net):
        return net.dn.unpack(net.m), net.dn.unpack(net.v), net.step
