"""Edge cases of the drop-in boundary (advisor findings, round 1):

  * `actor_rollout(..., t_hor=0)` from t0 < t_max returns the reference's 1-row
    trajectory (nets.py:403-423) and writes nothing past its outputs -- the C ABI
    uses CACTO_FULL_HORIZON (-1), not 0, for "every start to its own horizon";
  * `cacto_select_merge` with several padded runs (keep > shard size) is exact
    (the merge is stable for equal elements, so equal padding pairs of different
    runs land in distinct slots);
  * the UpdateEngine's Adam bias-correction tables grow on demand: a restored
    Adam step beyond the initial 2^17 table runs, with the reference's
    1 - beta**t values (nets.py:380-381).
"""

import numpy as np
from pathlib import Path
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import _lib, nets as B_nets, specs as B_specs, trainer as B_trainer  # noqa: E402
from oracle import nets as O_nets, envs as O_envs  # noqa: E402


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("t0", [0, 37, 100])
def test_rollout_t_hor_zero_is_one_row(prec, t0):
    old = P.get_precision()
    P.set_precision(prec)
    try:
        spec, fld = B_specs.config("dubins")
        rng = np.random.default_rng(3)
        c, h = B_specs.normalisation(spec)
        actor = B_nets.init_mlp([6, 64, 64, 64, 2], rng, head="tanh", out_scale=spec.u_bound, in_center=c, in_half=h)
        x0 = B_specs.TimeState(np.array([1.0, -2.0, 0.3, 0.1, -0.2]), t0)
        tr = B_nets.actor_rollout(actor, spec, x0, 0, fld)
        X, U, sc = O_nets.actor_rollout(actor, spec, x0.x, t0, 0, fld)
        assert tr.X.shape == (1, 5) and tr.U.shape == (0, 2) and tr.step_costs.shape == (1,)
        np.testing.assert_array_equal(tr.X, X.astype(np.float32) if prec == "fp32" else X)
        np.testing.assert_allclose(tr.step_costs, sc, rtol=1e-6 if prec == "fp32" else 1e-12)
        # batched, canaries around the outputs stay untouched
        N = 300
        xs = O_envs.sample_initial_states(spec, N, 5)
        r = B_nets.actor_rollout_batch(actor, spec, xs, t0, 0, fld, as_numpy=False)
        assert tuple(r["X"].shape) == (N, 1, 5) and tuple(r["step_costs"].shape) == (N, 1)
        np.testing.assert_array_equal(r["X"][:, 0].cpu().double().numpy(),
                                      torch.as_tensor(xs).to(r["X"].dtype).double().numpy())
        _, _, scr, Jr = O_nets.actor_rollout_batch(actor, spec, xs, t0, 0, fld)
        np.testing.assert_allclose(r["cost"].cpu().numpy(), Jr, rtol=1e-5 if prec == "fp32" else 1e-12)
    finally:
        P.set_precision(old)


def test_rollout_t_hor_zero_does_not_write_past_outputs():
    spec, fld = B_specs.config("pointmass")
    actor = B_nets.init_mlp([5, 64, 64, 64, 2], np.random.default_rng(1), head="tanh", out_scale=spec.u_bound)
    from paper_2602_19699_b200.device import device_net
    dn = device_net(actor, "fp32")
    N = 1000
    x0 = torch.as_tensor(O_envs.sample_initial_states(spec, N, 2)).cuda()
    arena = torch.full((4 * N * 8,), 7.0, device="cuda")   # X [N, 1, n] in the middle, canaries around
    X = arena[N * 8:N * 8 + N * 4]
    sc_arena = torch.full((3 * N,), 7.0, device="cuda")
    SC = sc_arena[N:2 * N]
    _lib.call("cacto_rollout", B_specs.system_struct(spec), B_specs.cost_struct(spec, fld), dn.desc, x0.data_ptr(),
              None, 5, N, 0, None, X.data_ptr(), SC.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.all(arena[:N * 8] == 7.0) and torch.all(arena[N * 8 + N * 4:] == 7.0)
    assert torch.all(sc_arena[:N] == 7.0) and torch.all(sc_arena[2 * N:] == 7.0)
    np.testing.assert_array_equal(X.view(N, 4).cpu().numpy(), x0.float().cpu().numpy())


def test_rollout_rejects_bad_sentinels():
    spec, fld = B_specs.config("pointmass")
    actor = B_nets.init_mlp([5, 8, 2], np.random.default_rng(1), head="tanh", out_scale=spec.u_bound)
    from paper_2602_19699_b200.device import device_net
    dn = device_net(actor, "fp32")
    x0 = torch.zeros((4, 4), device="cuda", dtype=torch.float64)
    with pytest.raises(ValueError):
        _lib.call("cacto_rollout", B_specs.system_struct(spec), None, dn.desc, x0.data_ptr(), None, 0, 4, -2,
                  None, None, None, None, torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("R,shard,keep", [(4, 100, 300), (3, 1000, 2500), (5, 7, 30), (4, 5000, 4096)])
def test_select_merge_padded_runs(dtype, R, shard, keep):
    """Each shard's local top-min(keep, shard) padded to `keep` rows (parallel.gather_winners
    layout: padding carries index -1), merged on device == the global stable argsort."""
    rng = np.random.default_rng(R * shard + keep)
    npdt, tdt = (np.float32, torch.float32) if dtype == "f32" else (np.float64, torch.float64)
    N = R * shard
    s = np.round(rng.normal(0, 1, N), 1).astype(npdt)
    s[rng.integers(0, N, 3)] = np.nan
    keep = min(keep, N)
    rs = np.full(R * keep, np.nan, dtype=npdt)
    ri = np.full(R * keep, -1, dtype=np.int64)
    for r in range(R):
        loc = s[r * shard:(r + 1) * shard]
        k = min(keep, shard)
        o = np.argsort(-loc, kind="stable")[:k]
        rs[r * keep:r * keep + k] = loc[o]
        ri[r * keep:r * keep + k] = r * keep + np.arange(k)          # positions (merge_positions)
    M = R * keep
    ws_bytes = 2 * (((M * 16) + 255) // 256) * 256
    ws = torch.full((ws_bytes,), 0xAB, device="cuda", dtype=torch.uint8)   # stale workspace bytes
    order = torch.empty(keep, device="cuda", dtype=torch.int64)
    top = torch.empty(keep, device="cuda", dtype=tdt)
    rs_d, ri_d = torch.as_tensor(rs).cuda(), torch.as_tensor(ri).cuda()   # alive across the launch
    _lib.call("cacto_select_merge", _lib.F32 if dtype == "f32" else _lib.F64, rs_d.data_ptr(), ri_d.data_ptr(), R,
              keep, order.data_ptr(), top.data_ptr(), ws.data_ptr(), ws_bytes, torch.cuda.current_stream().cuda_stream)
    pos = order.cpu().numpy()
    run, j = pos // keep, pos % keep
    got = np.array([r * shard + np.argsort(-s[r * shard:(r + 1) * shard], kind="stable")[jj]
                    for r, jj in zip(run, j)])
    np.testing.assert_array_equal(got, np.argsort(-s, kind="stable")[:keep])


def test_adam_tables_grow_past_initial_cap():
    from dp_setup import engine_setup
    old = P.get_precision()
    P.set_precision("fp64")
    try:
        eng, seed = engine_setup(32)
        start = (1 << 17) - 3
        for n in (eng.actor, eng.critic, eng.std):
            n.step = start
        closs, _ = eng.run(6, np.random.default_rng(seed))
        assert np.all(np.isfinite(closs))
        assert eng.critic.step == start + 6 and eng.max_steps >= start + 8
        bc1, bc2 = eng.bc[(0.9, 0.999)]
        t = start + 6
        assert bc1[t].item() == 1.0 - 0.9 ** float(t) and bc2[t].item() == 1.0 - 0.999 ** float(t)
    finally:
        P.set_precision(old)


@pytest.mark.parametrize("name,count,keep", [("pointmass", 750, 75), ("dubins", 65536, 6553),
                                             ("manipulator3", 20000, 2000)])
def test_device_sampled_bic_equals_host_sampled(name, count, keep):
    """trainer.py:183-186 on the device: the PCG64 replay gives the reference's
    candidates bit-exactly, so the kept starts (rows and order) equal the host
    path's select_initial_states_bic(sample_initial_states(...)) on the same scores."""
    from paper_2602_19699_b200 import specs
    spec, _ = B_specs.config(name)
    rng = np.random.default_rng(7)
    c, h = B_specs.normalisation(spec)
    std = B_nets.init_mlp([spec.n + 1, 64, 64, 64, 1], rng, head="std", in_center=c, in_half=h)
    seed = O_envs.seed_int(3, 1, 5)
    kept, order = B_trainer.sample_select_bic(spec, count, seed, std, keep)
    cands = [specs.TimeState(x, 0) for x in O_envs.sample_initial_states(spec, count, seed)]
    ref = B_trainer.select_initial_states_bic(cands, std, keep)
    np.testing.assert_array_equal(kept, np.stack([s.x for s in ref]))
    # and the device block itself is the host draw, bit for bit
    from paper_2602_19699_b200.sampling import sample_initial_states_device
    x = sample_initial_states_device(spec, count, seed, first_row=count // 3, rows=count // 2).cpu().numpy()
    np.testing.assert_array_equal(x, O_envs.sample_initial_states(spec, count, seed)[count // 3:count // 3 + count // 2])


@pytest.mark.parametrize("graphs", [True, False])
def test_training_state_resume_is_bitwise(graphs, tmp_path):
    """save_training_state / load_training_state (checkpoint.py): networks in the
    reference's JSON format, Adam moments + steps, the ring in physical slot order
    and the minibatch generator state -> the resumed run equals the uninterrupted
    one bit for bit (fp64)."""
    from dp_setup import engine_setup
    from paper_2602_19699_b200 import checkpoint
    old = P.get_precision()
    P.set_precision("fp64")
    try:
        eng, seed = engine_setup(40)
        eng.use_graphs = graphs
        rng = np.random.default_rng(seed)
        eng.run(3, rng)
        checkpoint.save_training_state(tmp_path, eng, rng, model_name="pointmass")
        c1, s1 = eng.run(4, rng)
        ref = [np.asarray(p) for n in eng.networks() for p in n.flat_params()]
        spec, fld = B_specs.config("pointmass")
        eng2, rng2 = checkpoint.load_training_state(tmp_path, spec, fld, use_graphs=graphs)
        c2, s2 = eng2.run(4, rng2)
        np.testing.assert_array_equal(c1, c2)
        np.testing.assert_array_equal(s1, s2)
        got = [np.asarray(p) for n in eng2.networks() for p in n.flat_params()]
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)
        assert eng2.critic.step == eng.critic.step
    finally:
        P.set_precision(old)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_pipelined_update_loop_is_bitwise_the_sequential_one(prec):
    """The graph schedule runs the critic chain ahead of the actor chain (each actor
    update reads a ring copy of the critic of its own cycle) and the std chain beside
    the actor chain's tail: same kernels on the same inputs, so the losses and every
    parameter equal the plain sequential loop bit for bit (M = 37: two full 16-cycle
    chunks, a partial one, and a ring wrap)."""
    from dp_setup import engine_setup
    old = P.get_precision()
    P.set_precision(prec)
    try:
        res = []
        for graphs in (False, True):
            eng, seed = engine_setup(64)
            eng.use_graphs = graphs
            rng = np.random.default_rng(seed)
            c1, s1 = eng.run(37, rng)
            c2, s2 = eng.run(5, rng)           # a second run continues the streams
            res.append((c1, s1, c2, s2, [np.asarray(p) for n in eng.networks() for p in n.flat_params()],
                        eng.actor.step))
        a, b = res
        for x, y in zip(a[:4], b[:4]):
            np.testing.assert_array_equal(x, y)
        for x, y in zip(a[4], b[4]):
            np.testing.assert_array_equal(x, y)
        assert a[5] == b[5] == 42
    finally:
        P.set_precision(old)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_std_loss_from_precomputed_errors_is_bitwise(prec):
    """cacto_value_errors + cacto_std_loss_err (the update loop's std phase) equal
    cacto_std_loss (critic forward inside) bit for bit, cycle by cycle."""
    import ctypes
    from paper_2602_19699_b200.device import DeviceNet, torch_dtype
    from dp_setup import engine_setup
    old = P.get_precision()
    P.set_precision(prec)
    try:
        eng, seed = engine_setup(64)
        M, B = 5, 64
        rng = np.random.default_rng(seed)
        lists = np.stack([eng.buffer.draw_indices(B, rng) for _ in range(M)])
        idx = torch.as_tensor(lists).cuda()
        cnt = torch.zeros(1, device="cuda", dtype=torch.int64)
        st = torch.cuda.current_stream().cuda_stream
        ws = torch.empty(_lib.load().cacto_loss_workspace_bytes(eng.std.dn.desc, B), device="cuda", dtype=torch.uint8)
        dall = eng.buffer.ring_desc(idx, rows=M * B)
        err = torch.empty(M * B, device="cuda", dtype=torch_dtype(prec))
        _lib.call("cacto_value_errors", eng.critic.dn.desc, dall, err.data_ptr(), st)
        for c in range(M):
            cnt.fill_(c)
            d = eng.buffer.ring_desc(idx, rows=B)
            d.cycle = cnt.data_ptr()
            d.idx_stride = B
            g = []
            for fn, args in (("cacto_std_loss", (eng.std.dn.desc, eng.critic.dn.desc, d)),
                             ("cacto_std_loss_err", (eng.std.dn.desc, err.data_ptr(), d))):
                npart = ctypes.c_int32(0)
                _lib.call(fn, *args, ws.data_ptr(), ws.numel(), npart, st)
                out = torch.empty(eng.std.dn.count + 1, device="cuda", dtype=torch_dtype(prec))
                _lib.call("cacto_reduce_grads", eng.std.dn.desc.dtype, ws.data_ptr(), npart.value, eng.std.dn.count,
                          out.data_ptr(), out[eng.std.dn.count:].data_ptr(), st)
                g.append(out.cpu().numpy())
            np.testing.assert_array_equal(g[0], g[1])
    finally:
        P.set_precision(old)


def test_critic_wgrad_reduction_matches_gemm_path():
    """The fp16-pair tensor-core weight-gradient reduction (default) and the 3xTF32 GEMM
    reductions (CACTO_CRITIC_WGRAD=0) agree to fp32 accuracy, and both match the
    float64 oracle within the SURVEY 8(c) bounds (loss 1e-5, grads 1e-4 of max|g|)."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2602_19699_b200 as P
from paper_2602_19699_b200 import nets as B_nets, specs as B_specs
from oracle import nets as O_nets
from types import SimpleNamespace
P.set_precision('fp32')
spec, fld = B_specs.config('manipulator3')
rng = np.random.default_rng(21)
c, h = B_specs.normalisation(spec)
critic = B_nets.init_mlp([7, 64, 64, 64, 1], rng, in_center=c, in_half=h)
target = B_nets.init_mlp([7, 64, 64, 64, 1], rng, in_center=c, in_half=h)
B = 20000
lo, hi = B_specs.region_box(spec)
xa = np.concatenate([rng.uniform(size=(B, 6)) * (hi - lo) + lo, rng.integers(0, 100, (B, 1))], 1)
xk = np.concatenate([rng.uniform(size=(B, 6)) * (hi - lo) + lo, rng.integers(1, 101, (B, 1))], 1)
b = SimpleNamespace(xa=xa, u=rng.normal(size=(B, 3)), v_bar=rng.normal(size=B) * 30, v_bar_x=rng.normal(size=(B, 6)),
                    xa_plus_k=xk, t_max=100)
loss, g = B_nets.critic_loss(critic, target, b, 0.7, True)
np.savez(sys.argv[1], loss=loss, *g)
"""
    outs = []
    for v in ("1", "0"):
        path = f"/tmp/wgrad_{v}.npz"
        env = dict(os.environ, CACTO_CRITIC_WGRAD=v)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, cwd=str(Path(__file__).parents[1]))
        outs.append(np.load(path))
    from types import SimpleNamespace
    spec, fld = B_specs.config("manipulator3")
    rng = np.random.default_rng(21)
    c, h = B_specs.normalisation(spec)
    critic = B_nets.init_mlp([7, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    target = B_nets.init_mlp([7, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    B = 20000
    lo, hi = B_specs.region_box(spec)
    xa = np.concatenate([rng.uniform(size=(B, 6)) * (hi - lo) + lo, rng.integers(0, 100, (B, 1))], 1)
    xk = np.concatenate([rng.uniform(size=(B, 6)) * (hi - lo) + lo, rng.integers(1, 101, (B, 1))], 1)
    b = SimpleNamespace(xa=xa, u=rng.normal(size=(B, 3)), v_bar=rng.normal(size=B) * 30,
                        v_bar_x=rng.normal(size=(B, 6)), xa_plus_k=xk, t_max=100)
    ref_loss, ref_g = O_nets.critic_loss(critic, target, b, 0.7, True)
    scale = max(np.abs(r).max() for r in ref_g)
    for o in outs:
        assert abs(float(o["loss"]) - ref_loss) <= 1e-5 * abs(ref_loss)
        for i, r in enumerate(ref_g):
            assert np.abs(o[f"arr_{i}"] - r).max() <= 1e-4 * scale, i


@pytest.mark.parametrize("zero_copy", [False, True])
def test_bic_pipeline_host_buffers_zero_copy(zero_copy, monkeypatch):
    """BicPipeline.run with a pinned HOST x0 (read zero-copy by the rollout kernel) and
    a pinned host warm-start buffer (chunked take + copy-engine copies overlapped on a
    side stream, or written zero-copy by the take kernel) gives exactly the
    device-resident results."""
    from bench import make_nets, candidates
    monkeypatch.setattr(B_trainer, "_WARM_ZC", zero_copy)
    old = P.get_precision()
    P.set_precision("fp32")
    try:
        spec, fld = B_specs.config("dubins")
        actor, critic, std = make_nets(spec)
        N, keep = 20000, 2000
        x0h = torch.from_numpy(candidates(spec, 0, N)).pin_memory()
        pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
        ref = pipe.run(x0h.cuda(), keep)
        Uh = torch.empty((keep, spec.t_max, spec.m), dtype=torch.float32).pin_memory()
        got = pipe.run(x0h, keep, u_out=Uh)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got["order"].cpu().numpy(), ref["order"].cpu().numpy())
        np.testing.assert_array_equal(got["scores"].cpu().numpy(), ref["scores"].cpu().numpy())
        np.testing.assert_array_equal(Uh.numpy(), ref["U"].cpu().numpy())
        assert got["U"].data_ptr() == Uh.data_ptr()
    finally:
        P.set_precision(old)
