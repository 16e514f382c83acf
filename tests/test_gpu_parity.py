"""GPU parity: the sm_100a kernels (through the C ABI) against the golden
fixtures produced by the reference and against the CPU oracle.

Tolerances (stated per test):
  fp64 mode  rollouts 1e-10 rel (manipulator3 1e-8: chaotic amplification of the
             closed-form 3x3 solve vs LAPACK), losses / grads 1e-10, Adam and
             Polyak bit-exact, select / gather / sampling bit-exact.
  fp32 mode  rollout cost rel 2e-5 (pointmass, dubins, aliengo; 3000-start dubins
             batch: median 1e-6 / p99 1e-4 / max 2e-3, chaotic tail); manipulator3
             median 1e-4 / max 0.1 (chaotic tail); losses 1e-6 rel;
             grads 1e-5 of max|grad| (the reference FD metric, test_nets.py:45-49).
  The SURVEY 8(c) contract itself, on the bench path at bench sizes, is
  tests/test_gpu_contract.py.
"""

import numpy as np
import pytest

import golden_utils as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the -m gpu suite only runs on the B200 box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import buffer as B_buffer  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets  # noqa: E402
from paper_2602_19699_b200 import specs as B_specs  # noqa: E402
from paper_2602_19699_b200 import trainer as B_trainer  # noqa: E402
from oracle import nets as O_nets  # noqa: E402
from oracle import select as O_select  # noqa: E402
from oracle import envs as O_envs  # noqa: E402


class Net(G.Net):
    def with_params(self, params):
        from dataclasses import replace
        L = len(self.weights)
        return replace(self, weights=tuple(params[2 * i] for i in range(L)),
                       biases=tuple(params[2 * i + 1] for i in range(L)))


def net(d, prefix):
    g = G.net(d, prefix)
    return Net(**{k: getattr(g, k) for k in ("weights", "biases", "activation", "head", "out_scale",
                                             "sigma_min", "in_center", "in_half")})


@pytest.fixture(params=["fp64", "fp32"])
def precision(request):
    old = P.get_precision()
    P.set_precision(request.param)
    yield request.param
    P.set_precision(old)


@pytest.fixture
def fp64():
    old = P.get_precision()
    P.set_precision("fp64")
    yield "fp64"
    P.set_precision(old)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def grads_close(got, ref, tol):
    scale = max(1e-12, max(np.abs(r).max() for r in ref))
    for g, r in zip(got, ref):
        assert g.shape == r.shape
        assert np.abs(g - r).max() / scale < tol


# ---- K1 rollouts -----------------------------------------------------------------

@pytest.mark.parametrize("name", G.SYSTEMS)
@pytest.mark.parametrize("tag", ["init", "trained"])
def test_batched_rollout_vs_reference(name, tag, precision):
    d = G.load("rollout")
    spec, fld = G.spec(d, f"{name}_spec"), G.field(d, f"{name}_field")
    key = f"{name}_{tag}"
    x0, t0 = d[f"{key}_x0"], d[f"{key}_t0"]
    r = B_nets.actor_rollout_batch(net(d, f"{key}_actor"), spec, x0, t0, None, fld)
    ref_cost = d[f"{key}_cost"]
    err = np.abs(r["cost"] - ref_cost) / np.maximum(1.0, np.abs(ref_cost))
    if precision == "fp64":
        tol = 1e-8 if name == "manipulator3" else 1e-10
        assert err.max() < tol
        mask = ~np.isnan(d[f"{key}_X"])
        assert rel(r["X"][mask], d[f"{key}_X"][mask]) < tol
        mu = ~np.isnan(d[f"{key}_U"])
        assert rel(r["U"][mu], d[f"{key}_U"][mu]) < tol
        ms = ~np.isnan(d[f"{key}_step_costs"])
        np.testing.assert_array_equal(np.isnan(r["step_costs"]), ~ms)
    elif name == "manipulator3":
        assert np.median(err) < 1e-4 and err.max() < 1e-1
    else:
        assert err.max() < 2e-5


def test_single_rollout_dropin_and_no_field(fp64):
    d = G.load("rollout")
    spec, fld = G.spec(d, "dubins_spec"), G.field(d, "dubins_field")
    from paper_2602_19699_b200.specs import TimeState
    x0 = TimeState(d["dubins_init_x0"][0], 0)
    tr = B_nets.actor_rollout(net(d, "dubins_init_actor"), spec, x0, spec.t_max)
    np.testing.assert_array_equal(tr.step_costs, np.zeros(spec.t_max + 1))
    assert rel(tr.U, d["dubins_nofield_U"]) < 1e-9
    tr2 = B_nets.actor_rollout(net(d, "dubins_init_actor"), spec, x0, spec.t_max, fld)
    assert abs(tr2.cost - d["dubins_init_cost"][0]) < 1e-9 * max(1.0, abs(d["dubins_init_cost"][0]))


def test_rollout_rejects_horizon_overflow():
    d = G.load("rollout")
    spec = G.spec(d, "pointmass_spec")
    from paper_2602_19699_b200.specs import TimeState
    with pytest.raises(ValueError):
        B_nets.actor_rollout(net(d, "pointmass_init_actor"), spec, TimeState(np.zeros(4), 30), 31)


def test_zero_actor_rollout_is_naive_warm_start_bitwise(fp64):
    # test_nets.py:352-367
    spec = B_specs.default_model("pointmass")
    actor = B_nets.init_mlp([5, 8, 2], np.random.default_rng(19), head="tanh", out_scale=spec.u_bound)
    p = list(actor.flat_params())
    p[-2] = np.zeros_like(p[-2])
    p[-1] = np.zeros_like(p[-1])
    actor = actor.with_params(p)
    x0 = B_specs.TimeState(np.array([3.0, -2.0, 1.0, 0.5]), 0)
    tr = B_nets.actor_rollout(actor, spec, x0, spec.t_max)
    np.testing.assert_array_equal(tr.U, np.zeros((spec.t_max, 2)))
    x = x0.x
    for k in range(spec.t_max):
        x = O_envs.step_x(spec, x, np.zeros(2))
        np.testing.assert_array_equal(tr.X[k + 1], x)


def test_rollout_large_batch_vs_oracle(precision):
    spec, fld = B_specs.config("dubins")
    rng = np.random.default_rng(5)
    c, h = B_specs.normalisation(spec)
    actor = B_nets.init_mlp([6, 64, 64, 64, 2], rng, head="tanh", out_scale=spec.u_bound, in_center=c,
                            in_half=h)
    actor = actor.with_params([q * (5.0 if i == 6 else 1.0) for i, q in enumerate(actor.flat_params())])
    x0 = O_envs.sample_initial_states(spec, 3000, 77)
    r = B_nets.actor_rollout_batch(actor, spec, x0, 0, None, fld, emit=("cost",))
    _, _, _, ref = O_nets.actor_rollout_batch(actor, spec, x0, 0, spec.t_max, fld)
    err = np.abs(r["cost"] - ref) / np.maximum(1.0, np.abs(ref))
    if precision == "fp64":
        assert err.max() < 1e-9
    else:
        # fp32 (3xTF32 tensor-core or FFMA): most trajectories agree to ~1e-6;
        # the few that graze an obstacle boundary amplify rounding (chaotic tail)
        assert np.median(err) < 1e-5 and np.quantile(err, 0.99) < 1e-4 and err.max() < 2e-3


# ---- forward / jacobian -----------------------------------------------------------

@pytest.mark.parametrize("key", ["lin3", "tanh", "std", "lin1", "tanh3", "single"])
def test_forward_and_jacobian(key, precision):
    d = G.load("nets")
    n_ = net(d, f"fwd_{key}")
    x = d[f"fwd_{key}_x"]
    tol = 1e-12 if precision == "fp64" else 1e-5
    assert rel(B_nets.mlp_forward(n_, x), d[f"fwd_{key}_y"]) < tol
    assert rel(B_nets.mlp_input_gradient(n_, x), d[f"fwd_{key}_jac"]) < tol * 10
    if f"fwd_{key}_v" in d:
        v, g = B_nets.value_and_state_grad(n_, x)
        assert rel(v, d[f"fwd_{key}_v"]) < tol
        assert rel(g, d[f"fwd_{key}_g"]) < tol * 10


def test_forward_rejects_dim_mismatch():
    d = G.load("nets")
    with pytest.raises(ValueError):
        B_nets.mlp_forward(net(d, "fwd_lin3"), np.ones(5))


# ---- losses ----------------------------------------------------------------------

@pytest.mark.parametrize("key", ["b64", "b200"])
@pytest.mark.parametrize("boot", [0, 1])
def test_critic_loss(key, boot, precision):
    d = G.load("losses")
    critic, target = net(d, "critic_net"), net(d, "critic_target")
    batch = G.batch(d, f"critic_{key}")
    loss, grads = B_nets.critic_loss(critic, target if boot else None, batch, 0.7, bool(boot))
    ref = float(d[f"critic_{key}_boot{boot}_loss"])
    ref_g = G.grads(d, f"critic_{key}_boot{boot}", 8)
    if precision == "fp64":
        assert loss == pytest.approx(ref, rel=1e-11)
        grads_close(grads, ref_g, 1e-10)
    else:
        assert loss == pytest.approx(ref, rel=1e-6)
        grads_close(grads, ref_g, 1e-5)


def test_critic_loss_small_odd_shape(precision):
    d = G.load("losses")
    loss, grads = B_nets.critic_loss(net(d, "critic_small_net"), net(d, "critic_small_target"),
                                     G.batch(d, "critic_small"), 0.5, True)
    assert loss == pytest.approx(float(d["critic_small_loss"]), rel=1e-11 if precision == "fp64" else 1e-6)
    grads_close(grads, G.grads(d, "critic_small", 6), 1e-10 if precision == "fp64" else 1e-5)


def test_critic_loss_perfect_critic_is_zero(fp64):
    # test_nets.py:108-118
    rng = np.random.default_rng(5)
    critic = B_nets.init_mlp([4, 10, 1], rng)
    xa = rng.normal(0.0, 1.0, (6, 4))
    xa[:, -1] = 3.0
    v, g = O_nets.value_and_state_grad(critic, xa)
    batch = B_buffer.SampleBatch(xa, np.zeros((6, 1)), v, g[:, :-1], xa, t_max=50)
    loss, grads = B_nets.critic_loss(critic, None, batch, k_s=0.7, gamma_bootstrap=False)
    assert loss < 1e-24
    assert max(np.abs(x).max() for x in grads) < 1e-11


def test_critic_loss_rejects_empty_batch():
    critic = B_nets.init_mlp([3, 8, 1], np.random.default_rng(0))
    empty = B_buffer.SampleBatch(np.zeros((0, 3)), np.zeros((0, 1)), np.zeros(0), np.zeros((0, 2)),
                                 np.zeros((0, 3)), t_max=5)
    with pytest.raises(ValueError):
        B_nets.critic_loss(critic, None, empty, 1.0, False)


@pytest.mark.parametrize("key", ["b64", "b200"])
def test_std_loss(key, precision):
    d = G.load("losses")
    loss, grads = B_nets.std_critic_loss(net(d, "std_net"), net(d, "critic_net"), G.batch(d, f"critic_{key}"))
    assert loss == pytest.approx(float(d[f"std_{key}_loss"]), rel=1e-11 if precision == "fp64" else 1e-6)
    grads_close(grads, G.grads(d, f"std_{key}", 8), 1e-10 if precision == "fp64" else 1e-5)


@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3", "aliengo_lipm"])
def test_actor_loss(name, precision):
    d = G.load("losses")
    r = G.load("rollout")
    spec, fld = G.spec(r, f"{name}_spec"), G.field(r, f"{name}_field")
    batch = type("B", (), {"xa": d[f"actor_{name}_xa"]})()
    loss, grads, skipped = B_nets.actor_loss(net(d, f"actor_{name}_actor"), net(d, f"actor_{name}_critic"),
                                             spec, fld, batch)
    assert skipped == int(d[f"actor_{name}_skipped"])
    ref = float(d[f"actor_{name}_loss"])
    if precision == "fp64":
        assert loss == pytest.approx(ref, rel=1e-10)
        grads_close(grads, G.grads(d, f"actor_{name}", 8), 1e-9)
    else:
        assert loss == pytest.approx(ref, rel=1e-6)
        grads_close(grads, G.grads(d, f"actor_{name}", 8), 1e-5)


def test_actor_loss_all_at_horizon_raises():
    spec = B_specs.default_model("pointmass")
    _, fld = B_specs.config("pointmass")
    a = B_nets.init_mlp([5, 10, 8, 2], np.random.default_rng(11), head="tanh", out_scale=spec.u_bound)
    c = B_nets.init_mlp([5, 10, 1], np.random.default_rng(12))
    with pytest.raises(ValueError):
        B_nets.actor_loss(a, c, spec, fld, [B_specs.TimeState(np.zeros(4), 60)])


# ---- optimizer --------------------------------------------------------------------

def test_adam_sequence_bitwise(fp64):
    d = G.load("optim")
    params = [d["adam_p0_0"], d["adam_p0_1"]]
    state = B_nets.AdamState.init(params, lr=3e-3)
    for k in range(5):
        params, state = B_nets.adam_step(params, state, [d[f"adam_g{k}_0"], d[f"adam_g{k}_1"]])
        np.testing.assert_array_equal(params[0], d[f"adam_p{k + 1}_0"])
        np.testing.assert_array_equal(params[1], d[f"adam_p{k + 1}_1"])


def test_polyak_bitwise(fp64):
    d = G.load("optim")
    mixed = B_nets.polyak(net(d, "polyak_a"), net(d, "polyak_b"), 0.25)
    for a, b in zip(mixed.flat_params(), G.grads(d, "polyak_mix", 4)):
        np.testing.assert_array_equal(a, b)


# ---- select ------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3"])
def test_select_bitwise_given_reference_scores(name, precision):
    d = G.load("select")
    dt = torch.float64 if precision == "fp64" else torch.float32
    s = d[f"select_{name}_scores"]
    order, _ = B_trainer.select_topk_device(torch.as_tensor(s).to("cuda", dt), 75)
    ref = O_select.select_order(s.astype(np.float32) if precision == "fp32" else s, 75)
    np.testing.assert_array_equal(order.cpu().numpy(), ref)
    if precision == "fp64":
        np.testing.assert_array_equal(order.cpu().numpy(), d[f"select_{name}_order"])


@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3"])
def test_select_initial_states_bic_dropin(name, fp64):
    d = G.load("select")
    cands = [B_specs.TimeState(x, 0) for x in d[f"select_{name}_cands"]]
    kept = B_trainer.select_initial_states_bic(cands, net(d, f"select_{name}_std"), 75)
    got = [next(i for i, c in enumerate(cands) if c is k) for k in kept]
    np.testing.assert_array_equal(got, d[f"select_{name}_order"])


def test_select_ties_nan_signed_zero(precision):
    d = G.load("select")
    dt = torch.float64 if precision == "fp64" else torch.float32
    vals = d["select_ties_vals"]
    order, _ = B_trainer.select_topk_device(torch.as_tensor(vals).to("cuda", dt), 12)
    np.testing.assert_array_equal(order.cpu().numpy(), d["select_ties_order"])


@pytest.mark.parametrize("N,keep", [(1, 1), (65, 3), (750, 75), (1000, 1000), (2048, 300), (2049, 2049), (65536, 6553),
                                    (1 << 20, 104857), (300001, 7)])
def test_select_large_with_heavy_ties(N, keep, precision):
    rng = np.random.default_rng(N)
    s = np.round(rng.normal(0, 1, N), 2)          # ~600 distinct values -> massive ties
    s[rng.integers(0, N, N // 100)] = np.nan
    s[rng.integers(0, N, N // 100)] = -0.0
    dt = torch.float64 if precision == "fp64" else torch.float32
    ref_s = s.astype(np.float32) if precision == "fp32" else s
    order, top = B_trainer.select_topk_device(torch.as_tensor(ref_s).to("cuda", dt), keep)
    want = np.argsort(-ref_s, kind="stable")[:keep]
    np.testing.assert_array_equal(order.cpu().numpy(), want)
    np.testing.assert_array_equal(top.cpu().numpy(), ref_s[want])  # NaN == NaN, -0.0 == 0.0


def test_select_rejects_keep_too_large():
    with pytest.raises(ValueError):
        B_trainer.select_topk_device(torch.zeros(3, device="cuda"), 4)


def test_select_merge_of_shards_equals_global(precision):
    from paper_2602_19699_b200 import _lib
    rng = np.random.default_rng(3)
    dt = torch.float64 if precision == "fp64" else torch.float32
    N, R, keep = 40000, 4, 3000
    s = np.round(rng.normal(0, 1, N), 2).astype(np.float32 if precision == "fp32" else np.float64)
    shard = N // R
    runs_s, runs_i = [], []
    for r in range(R):
        o, t = B_trainer.select_topk_device(torch.as_tensor(s[r * shard:(r + 1) * shard]).to("cuda", dt), keep,
                                            base_index=r * shard)
        runs_s.append(t)
        runs_i.append(o)
    rs, ri = torch.cat(runs_s), torch.cat(runs_i)
    ws = torch.empty(2 * 256 + 2 * R * keep * 16 + 4096, device="cuda", dtype=torch.uint8)
    order = torch.empty(keep, device="cuda", dtype=torch.int64)
    top = torch.empty(keep, device="cuda", dtype=dt)
    _lib.call("cacto_select_merge", _lib.F32 if precision == "fp32" else _lib.F64, rs.data_ptr(), ri.data_ptr(),
              R, keep, order.data_ptr(), top.data_ptr(), ws.data_ptr(), ws.numel(),
              torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(order.cpu().numpy(), np.argsort(-s, kind="stable")[:keep])


# ---- gather / ring / sampling --------------------------------------------------------

def test_buffer_ring_and_minibatches_bitwise(fp64):
    d = G.load("buffer")
    rows = G.batch(d, "buf_rows")
    buf = B_buffer.ReplayBuffer(3, 2, 60, capacity=int(d["buf_capacity"]))
    cut = lambda a, b: B_buffer.SampleBatch(rows.xa[a:b], rows.u[a:b], rows.v_bar[a:b], rows.v_bar_x[a:b],  # noqa
                                            rows.xa_plus_k[a:b], 60)
    buf.push_many(cut(0, 40))
    buf.push_many(cut(40, 83))
    g = np.random.default_rng(int(d["buf_rng_seed"]))
    for mb, bsz in (("buf_mb1", 64), ("buf_mb2", 7)):
        got = buf.sample_minibatch(bsz, g)
        ref = G.batch(d, mb)
        for k in ("xa", "u", "v_bar", "v_bar_x", "xa_plus_k"):
            np.testing.assert_array_equal(getattr(got, k), getattr(ref, k))


def test_buffer_empty_raises():
    buf = B_buffer.ReplayBuffer(3, 2, 60, capacity=4)
    with pytest.raises(ValueError):
        buf.sample_minibatch(4, np.random.default_rng(0))


@pytest.mark.parametrize("name", G.SYSTEMS)
def test_device_pcg64_sampling_bitwise(name):
    from paper_2602_19699_b200 import _lib
    d, r = G.load("sampling"), G.load("rollout")
    spec = G.spec(r, f"{name}_spec")
    st = np.random.PCG64(int(d[f"sample_{name}_seed"])).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    lo, hi = O_envs.region_box(spec)
    x = torch.empty((40, spec.n), device="cuda", dtype=torch.float64)
    lo_d, hi_d = torch.as_tensor(lo).cuda(), torch.as_tensor(hi).cuda()
    M = (1 << 64) - 1
    _lib.call("cacto_sample_states", s >> 64, s & M, inc >> 64, inc & M, 0, 40, spec.n, lo_d.data_ptr(),
              hi_d.data_ptr(), x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(x.cpu().numpy(), d[f"sample_{name}_x"])
    # a shard starting at row 13 reproduces rows 13.. of the same stream
    x2 = torch.empty((27, spec.n), device="cuda", dtype=torch.float64)
    _lib.call("cacto_sample_states", s >> 64, s & M, inc >> 64, inc & M, 13, 27, spec.n, lo_d.data_ptr(),
              hi_d.data_ptr(), x2.data_ptr(), torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(x2.cpu().numpy(), d[f"sample_{name}_x"][13:])


# ---- pipeline -------------------------------------------------------------------------

@pytest.mark.parametrize("mode", ["gap", "std", "std_x_gap"])
def test_bic_pipeline_vs_oracle_composition(mode, fp64):
    spec, fld = B_specs.config("pointmass")
    rng = np.random.default_rng(8)
    c, h = B_specs.normalisation(spec)
    actor = B_nets.init_mlp([5, 64, 64, 64, 2], rng, head="tanh", out_scale=spec.u_bound, in_center=c, in_half=h)
    critic = B_nets.init_mlp([5, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    std = B_nets.init_mlp([5, 64, 64, 64, 1], rng, head="std", in_center=c, in_half=h)
    x0 = O_envs.sample_initial_states(spec, 750, 4)
    pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode=mode)
    out = pipe.run(torch.as_tensor(x0).cuda(), keep=75)
    xa = O_select.augmented(x0)
    _, _, _, J = O_nets.actor_rollout_batch(actor, spec, x0, 0, spec.t_max, fld)
    if mode == "gap":
        s = O_select.gap_scores(critic, xa, J)
    elif mode == "std":
        s = O_select.std_scores(std, xa)
    else:
        s = O_select.std_scores(std, xa) * O_select.gap_scores(critic, xa, J)
    ref = O_select.select_order(s, 75)
    got = out["order"].cpu().numpy()
    # identical up to near-ties (|ds| < 1e-9 relative) -- check set and scores
    np.testing.assert_allclose(out["scores"].cpu().numpy(), s[ref], rtol=1e-9)
    assert (got == ref).mean() > 0.97
    U = out["U"].cpu().numpy()
    _, U_ref, _, _ = O_nets.actor_rollout_batch(actor, spec, x0[got], 0, spec.t_max, None)
    assert rel(U, U_ref) < 1e-9


@pytest.mark.parametrize("mode", ["gap", "std_x_gap"])
def test_bic_pipeline_warm_starts_equal_rerollout(mode, precision):
    # gap modes keep every candidate's controls from the cost rollout (time-major)
    # and take the kept columns: identical to rolling the kept starts out again
    spec, fld = B_specs.config("dubins")
    rng = np.random.default_rng(18)
    c, h = B_specs.normalisation(spec)
    d = spec.n + 1
    actor = B_nets.init_mlp([d, 64, 64, 64, spec.m], rng, head="tanh", out_scale=spec.u_bound, in_center=c,
                            in_half=h)
    actor = actor.with_params([q * (5.0 if i == 6 else 1.0) for i, q in enumerate(actor.flat_params())])
    critic = B_nets.init_mlp([d, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    std = B_nets.init_mlp([d, 64, 64, 64, 1], rng, head="std", in_center=c, in_half=h)
    x0 = torch.as_tensor(O_envs.sample_initial_states(spec, 40000, 3)).cuda()
    pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode=mode)
    out = pipe.run(x0, keep=4000)
    kept = x0.index_select(0, out["order"]).cpu().numpy()
    U = B_nets.actor_rollout_batch(actor, spec, kept, 0, None, None, emit=("U",))["U"]
    np.testing.assert_array_equal(out["U"].cpu().numpy(), U)


@pytest.mark.parametrize("mode", ["gap", "std_x_gap"])
def test_fused_rollout_scores_match_separate_kernels(mode):
    # cacto_rollout_score (K1 + K2 in one tensor-core launch) against the rollout
    # followed by the separate score kernel on the same starts (fp32)
    old = P.get_precision()
    P.set_precision("fp32")
    try:
        spec, fld = B_specs.config("dubins")
        rng = np.random.default_rng(19)
        c, h = B_specs.normalisation(spec)
        d = spec.n + 1
        actor = B_nets.init_mlp([d, 64, 64, 64, spec.m], rng, head="tanh", out_scale=spec.u_bound, in_center=c,
                                in_half=h)
        critic = B_nets.init_mlp([d, 64, 64, 64, 1], rng, in_center=c, in_half=h)
        std = B_nets.init_mlp([d, 64, 64, 64, 1], rng, head="std", in_center=c, in_half=h)
        x0 = torch.as_tensor(O_envs.sample_initial_states(spec, 20000, 5)).cuda()
        pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode=mode)
        scores, cost = pipe._fused(x0, 0, False)
        assert scores is not None, "tensor-core fused path expected for fp32 3x64 nets"
        cost2 = pipe.rollout_costs(x0, 0)
        np.testing.assert_array_equal(cost.cpu().numpy(), cost2.cpu().numpy())
        xa = torch.cat([x0.float(), torch.zeros(x0.shape[0], 1, device="cuda")], 1)
        s2 = B_trainer.score_device(mode, xa, pipe.std, pipe.critic, cost2)
        np.testing.assert_allclose(scores.cpu().numpy(), s2.cpu().numpy(), rtol=2e-5, atol=1e-5)
    finally:
        P.set_precision(old)


# ---- device-resident update loop (trainer.py:208-234) ------------------------------

def _oracle_update_loop(spec, fld, nets0, rows, B, M, seed, k_s=1.0, tau=0.005, lrs=(5e-4, 1e-3, 1e-3)):
    from types import SimpleNamespace
    from oracle import buffer as O_buffer
    actor, critic, target, std = [list(n.flat_params()) for n in nets0]
    mk = lambda tmpl, p: tmpl.with_params(p)  # noqa: E731
    ring = O_buffer.Ring(spec.n, spec.m, 1 << 12)
    ring.push_many(rows)
    rng = np.random.default_rng(seed)
    st = {k: ([np.zeros_like(p) for p in v], [np.zeros_like(p) for p in v], 0)
          for k, v in (("a", actor), ("c", critic), ("s", std))}
    closs, sloss = [], []
    lists = [ring.draw_indices(B, rng) for _ in range(2 * M)]

    def batch(idx):
        g = ring.gather(idx)
        return SimpleNamespace(t_max=spec.t_max, **g)

    for i in range(M):
        b = batch(lists[i])
        l, g = O_nets.critic_loss(mk(nets0[1], critic), mk(nets0[2], target), b, k_s, True)
        m_, v_, t_ = st["c"]
        critic, m_, v_ = O_nets.adam_step(critic, m_, v_, g, t_, lrs[1])
        st["c"] = (m_, v_, t_ + 1)
        target = O_nets.polyak(target, critic, tau)
        _, ga, _ = O_nets.actor_loss(mk(nets0[0], actor), mk(nets0[1], critic), spec, fld, b.xa)
        m_, v_, t_ = st["a"]
        actor, m_, v_ = O_nets.adam_step(actor, m_, v_, ga, t_, lrs[0])
        st["a"] = (m_, v_, t_ + 1)
        closs.append(l)
    for i in range(M):
        b = batch(lists[M + i])
        l, g = O_nets.std_critic_loss(mk(nets0[3], std), mk(nets0[1], critic), b)
        m_, v_, t_ = st["s"]
        std, m_, v_ = O_nets.adam_step(std, m_, v_, g, t_, lrs[2])
        st["s"] = (m_, v_, t_ + 1)
        sloss.append(l)
    return (actor, critic, target, std), np.array(closs), np.array(sloss)


@pytest.mark.parametrize("graphs", [True, False])
def test_update_engine_matches_oracle_loop(graphs, fp64):
    from paper_2602_19699_b200.engine import UpdateEngine
    spec, fld = B_specs.config("pointmass")
    rng = np.random.default_rng(44)
    c, h = B_specs.normalisation(spec)
    d = spec.n + 1
    actor = B_nets.init_mlp([d, 64, 64, 64, spec.m], rng, head="tanh", out_scale=spec.u_bound, in_center=c,
                            in_half=h)
    critic = B_nets.init_mlp([d, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    target = B_nets.init_mlp([d, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    std = B_nets.init_mlp([d, 64, 64, 64, 1], rng, head="std", in_center=c, in_half=h)
    R = 700
    lo, hi = O_envs.region_box(spec)
    xa = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(0, spec.t_max + 1, (R, 1))], 1)
    xk = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(1, spec.t_max + 1, (R, 1))], 1)
    rows = {"xa": xa, "u": rng.normal(size=(R, spec.m)), "v_bar": rng.normal(size=R) * 10,
            "v_bar_x": rng.normal(size=(R, spec.n)), "xa_plus_k": xk}
    B, M = 48, 6
    ref, ref_c, ref_s = _oracle_update_loop(spec, fld, (actor, critic, target, std), rows, B, M, seed=9)
    buf = B_buffer.ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=1 << 12)
    buf.push_many(B_buffer.SampleBatch(rows["xa"], rows["u"], rows["v_bar"], rows["v_bar_x"], rows["xa_plus_k"],
                                       spec.t_max))
    eng = UpdateEngine(spec, fld, actor, critic, target, std, buf, minibatch=B, use_graphs=graphs)
    closs, sloss = eng.run(M, np.random.default_rng(9))
    np.testing.assert_allclose(closs, ref_c, rtol=1e-10)
    np.testing.assert_allclose(sloss, ref_s, rtol=1e-10)
    got = eng.networks()
    for g_net, r_params in zip((got[0], got[1], got[2], got[3]), ref):
        for a, b in zip(g_net.flat_params(), r_params):
            np.testing.assert_allclose(a, b, rtol=1e-8, atol=1e-12)
    # a second run continues the streams (Adam steps, buffer) like the reference's next iteration
    closs2, _ = eng.run(M, np.random.default_rng(10))
    assert np.all(np.isfinite(closs2))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("n,m,cap,pushes,bsz", [(4, 2, 777, (500, 700, 3), 1000), (15, 6, 64, (64, 1), 33),
                                                (6, 3, 4096, (4096, 2049), 4097)])
def test_ring_push_wrap_and_gather_bitwise(prec, n, m, cap, pushes, bsz):
    """FIFO push with wrap-around (buffer.py:108-130) and the warp-per-32-rows gather
    (buffer.py:132-138) vs the same ring restated in NumPy, ragged batch sizes."""
    from paper_2602_19699_b200.device import set_precision, get_precision
    old = get_precision()
    set_precision(prec)
    try:
        rng = np.random.default_rng(cap + bsz)
        buf = B_buffer.ReplayBuffer(n, m, 60, capacity=cap)
        widths = (n + 1, m, None, n, n + 1)
        ring = [np.zeros((cap,) + ((w,) if w else ())) for w in widths]
        cursor = size = 0
        for cnt in pushes:
            cols = [rng.standard_normal((cnt,) + ((w,) if w else ())) for w in widths]
            buf.push_many(B_buffer.SampleBatch(*cols, 60))
            first = max(0, cnt - cap)
            for r in range(first, cnt):
                for c, col in zip(ring, cols):
                    c[(cursor + r - first) % cap] = col[r]
            cursor = (cursor + cnt - first) % cap
            size = min(size + cnt - first, cap)
        assert len(buf) == size
        dt = torch.float32 if prec == "fp32" else torch.float64
        idx = rng.integers(0, size, size=bsz)
        got = buf.gather_device(torch.as_tensor(idx, device="cuda"))
        for g, c in zip(got, ring):
            want = torch.as_tensor(c[idx]).to(dt).numpy()
            np.testing.assert_array_equal(g.cpu().numpy().reshape(want.shape), want)
    finally:
        set_precision(old)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("R,N,K", [(200, 65536, 6553), (7, 100, 33), (64, 5000, 5000), (1, 3, 1)])
def test_take_columns_bitwise(dtype, R, N, K):
    """cacto_take_columns (kept warm starts out of K1's time-major U): dst[k, r] = src[r, idx[k]]."""
    from paper_2602_19699_b200 import _lib
    dt = torch.float32 if dtype == "f32" else torch.float64
    g = torch.Generator(device="cuda").manual_seed(R * 7 + K)
    src = torch.randn((R, N), device="cuda", dtype=dt, generator=g)
    idx = torch.randint(0, N, (K,), device="cuda", generator=g)
    dst = torch.empty((K, R), device="cuda", dtype=dt)
    _lib.call("cacto_take_columns", _lib.F32 if dtype == "f32" else _lib.F64, src.data_ptr(), R, N, idx.data_ptr(),
              K, dst.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert torch.equal(dst, src[:, idx].T)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("T,N,M,K", [(100, 65536, 3, 6553), (7, 100, 2, 33), (33, 5000, 6, 5000), (1, 3, 1, 1)])
def test_take_steps_bitwise(dtype, T, N, M, K):
    """cacto_take_steps (kept warm starts out of K1's step-major U [T, N, m]):
    dst[k, t, :] = src[t, idx[k], :]."""
    from paper_2602_19699_b200 import _lib
    dt = torch.float32 if dtype == "f32" else torch.float64
    g = torch.Generator(device="cuda").manual_seed(T * 7 + K)
    src = torch.randn((T, N, M), device="cuda", dtype=dt, generator=g)
    idx = torch.randint(0, N, (K,), device="cuda", generator=g)
    dst = torch.empty((K, T, M), device="cuda", dtype=dt)
    _lib.call("cacto_take_steps", _lib.F32 if dtype == "f32" else _lib.F64, src.data_ptr(), T, N, M, idx.data_ptr(),
              K, dst.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert torch.equal(dst, src[:, idx, :].transpose(0, 1))
