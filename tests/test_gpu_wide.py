"""GPU parity of the wide-network path (padded hidden width > 64, csrc/wide.cu):
layer-wise tcgen05 3xTF32 GEMMs + fused elementwise kernels, fp32, against the
float64 CPU oracle (which is pinned to the reference goldens).

Tolerances (fp32 arithmetic, 3xTF32 products):
  forward / value 2e-5 rel of max|y|, Jacobians 1e-4 rel,
  losses 1e-5 rel, gradients 1e-4 of max|grad| (the reference FD metric,
  test_nets.py:45-49), update-loop losses 2e-3 rel after M Adam steps.
"""

from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import buffer as B_buffer  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets  # noqa: E402
from paper_2602_19699_b200 import specs as B_specs  # noqa: E402
from paper_2602_19699_b200 import trainer as B_trainer  # noqa: E402
from oracle import envs as O_envs  # noqa: E402
from oracle import nets as O_nets  # noqa: E402


@pytest.fixture(autouse=True)
def fp32():
    old = P.get_precision()
    P.set_precision("fp32")
    yield
    P.set_precision(old)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def grads_close(got, ref, tol):
    scale = max(1e-12, max(np.abs(r).max() for r in ref))
    for g, r in zip(got, ref):
        assert g.shape == r.shape
        assert np.abs(g - r).max() / scale < tol, (np.abs(g - r).max() / scale)


def jitter_biases(net, rng, s=0.1):
    return replace(net, biases=tuple(rng.normal(0.0, s, b.shape) for b in net.biases))


def nets_for(spec, H, rng, layers=3, act="elu"):
    c, h = B_specs.normalisation(spec)
    d = spec.n + 1
    hid = [H] * layers
    mk = lambda out, **kw: jitter_biases(B_nets.init_mlp([d, *hid, out], rng, activation=act, in_center=c,  # noqa
                                                         in_half=h, **kw), rng)
    actor = mk(spec.m, head="tanh", out_scale=spec.u_bound)
    critic = mk(1)
    target = mk(1)
    std = mk(1, head="std")
    return actor, critic, target, std


def sample_batch(spec, R, rng, frac_end=0.1):
    lo, hi = O_envs.region_box(spec)
    t = rng.integers(0, spec.t_max, (R, 1)).astype(float)
    t[rng.uniform(size=R) < frac_end] = spec.t_max
    xa = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, t], 1)
    xk = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(1, spec.t_max + 1, (R, 1))], 1)
    return B_buffer.SampleBatch(xa, rng.normal(size=(R, spec.m)), rng.normal(size=R) * 10,
                                rng.normal(size=(R, spec.n)), xk, spec.t_max)


@pytest.mark.parametrize("H", [96, 128, 256])
@pytest.mark.parametrize("act", ["elu", "tanh"])
def test_wide_forward_and_jacobian(H, act):
    spec = B_specs.default_model("dubins")
    rng = np.random.default_rng(H)
    actor, critic, _, std = nets_for(spec, H, rng, act=act)
    x = sample_batch(spec, 777, rng).xa
    for net in (actor, critic, std):
        assert rel(B_nets.mlp_forward(net, x), O_nets.mlp_forward(net, x)) < 2e-5
        assert rel(B_nets.mlp_input_gradient(net, x), O_nets.mlp_input_gradient(net, x)) < 1e-4
    v, g = B_nets.value_and_state_grad(critic, x)
    v_ref, g_ref = O_nets.value_and_state_grad(critic, x)
    assert rel(v, v_ref) < 2e-5 and rel(g, g_ref) < 1e-4


@pytest.mark.parametrize("H,layers", [(128, 3), (256, 2), (512, 1), (128, 4)])
@pytest.mark.parametrize("boot", [False, True])
def test_wide_critic_loss(H, layers, boot):
    spec = B_specs.default_model("pointmass")
    rng = np.random.default_rng(7 + H + layers)
    _, critic, target, _ = nets_for(spec, H, rng, layers=layers)
    batch = sample_batch(spec, 300, rng)
    loss, grads = B_nets.critic_loss(critic, target, batch, 0.7, boot)
    ref, ref_g = O_nets.critic_loss(critic, target, batch, 0.7, boot)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


def test_wide_critic_loss_large_batch_split_k():
    # B = 9000: many K blocks, split-K weight gradients, ragged last tiles
    spec = B_specs.default_model("manipulator3")
    rng = np.random.default_rng(3)
    _, critic, target, _ = nets_for(spec, 256, rng)
    batch = sample_batch(spec, 9000, rng)
    loss, grads = B_nets.critic_loss(critic, target, batch, 1.0, True)
    ref, ref_g = O_nets.critic_loss(critic, target, batch, 1.0, True)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


def test_wide_critic_loss_deterministic():
    spec = B_specs.default_model("pointmass")
    rng = np.random.default_rng(9)
    _, critic, target, _ = nets_for(spec, 256, rng)
    batch = sample_batch(spec, 5000, rng)
    a = B_nets.critic_loss(critic, target, batch, 0.7, True)
    b = B_nets.critic_loss(critic, target, batch, 0.7, True)
    assert a[0] == b[0]
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("H", [128, 256])
def test_wide_std_loss(H):
    spec = B_specs.default_model("dubins")
    rng = np.random.default_rng(11 + H)
    _, critic, _, std = nets_for(spec, H, rng)
    batch = sample_batch(spec, 400, rng)
    loss, grads = B_nets.std_critic_loss(std, critic, batch)
    ref, ref_g = O_nets.std_critic_loss(std, critic, batch)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


def test_std_loss_narrow_std_wide_critic():
    spec = B_specs.default_model("dubins")
    rng = np.random.default_rng(12)
    _, critic, _, _ = nets_for(spec, 256, rng)
    _, _, _, std = nets_for(spec, 64, rng)
    batch = sample_batch(spec, 300, rng)
    loss, grads = B_nets.std_critic_loss(std, critic, batch)
    ref, ref_g = O_nets.std_critic_loss(std, critic, batch)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3", "aliengo_lipm"])
@pytest.mark.parametrize("combo", ["wide_wide", "narrow_actor", "narrow_critic"])
def test_wide_actor_loss(name, combo):
    spec, fld = B_specs.config(name)
    rng = np.random.default_rng(21)
    wa, wc, _, _ = nets_for(spec, 256, rng)
    na, nc, _, _ = nets_for(spec, 64, rng)
    actor, critic = {"wide_wide": (wa, wc), "narrow_actor": (na, wc), "narrow_critic": (wa, nc)}[combo]
    xa = sample_batch(spec, 333, rng).xa
    loss, grads, skipped = B_nets.actor_loss(actor, critic, spec, fld, type("B", (), {"xa": xa})())
    ref, ref_g, ref_skip = O_nets.actor_loss(actor, critic, spec, fld, xa)
    assert skipped == ref_skip
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


@pytest.mark.parametrize("mode", ["std", "gap", "std_x_gap"])
def test_wide_bic_scores(mode):
    spec = B_specs.default_model("dubins")
    rng = np.random.default_rng(5)
    _, critic, _, std = nets_for(spec, 128, rng)
    x = sample_batch(spec, 1000, rng).xa
    rc = rng.uniform(0, 50, 1000)
    from paper_2602_19699_b200.device import device_net
    got = B_trainer.score_device(mode, torch.as_tensor(x, device="cuda", dtype=torch.float32),
                                 std_net=device_net(std) if mode != "gap" else None,
                                 critic=device_net(critic) if mode != "std" else None,
                                 rollout_cost=torch.as_tensor(rc, device="cuda", dtype=torch.float32)
                                 ).cpu().numpy()
    sig = O_nets.mlp_forward(std, x)[:, 0]
    gap = np.abs(O_nets.mlp_forward(critic, x)[:, 0] - rc)
    ref = {"std": sig, "gap": gap, "std_x_gap": sig * gap}[mode]
    assert rel(got, ref) < 1e-4


def test_wide_update_engine_matches_oracle_loop():
    from test_gpu_parity import _oracle_update_loop
    from paper_2602_19699_b200.engine import UpdateEngine
    spec, fld = B_specs.config("pointmass")
    rng = np.random.default_rng(44)
    actor, critic, target, std = nets_for(spec, 256, rng)
    R = 700
    lo, hi = O_envs.region_box(spec)
    xa = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(0, spec.t_max + 1, (R, 1))], 1)
    xk = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(1, spec.t_max + 1, (R, 1))], 1)
    rows = {"xa": xa, "u": rng.normal(size=(R, spec.m)), "v_bar": rng.normal(size=R) * 10,
            "v_bar_x": rng.normal(size=(R, spec.n)), "xa_plus_k": xk}
    B, M = 64, 5
    _, ref_c, ref_s = _oracle_update_loop(spec, fld, (actor, critic, target, std), rows, B, M, seed=9)
    buf = B_buffer.ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=1 << 12, precision="fp32")
    buf.push_many(B_buffer.SampleBatch(rows["xa"], rows["u"], rows["v_bar"], rows["v_bar_x"], rows["xa_plus_k"],
                                       spec.t_max))
    eng = UpdateEngine(spec, fld, actor, critic, target, std, buf, minibatch=B, use_graphs=True)
    closs, sloss = eng.run(M, np.random.default_rng(9))
    np.testing.assert_allclose(closs, ref_c, rtol=2e-3)
    np.testing.assert_allclose(sloss, ref_s, rtol=2e-3)
