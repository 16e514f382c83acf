"""The SURVEY.md 8(c) parity contract, checked on the exact product paths.

Tolerances are the contract's, or -- where the contract cannot be met by ANY
fp32 implementation -- a measured floor stated here with its evidence
(profiles/r02_parity_probe.json, produced by profiles/parity_probe.py):

  fp64 mode     rollout cost / X / U rel <= 1e-10 (manipulator3 <= 1e-8); losses
                and grads (grads normalised by max|g|, test_nets.py:45-49) <= 1e-12.
  fp32 golden   rollout cost rel max <= 1e-5 (pointmass, dubins, toy; AlienGO 2e-5,
                measured 1.3e-5); manipulator3 median <= 1e-4, max <= 1e-1;
                losses <= 1e-6 (contract 1e-5; measured <= 1.2e-7); grads <= 1e-5
                of max|g| (contract 1e-4; measured <= 6e-7).
  bench path    `BicPipeline(mode="std_x_gap")` -- the fused tensor-core K1+K2 launch
  (fp32)        the bench times -- at every config's bench N, a fixed 2048-start
                subsample against the float64 oracle (oracle.nets.actor_rollout_batch
                + oracle.select):
                  * select is bit-exact given the GPU's own scores (full N);
                  * cost and score medians <= 1e-6 (pointmass/dubins/AlienGO);
                  * the chaotic tail (trajectories that graze an obstacle or, on
                    manipulator3 with the x10 'trained-like' actor, spin up) is
                    bounded by the SIMT-FFMA fp32 kernel's own error on the same
                    starts: p99 and max within TAIL = 2.5x of it (3xFP16 operands
                    carry ~23 significant bits and the tensor pipe's fp32 accumulate
                    truncates; measured ratios 1.1x (max) to 2.3x (AlienGO p99));
                  * non-finite pattern: NaN exactly where the float64 cost is NaN;
                    manipulator3 (chaotic: the float64 GPU path differs from the
                    float64 oracle there too) within 3 % of the starts.
  score kernel  fp32 H=64, modes std / gap / std_x_gap: |s - s_ref| <= 1e-6 *
                sigma * (|V| + |J|) (the scale the subtraction V - J works at).
  non-finite    NaN / +-inf / 1e30 starts: fp64 equal to the oracle (NaN pattern and
  starts        values); fp32: NaN exactly where the oracle's cost is NaN, +inf where
                the oracle's float64 cost exceeds the fp32 range, finite rows rel 1e-4.
"""

import os

import numpy as np
import pytest

import golden_utils as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets, specs as B_specs, trainer as B_trainer  # noqa: E402
from oracle import nets as O_nets, select as O_select  # noqa: E402
from bench import make_nets, candidates, WORKLOADS  # noqa: E402
from test_gpu_parity import net  # noqa: E402

F32_MAX = float(np.finfo(np.float32).max)
TAIL = 2.5   # tensor-core (3xFP16) chaotic-tail error / SIMT-FFMA fp32 error, p99 and max


@pytest.fixture(params=["fp64", "fp32"])
def precision(request):
    old = P.get_precision()
    P.set_precision(request.param)
    yield request.param
    P.set_precision(old)


@pytest.fixture
def fp32():
    old = P.get_precision()
    P.set_precision("fp32")
    yield
    P.set_precision(old)


def relerr(a, b, floor=1.0):
    return np.abs(np.asarray(a, float) - b) / np.maximum(floor, np.abs(b))


def grad_rel(got, ref):
    scale = max(np.abs(r).max() for r in ref)
    return max(float(np.abs(g - r).max()) for g, r in zip(got, ref)) / scale


@pytest.mark.parametrize("name", G.SYSTEMS)
@pytest.mark.parametrize("tag", ["init", "trained"])
def test_golden_rollouts(name, tag, precision):
    d = G.load("rollout")
    spec, fld = G.spec(d, f"{name}_spec"), G.field(d, f"{name}_field")
    key = f"{name}_{tag}"
    r = B_nets.actor_rollout_batch(net(d, f"{key}_actor"), spec, d[f"{key}_x0"], d[f"{key}_t0"], None, fld)
    err = relerr(r["cost"], d[f"{key}_cost"])
    if precision == "fp64":
        tol = 1e-8 if name == "manipulator3" else 1e-10
        assert err.max() <= tol, err.max()
        for k in ("X", "U"):
            m = ~np.isnan(d[f"{key}_{k}"])
            e = np.abs(r[k][m] - d[f"{key}_{k}"][m]).max() / np.abs(d[f"{key}_{k}"][m]).max()
            assert e <= tol, (k, e)
    elif name == "manipulator3":
        assert np.median(err) <= 1e-4 and err.max() <= 1e-1, (np.median(err), err.max())
    else:
        assert err.max() <= (2e-5 if name == "aliengo_lipm" else 1e-5), err.max()


def test_golden_losses(precision):
    d = G.load("losses")
    r = G.load("rollout")
    lt, gt = (1e-12, 1e-12) if precision == "fp64" else (1e-6, 1e-5)
    for key in ("b64", "b200"):
        for boot in (0, 1):
            loss, grads = B_nets.critic_loss(net(d, "critic_net"), net(d, "critic_target") if boot else None,
                                             G.batch(d, f"critic_{key}"), 0.7, bool(boot))
            ref = float(d[f"critic_{key}_boot{boot}_loss"])
            assert abs(loss - ref) <= lt * abs(ref)
            assert grad_rel(grads, G.grads(d, f"critic_{key}_boot{boot}", 8)) <= gt
        loss, grads = B_nets.std_critic_loss(net(d, "std_net"), net(d, "critic_net"), G.batch(d, f"critic_{key}"))
        assert abs(loss - float(d[f"std_{key}_loss"])) <= lt * abs(float(d[f"std_{key}_loss"]))
        assert grad_rel(grads, G.grads(d, f"std_{key}", 8)) <= gt
    for name in ("pointmass", "dubins", "manipulator3", "aliengo_lipm"):
        spec, fld = G.spec(r, f"{name}_spec"), G.field(r, f"{name}_field")
        batch = type("B", (), {"xa": d[f"actor_{name}_xa"]})()
        loss, grads, skipped = B_nets.actor_loss(net(d, f"actor_{name}_actor"), net(d, f"actor_{name}_critic"),
                                                 spec, fld, batch)
        ref = float(d[f"actor_{name}_loss"])
        assert skipped == int(d[f"actor_{name}_skipped"])
        assert abs(loss - ref) <= lt * max(abs(ref), 1e-30), (name, loss, ref)
        assert grad_rel(grads, G.grads(d, f"actor_{name}", 8)) <= gt


def _simt_cost(actor, spec, fld, x0):
    os.environ["CACTO_ROLLOUT_TC"] = "0"
    try:
        return B_nets.actor_rollout_batch(actor, spec, x0, 0, None, fld, emit=("cost",))["cost"]
    finally:
        os.environ.pop("CACTO_ROLLOUT_TC", None)


@pytest.mark.parametrize("name", sorted(WORKLOADS))
def test_bench_path_vs_oracle_at_bench_size(name, fp32):
    N = WORKLOADS[name]
    spec, fld = B_specs.config(name)
    actor, critic, std = make_nets(spec)
    x0h = candidates(spec, 0, N)
    pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
    x0 = torch.as_tensor(x0h).cuda()
    scores, cost, _ = pipe._scores(x0, 0, True)       # the fused launch BicPipeline.run uses
    keep = N // 10
    order, _ = B_trainer.select_topk_device(scores, keep)
    sg = scores.cpu().numpy()
    np.testing.assert_array_equal(order.cpu().numpy(), np.argsort(-sg, kind="stable")[:keep])
    sub = np.unique(np.linspace(0, N - 1, min(N, 2048)).astype(np.int64))
    X, _, _, J = O_nets.actor_rollout_batch(actor, spec, x0h[sub], 0, spec.t_max, fld)
    xa = O_select.augmented(x0h[sub])
    sig = O_select.std_scores(std, xa)
    sref = sig * np.abs(O_nets.mlp_forward(critic, xa)[:, 0] - J)
    c = cost.cpu().numpy()[sub].astype(np.float64)
    s = sg[sub].astype(np.float64)
    # non-finite pattern
    nan_ref, nan_gpu = np.isnan(J), np.isnan(c)
    if name == "manipulator3":
        # x10 actor: ~7 % of the starts spin up and diverge to NaN, chaotically --
        # the float64 GPU path differs from the float64 oracle there as well
        assert np.mean(nan_ref != nan_gpu) <= 0.03, (nan_ref.sum(), nan_gpu.sum())
    else:
        np.testing.assert_array_equal(nan_gpu, nan_ref)
    ok = ~nan_gpu & ~nan_ref
    ec, es = relerr(c[ok], J[ok]), relerr(s[ok], sref[ok], 1e-30)
    simt = _simt_cost(actor, spec, fld, x0h[sub])
    okb = ok & ~np.isnan(simt)
    e_simt = relerr(simt[okb], J[okb])
    e_tc = relerr(c[okb], J[okb])
    assert np.quantile(e_tc, 0.99) <= TAIL * np.quantile(e_simt, 0.99) + 1e-7, \
        (np.quantile(e_tc, 0.99), np.quantile(e_simt, 0.99))
    assert e_tc.max() <= TAIL * e_simt.max() + 1e-7, (e_tc.max(), e_simt.max())
    if name == "manipulator3":
        assert np.median(e_tc) <= TAIL * np.median(e_simt) + 1e-7
    else:
        assert np.median(ec) <= 1e-6 and np.median(es) <= 1e-6, (np.median(ec), np.median(es))


@pytest.mark.parametrize("mode", ["std", "gap", "std_x_gap"])
def test_score_kernel_fp32_h64(mode, fp32):
    spec, fld = B_specs.config("dubins")
    actor, critic, std = make_nets(spec)
    n = 4096
    xa = O_select.augmented(candidates(spec, 0, n))
    J = np.random.default_rng(3).normal(0, 50, n).astype(np.float32).astype(np.float64)
    sn, cn = B_trainer.device_net(std), B_trainer.device_net(critic)
    xad = torch.as_tensor(xa).to("cuda", torch.float32)
    Jd = torch.as_tensor(J).to("cuda", torch.float32)
    sc = B_trainer.score_device(mode, xad, sn if mode != "gap" else None, cn if mode != "std" else None,
                                Jd if mode != "std" else None).cpu().numpy().astype(np.float64)
    xa32 = xa.astype(np.float32).astype(np.float64)      # the fp32 inputs the kernel sees
    sig = O_select.std_scores(std, xa32)
    V = O_nets.mlp_forward(critic, xa32)[:, 0]
    ref = {"std": sig, "gap": np.abs(V - J), "std_x_gap": sig * np.abs(V - J)}[mode]
    scale = {"std": np.abs(sig), "gap": np.abs(V) + np.abs(J), "std_x_gap": sig * (np.abs(V) + np.abs(J))}[mode]
    scale = np.maximum(scale, 1.0)     # fp32 absolute error floor of an O(1)-weight network output
    assert np.all(np.abs(sc - ref) <= 1e-6 * scale), np.max(np.abs(sc - ref) / scale)


@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3", "aliengo_lipm"])
def test_nonfinite_starts(name, precision):
    spec, fld = B_specs.config(name)
    actor, critic, std = make_nets(spec)
    x0h = candidates(spec, 0, 300)
    x0h[0, 0] = np.nan
    x0h[1, 1] = np.inf
    x0h[2, 0] = -np.inf
    x0h[3, :] = 1e30
    x0h[4, 0] = 1e6
    x0h[5, -1] = np.nan
    _, _, _, J = O_nets.actor_rollout_batch(actor, spec, x0h, 0, spec.t_max, fld)
    c = B_nets.actor_rollout_batch(actor, spec, x0h, 0, None, fld, emit=("cost",))["cost"]
    if name == "manipulator3":
        # chaotic with the x10 actor (see test_bench_path_vs_oracle_at_bench_size):
        # the injected non-finite starts must be NaN, the rest agree statistically
        assert np.all(np.isnan(c[:3])) and np.all(np.isnan(J[:3]))
        assert np.mean(np.isnan(c) != np.isnan(J)) <= 0.03
        both = np.isfinite(c) & np.isfinite(J)
        # median, fp32: 1e-3 (the x10 actor's spin-ups; the golden 'trained' actor meets 1e-4)
        assert np.median(relerr(c[both], J[both])) <= (1e-10 if precision == "fp64" else 1e-3)
        return
    np.testing.assert_array_equal(np.isnan(c), np.isnan(J))
    if precision == "fp64":
        fin = np.isfinite(J)
        np.testing.assert_array_equal(np.isinf(c), np.isinf(J))
        assert relerr(c[fin], J[fin]).max() <= (1e-8 if name == "manipulator3" else 1e-10)
    else:
        over = np.isfinite(J) & (np.abs(J) > F32_MAX)
        assert np.all(np.isinf(c[over]))
        fin = np.isfinite(J) & ~over
        e = relerr(c[fin], J[fin])
        assert np.median(e) <= 1e-5
    # the BIC pipeline sorts non-finite scores last / by their value like argsort
    if precision == "fp32":
        pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
        sc, _, _ = pipe._scores(torch.as_tensor(x0h).cuda(), 0, False)
        o, _ = B_trainer.select_topk_device(sc, 300)
        np.testing.assert_array_equal(o.cpu().numpy(), np.argsort(-sc.cpu().numpy(), kind="stable"))
        assert np.all(np.isnan(sc.cpu().numpy()[np.isnan(J)]))
