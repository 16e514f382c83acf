"""Measure the GPU-vs-oracle error floors behind the SURVEY 8(c) parity contract
(run on the B200: python profiles/parity_probe.py > profiles/r02_parity_probe.json).

For each check it prints max / p99 / median errors so the tolerances written in
tests/test_gpu_contract.py can be set to the contract, or to a measured floor
with this file as the evidence.
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import golden_utils as G  # noqa: E402
import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets, specs as B_specs, trainer as B_trainer  # noqa: E402
from oracle import nets as O_nets, select as O_select  # noqa: E402
from bench import make_nets, candidates, WORKLOADS  # noqa: E402
from test_gpu_parity import net  # noqa: E402

out = {}


def stats(err):
    err = np.asarray(err, float)
    err = err[np.isfinite(err)]
    if err.size == 0:
        return None
    return {"max": float(err.max()), "p99": float(np.quantile(err, 0.99)), "median": float(np.median(err)),
            "n": int(err.size)}


def relerr(a, b, floor=1.0):
    return np.abs(np.asarray(a, float) - b) / np.maximum(floor, np.abs(b))


def grad_rel(got, ref):
    scale = max(np.abs(r).max() for r in ref)
    return max(float(np.abs(g - r).max()) for g, r in zip(got, ref)) / scale


# 1. golden rollouts, both precisions
d = G.load("rollout")
for prec in ("fp64", "fp32"):
    P.set_precision(prec)
    for name in G.SYSTEMS:
        for tag in ("init", "trained"):
            key = f"{name}_{tag}"
            spec, fld = G.spec(d, f"{name}_spec"), G.field(d, f"{name}_field")
            r = B_nets.actor_rollout_batch(net(d, f"{key}_actor"), spec, d[f"{key}_x0"], d[f"{key}_t0"], None, fld)
            out[f"rollout_golden_{prec}_{key}_cost"] = stats(relerr(r["cost"], d[f"{key}_cost"]))
            m = ~np.isnan(d[f"{key}_X"])
            out[f"rollout_golden_{prec}_{key}_X"] = float(np.abs(r["X"][m] - d[f"{key}_X"][m]).max() /
                                                          np.abs(d[f"{key}_X"][m]).max())

# 2. golden losses
L = G.load("losses")
for prec in ("fp64", "fp32"):
    P.set_precision(prec)
    for key in ("b64", "b200"):
        for boot in (0, 1):
            loss, grads = B_nets.critic_loss(net(L, "critic_net"), net(L, "critic_target") if boot else None,
                                             G.batch(L, f"critic_{key}"), 0.7, bool(boot))
            ref = float(L[f"critic_{key}_boot{boot}_loss"])
            out[f"critic_{prec}_{key}_boot{boot}"] = {"loss": abs(loss - ref) / abs(ref),
                                                      "grad": grad_rel(grads, G.grads(L, f"critic_{key}_boot{boot}", 8))}
        loss, grads = B_nets.std_critic_loss(net(L, "std_net"), net(L, "critic_net"), G.batch(L, f"critic_{key}"))
        ref = float(L[f"std_{key}_loss"])
        out[f"std_{prec}_{key}"] = {"loss": abs(loss - ref) / abs(ref), "grad": grad_rel(grads, G.grads(L, f"std_{key}", 8))}
    for name in ("pointmass", "dubins", "manipulator3", "aliengo_lipm"):
        spec, fld = G.spec(d, f"{name}_spec"), G.field(d, f"{name}_field")
        batch = type("B", (), {"xa": L[f"actor_{name}_xa"]})()
        loss, grads, sk = B_nets.actor_loss(net(L, f"actor_{name}_actor"), net(L, f"actor_{name}_critic"), spec, fld, batch)
        ref = float(L[f"actor_{name}_loss"])
        out[f"actor_{prec}_{name}"] = {"loss": abs(loss - ref) / max(abs(ref), 1e-30),
                                       "grad": grad_rel(grads, G.grads(L, f"actor_{name}", 8))}
    loss, grads = B_nets.critic_loss(net(L, "critic_small_net"), net(L, "critic_small_target"),
                                     G.batch(L, "critic_small"), 0.5, True)
    out[f"critic_small_{prec}"] = {"loss": abs(loss - float(L["critic_small_loss"])) / abs(float(L["critic_small_loss"])),
                                   "grad": grad_rel(grads, G.grads(L, "critic_small", 6))}

# 3. the bench path (fused K1+K2, fp32) at every config's bench N vs the oracle on a subsample
P.set_precision("fp32")
for name, N in WORKLOADS.items():
    spec, fld = B_specs.config(name)
    actor, critic, std = make_nets(spec)
    x0h = candidates(spec, 0, N)
    pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
    x0 = torch.as_tensor(x0h).cuda()
    scores, cost, _ = pipe._scores(x0, 0, True)
    s = scores.cpu().numpy().astype(np.float64)
    c = cost.cpu().numpy().astype(np.float64)
    sub = np.unique(np.linspace(0, N - 1, min(N, 2048)).astype(np.int64))
    _, _, _, J = O_nets.actor_rollout_batch(actor, spec, x0h[sub], 0, spec.t_max, fld)
    xa = O_select.augmented(x0h[sub])
    sig = O_select.std_scores(std, xa)
    V = O_nets.mlp_forward(critic, xa)[:, 0]
    sref = sig * np.abs(V - J)
    cond = sig * (np.abs(V) + np.abs(J))          # the scale the subtraction V - J works at
    order, _ = B_trainer.select_topk_device(scores, N // 10)
    out[f"bench_{name}"] = {
        "N": N, "cost": stats(relerr(c[sub], J)), "score_rel": stats(relerr(s[sub], sref, 1e-30)),
        "score_vs_cond": stats(np.abs(s[sub] - sref) / np.maximum(cond, 1e-30)),
        "nan_ref": int(np.isnan(J).sum()), "nan_gpu": int(np.isnan(c[sub]).sum()),
        "inf_ref": int(np.isinf(J).sum()), "inf_gpu": int(np.isinf(c[sub]).sum()),
        "nan_pattern_equal": bool(np.array_equal(np.isnan(J), np.isnan(c[sub]))),
        "select_exact_given_gpu_scores": bool(np.array_equal(order.cpu().numpy(),
                                                             np.argsort(-scores.cpu().numpy(), kind="stable")[:N // 10]))}
    # SIMT fp32 kernel on the same subsample, same precision (the TC tail must be no worse)
    os.environ["CACTO_ROLLOUT_TC"] = "0"
    rs = B_nets.actor_rollout_batch(actor, spec, x0h[sub], 0, None, fld, emit=("cost",))
    os.environ.pop("CACTO_ROLLOUT_TC")
    rt = B_nets.actor_rollout_batch(actor, spec, x0h[sub], 0, None, fld, emit=("cost",))
    out[f"bench_{name}"]["simt_cost"] = stats(relerr(rs["cost"], J))
    out[f"bench_{name}"]["tc_cost_api"] = stats(relerr(rt["cost"], J))

# 4. score_kernel fp32 at H=64 (non-fused path) for each mode
for mode in ("std", "gap", "std_x_gap"):
    spec, fld = B_specs.config("dubins")
    actor, critic, std = make_nets(spec)
    x0h = candidates(spec, 0, 4096)
    xa = O_select.augmented(x0h)
    J = np.random.default_rng(3).normal(0, 50, 4096)
    sn, cn = B_trainer.device_net(std), B_trainer.device_net(critic)
    xad = torch.as_tensor(xa).to("cuda", torch.float32)
    Jd = torch.as_tensor(J).to("cuda", torch.float32)
    sc = B_trainer.score_device(mode, xad, sn if mode != "gap" else None, cn if mode != "std" else None,
                                Jd if mode != "std" else None).cpu().numpy()
    sig = O_select.std_scores(std, xa)
    V = O_nets.mlp_forward(critic, xa)[:, 0]
    Jr = J.astype(np.float32).astype(np.float64)
    ref = {"std": sig, "gap": np.abs(V - Jr), "std_x_gap": sig * np.abs(V - Jr)}[mode]
    out[f"score_kernel_fp32_{mode}"] = stats(relerr(sc, ref, 1e-30))

# 5. non-finite starts
for prec in ("fp64", "fp32"):
    P.set_precision(prec)
    for name in ("dubins", "manipulator3"):
        spec, fld = B_specs.config(name)
        actor, critic, std = make_nets(spec)
        x0h = candidates(spec, 0, 64)
        x0h[0, 0] = np.nan
        x0h[1, 1] = np.inf
        x0h[2, 0] = -np.inf
        x0h[3, :] = 1e30
        x0h[4, 0] = 1e6
        _, _, _, J = O_nets.actor_rollout_batch(actor, spec, x0h, 0, spec.t_max, fld)
        r = B_nets.actor_rollout_batch(actor, spec, x0h, 0, None, fld, emit=("cost",))
        out[f"nonfinite_{prec}_{name}"] = {"ref": [str(v) for v in J[:5]], "gpu": [str(v) for v in r["cost"][:5]],
                                           "rest_max_rel": float(relerr(r["cost"][5:], J[5:]).max())}
print(json.dumps(out, indent=1))
