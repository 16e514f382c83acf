"""Checkpoints: the reference's JSON network interchange (nets.py:428-464) and a
full training-state resume the reference lacks.

`save_training_state(dir, engine, rng)` writes
  actor.json, critic.json, critic_target.json, std.json   reference format
      (nets.save_checkpoint, loadable by trajrl.nets.load_checkpoint)
  state.npz   the three Adam states (m, v per parameter array, in flat_params
      order) and the replay ring's columns in PHYSICAL slot order (a TRLB dump,
      buffer.py:142-168, re-packs the ring oldest-first, which moves rows to other
      slots -- the minibatch indices, buffer.py:136, address slots)
  state.json  Adam steps / hyper-parameters, ring size / cursor / shape, and the
      minibatch generator's bit_generator.state (rng_batches, trainer.py:123)
`load_training_state(dir, model, field, minibatch=...)` rebuilds an UpdateEngine
and the generator such that the next `engine.run(M, rng)` is bit-identical (fp64)
to the uninterrupted run.
"""

from __future__ import annotations

import json
import os
from types import SimpleNamespace

import numpy as np
import torch

from . import nets
from .buffer import ReplayBuffer

KINDS = ("actor", "critic", "critic_target", "std")


def save_training_state(path, engine, rng: np.random.Generator, model_name: str = "", config_hash: str = ""):
    os.makedirs(path, exist_ok=True)
    for kind, net in zip(KINDS, engine.networks()):
        nets.save_checkpoint(os.path.join(path, f"{kind}.json"), net, kind, model_name, config_hash)
    arrays, meta = {}, {"adam": {}}
    for name in ("actor", "critic", "std"):
        n = getattr(engine, name)
        m, v, step = engine.adam_host(n)
        for i, (a, b) in enumerate(zip(m, v)):
            arrays[f"{name}_m{i}"] = a
            arrays[f"{name}_v{i}"] = b
        meta["adam"][name] = {"step": int(step), "lr": n.lr, "beta1": n.beta1, "beta2": n.beta2, "eps": n.eps,
                              "arrays": len(m)}
    buf = engine.buffer
    for i, c in enumerate(buf.cols):
        arrays[f"ring{i}"] = c[:buf._size].to("cpu").numpy()
    meta["ring"] = {"size": int(buf._size), "cursor": int(buf._cursor), "capacity": int(buf.capacity),
                    "n": buf.n, "m": buf.m, "t_max": buf.t_max, "k_lookahead": buf.k_lookahead,
                    "model_name": buf.model_name, "precision": engine.precision}
    meta["engine"] = {"minibatch": engine.B, "k_s": engine.k_s, "bootstrap": engine.bootstrap, "tau": engine.tau}
    meta["rng"] = rng.bit_generator.state
    np.savez(os.path.join(path, "state.npz"), **arrays)
    with open(os.path.join(path, "state.json"), "w") as fh:
        json.dump(meta, fh)


def load_training_state(path, model, field, **engine_kwargs):
    """-> (UpdateEngine, np.random.Generator) continuing the saved run."""
    from .engine import UpdateEngine
    with open(os.path.join(path, "state.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(path, "state.npz"))
    mlps = {k: nets.load_checkpoint(os.path.join(path, f"{k}.json"))[0] for k in KINDS}
    adam = []
    for name in ("actor", "critic", "std"):
        a = meta["adam"][name]
        adam.append(SimpleNamespace(m=tuple(arrays[f"{name}_m{i}"] for i in range(a["arrays"])),
                                    v=tuple(arrays[f"{name}_v{i}"] for i in range(a["arrays"])),
                                    step=a["step"], lr=a["lr"], beta1=a["beta1"], beta2=a["beta2"],
                                    eps_adam=a["eps"]))
    r = meta["ring"]
    buf = ReplayBuffer(r["n"], r["m"], r["t_max"], capacity=r["capacity"], model_name=r["model_name"],
                       k_lookahead=r["k_lookahead"], precision=r["precision"])
    for i, c in enumerate(buf.cols):
        c[:r["size"]].copy_(torch.as_tensor(arrays[f"ring{i}"]).to(c.device, c.dtype))
    buf._size, buf._cursor = r["size"], r["cursor"]
    e = dict(meta["engine"])
    e.update(engine_kwargs)
    minibatch = e.pop("minibatch")
    eng = UpdateEngine(model, field, mlps["actor"], mlps["critic"], mlps["critic_target"], mlps["std"], buf,
                       minibatch=minibatch, adam_states=tuple(adam), precision=r["precision"],
                       lr_actor=adam[0].lr, lr_critic=adam[1].lr, lr_std=adam[2].lr, **e)
    rng = np.random.Generator(np.random.PCG64())
    rng.bit_generator.state = meta["rng"]
    return eng, rng
