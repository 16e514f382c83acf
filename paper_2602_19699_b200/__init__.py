"""B200-native CACTO-BIC hot path (arXiv 2602.19699): batched actor rollouts,
BIC scoring + stable top-k, Sobolev critic / actor / std training and the
replay gather as hand-written sm_100a kernels behind a C ABI
(include/cacto_b200.h), with the reference `trajrl` Python API on top.

Modules mirror the reference: `nets` (trajrl.nets), `trainer`
(trajrl.trainer select/rollout call sites), `buffer` (trajrl.buffer),
`specs` (trajrl.envs types).  `engine` runs the device-resident M-cycle update
loop; `install()` rebinds the reference's hot functions onto this package.
"""

from .device import get_precision, set_precision  # noqa: F401

__version__ = "0.1.0"


def library_path():
    from . import _lib
    return str(_lib.LIB_PATH)


def install(trajrl_module, iteration: bool = True):
    """Rebind the reference's hot-path functions onto the B200 implementation:
    trajrl.nets.{mlp_forward, critic_loss, actor_loss, std_critic_loss,
    adam_step, polyak, actor_rollout} and trajrl.trainer.select_initial_states_bic
    (call sites trainer.py:186, 192-193, 211-233, 267-268), and -- with
    `iteration=True` (default) -- trajrl.trainer.run_iteration (trainer.py:168-255)
    by the batched device iteration (iteration.run_iteration: one launch per
    phase, the replay producer, the CUDA-graph update engine), so
    `trajrl.trainer.train` runs the whole hot path on the B200.  Returns
    `uninstall()`."""
    from . import nets, trainer
    tn = trajrl_module.nets
    tt = trajrl_module.trainer
    saved = {}

    def swap(mod, name, fn):
        saved[(mod, name)] = getattr(mod, name)
        setattr(mod, name, fn)

    for name in ("mlp_forward", "critic_loss", "actor_loss", "std_critic_loss", "polyak"):
        swap(tn, name, getattr(nets, name))

    def adam_step(params, state, grads):
        p, st = nets.adam_step(params, nets.AdamState(state.m, state.v, state.step, state.lr, state.beta1,
                                                      state.beta2, state.eps_adam), grads)
        from dataclasses import replace
        return p, replace(state, m=st.m, v=st.v, step=st.step)

    def actor_rollout(actor, model, x0, t_hor, field=None):
        t = nets.actor_rollout(actor, model, x0, t_hor, field)
        return trajrl_module.ilqr.Trajectory(X=t.X, U=t.U, step_costs=t.step_costs, t0=t.t0)

    swap(tn, "adam_step", adam_step)
    swap(tn, "actor_rollout", actor_rollout)
    swap(tt, "select_initial_states_bic", trainer.select_initial_states_bic)
    if iteration:
        from . import iteration as _it
        swap(tt, "run_iteration", lambda state, iter_idx: _it.run_iteration(state, iter_idx, trajrl_module))

    def uninstall():
        for (mod, name), fn in saved.items():
            setattr(mod, name, fn)
    return uninstall
