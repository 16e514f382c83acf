"""ctypes binding of the C-ABI in include/cacto_b200.h (libcacto_b200.so).

The shared library is built in-tree (`make`, or `__graft_entry__.build()`).
There is no CPU fallback: importing the product API on a machine without the
library raises, and every call without a CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("CACTO_B200_LIB", _HERE / "libcacto_b200.so"))

MAX_LAYERS = 5
MAX_IN = 32
MAX_OUT = 8
MAX_OBST = 4

OK, EVALUE, EUNSUPPORTED, ECUDA = 0, -1, -2, -3
F32, F64 = 0, 1
ACT = {"elu": 0, "tanh": 1}
HEAD = {"linear": 0, "tanh": 1, "std": 2}
SYS = {"toy1d": 0, "pointmass": 1, "dubins": 2, "manipulator3": 3, "aliengo_lipm": 4}
COST_TASK, COST_TOY1D, COST_LIPM = 0, 1, 2
SCORE = {"std": 0, "gap": 1, "std_x_gap": 2}


class CactoMlp(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("n_layers", ctypes.c_int32),
                ("sizes", ctypes.c_int32 * (MAX_LAYERS + 1)), ("hp", ctypes.c_int32),
                ("activation", ctypes.c_int32), ("head", ctypes.c_int32), ("has_norm", ctypes.c_int32),
                ("sigma_min", ctypes.c_double), ("in_center", ctypes.c_double * MAX_IN),
                ("in_half", ctypes.c_double * MAX_IN), ("out_scale", ctypes.c_double * MAX_OUT),
                ("params", ctypes.c_void_p)]


class CactoSystem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n", ctypes.c_int32), ("m", ctypes.c_int32),
                ("t_max", ctypes.c_int32), ("dt", ctypes.c_double),
                ("u_max", ctypes.c_double * MAX_OUT), ("p", ctypes.c_double * 16)]


class CactoCost(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_obstacles", ctypes.c_int32),
                ("target", ctypes.c_double * 2), ("obs_center", (ctypes.c_double * 2) * MAX_OBST),
                ("obs_form", (ctypes.c_double * 4) * MAX_OBST), ("w_obstacle", ctypes.c_double),
                ("w_reward", ctypes.c_double), ("reward_radius", ctypes.c_double),
                ("w_control", ctypes.c_double), ("w_distance", ctypes.c_double),
                ("extra", ctypes.c_double * 8)]


class CactoBatch(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("n", ctypes.c_int32), ("m", ctypes.c_int32),
                ("t_max", ctypes.c_int32), ("rows", ctypes.c_int64), ("denom", ctypes.c_int64),
                ("idx", ctypes.c_void_p), ("xa", ctypes.c_void_p), ("u", ctypes.c_void_p),
                ("v_bar", ctypes.c_void_p), ("v_bar_x", ctypes.c_void_p), ("xa_plus_k", ctypes.c_void_p),
                ("cycle", ctypes.c_void_p), ("idx_stride", ctypes.c_int64)]


class CactoSolutions(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("count", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("offsets", ctypes.c_void_p), ("t0", ctypes.c_void_p), ("X", ctypes.c_void_p),
                ("U", ctypes.c_void_p), ("step_costs", ctypes.c_void_p), ("v_bar", ctypes.c_void_p),
                ("v_bar_x", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_U64 = ctypes.c_uint64
_PMLP = ctypes.POINTER(CactoMlp)
_PSYS = ctypes.POINTER(CactoSystem)
_PCOST = ctypes.POINTER(CactoCost)
_PBATCH = ctypes.POINTER(CactoBatch)
_PI32 = ctypes.POINTER(ctypes.c_int32)

ROLLOUT_U_TIME_MAJOR = 1   # CACTO_ROLLOUT_U_TIME_MAJOR
ROLLOUT_U_STEP_MAJOR = 2   # CACTO_ROLLOUT_U_STEP_MAJOR
FULL_HORIZON = -1          # CACTO_FULL_HORIZON

# symbol -> (restype, argtypes); mirrors include/cacto_b200.h one to one
SIGNATURES = {
    "cacto_abi_version": (ctypes.c_int, []),
    "cacto_last_error": (ctypes.c_char_p, []),
    "cacto_padded_in": (_I32, [_I32]),
    "cacto_mlp_param_count": (_I64, [_PMLP]),
    "cacto_mlp_forward": (ctypes.c_int, [_PMLP, _P, _I64, _P, _P]),
    "cacto_mlp_jacobian": (ctypes.c_int, [_PMLP, _P, _I64, _P, _P, _P]),
    "cacto_rollout": (ctypes.c_int, [_PSYS, _PCOST, _PMLP, _P, _P, _I32, _I64, _I32, _P, _P, _P, _P, _P]),
    "cacto_rollout_ex": (ctypes.c_int, [_PSYS, _PCOST, _PMLP, _P, _P, _I32, _I64, _I32, _I32, _P, _P, _P, _P,
                                         _P]),
    "cacto_take_columns": (ctypes.c_int, [_I32, _P, _I64, _I64, _P, _I64, _P, _P]),
    "cacto_take_rows": (ctypes.c_int, [_I32, _P, _I64, _P, _I64, _P, _P]),
    "cacto_take_steps": (ctypes.c_int, [_I32, _P, _I64, _I64, _I32, _P, _I64, _P, _P]),
    "cacto_rollout_score": (ctypes.c_int, [_PSYS, _PCOST, _PMLP, _I32, _PMLP, _PMLP, _P, _I32, _I64, _I32, _I32,
                                            _P, _P, _P, _P]),
    "cacto_score": (ctypes.c_int, [_I32, _PMLP, _PMLP, _P, _P, _I64, _P, _P]),
    "cacto_select_workspace_bytes": (_SZ, [_I32, _I64, _I64]),
    "cacto_select_topk": (ctypes.c_int, [_I32, _P, _I64, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "cacto_select_merge": (ctypes.c_int, [_I32, _P, _P, _I32, _I64, _P, _P, _P, _SZ, _P]),
    "cacto_dselect_workspace_bytes": (_SZ, [_I32, _I64, _I64]),
    "cacto_dselect_begin": (ctypes.c_int, [_I32, _I64, _I64, _I64, _P, _SZ, _P]),
    "cacto_dselect_pass": (ctypes.c_int, [_I32, _P, _I64, _I64, _I32, _P, _P, _P]),
    "cacto_dselect_digit": (ctypes.c_int, [_I32, _I64, _I64, _I32, _P, _P, _P, _P]),
    "cacto_dselect_local": (ctypes.c_int, [_I32, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "cacto_dselect_finish": (ctypes.c_int, [_I32, _P, _I64, _P, _P, _P, _SZ, _P]),
    "cacto_gather": (ctypes.c_int, [_PBATCH, _P, _P, _P, _P, _P, _P]),
    "cacto_ring_push": (ctypes.c_int, [_PBATCH, _P, _P, _P, _P, _P, _I64, _I64, _P]),
    "cacto_kstep_push": (ctypes.c_int, [ctypes.POINTER(CactoSolutions), _I32, _I32, _P, _P, _P, _P, _P, _I64, _I64,
                                         _I64, _P, _P]),
    "cacto_loss_workspace_bytes": (_SZ, [_PMLP, _I64]),
    "cacto_critic_loss": (ctypes.c_int, [_PMLP, _PMLP, _PBATCH, _D, _I32, _P, _SZ, _PI32, _P]),
    "cacto_actor_loss": (ctypes.c_int, [_PMLP, _PMLP, _PSYS, _PCOST, _PBATCH, _P, _P, _SZ, _PI32, _P]),
    "cacto_std_loss": (ctypes.c_int, [_PMLP, _PMLP, _PBATCH, _P, _SZ, _PI32, _P]),
    "cacto_count_live": (ctypes.c_int, [_PBATCH, _P, _P]),
    "cacto_reduce_grads": (ctypes.c_int, [_I32, _P, _I32, _I64, _P, _P, _P]),
    "cacto_adam_step": (ctypes.c_int, [_I32, _P, _P, _P, _P, _I64, _I64, _D, _D, _D, _D, _P]),
    "cacto_polyak": (ctypes.c_int, [_I32, _P, _P, _I64, _D, _P]),
    "cacto_reduce_adam": (ctypes.c_int, [_I32, _P, _I32, _I64, _P, _P, _P, _I64, _D, _D, _D, _D, _P, _D,
                                         _P, _P, _P]),
    "cacto_reduce_adam_graph": (ctypes.c_int, [_I32, _P, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _D, _D,
                                                _D, _P, _D, _P, _P]),
    "cacto_reduce_adam_graph_ring": (ctypes.c_int, [_I32, _P, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _D, _D,
                                                     _D, _P, _D, _P, _P, _I64, _I64, _P]),
    "cacto_counter_tick": (ctypes.c_int, [_P, _P]),
    "cacto_ring_copy": (ctypes.c_int, [_I32, _P, _P, _I64, _I64, _I64, _P, _I32, _P]),
    "cacto_counter_span": (ctypes.c_int, [_P, _P, _I32, _P]),
    "cacto_value_errors": (ctypes.c_int, [_PMLP, _PBATCH, _P, _P]),
    "cacto_std_loss_err": (ctypes.c_int, [_PMLP, _P, _PBATCH, _P, _SZ, _PI32, _P]),
    "cacto_sample_states": (ctypes.c_int, [_U64, _U64, _U64, _U64, _I64, _I64, _I32, _P, _P, _P, _P]),
    "cacto_gemm_workspace_bytes": (_SZ, [_I32, _I32, _I32]),
    "cacto_gemm_tf32": (ctypes.c_int, [_I32, _I32, _I32, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I32,
                                        ctypes.c_float, _I32, _P, _SZ, _P]),
    "cacto_fma_peak": (ctypes.c_int, [_I32, _I32, _I32, _P, _P]),
    "cacto_fma_peak_mode": (ctypes.c_int, [_I32, _I32, _I32, _P, _P]),
}


class CactoError(RuntimeError):
    pass


_lib = None


def load():
    """Load and type the shared library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} not built; run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cacto_abi_version() != 1:
        raise ImportError("libcacto_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str = ""):
    """Map a C-ABI status onto the reference's exception types."""
    if rc == OK:
        return
    msg = load().cacto_last_error().decode(errors="replace")
    if rc in (EVALUE, EUNSUPPORTED):
        raise ValueError(msg or what)
    raise CactoError(msg or what)


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)
