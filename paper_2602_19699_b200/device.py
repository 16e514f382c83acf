"""Device residency: padded network buffers, precision policy, streams.

`DeviceNet` holds one network (reference `nets.Mlp`, nets.py:63-103) as a
single padded parameter buffer in HBM plus its `cacto_mlp_t` descriptor.  The
padded layout (include/cacto_b200.h) pads every hidden width to 32 or 64 and
the input width to 8/16/32 with zeros; padded entries contribute exact zeros
and receive zero gradients, so the device network is the reference network.
"""

from __future__ import annotations

import os
import weakref

import numpy as np
import torch

from . import _lib

_PRECISION = os.environ.get("CACTO_PRECISION", "fp32")


def set_precision(p: str):
    """'fp32' (default, the measured hot path) or 'fp64' (bit-faithful parity mode)."""
    global _PRECISION
    if p not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {p!r}")
    _PRECISION = p


def get_precision() -> str:
    return _PRECISION


def torch_dtype(precision=None):
    return torch.float32 if (precision or _PRECISION) == "fp32" else torch.float64


def abi_dtype(precision=None):
    return _lib.F32 if (precision or _PRECISION) == "fp32" else _lib.F64


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_19699_b200 needs a CUDA device (B200); there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return ctypes_void(torch.cuda.current_stream().cuda_stream)


def ctypes_void(v):
    import ctypes
    return ctypes.c_void_p(int(v))


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def padded_in(d: int) -> int:
    return 8 if d <= 8 else (16 if d <= 16 else 32)


MAX_HIDDEN = 1024   # CACTO_MAX_HIDDEN


def padded_hidden(widths) -> int:
    w = max(widths) if widths else 0
    if w <= 32:
        return 32
    if w <= 64:
        return 64
    if w <= MAX_HIDDEN:
        return (w + 31) // 32 * 32     # layer-wise tcgen05 path (fp32), csrc/wide.cu
    raise ValueError(f"hidden width {w} > {MAX_HIDDEN} is not supported by libcacto_b200")


def layer_layout(sizes, hp):
    """[(w_off, rows_p, cols_p, b_off, rows, cols)] per layer and the total, mirroring
    layer_offsets() in csrc/common.cuh."""
    L = len(sizes) - 1
    ip = padded_in(sizes[0])
    out, off = [], 0
    for i in range(L):
        cols_p = ip if i == 0 else hp
        rows_p = sizes[-1] if i == L - 1 else hp
        w_off = off
        off += rows_p * cols_p
        b_off = off
        off += rows_p
        out.append((w_off, rows_p, cols_p, b_off, sizes[i + 1], sizes[i]))
    return out, off


def net_sizes(mlp):
    return [int(mlp.weights[0].shape[1])] + [int(w.shape[0]) for w in mlp.weights]


class DeviceNet:
    """A network resident in HBM in the padded layout + its C descriptor."""

    def __init__(self, mlp, precision=None, params: torch.Tensor | None = None):
        self.precision = precision or _PRECISION
        self.sizes = net_sizes(mlp)
        if len(self.sizes) - 1 > _lib.MAX_LAYERS:
            raise ValueError(f"{len(self.sizes) - 1} layers > {_lib.MAX_LAYERS}")
        if self.sizes[0] > _lib.MAX_IN or self.sizes[-1] > _lib.MAX_OUT:
            raise ValueError("network input/output width not supported by libcacto_b200")
        self.L = len(self.sizes) - 1
        self.hp = padded_hidden(self.sizes[1:-1]) if self.L > 1 else 0
        self.layout, self.count = layer_layout(self.sizes, self.hp)
        self.activation = mlp.activation
        self.head = mlp.head
        self._template = mlp
        self._template_ref = None
        dev = device()
        if params is None:
            params = torch.from_numpy(self.pack(mlp.flat_params())).to(dev, torch_dtype(self.precision))
        self.params = params
        self.desc = self._descriptor(mlp)

    # -- layout conversion --------------------------------------------------------
    def pack(self, flat):
        """reference flat_params order [W0, b0, ...] -> padded host vector (float64)."""
        buf = np.zeros(self.count)
        for i, (w_off, rp, cp, b_off, rows, cols) in enumerate(self.layout):
            W = np.zeros((rp, cp))
            W[:rows, :cols] = np.asarray(flat[2 * i], dtype=float).reshape(rows, cols)
            buf[w_off:w_off + rp * cp] = W.reshape(-1)
            buf[b_off:b_off + rows] = np.asarray(flat[2 * i + 1], dtype=float).reshape(-1)
        return buf

    def unpack(self, vec):
        """padded vector (tensor or array) -> reference flat_params order (float64 numpy)."""
        if isinstance(vec, torch.Tensor):
            vec = vec.detach().to("cpu", torch.float64).numpy()
        out = []
        for (w_off, rp, cp, b_off, rows, cols) in self.layout:
            W = np.asarray(vec[w_off:w_off + rp * cp], dtype=float).reshape(rp, cp)[:rows, :cols].copy()
            out += [W, np.asarray(vec[b_off:b_off + rows], dtype=float).copy()]
        return out

    def _descriptor(self, mlp):
        d = _lib.CactoMlp()
        d.dtype = _lib.F32 if self.precision == "fp32" else _lib.F64
        d.n_layers = self.L
        for i, s in enumerate(self.sizes):
            d.sizes[i] = s
        d.hp = self.hp
        d.activation = _lib.ACT[mlp.activation]
        d.head = _lib.HEAD[mlp.head]
        d.has_norm = int(mlp.in_center is not None)
        d.sigma_min = float(mlp.sigma_min)
        if mlp.in_center is not None:
            for i, (c, h) in enumerate(zip(np.asarray(mlp.in_center, float), np.asarray(mlp.in_half, float))):
                d.in_center[i], d.in_half[i] = float(c), float(h)
        if mlp.out_scale is not None:
            for j, s in enumerate(np.asarray(mlp.out_scale, float).reshape(-1)):
                d.out_scale[j] = float(s)
        d.params = self.params.data_ptr()
        return d

    def rebind(self, params: torch.Tensor):
        self.params = params
        self.desc.params = params.data_ptr()

    @property
    def template(self):
        return self._template if self._template is not None else self._template_ref()

    def to_mlp(self, vec=None):
        """Reference-style network with these parameters (uses the template's
        `with_params` when it is a reference Mlp)."""
        flat = self.unpack(self.params if vec is None else vec)
        return self.template.with_params(flat)


# cache: immutable reference networks -> device copies (per precision)
_CACHE: dict = {}


def device_net(mlp, precision=None) -> DeviceNet:
    precision = precision or _PRECISION
    key = (id(mlp), precision)
    hit = _CACHE.get(key)
    if hit is not None and hit[0]() is mlp:
        return hit[1]
    dn = DeviceNet(mlp, precision)
    try:
        ref = weakref.ref(mlp, lambda _r, k=key, c=_CACHE: c.pop(k, None))
    except TypeError:  # not weak-referenceable: do not cache
        return dn
    dn._template, dn._template_ref = None, ref   # the cache must not keep `mlp` alive
    _CACHE[key] = (ref, dn)
    return dn


def to_device(a, precision=None, dtype=None):
    """host array -> device tensor in the compute precision (or `dtype`)."""
    t = torch.as_tensor(np.ascontiguousarray(a))
    return t.to(device(), dtype or torch_dtype(precision))
