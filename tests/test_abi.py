"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, the ctypes structs match the C layout, and the padded
parameter layout agrees between C and Python.  No kernel is launched here."""

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "cacto_b200.h"


def _lib():
    from paper_2602_19699_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("libcacto_b200.so not built (run make)")
    return _lib


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*[a-z_0-9 \*]+?\b(cacto_[a-z_0-9]+)\(", text, re.M)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("cacto_rollout", "cacto_score", "cacto_select_topk", "cacto_gather", "cacto_critic_loss",
              "cacto_actor_loss", "cacto_std_loss", "cacto_adam_step", "cacto_polyak", "cacto_mlp_forward"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(cacto_[a-z_0-9]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_ctypes_signatures_cover_the_header():
    lib = _lib()
    assert sorted(lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_padding():
    lib = _lib()
    L = lib.load()
    assert L.cacto_abi_version() == 1
    assert [L.cacto_padded_in(d) for d in (1, 5, 8, 9, 16, 17, 32)] == [8, 8, 8, 16, 16, 32, 32]


def test_struct_layout_matches_c(tmp_path):
    lib = _lib()
    import ctypes
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "cacto_b200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(cacto_mlp_t), '
                   'offsetof(cacto_mlp_t, params), sizeof(cacto_system_t), sizeof(cacto_cost_t), '
                   'sizeof(cacto_batch_t), offsetof(cacto_batch_t, xa_plus_k));'
                   'printf("%zu %zu\\n", sizeof(cacto_solutions_t), offsetof(cacto_solutions_t, v_bar_x));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    want = [ctypes.sizeof(lib.CactoMlp), lib.CactoMlp.params.offset, ctypes.sizeof(lib.CactoSystem),
            ctypes.sizeof(lib.CactoCost), ctypes.sizeof(lib.CactoBatch), lib.CactoBatch.xa_plus_k.offset,
            ctypes.sizeof(lib.CactoSolutions), lib.CactoSolutions.v_bar_x.offset]
    assert got == want


@pytest.mark.parametrize("sizes", [[7, 64, 64, 64, 1], [6, 64, 64, 64, 2], [16, 64, 64, 64, 6],
                                   [4, 10, 8, 1], [5, 8, 2], [4, 3], [2, 16, 1]])
def test_param_count_c_equals_python(sizes):
    lib = _lib()
    from paper_2602_19699_b200.device import layer_layout, padded_hidden
    hp = padded_hidden(sizes[1:-1]) if len(sizes) > 2 else 0
    d = lib.CactoMlp()
    d.n_layers = len(sizes) - 1
    d.hp = hp
    for i, s in enumerate(sizes):
        d.sizes[i] = s
    assert lib.load().cacto_mlp_param_count(d) == layer_layout(sizes, hp)[1]


def test_pack_unpack_roundtrip_host_only():
    _lib()
    from paper_2602_19699_b200 import nets
    from paper_2602_19699_b200.device import DeviceNet
    net = nets.init_mlp([7, 40, 64, 12, 3], np.random.default_rng(0), head="tanh", out_scale=np.ones(3))
    dn = DeviceNet.__new__(DeviceNet)
    from paper_2602_19699_b200.device import layer_layout, net_sizes, padded_hidden
    dn.sizes = net_sizes(net)
    dn.hp = padded_hidden(dn.sizes[1:-1])
    dn.layout, dn.count = layer_layout(dn.sizes, dn.hp)
    vec = dn.pack(net.flat_params())
    back = dn.unpack(vec)
    for a, b in zip(back, net.flat_params()):
        np.testing.assert_array_equal(a, b)
    # padding stays zero: only the true entries are non-zero
    assert np.count_nonzero(vec) == sum(np.count_nonzero(p) for p in net.flat_params())


def test_product_refuses_to_run_without_a_gpu():
    _lib()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_19699_b200 import nets
    net = nets.init_mlp([5, 8, 1], np.random.default_rng(0))
    with pytest.raises(RuntimeError):
        nets.mlp_forward(net, np.zeros((3, 5)))


def test_specs_mirror_reference_defaults():
    from oracle import envs as O
    from paper_2602_19699_b200 import specs
    for name, d in O.DEFAULTS.items():
        s = specs.default_model(name)
        for k, v in d.items():
            assert getattr(s, k) == v, (name, k)


def test_oracle_is_not_imported_by_the_product():
    pkg = ROOT / "paper_2602_19699_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "import oracle" not in text and "from oracle" not in text, py
