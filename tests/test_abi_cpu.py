"""CPU checks of the boundary: libnpm.so loads without a GPU and exports every
symbol include/npm.h declares; the binding's struct layouts match the header."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "npm.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(npm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_five_hot_path_calls():
    syms = declared_symbols()
    for s in ("npm_encode", "npm_decode", "npm_pdf", "npm_sample", "npm_train_step"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2504_04315_b200 import npm
    lib = ctypes.CDLL(npm.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_struct_sizes_match_c_layout():
    from paper_2504_04315_b200 import npm
    # the library reports its compiled struct sizes (npm_abi_sizes)
    assert npm.npm_abi_sizes() == (ctypes.sizeof(npm.npm_config), ctypes.sizeof(npm.npm_query),
                                   ctypes.sizeof(npm.npm_step_stats))
    # npm_config: 10 int32 + 6 float + 7 float + pad + uint64 + int32 divergence + int32 learn_alpha
    assert ctypes.sizeof(npm.npm_config) == 10 * 4 + 6 * 4 + 7 * 4 + 4 + 8 + 4 + 4
    # npm_query: n + 11 pointers (px..rough, bsdf_pdf)
    assert ctypes.sizeof(npm.npm_query) == 8 + 11 * 8
    assert ctypes.sizeof(npm.npm_step_stats) == 6 * 8


def test_default_config_is_the_papers_model():
    from paper_2504_04315_b200 import npm
    c = npm.npm_default_config()
    # K = 8, L = 8, D_1 = 8, D_8 = 86, F = 4, 3 linear layers of width 64; lr 0.005
    assert (c.n_lobes, c.n_levels, c.base_res, c.max_res, c.n_features) == (8, 8, 8, 86, 4)
    assert (c.mlp_linear_layers, c.mlp_width) == (3, 64)
    assert abs(c.lr - 0.005) < 1e-9 and abs(c.ema_decay - 0.99) < 1e-7


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_04315_b200 import npm
    with pytest.raises(npm.NpmError):
        npm.npm_create(npm.npm_default_config(), 0)


def test_invalid_config_rejected_before_device_use():
    from paper_2504_04315_b200 import npm
    for bad in (dict(n_features=2), dict(base_res=90), dict(aabb_lo=(1, 1, 1), aabb_hi=(1, 2, 2)),
                dict(n_lobes=0), dict(mlp_width=48)):
        with pytest.raises(npm.NpmError) as e:
            npm.npm_create(npm.npm_default_config(**bad), 0)
        assert e.value.status == 1   # NPM_ERR_INVALID
