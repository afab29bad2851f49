"""CPU checks of the C ABI: the library loads, exports every symbol include/lg.h declares, and the
host-side validation/size logic behaves as documented (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lgmod():
    from paper_2109_11978_b200 import build
    build.build()
    from paper_2109_11978_b200 import lg
    return lg


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:lg_status|int64_t|int32_t|const char\*)\s+(\w+)\s*\(", src, flags=re.M)))


def test_exports_every_header_symbol(lgmod):
    syms = header_symbols()
    assert len(syms) >= 24
    lib = ctypes.CDLL(lgmod.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(lgmod.EXPORTS)


def _cfg(lgmod, **kw):
    from paper_2109_11978_b200.context import Config
    return Config.make(**kw).to_c()


def test_param_count_and_sizes(lgmod):
    assert lgmod.lg_num_params(_cfg(lgmod)) == 571801
    assert lgmod.lg_num_params(_cfg(lgmod, scan_nx=0, scan_ny=0)) == 380313
    assert lgmod.lg_num_params(_cfg(lgmod, scan_nx=0, scan_ny=0, hidden=(128, 64, 32))) == 33657
    c = _cfg(lgmod)
    assert lgmod.lg_obs_dim(c) == 235 and lgmod.lg_obs_stride(c) == 240
    st, sizes = lgmod.lg_required_sizes(c)
    assert st == 0
    assert sizes[lgmod.BUF["OBS"]] >= 25 * 4096 * 240 * 2
    assert sizes[lgmod.BUF["STATE"]] >= 66 * 4096 * 4
    assert sizes[lgmod.BUF["HEIGHTFIELD"]] == 800 * 1600 * 4


@pytest.mark.parametrize("kw,code", [(dict(n_envs=0), 1), (dict(n_minibatches=5), 1), (dict(hidden=(500, 256, 128)), 3),
                                     (dict(gamma=1.5), 2), (dict(n_levels=0), 2), (dict(scan_nx=17, scan_ny=0), 3),
                                     (dict(lr_init=0.5), 2), (dict(rank=2, world_size=2), 2)])
def test_validation_errors(lgmod, kw, code):
    st, _ = lgmod.lg_required_sizes(_cfg(lgmod, **kw))
    assert st == code


def test_config_rejects_unknown_keys(lgmod):
    from paper_2109_11978_b200.context import Config
    with pytest.raises(ValueError):
        Config.make(n_robots=10)


def test_create_without_gpu_fails_loudly(lgmod):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, sizes = lgmod.lg_required_sizes(_cfg(lgmod))
    bufs = [256 * (i + 1) for i in range(lgmod.NUM_BUFFERS)]  # fake aligned addresses; never dereferenced
    st, ctx = lgmod.lg_create(_cfg(lgmod), bufs, 0)
    assert st == 7  # LG_ERR_UNSUPPORTED: no silent CPU fallback


def test_terrain_generate_validation_and_no_cpu_fallback(lgmod):
    import torch
    f = lgmod._lib.lg_terrain_generate
    assert f(None, 10, 20, 0, None) == 1          # LG_ERR_INVALID_ARG: no buffer
    assert f(4096, 0, 20, 0, None) == 1           # no levels
    assert f(4096, 10, 0, 0, None) == 1           # no columns
    assert f(4096, 65, 20, 0, None) == 2          # LG_ERR_RANGE: more levels than the kernel's slope table
    if not torch.cuda.is_available():
        assert f(4096, 10, 20, 0, None) == 7      # LG_ERR_UNSUPPORTED: no device, no CPU fallback
