"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
entry point include/tilefield_gpu.h declares, and fails loudly (no CPU
fallback) when no sm_100 device is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tilefield_gpu.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"TFG_API\s+[\w\s\*]+?\b(tfg_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_01631_b200 import tilefield

    if not os.path.exists(tilefield.LIB_PATH):
        from paper_2507_01631_b200 import build

        build.build()
    return tilefield.lib()


def test_every_declared_symbol_exported(lib):
    names = declared()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

    h = C.c_void_p()
    rc = lib.tfg_create(C.byref(FieldConfig.defaults()), C.byref(TrainConfig.defaults()), 0, 1024, C.byref(h))
    assert rc == 4  # TFG_ERR_NO_DEVICE
    assert b"no CPU fallback" in lib.tfg_last_error() or b"device" in lib.tfg_last_error()


def test_field_config_validation(lib):
    """tfg_create accepts any hash-grid geometry (n_min, n_max, power-of-two
    table_size) and rejects other widths, before it looks for a device."""
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

    def rc_of(**kw):
        cfg = FieldConfig.defaults()
        for k, v in kw.items():
            setattr(cfg, k, v)
        h = C.c_void_p()
        rc = lib.tfg_create(C.byref(cfg), C.byref(TrainConfig.defaults()), 99, 1024, C.byref(h))
        return rc, lib.tfg_last_error()

    for bad in (dict(levels=6), dict(features=4), dict(density_hidden=32), dict(color_hidden=128),
                dict(view_freqs=6), dict(occupancy_resolution=64), dict(table_size=3 << 12),
                dict(table_size=1 << 23), dict(n_min=0), dict(n_min=64, n_max=32)):
        rc, msg = rc_of(**bad)
        assert rc == 1, (bad, rc, msg)  # TFG_ERR_INVALID
    for ok in (dict(table_size=1 << 14), dict(table_size=1 << 19, n_max=2048), dict(n_min=8, n_max=512)):
        rc, msg = rc_of(**ok)
        assert rc == 4, (ok, rc, msg)  # accepted; no device 99 (here or on a GPU box)


def test_param_counts(lib):
    from paper_2507_01631_b200.abi import FieldConfig, field_sizes

    cfg = FieldConfig.defaults()
    e, d, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    assert lib.tfg_param_counts(C.byref(cfg), C.byref(e), C.byref(d), C.byref(c)) == 0
    assert (e.value, d.value, c.value) == field_sizes(cfg)[:3] == (434292, 2128, 6915)
    assert 4 * (e.value + d.value) + c.value == 1752595  # SURVEY.md §8 window size


def test_snake_path_abi(lib):
    from paper_2507_01631_b200.tilefield import snake_path

    assert snake_path(4, 4) == [(0, 0), (0, 1), (0, 2), (1, 2), (1, 1), (1, 0), (2, 0), (2, 1), (2, 2)]
