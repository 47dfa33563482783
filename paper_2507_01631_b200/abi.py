"""ctypes mirrors of the C-ABI structs in include/tilefield_gpu.h.

These are plain data layouts of the reference types (RationalCamera,
camera.hpp:22-33; Roi, tiler.hpp:10-19; FieldConfig, nn.hpp:14-37; ...) and are
shared by the product host code (paper_2507_01631_b200.tilefield) and by the
test-side oracle binding (oracle/pyoracle.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


class Rpc(C.Structure):
    """RationalCamera (camera.hpp:22-33)."""

    _fields_ = [
        ("line_num", C.c_double * 20),
        ("line_den", C.c_double * 20),
        ("samp_num", C.c_double * 20),
        ("samp_den", C.c_double * 20),
        ("line_off", C.c_double),
        ("samp_off", C.c_double),
        ("lat_off", C.c_double),
        ("long_off", C.c_double),
        ("height_off", C.c_double),
        ("line_scale", C.c_double),
        ("samp_scale", C.c_double),
        ("lat_scale", C.c_double),
        ("long_scale", C.c_double),
        ("height_scale", C.c_double),
        ("image_rows", C.c_int32),
        ("image_cols", C.c_int32),
    ]

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        if not args:  # reference defaults: scales 1 (camera.hpp:25)
            for f in ("line_scale", "samp_scale", "lat_scale", "long_scale", "height_scale"):
                if f not in kw:
                    setattr(self, f, 1.0)


class Roi(C.Structure):
    """Roi (tiler.hpp:10-19)."""

    _fields_ = [
        ("easting_min", C.c_double),
        ("easting_max", C.c_double),
        ("northing_min", C.c_double),
        ("northing_max", C.c_double),
        ("z_min", C.c_double),
        ("z_max", C.c_double),
    ]


class FieldConfig(C.Structure):
    """FieldConfig (nn.hpp:14-37); defaults() returns the reference defaults."""

    _fields_ = [
        ("levels", C.c_int32),
        ("table_size", C.c_int32),
        ("features", C.c_int32),
        ("n_min", C.c_int32),
        ("n_max", C.c_int32),
        ("density_hidden", C.c_int32),
        ("embedding", C.c_int32),
        ("color_hidden", C.c_int32),
        ("color_layers", C.c_int32),
        ("view_freqs", C.c_int32),
        ("density_max", C.c_float),
        ("occupancy_resolution", C.c_int32),
        ("occupancy_decay", C.c_float),
        ("occupancy_threshold", C.c_float),
        ("occupancy_interval", C.c_int32),
    ]

    @classmethod
    def defaults(cls) -> "FieldConfig":
        return cls(8, 1 << 15, 2, 16, 256, 64, 15, 64, 2, 4, 1e4, 32, 0.95, 0.02, 16)


class TrainConfig(C.Structure):
    """Trainer/sampler knobs (AdamConfig, LrSchedule field.hpp:16-31)."""

    _fields_ = [
        ("seed", C.c_uint64),
        ("samples_per_meter", C.c_double),
        ("max_samples_per_ray", C.c_int32),
        ("delta_cap", C.c_double),
        ("background", C.c_float * 3),
        ("margin_px", C.c_int32),
        ("lr_field", C.c_double),
        ("lr_color", C.c_double),
        ("lr_decay_rate", C.c_double),
        ("lr_decay_steps", C.c_uint64),
        ("beta1", C.c_float),
        ("beta2", C.c_float),
        ("eps", C.c_float),
        ("batch_rays", C.c_int32),
    ]

    @classmethod
    def defaults(cls, batch_rays: int = 4096, seed: int = 2) -> "TrainConfig":
        t = cls()
        t.seed = seed
        # 63 intervals over the 40 m z-extent -> 64 samples on a nadir ray.
        t.samples_per_meter = 63.0 / 40.0
        t.max_samples_per_ray = 1024
        t.delta_cap = 10.0
        t.background[:] = (0.5, 0.5, 0.5)
        t.margin_px = 4
        t.lr_field = 1e-2
        t.lr_color = 1e-3
        t.lr_decay_rate = 1.0
        t.lr_decay_steps = 1000
        t.beta1, t.beta2, t.eps = 0.9, 0.99, 1e-15
        t.batch_rays = batch_rays
        return t


class RayEntry(C.Structure):
    """RaySegmentBatch::RayEntry (ray_batch.hpp:14-20)."""

    _fields_ = [
        ("origin", C.c_double * 3),
        ("direction", C.c_double * 3),
        ("target", C.c_float * 3),
        ("image_id", C.c_int32),
        ("row", C.c_int32),
        ("col", C.c_int32),
    ]


RAY_DTYPE = np.dtype(
    [
        ("origin", "<f8", 3),
        ("direction", "<f8", 3),
        ("target", "<f4", 3),
        ("image_id", "<i4"),
        ("row", "<i4"),
        ("col", "<i4"),
    ],
    align=True,
)
assert RAY_DTYPE.itemsize == C.sizeof(RayEntry)


class BatchView(C.Structure):
    _fields_ = [
        ("rays", C.c_void_p),
        ("offsets", C.c_void_p),
        ("t", C.c_void_p),
        ("delta", C.c_void_p),
        ("local", C.c_void_p),
        ("slot", C.c_void_p),
        ("endpoint", C.c_void_p),
        ("capacity", C.c_uint64),
    ]


class TileState(C.Structure):
    _fields_ = [
        ("enc", C.c_void_p),
        ("dnet", C.c_void_p),
        ("enc_m", C.c_void_p),
        ("enc_v", C.c_void_p),
        ("dnet_m", C.c_void_p),
        ("dnet_v", C.c_void_p),
        ("enc_step", C.c_uint64),
        ("dnet_step", C.c_uint64),
        ("occupancy", C.c_void_p),
    ]


class MemoryReport(C.Structure):
    _fields_ = [
        (n, C.c_uint64)
        for n in (
            "tile_params",
            "optimizer_moments",
            "occupancy",
            "crops",
            "accept_list",
            "batch_buffers",
            "color_net",
            "staging",
            "total_device",
        )
    ]


def ptr(a: np.ndarray | None) -> C.c_void_p | None:
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    # data_as keeps a reference to the array, so temporaries outlive the call
    return a.ctypes.data_as(C.c_void_p)


def field_sizes(cfg: FieldConfig) -> tuple[int, int, int, list[int]]:
    """(enc params, dnet params, colour params, level resolutions) per
    HashGridT::init / MlpT::param_count (nn.hpp:40-45, 57-62, 180-195)."""
    import math

    res = []
    total = 0
    for l in range(cfg.levels):
        if cfg.levels <= 1:
            r = cfg.n_min
        else:
            b = math.exp((math.log(float(cfg.n_max)) - math.log(float(cfg.n_min))) / (cfg.levels - 1))
            r = int(math.floor(cfg.n_min * math.pow(b, l) + 0.5))
        res.append(r)
        total += min((r + 1) ** 3, cfg.table_size)
    enc = total * cfg.features

    def mlp(w):
        return sum(w[i + 1] * w[i] + w[i + 1] for i in range(len(w) - 1))

    dnet = mlp([cfg.levels * cfg.features, cfg.density_hidden, 1 + cfg.embedding])
    cw = [cfg.embedding + 6 * cfg.view_freqs] + [cfg.color_hidden] * cfg.color_layers + [3]
    return enc, dnet, mlp(cw), res
