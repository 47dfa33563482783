"""Host-side mirror of the reference's tile-grid / window / sampler / trainer
API over the C-ABI of libtilefield_gpu.so (include/tilefield_gpu.h).

Names follow the reference (proj/src/core): ``snake_path``/``set_window``
(scheduler ``snake_path``/``advance``), ``accept_list``
(``accept_rays``), ``sample`` (``sample_segments``,
SPEC.md:352-360, into a ``RaySegmentBatch``, ray_batch.hpp:13-49),
``field_forward``/``field_backward`` (``forward_batch``/``backward_batch``,
field.hpp:186-197), ``composite`` (``render`` + ``color_loss``),
``optimizer_step`` (``adam_step``, field.hpp:47-48) and ``train_step`` (one
trainer iteration).  Errors raise ``TileFieldError`` (the
reference's ``tilefield::Error``, common.hpp:27-34).

There is no CPU fallback: without the built library or an sm_100 device the
constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .abi import (
    RAY_DTYPE,
    BatchView,
    FieldConfig,
    MemoryReport,
    Roi,
    Rpc,
    TileState,
    TrainConfig,
    field_sizes,
    ptr,
)

LIB_PATH = os.environ.get(
    "TFG_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtilefield_gpu.so"))
_lib = None
_vp = C.c_void_p


class TileFieldError(RuntimeError):
    """tilefield::Error (common.hpp:27-30)."""


class NonFiniteGradient(TileFieldError):
    pass


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TileFieldError(
            f"{LIB_PATH} is not built; run paper_2507_01631_b200/build.py (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    L.tfg_last_error.restype = C.c_char_p
    sig = {
        "tfg_create": [_vp, _vp, C.c_int, C.c_int, _vp],
        "tfg_destroy": [_vp],
        "tfg_set_stream": [_vp, _vp],
        "tfg_set_scene": [_vp, _vp, C.c_int, _vp, _vp, C.c_int, C.c_int],
        "tfg_set_window": [_vp, C.c_int, C.c_int],
        "tfg_prefetch_window": [_vp, C.c_int, C.c_int],
        "tfg_window_tiles": [_vp, _vp, _vp],
        "tfg_snake_path": [C.c_int, C.c_int, _vp, _vp],
        "tfg_accept_count": [_vp, _vp],
        "tfg_accept_export": [_vp, _vp, C.c_uint64],
        "tfg_forward_backward": [_vp, C.c_uint64, C.c_uint64, C.c_int],
        "tfg_optimizer_step": [_vp, C.c_uint64],
        "tfg_train_step": [_vp, C.c_uint64, C.c_uint64, C.c_int, _vp],
        "tfg_grad_buffer": [_vp, _vp, _vp],
        "tfg_read_loss": [_vp, _vp],
        "tfg_loss_request": [_vp],
        "tfg_loss_poll": [_vp, _vp],
        "tfg_sample": [_vp, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _vp],
        "tfg_sample_pixels": [_vp, _vp, C.c_int, _vp],
        "tfg_batch_export": [_vp, _vp],
        "tfg_field_forward": [_vp, _vp, _vp],
        "tfg_composite": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
        "tfg_field_backward": [_vp],
        "tfg_batch_import": [_vp, _vp, C.c_int],
        "tfg_set_slot_params": [_vp, C.c_int, _vp, _vp],
        "tfg_set_color_params": [_vp, _vp],
        "tfg_set_field_outputs": [_vp, _vp, _vp],
        "tfg_field_backward_from": [_vp, _vp, _vp],
        "tfg_adam_step": [_vp, _vp, _vp, _vp, _vp, C.c_uint64, _vp, C.c_double, C.c_double, C.c_uint64,
                          C.c_float, C.c_float, C.c_float, C.c_char_p],
        "tfg_get_tile_state": [_vp, C.c_int, _vp],
        "tfg_set_tile_state": [_vp, C.c_int, _vp],
        "tfg_get_color": [_vp, _vp, _vp, _vp, _vp],
        "tfg_set_color": [_vp, _vp, _vp, _vp, C.c_uint64],
        "tfg_get_grads": [_vp, C.c_int, _vp, _vp, _vp],
        "tfg_update_occupancy": [_vp],
        "tfg_get_memory_report": [_vp, _vp],
        "tfg_render_setup": [_vp, _vp, _vp, C.c_int, _vp, _vp],
        "tfg_render_pixels": [_vp, _vp, _vp, C.c_int, _vp, _vp, _vp],
        "tfg_kernel_launch_count": [_vp, _vp],
        "tfg_copy_bytes": [_vp, _vp, _vp],
        "tfg_last_batch": [_vp, _vp, _vp],
        "tfg_tile_init": [_vp, C.c_uint64, C.c_int, C.c_int, _vp],
        "tfg_profile_enable": [_vp, C.c_int],
        "tfg_profile_read": [_vp, _vp, _vp, _vp, C.c_int, _vp],
        "tfg_param_counts": [_vp, _vp, _vp, _vp],
        "tfg_default_field_config": [_vp],
        "tfg_default_train_config": [_vp],
        "tfg_save_tile_checkpoint": [C.c_char_p, _vp, C.c_int, C.c_int, _vp],
        "tfg_load_tile_checkpoint": [C.c_char_p, _vp, _vp, _vp, _vp],
        "tfg_save_color_checkpoint": [C.c_char_p, _vp, _vp, _vp, _vp, C.c_uint64],
        "tfg_load_color_checkpoint": [C.c_char_p, _vp, _vp, _vp, _vp, _vp],
        "tfg_save_run": [_vp, C.c_char_p],
        "tfg_psnr": [_vp, _vp, _vp, C.c_uint64, _vp],
        "tfg_ssim": [_vp, _vp, _vp, C.c_int, C.c_int, _vp],
        "tfg_depth_mae": [_vp, _vp, _vp, _vp, C.c_uint64, _vp],
        "tfg_edge_band_mask": [_vp, _vp, C.c_int, _vp],
        "tfg_render_view": [_vp, _vp, _vp, _vp, _vp],
        "tfg_load_run": [_vp, C.c_char_p],
        "tfg_build_crop_cache": [_vp, C.c_char_p, _vp],
        "tfg_load_crop_cache": [_vp, C.c_char_p],
        "tfg_crop_rect": [_vp, C.c_int, C.c_int, C.c_int, _vp],
        "tfg_comm_unique_id": [_vp],
        "tfg_comm_init": [_vp, _vp, C.c_int, C.c_int],
        "tfg_allreduce_grads": [_vp],
        "tfg_comm_destroy": [_vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().tfg_last_error().decode()
        if rc == 3:
            raise NonFiniteGradient(msg)
        raise TileFieldError(msg or f"tilefield_gpu error {rc}")


def tile_init(fcfg: FieldConfig, seed: int, row: int, col: int) -> dict:
    """TileField::create (field.hpp:93): fresh params, zero moments, occupancy 1."""
    enc_n, dnet_n, _, _ = field_sizes(fcfg)
    a = {k: np.zeros(enc_n, np.float32) for k in ("enc", "enc_m", "enc_v")}
    a.update({k: np.zeros(dnet_n, np.float32) for k in ("dnet", "dnet_m", "dnet_v")})
    a["occupancy"] = np.zeros(fcfg.occupancy_resolution ** 3, np.float32)
    ts = TileState(*[a[k].ctypes.data for k in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v")],
                   0, 0, a["occupancy"].ctypes.data)
    _check(lib().tfg_tile_init(C.byref(fcfg), seed, row, col, C.byref(ts)))
    a["enc_step"], a["dnet_step"] = 0, 0
    return a


def _state_struct(a: dict) -> TileState:
    return TileState(*[ptr(a.get(k)) for k in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v")],
                     a.get("enc_step", 0), a.get("dnet_step", 0), ptr(a.get("occupancy")))


def save_tile_checkpoint(path: str, fcfg: FieldConfig, row: int, col: int, state: dict) -> None:
    """save_tile_checkpoint (field.hpp:206); layout in include/tilefield_gpu.h."""
    _check(lib().tfg_save_tile_checkpoint(os.fsencode(path), C.byref(fcfg), row, col, C.byref(_state_struct(state))))


def load_tile_checkpoint(path: str, fcfg: FieldConfig) -> tuple[int, int, dict]:
    """load_tile_checkpoint (field.hpp:207): rejects a mismatching FieldConfig."""
    enc_n, dnet_n, _, _ = field_sizes(fcfg)
    a = {k: np.zeros(enc_n, np.float32) for k in ("enc", "enc_m", "enc_v")}
    a.update({k: np.zeros(dnet_n, np.float32) for k in ("dnet", "dnet_m", "dnet_v")})
    a["occupancy"] = np.zeros(fcfg.occupancy_resolution ** 3, np.float32)
    ts = _state_struct(a)
    r, c = C.c_int(), C.c_int()
    _check(lib().tfg_load_tile_checkpoint(os.fsencode(path), C.byref(fcfg), C.byref(r), C.byref(c), C.byref(ts)))
    a["enc_step"], a["dnet_step"] = ts.enc_step, ts.dnet_step
    return r.value, c.value, a


def save_color_checkpoint(path: str, fcfg: FieldConfig, p, m=None, v=None, step: int = 0) -> None:
    """save_color_checkpoint (field.hpp:209)."""
    _check(lib().tfg_save_color_checkpoint(os.fsencode(path), C.byref(fcfg), ptr(p), ptr(m), ptr(v), step))


def load_color_checkpoint(path: str, fcfg: FieldConfig):
    """load_color_checkpoint (field.hpp:210) -> (params, m, v, step)."""
    n = field_sizes(fcfg)[2]
    p, m, v = (np.zeros(n, np.float32) for _ in range(3))
    st = C.c_uint64()
    _check(lib().tfg_load_color_checkpoint(os.fsencode(path), C.byref(fcfg), ptr(p), ptr(m), ptr(v), C.byref(st)))
    return p, m, v, st.value


def snake_path(H: int, W: int) -> list[tuple[int, int]]:
    """Window positions: rows south->north, serpentine."""
    n = C.c_int()
    _check(lib().tfg_snake_path(H, W, None, C.byref(n)))
    out = np.zeros(2 * n.value, np.int32)
    _check(lib().tfg_snake_path(H, W, ptr(out), C.byref(n)))
    return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(n.value)]


class Context:
    """One GPU's window trainer state (a tfg_ctx)."""

    def __init__(self, scene, fcfg: FieldConfig | None = None, tcfg: TrainConfig | None = None,
                 device: int = 0, max_rays: int = 65536, stream=None):
        self.fcfg = fcfg or FieldConfig.defaults()
        self.tcfg = tcfg or TrainConfig.defaults(batch_rays=max_rays)
        self.enc_n, self.dnet_n, self.color_n, _ = field_sizes(self.fcfg)
        h = C.c_void_p()
        _check(lib().tfg_create(C.byref(self.fcfg), C.byref(self.tcfg), device, max_rays, C.byref(h)))
        self.h = h
        self.max_rays = max_rays
        if stream is not None:
            _check(lib().tfg_set_stream(self.h, C.c_void_p(stream)))
        self._set_scene(scene)
        self.n_rays = 0
        self.n_samples = 0

    def _set_scene(self, scene) -> None:
        """tfg_set_scene: cameras, pinned host images, grid (re-callable)."""
        self.scene = scene
        self._cams = (Rpc * scene.n_views)(*scene.cams)
        # images may be None: the pinned host images start black and a crop
        # cache (load_crop_cache) fills the only pixels training reads
        imgs = [None if im is None else np.ascontiguousarray(im) for im in (scene.images or [None] * scene.n_views)]
        imgp = (C.c_void_p * scene.n_views)(*[None if im is None else im.ctypes.data for im in imgs])
        _check(lib().tfg_set_scene(self.h, self._cams, scene.n_views, imgp, C.byref(scene.roi),
                                   scene.grid_rows, scene.grid_cols))

    def close(self):
        if getattr(self, "h", None):
            lib().tfg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- window ------------------------------------------------------------
    def set_window(self, r: int, c: int) -> None:
        _check(lib().tfg_set_window(self.h, r, c))

    def prefetch_window(self, r: int, c: int) -> None:
        _check(lib().tfg_prefetch_window(self.h, r, c))

    def window_tiles(self) -> list[tuple[int, int]]:
        rr, cc = np.zeros(4, np.int32), np.zeros(4, np.int32)
        n = lib().tfg_window_tiles(self.h, ptr(rr), ptr(cc))
        return [(int(rr[k]), int(cc[k])) for k in range(n)]

    def accept_count(self) -> int:
        n = C.c_uint64()
        _check(lib().tfg_accept_count(self.h, C.byref(n)))
        return n.value

    def accept_list(self) -> np.ndarray:
        n = self.accept_count()
        out = np.zeros(max(n, 1), np.uint64)
        _check(lib().tfg_accept_export(self.h, ptr(out), n))
        return out[:n]

    # ---- sub-steps ---------------------------------------------------------
    def sample(self, it: int, ray_begin: int, n_rays: int, jitter: bool = True) -> int:
        n = C.c_uint64()
        _check(lib().tfg_sample(self.h, it, ray_begin, n_rays, int(jitter), C.byref(n)))
        self.n_rays, self.n_samples = n_rays, n.value
        return n.value

    def sample_pixels(self, pixels) -> int:
        px = np.ascontiguousarray(pixels, np.int32).reshape(-1, 3)
        n = C.c_uint64()
        _check(lib().tfg_sample_pixels(self.h, ptr(px), px.shape[0], C.byref(n)))
        self.n_rays, self.n_samples = px.shape[0], n.value
        return n.value

    def batch(self) -> dict:
        R, S = self.n_rays, self.n_samples
        rays = np.zeros(R, RAY_DTYPE)
        off = np.zeros(R + 1, np.uint32)
        t, de = np.zeros(S, np.float32), np.zeros(S, np.float32)
        lc = np.zeros(3 * S, np.float32)
        sl, ep = np.zeros(S, np.uint8), np.zeros(S, np.uint8)
        bv = BatchView(rays.ctypes.data, off.ctypes.data, t.ctypes.data, de.ctypes.data,
                       lc.ctypes.data, sl.ctypes.data, ep.ctypes.data, S)
        _check(lib().tfg_batch_export(self.h, C.byref(bv)))
        return dict(rays=rays, offsets=off, t=t, delta=de, local=lc.reshape(S, 3), slot=sl, endpoint=ep)

    def batch_import(self, b: dict) -> int:
        """A caller-built RaySegmentBatch (dict as batch() returns) becomes the
        current batch (the batch argument of forward_batch / backward_batch)."""
        rays = np.ascontiguousarray(b["rays"], RAY_DTYPE)
        off = np.ascontiguousarray(b["offsets"], np.uint32)
        arrs = [np.ascontiguousarray(b[k], dt) for k, dt in
                (("t", np.float32), ("delta", np.float32), ("local", np.float32), ("slot", np.uint8),
                 ("endpoint", np.uint8))]
        R = rays.shape[0]
        S = int(off[-1])
        bv = BatchView(rays.ctypes.data, off.ctypes.data, *[a.ctypes.data for a in arrs], S)
        _check(lib().tfg_batch_import(self.h, C.byref(bv), R))
        self.n_rays, self.n_samples = R, S
        return S

    def set_slot_params(self, slot: int, enc=None, dnet=None) -> None:
        """FieldParamView (field.hpp:130-137): caller parameters into a slot."""
        e = None if enc is None else np.ascontiguousarray(enc, np.float32)
        d = None if dnet is None else np.ascontiguousarray(dnet, np.float32)
        _check(lib().tfg_set_slot_params(self.h, slot, ptr(e), ptr(d)))

    def set_color_params(self, params) -> None:
        """ColorParamView (field.hpp:139-144)."""
        _check(lib().tfg_set_color_params(self.h, ptr(np.ascontiguousarray(params, np.float32))))

    def set_field_outputs(self, sigma, rgb) -> None:
        """Per-sample sigma / rgb (ray order) as the batch's field outputs."""
        sg = np.ascontiguousarray(sigma, np.float32)
        rg = np.ascontiguousarray(rgb, np.float32).reshape(-1)
        if sg.size != self.n_samples or rg.size != 3 * self.n_samples:
            raise ValueError("set_field_outputs: one sigma and three rgb per sample")
        _check(lib().tfg_set_field_outputs(self.h, ptr(sg), ptr(rg)))

    def field_backward_from(self, d_sigma, d_rgb) -> None:
        """backward_batch from caller d_sigma / d_rgb (field.hpp:193-197)."""
        ds = np.ascontiguousarray(d_sigma, np.float32)
        dr = np.ascontiguousarray(d_rgb, np.float32).reshape(-1)
        if ds.size != self.n_samples or dr.size != 3 * self.n_samples:
            raise ValueError("field_backward_from: one d_sigma and three d_rgb per sample")
        _check(lib().tfg_field_backward_from(self.h, ptr(ds), ptr(dr)))

    def adam_step(self, params, grads, m, v, step: int, lr: float = 1e-2, decay_rate: float = 1.0,
                  decay_steps: int = 1000, beta1: float = 0.9, beta2: float = 0.99, eps: float = 1e-15,
                  group: str = "params") -> int:
        """adam_step (field.hpp:45-48) in place on float32 arrays (numpy, or
        torch CUDA tensors); returns the new step count."""
        def addr(a):
            if hasattr(a, "data_ptr"):
                return C.c_void_p(a.data_ptr())
            return ptr(a)
        n = params.numel() if hasattr(params, "numel") else params.size
        st = C.c_uint64(step)
        _check(lib().tfg_adam_step(self.h, addr(params), addr(grads), addr(m), addr(v), n, C.byref(st), lr,
                                   decay_rate, decay_steps, beta1, beta2, eps, group.encode()))
        return st.value

    def field_forward(self):
        S = self.n_samples
        sg, rgb = np.zeros(S, np.float32), np.zeros(3 * S, np.float32)
        _check(lib().tfg_field_forward(self.h, ptr(sg), ptr(rgb)))
        return sg, rgb.reshape(S, 3)

    def composite(self) -> dict:
        R, S = self.n_rays, self.n_samples
        rr, dep, op = np.zeros(3 * R, np.float32), np.zeros(R, np.float32), np.zeros(R, np.float32)
        ds, dr = np.zeros(S, np.float32), np.zeros(3 * S, np.float32)
        loss = C.c_float()
        _check(lib().tfg_composite(self.h, ptr(rr), ptr(dep), ptr(op), ptr(ds), ptr(dr), C.byref(loss)))
        return dict(rgb=rr.reshape(R, 3), depth=dep, opacity=op, d_sigma=ds, d_rgb=dr.reshape(S, 3),
                    loss=loss.value)

    def field_backward(self) -> None:
        _check(lib().tfg_field_backward(self.h))

    def grads(self, slot: int):
        e = np.zeros(self.enc_n, np.float32)
        d = np.zeros(self.dnet_n, np.float32)
        c = np.zeros(self.color_n, np.float32)
        _check(lib().tfg_get_grads(self.h, slot, ptr(e), ptr(d), ptr(c)))
        return e, d, c

    def optimizer_step(self, it: int) -> None:
        _check(lib().tfg_optimizer_step(self.h, it))

    def forward_backward(self, it: int, ray_begin: int, n_rays: int) -> None:
        _check(lib().tfg_forward_backward(self.h, it, ray_begin, n_rays))

    def read_loss(self) -> float:
        l = C.c_float()
        _check(lib().tfg_read_loss(self.h, C.byref(l)))
        return l.value

    def request_loss(self) -> None:
        """Asynchronous snapshot of the loss / status so far (poll_loss reads it)."""
        _check(lib().tfg_loss_request(self.h))

    def poll_loss(self) -> float:
        """The oldest requested loss (waits for it); raises like read_loss."""
        l = C.c_float()
        _check(lib().tfg_loss_poll(self.h, C.byref(l)))
        return l.value

    def train_step(self, it: int, ray_begin: int = 0, n_rays: int | None = None) -> float:
        l = C.c_float()
        _check(lib().tfg_train_step(self.h, it, ray_begin, n_rays or self.max_rays, C.byref(l)))
        return l.value

    # ---- multi-GPU through the C-ABI's own NCCL communicator.  torch is
    # imported first so that the library binds torch's libnccl.so.2 instead of
    # loading the system copy under the same soname (torch would then fail to
    # import against the older one).
    @staticmethod
    def comm_unique_id() -> bytes:
        """128-byte NCCL id (rank 0 creates it; the host distributes it)."""
        import torch  # noqa: F401  (see above)

        buf = (C.c_uint8 * 128)()
        _check(lib().tfg_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes, rank: int, nranks: int) -> None:
        if len(uid) != 128:
            raise ValueError("comm_init: the NCCL id is 128 bytes")
        import torch  # noqa: F401  (see comm_unique_id)

        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().tfg_comm_init(self.h, buf, rank, nranks))

    def allreduce_grads(self) -> None:
        """In-place sum of the flat gradient buffer over the ranks (context stream)."""
        _check(lib().tfg_allreduce_grads(self.h))

    def comm_destroy(self) -> None:
        _check(lib().tfg_comm_destroy(self.h))

    def grad_buffer(self) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib().tfg_grad_buffer(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def grad_tensor(self):
        """The flat gradient buffer as a torch CUDA tensor (allreduce target)."""
        import torch

        p, n = self.grad_buffer()

        class _Cai:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (p, False), "version": 3}

        return torch.as_tensor(_Cai(), device="cuda")

    # ---- state ---------------------------------------------------------------
    def tile_state(self, slot: int) -> dict:
        occn = self.fcfg.occupancy_resolution ** 3
        a = {k: np.zeros(self.enc_n, np.float32) for k in ("enc", "enc_m", "enc_v")}
        a.update({k: np.zeros(self.dnet_n, np.float32) for k in ("dnet", "dnet_m", "dnet_v")})
        a["occupancy"] = np.zeros(occn, np.float32)
        ts = TileState(*[a[k].ctypes.data for k in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v")],
                       0, 0, a["occupancy"].ctypes.data)
        _check(lib().tfg_get_tile_state(self.h, slot, C.byref(ts)))
        a["enc_step"], a["dnet_step"] = ts.enc_step, ts.dnet_step
        return a

    def set_tile_state(self, slot: int, a: dict) -> None:
        ts = TileState(*[ptr(a.get(k)) for k in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v")],
                       a.get("enc_step", 0), a.get("dnet_step", 0), ptr(a.get("occupancy")))
        _check(lib().tfg_set_tile_state(self.h, slot, C.byref(ts)))

    def color(self):
        p, m, v = (np.zeros(self.color_n, np.float32) for _ in range(3))
        st = C.c_uint64()
        _check(lib().tfg_get_color(self.h, ptr(p), ptr(m), ptr(v), C.byref(st)))
        return p, m, v, st.value

    def set_color(self, p, m=None, v=None, step=0) -> None:
        _check(lib().tfg_set_color(self.h, ptr(p), ptr(m), ptr(v), step))

    def save_run(self, directory: str) -> None:
        """Checkpoint every materialised tile (tiles/r{R}_c{C}.ckpt) and the
        colour net (color_net.ckpt) — the run layout of SPEC.md:470."""
        os.makedirs(os.path.join(directory, "tiles"), exist_ok=True)
        _check(lib().tfg_save_run(self.h, os.fsencode(directory)))

    def load_run(self, directory: str) -> None:
        """Resume a saved run (before the first set_window)."""
        _check(lib().tfg_load_run(self.h, os.fsencode(directory)))

    def update_occupancy(self) -> None:
        _check(lib().tfg_update_occupancy(self.h))

    def memory_report(self) -> dict:
        m = MemoryReport()
        _check(lib().tfg_get_memory_report(self.h, C.byref(m)))
        return {k: getattr(m, k) for k, _ in MemoryReport._fields_}

    def launches(self) -> int:
        n = C.c_uint64()
        _check(lib().tfg_kernel_launch_count(self.h, C.byref(n)))
        return n.value

    def last_batch(self) -> tuple[int, int]:
        r, n = C.c_int(), C.c_uint64()
        _check(lib().tfg_last_batch(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value

    def copy_bytes(self) -> tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        _check(lib().tfg_copy_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile_enable(self, on: bool = True) -> None:
        _check(lib().tfg_profile_enable(self.h, int(on)))

    def profile_read(self) -> dict:
        """{phase: (device ms, kernel launches)} since profile_enable."""
        names = (C.c_char_p * 16)()
        ms = np.zeros(16, np.float64)
        ln = np.zeros(16, np.uint64)
        n = C.c_int()
        _check(lib().tfg_profile_read(self.h, names, ptr(ms), ptr(ln), 16, C.byref(n)))
        return {names[i].decode(): (float(ms[i]), int(ln[i])) for i in range(n.value)}

    # ---- render ---------------------------------------------------------------
    def render_setup(self, tiles: list[tuple[int, int]], states: list[dict], color) -> None:
        n = len(tiles)
        rows = np.array([t[0] for t in tiles], np.int32)
        cols = np.array([t[1] for t in tiles], np.int32)
        self._rkeep = states
        arr = (TileState * n)(*[
            TileState(ptr(s["enc"]), ptr(s["dnet"]), None, None, None, None, 0, 0, ptr(s.get("occupancy")))
            for s in states])
        self._rarr = arr
        _check(lib().tfg_render_setup(self.h, ptr(rows), ptr(cols), n, arr, ptr(np.ascontiguousarray(color, np.float32))))

    def render_pixels(self, cam: Rpc, pixels, out=None):
        """Renders (row, col) pixels of `cam`.  `out` = (rgb[n*3], depth[n],
        opacity[n]) float32 arrays to fill (reused buffers avoid the page
        faults of fresh ones); else new arrays are returned."""
        px = np.ascontiguousarray(pixels, np.int32).reshape(-1, 2)
        n = px.shape[0]
        if out is None:
            rgb, dep, op = np.empty(3 * n, np.float32), np.empty(n, np.float32), np.empty(n, np.float32)
        else:
            rgb, dep, op = out
            if not all(a.dtype == np.float32 and a.flags.c_contiguous for a in (rgb, dep, op)) or \
                    rgb.size != 3 * n or dep.size != n or op.size != n:
                raise ValueError("render_pixels: out must be contiguous float32 arrays of 3n, n, n")
        _check(lib().tfg_render_pixels(self.h, C.byref(cam), ptr(px), n, ptr(rgb), ptr(dep), ptr(op)))
        return rgb.reshape(n, 3), dep, op

    def render_view(self, cam: Rpc):
        """Full-frame render of `cam` (cmd_render): (rows, cols, 3)
        rgb, (rows, cols) depth and opacity."""
        R, W = cam.image_rows, cam.image_cols
        rgb = np.zeros((R, W, 3), np.float32)
        dep, op = np.zeros((R, W), np.float32), np.zeros((R, W), np.float32)
        _check(lib().tfg_render_view(self.h, C.byref(cam), ptr(rgb), ptr(dep), ptr(op)))
        return rgb, dep, op

    # ---- crop cache (build_crop_cache) ------------------------
    def build_crop_cache(self, path: str) -> int:
        """Writes every (view, tile) crop of the scene + an index; returns the
        total crop bytes."""
        n = C.c_uint64()
        _check(lib().tfg_build_crop_cache(self.h, os.fsencode(path), C.byref(n)))
        return n.value

    def load_crop_cache(self, path: str) -> None:
        """Fills the pinned host images from a crop cache of this scene (before
        the first set_window); training then reads only cached crops."""
        _check(lib().tfg_load_crop_cache(self.h, os.fsencode(path)))

    def crop_rect(self, view: int, row: int, col: int):
        """crop_for_tile of (view, tile) as (r0, r1, c0, c1); None if empty."""
        r = np.zeros(4, np.int32)
        _check(lib().tfg_crop_rect(self.h, view, row, col, ptr(r)))
        return None if r[0] >= r[1] or r[2] >= r[3] else tuple(int(x) for x in r)

    # ---- evaluation (evalio) ---------------------------------
    def psnr(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        if a.shape != b.shape:
            raise TileFieldError("psnr: shape mismatch")
        out = C.c_double()
        _check(lib().tfg_psnr(self.h, ptr(a), ptr(b), a.size, C.byref(out)))
        return out.value

    def ssim(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
            raise TileFieldError("ssim: expects two (rows, cols, 3) images")
        out = C.c_double()
        _check(lib().tfg_ssim(self.h, ptr(a), ptr(b), a.shape[0], a.shape[1], C.byref(out)))
        return out.value

    def depth_mae(self, d1, d2, mask=None) -> float:
        d1 = np.ascontiguousarray(d1, np.float32)
        d2 = np.ascontiguousarray(d2, np.float32)
        if d1.shape != d2.shape:
            raise TileFieldError("depth_mae: shape mismatch")
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        out = C.c_double()
        _check(lib().tfg_depth_mae(self.h, ptr(d1), ptr(d2), ptr(m), d1.size, C.byref(out)))
        return out.value

    def edge_band_mask(self, cam: Rpc, band_px: int = 8) -> np.ndarray:
        m = np.zeros((cam.image_rows, cam.image_cols), np.uint8)
        _check(lib().tfg_edge_band_mask(self.h, C.byref(cam), band_px, ptr(m)))
        return m
