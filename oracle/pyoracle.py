"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU parity checkers.

  Oracle  : oracle/build/libtforacle.so (restatement, tf_oracle.cpp)
  RefLib  : oracle/_ref/libtfref.so     (reference sources compiled verbatim)

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2507_01631_b200.abi import (
    RAY_DTYPE,
    BatchView,
    FieldConfig,
    Roi,
    Rpc,
    TileState,
    TrainConfig,
    field_sizes,
    ptr,
)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libtforacle.so")
REF_SO = os.path.join(HERE, "_ref", "libtfref.so")

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def build(ref: bool = True) -> None:
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if ref and os.path.isdir("/root/reference"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run oracle/Makefile)")
    return C.CDLL(path)


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class Oracle:
    def __init__(self):
        L = self.L = _load(ORACLE_SO)
        L.tfo_last_error.restype = C.c_char_p
        L.tfo_splitmix64.restype = C.c_uint64
        L.tfo_splitmix64.argtypes = [C.c_uint64]
        L.tfo_hash_combine.restype = C.c_uint64
        L.tfo_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
        L.tfo_create.restype = _vp
        L.tfo_create.argtypes = [_vp, _vp, _vp, C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int]
        L.tfo_destroy.argtypes = [_vp]
        for fn in ("tfo_build_accept", "tfo_accept_export", "tfo_sample", "tfo_sample_pixels"):
            getattr(L, fn).restype = C.c_int64
        L.tfo_accept_export.argtypes = [_vp, _vp, C.c_uint64]
        L.tfo_build_accept.argtypes = [_vp]
        L.tfo_sample.argtypes = [_vp, C.c_uint64, C.c_uint64, C.c_int, C.c_int]
        L.tfo_sample_pixels.argtypes = [_vp, _vp, C.c_int]
        L.tfo_set_window.argtypes = [_vp, C.c_int, C.c_int]
        L.tfo_window_tiles.argtypes = [_vp, _vp, _vp]
        L.tfo_batch_export.argtypes = [_vp, _vp]
        L.tfo_forward.argtypes = [_vp, _vp, _vp]
        L.tfo_composite.argtypes = [_vp] * 7
        L.tfo_backward.argtypes = [_vp]
        L.tfo_get_grads.argtypes = [_vp, C.c_int, _vp, _vp, _vp]
        L.tfo_optimizer_step.argtypes = [_vp, C.c_uint64]
        L.tfo_train_step.argtypes = [_vp, C.c_uint64, C.c_uint64, C.c_int, _vp]
        L.tfo_get_tile_state.argtypes = [_vp, C.c_int, _vp]
        L.tfo_set_tile_state.argtypes = [_vp, C.c_int, _vp]
        L.tfo_get_color.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.tfo_set_color.argtypes = [_vp, _vp, _vp, _vp, C.c_uint64]
        L.tfo_update_occupancy.argtypes = [_vp]
        L.tfo_set_workers.argtypes = [_vp, C.c_int]
        L.tfo_adam_step.argtypes = [_vp, _vp, _vp, _vp, C.c_uint64, _vp, C.c_double, C.c_double,
                                    C.c_uint64, C.c_float, C.c_float, C.c_float, C.c_char_p]
        L.tfo_render_ray.argtypes = [C.c_int] + [_vp] * 11
        L.tfo_render_ray.restype = None
        L.tfo_sample_ray.argtypes = [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp, _vp, C.c_int,
                                     C.c_float, C.c_double, C.c_int, C.c_double, C.c_double,
                                     C.c_int, C.c_uint64, _vp, _vp, _vp, _vp, _vp, C.c_int]
        L.tfo_tile_create.argtypes = [_vp, C.c_int, C.c_int, C.c_uint64, _vp, _vp, _vp]
        L.tfo_color_create.argtypes = [_vp, C.c_uint64, _vp]
        L.tfo_query_field.argtypes = [_vp] * 8
        L.tfo_level_resolution.argtypes = [_vp, C.c_int]
        L.tfo_snake_path.argtypes = [C.c_int, C.c_int, _vp, C.c_int]
        L.tfo_candidate_tiles.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int]
        L.tfo_grid_edges.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
        L.tfo_crop_for_tile.argtypes = [_vp, _vp, C.c_int, _vp]
        L.tfo_segments.argtypes = [_vp, _vp, _vp, C.c_int, _vp, _vp, _vp]
        L.tfo_intersect.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.tfo_ray_from_pixel.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double, _vp, _vp]
        L.tfo_localize.argtypes = [_vp, _vp, C.c_double, _vp, _vp, _vp]
        L.tfo_project.argtypes = [_vp, _vp, _vp]
        L.tfo_render_pixels.argtypes = [_vp, _vp, C.c_double, C.c_double, C.c_int, _vp, _vp, _vp, _vp, _vp,
                                         C.c_double, C.c_int, C.c_double, _vp, C.c_int, _vp, _vp, _vp, _vp, C.c_int]
        L.tfo_color_loss.argtypes = [_vp, _vp, C.c_int, C.c_int, _vp]
        L.tfo_color_loss.restype = C.c_double
        L.tfo_mlp_fwd_bwd.argtypes = [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
        L.tfo_hash_lookup_bwd.argtypes = [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp]
        L.tfo_shadow_loss_grad.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.tfo_shadow_loss_grad.restype = C.c_double

    def err(self) -> str:
        return self.L.tfo_last_error().decode()

    def render_pixels(self, cfg, cam, roi, boxes, states, color, px, spm=63.0 / 40.0, cap=1024, dcap=10.0,
                      bg=(0.5, 0.5, 0.5), workers=None):
        """cmd_render of (row, col) pixels over the given tile boxes / states
        (dicts with enc, dnet, occupancy): (rgb (n,3), depth, opacity)."""
        px = np.ascontiguousarray(px, np.int32).reshape(-1, 2)
        n, nt = px.shape[0], len(states)
        keep = [(np.ascontiguousarray(s["enc"], np.float32), np.ascontiguousarray(s["dnet"], np.float32),
                 np.ascontiguousarray(s["occupancy"], np.float32)) for s in states]
        arr = lambda i: (C.c_void_p * nt)(*[k[i].ctypes.data for k in keep])  # noqa: E731
        rgb, dep, op = np.zeros((n, 3), np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32)
        b = np.ascontiguousarray(boxes, np.float64).reshape(nt, 6)
        self.L.tfo_render_pixels(C.byref(cfg), C.byref(cam), roi.z_min, roi.z_max, nt, ptr(b), arr(0), arr(1),
                                 arr(2), ptr(np.ascontiguousarray(color, np.float32)), spm, cap, dcap,
                                 ptr(np.array(bg, np.float32)), n, ptr(px), ptr(rgb), ptr(dep), ptr(op),
                                 workers or os.cpu_count() or 1)
        return rgb, dep, op

    def color_loss(self, rgb, target, batch=None):
        """color_loss: (loss, gradient at rgb)."""
        r = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
        t = np.ascontiguousarray(target, np.float32).reshape(-1, 3)
        g = np.zeros_like(r)
        L = self.L.tfo_color_loss(ptr(r), ptr(t), r.shape[0], batch or r.shape[0], ptr(g))
        return L, g

    # -- backward primitives (same signatures as RefLib's) ---------------------
    def mlp_fwd_bwd(self, widths, params, x, d_out=None):
        w = np.array(widths, np.int32)
        out = np.zeros(widths[-1], np.float32)
        grad = np.zeros_like(params)
        d_in = np.zeros(widths[0], np.float32)
        do = None if d_out is None else np.ascontiguousarray(d_out, np.float32)
        self.L.tfo_mlp_fwd_bwd(ptr(w), len(widths), ptr(params), ptr(np.ascontiguousarray(x, np.float32)),
                               ptr(out), ptr(do), ptr(grad), ptr(d_in))
        return out, grad, d_in

    def hash_lookup_bwd(self, cfg, tables, pts, d_out=None):
        pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 3)
        n = pts.shape[0]
        out = np.zeros((n, cfg.levels * cfg.features), np.float32)
        grad = np.zeros_like(tables) if d_out is not None else None
        do = None if d_out is None else np.ascontiguousarray(d_out, np.float32)
        self.L.tfo_hash_lookup_bwd(C.byref(cfg), ptr(tables), n, ptr(pts), ptr(out), ptr(do), ptr(grad))
        return out, grad

    # -- primitives --------------------------------------------------------
    def project(self, cam: Rpc, xyz):
        x = _d(xyz)
        out = np.zeros(2)
        st = self.L.tfo_project(C.byref(cam), ptr(x), ptr(out))
        return None if st else out

    def localize(self, cam: Rpc, px, h):
        p = _d(px)
        xy = np.zeros(2)
        r = C.c_double()
        it = C.c_int()
        st = self.L.tfo_localize(C.byref(cam), ptr(p), C.c_double(h), ptr(xy), C.byref(r), C.byref(it))
        return (st, xy, r.value, it.value)

    def ray_from_pixel(self, cam: Rpc, row, col, zmin, zmax):
        o, d = np.zeros(3), np.zeros(3)
        st = self.L.tfo_ray_from_pixel(C.byref(cam), row, col, zmin, zmax, ptr(o), ptr(d))
        return None if st else (o, d)

    def intersect(self, o, d, box):
        t0, t1 = C.c_double(), C.c_double()
        st = self.L.tfo_intersect(ptr(_d(o)), ptr(_d(d)), ptr(_d(box)), C.byref(t0), C.byref(t1))
        return None if st else (t0.value, t1.value)

    def segments(self, o, d, boxes):
        b = _d(boxes).reshape(-1, 6)
        n = b.shape[0]
        sl = np.zeros(max(n, 1), np.int32)
        tn, tf = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        m = self.L.tfo_segments(ptr(_d(o)), ptr(_d(d)), ptr(b), n, ptr(sl), ptr(tn), ptr(tf))
        return [(int(sl[k]), float(tn[k]), float(tf[k])) for k in range(m)]

    def crop_for_tile(self, cam, box, margin):
        r = np.zeros(4, np.int32)
        st = self.L.tfo_crop_for_tile(C.byref(cam), ptr(_d(box)), margin, ptr(r))
        return None if st else tuple(int(v) for v in r)

    def grid_edges(self, roi: Roi, rows, cols):
        e, n = np.zeros(cols + 1), np.zeros(rows + 1)
        self.L.tfo_grid_edges(C.byref(roi), rows, cols, ptr(e), ptr(n))
        return e, n

    def candidate_tiles(self, roi, rows, cols, o, d):
        out = np.zeros(2 * 64, np.int32)
        m = self.L.tfo_candidate_tiles(C.byref(roi), rows, cols, ptr(_d(o)), ptr(_d(d)), ptr(out), 64)
        return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(min(m, 64))]

    def snake_path(self, rows, cols):
        out = np.zeros(2 * rows * cols, np.int32)
        m = self.L.tfo_snake_path(rows, cols, ptr(out), rows * cols)
        if m < 0:
            raise ValueError("snake_path: H, W must be >= 2")
        return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(m)]

    def sample_ray(self, o, d, segs, frames, spm, cap=1024, zmin=0.0, dcap=10.0, jitter=False,
                   key=0, occupancy=None, occ_res=32, occ_thr=0.02):
        n = len(segs)
        ss = np.array([s[0] for s in segs], np.int32)
        tn = np.array([s[1] for s in segs], np.float64)
        tf = np.array([s[2] for s in segs], np.float64)
        fr = _d(frames).reshape(-1, 6)
        occp = None
        if occupancy is not None:
            arrs = [np.ascontiguousarray(a, np.float32) for a in occupancy]
            occp = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
            self._keep = arrs
        capn = 4096
        t, de = np.zeros(capn, np.float32), np.zeros(capn, np.float32)
        lc = np.zeros(3 * capn, np.float32)
        sl, ep = np.zeros(capn, np.uint8), np.zeros(capn, np.uint8)
        m = self.L.tfo_sample_ray(ptr(_d(o)), ptr(_d(d)), n, ptr(ss), ptr(tn), ptr(tf), ptr(fr),
                                  C.cast(occp, C.c_void_p) if occp is not None else None,
                                  occ_res, occ_thr, spm, cap, zmin, dcap, int(jitter), key,
                                  ptr(t), ptr(de), ptr(lc), ptr(sl), ptr(ep), capn)
        return dict(t=t[:m], delta=de[:m], local=lc[: 3 * m].reshape(m, 3), slot=sl[:m], endpoint=ep[:m])

    def render_ray(self, sigma, rgb, t, delta, bg=(0.5, 0.5, 0.5), g=None):
        n = len(sigma)
        f = lambda a: np.ascontiguousarray(np.asarray(a, np.float32))
        sg, rg, tt, dl, b = f(sigma), f(rgb).reshape(-1), f(t), f(delta), f(bg)
        orgb, dep, op = np.zeros(3, np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32)
        ds = np.zeros(max(n, 1), np.float32)
        dr = np.zeros(max(3 * n, 1), np.float32)
        gg = f(g) if g is not None else None
        self.L.tfo_render_ray(n, ptr(sg), ptr(rg), ptr(tt), ptr(dl), ptr(b), ptr(orgb), ptr(dep),
                              ptr(op), ptr(gg), ptr(ds), ptr(dr))
        return orgb, float(dep[0]), float(op[0]), ds[:n], dr[: 3 * n].reshape(n, 3)

    def adam_step(self, p, g, m, v, step, lr=1e-2, rate=1.0, dsteps=1000, b1=0.9, b2=0.99,
                  eps=1e-15, group="g"):
        s = C.c_uint64(step)
        st = self.L.tfo_adam_step(ptr(p), ptr(g), ptr(m), ptr(v), p.size, C.byref(s), lr, rate,
                                  dsteps, b1, b2, eps, group.encode())
        if st:
            raise RuntimeError(self.err())
        return s.value

    def tile_create(self, cfg: FieldConfig, row, col, seed):
        enc_n, dnet_n, _, _ = field_sizes(cfg)
        enc = np.zeros(enc_n, np.float32)
        dnet = np.zeros(dnet_n, np.float32)
        occ = np.zeros(cfg.occupancy_resolution ** 3, np.float32)
        self.L.tfo_tile_create(C.byref(cfg), row, col, seed, ptr(enc), ptr(dnet), ptr(occ))
        return enc, dnet, occ

    def color_create(self, cfg: FieldConfig, seed):
        _, _, cn, _ = field_sizes(cfg)
        p = np.zeros(cn, np.float32)
        self.L.tfo_color_create(C.byref(cfg), seed, ptr(p))
        return p

    def query_field(self, cfg, enc, dnet, color, local3, dir3):
        s = np.zeros(1, np.float32)
        rgb = np.zeros(3, np.float32)
        l3 = np.ascontiguousarray(local3, np.float32)
        d3 = np.ascontiguousarray(dir3, np.float32)
        self.L.tfo_query_field(C.byref(cfg), ptr(enc), ptr(dnet), ptr(color), ptr(l3), ptr(d3),
                               ptr(s), ptr(rgb))
        return float(s[0]), rgb


class Session:
    """The oracle trainer's window state (scheduler + trainer restatement)."""

    def __init__(self, oracle: Oracle, scene, fcfg: FieldConfig, tcfg: TrainConfig, workers: int = 1):
        self.o = oracle
        self.fcfg, self.tcfg = fcfg, tcfg
        self.scene = scene
        self.enc_n, self.dnet_n, self.color_n, _ = field_sizes(fcfg)
        cams = (Rpc * scene.n_views)(*scene.cams)
        self._cams = cams
        self._imgs = [np.ascontiguousarray(im) for im in scene.images]
        imgp = (C.c_void_p * scene.n_views)(*[im.ctypes.data for im in self._imgs])
        self._imgp = imgp
        self._roi = scene.roi
        self.h = oracle.L.tfo_create(C.byref(fcfg), C.byref(tcfg), cams, scene.n_views, imgp,
                                     C.byref(scene.roi), scene.grid_rows, scene.grid_cols, workers)
        self.n_rays = 0
        self.n_samples = 0

    def __del__(self):
        try:
            self.o.L.tfo_destroy(self.h)
        except Exception:
            pass

    def _chk(self, st):
        if st != 0:
            raise RuntimeError(self.o.err())

    def set_workers(self, w):
        self.o.L.tfo_set_workers(self.h, w)

    def set_window(self, r, c):
        self._chk(self.o.L.tfo_set_window(self.h, r, c))

    def window_tiles(self):
        r, c = np.zeros(4, np.int32), np.zeros(4, np.int32)
        n = self.o.L.tfo_window_tiles(self.h, ptr(r), ptr(c))
        return [(int(r[k]), int(c[k])) for k in range(n)]

    def build_accept(self) -> np.ndarray:
        n = self.o.L.tfo_build_accept(self.h)
        out = np.zeros(max(n, 1), np.uint64)
        self.o.L.tfo_accept_export(self.h, ptr(out), n)
        return out[:n]

    def sample(self, it, ray_begin, n_rays, jitter=True):
        n = self.o.L.tfo_sample(self.h, it, ray_begin, n_rays, int(jitter))
        if n < 0:
            raise RuntimeError(self.o.err())
        self.n_rays, self.n_samples = n_rays, n
        return n

    def sample_pixels(self, pixels):
        px = np.ascontiguousarray(pixels, np.int32).reshape(-1, 3)
        n = self.o.L.tfo_sample_pixels(self.h, ptr(px), px.shape[0])
        if n < 0:
            raise RuntimeError(self.o.err())
        self.n_rays, self.n_samples = px.shape[0], n
        return n

    def batch(self) -> dict:
        R, S = self.n_rays, self.n_samples
        rays = np.zeros(R, RAY_DTYPE)
        off = np.zeros(R + 1, np.uint32)
        t, de = np.zeros(S, np.float32), np.zeros(S, np.float32)
        lc = np.zeros(3 * S, np.float32)
        sl, ep = np.zeros(S, np.uint8), np.zeros(S, np.uint8)
        bv = BatchView(rays.ctypes.data, off.ctypes.data, t.ctypes.data, de.ctypes.data,
                       lc.ctypes.data, sl.ctypes.data, ep.ctypes.data, S)
        self._chk(self.o.L.tfo_batch_export(self.h, C.byref(bv)))
        return dict(rays=rays, offsets=off, t=t, delta=de, local=lc.reshape(S, 3), slot=sl, endpoint=ep)

    def forward(self):
        S = self.n_samples
        sg, rgb = np.zeros(S, np.float32), np.zeros(3 * S, np.float32)
        self._chk(self.o.L.tfo_forward(self.h, ptr(sg), ptr(rgb)))
        return sg, rgb.reshape(S, 3)

    def composite(self):
        R, S = self.n_rays, self.n_samples
        rr, dep, op = np.zeros(3 * R, np.float32), np.zeros(R, np.float32), np.zeros(R, np.float32)
        ds, dr = np.zeros(S, np.float32), np.zeros(3 * S, np.float32)
        loss = C.c_double()
        self._chk(self.o.L.tfo_composite(self.h, ptr(rr), ptr(dep), ptr(op), ptr(ds), ptr(dr), C.byref(loss)))
        return dict(rgb=rr.reshape(R, 3), depth=dep, opacity=op, d_sigma=ds, d_rgb=dr.reshape(S, 3),
                    loss=loss.value)

    def backward(self):
        self._chk(self.o.L.tfo_backward(self.h))

    def grads(self, slot):
        e, d, c = np.zeros(self.enc_n, np.float32), np.zeros(self.dnet_n, np.float32), np.zeros(self.color_n, np.float32)
        self._chk(self.o.L.tfo_get_grads(self.h, slot, ptr(e), ptr(d), ptr(c)))
        return e, d, c

    def optimizer_step(self, it):
        self._chk(self.o.L.tfo_optimizer_step(self.h, it))

    def train_step(self, it, ray_begin, n_rays):
        loss = C.c_double()
        self._chk(self.o.L.tfo_train_step(self.h, it, ray_begin, n_rays, C.byref(loss)))
        return loss.value

    def tile_state(self, slot):
        occn = self.fcfg.occupancy_resolution ** 3
        a = {k: np.zeros(self.enc_n, np.float32) for k in ("enc", "enc_m", "enc_v")}
        a.update({k: np.zeros(self.dnet_n, np.float32) for k in ("dnet", "dnet_m", "dnet_v")})
        a["occupancy"] = np.zeros(occn, np.float32)
        ts = TileState(*[a[k].ctypes.data for k in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v")],
                       0, 0, a["occupancy"].ctypes.data)
        self._chk(self.o.L.tfo_get_tile_state(self.h, slot, C.byref(ts)))
        a["enc_step"], a["dnet_step"] = ts.enc_step, ts.dnet_step
        return a

    def set_tile_state(self, slot, a):
        ts = TileState(*[ptr(a[k]) for k in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v")],
                       a["enc_step"], a["dnet_step"], ptr(a["occupancy"]))
        self._chk(self.o.L.tfo_set_tile_state(self.h, slot, C.byref(ts)))

    def color(self):
        p, m, v = (np.zeros(self.color_n, np.float32) for _ in range(3))
        st = C.c_uint64()
        self.o.L.tfo_get_color(self.h, ptr(p), ptr(m), ptr(v), C.byref(st))
        return p, m, v, st.value

    def set_color(self, p, m, v, step):
        self.o.L.tfo_set_color(self.h, ptr(p), ptr(m), ptr(v), step)

    def update_occupancy(self):
        self._chk(self.o.L.tfo_update_occupancy(self.h))

    def shadow_loss_grad(self, enc, dnet, color, grad=True):
        """float64 shadow of the current batch: loss and (grad=True) the exact
        reverse-mode gradients, for per-slot float64 parameter arrays."""
        ns = len(enc)
        enc = [np.ascontiguousarray(e, np.float64) for e in enc]
        dnet = [np.ascontiguousarray(d, np.float64) for d in dnet]
        color = np.ascontiguousarray(color, np.float64)
        pe = (C.c_void_p * ns)(*[e.ctypes.data for e in enc])
        pd = (C.c_void_p * ns)(*[d.ctypes.data for d in dnet])
        if not grad:
            return self.o.L.tfo_shadow_loss_grad(self.h, pe, pd, ptr(color), None, None, None), None
        ge = [np.zeros_like(e) for e in enc]
        gd = [np.zeros_like(d) for d in dnet]
        gc = np.zeros_like(color)
        qe = (C.c_void_p * ns)(*[g.ctypes.data for g in ge])
        qd = (C.c_void_p * ns)(*[g.ctypes.data for g in gd])
        L = self.o.L.tfo_shadow_loss_grad(self.h, pe, pd, ptr(color), qe, qd, ptr(gc))
        return L, (ge, gd, gc)


class RefLib:
    """The reference sources compiled verbatim (oracle/_ref/libtfref.so)."""

    def __init__(self):
        L = self.L = _load(REF_SO)
        L.ref_project.argtypes = [_vp, _vp, _vp]
        L.ref_localize.argtypes = [_vp, _vp, C.c_double, _vp, _vp, _vp]
        L.ref_ray_from_pixel.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double, _vp, _vp]
        L.ref_intersect.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.ref_segments.argtypes = [_vp, _vp, _vp, C.c_int, _vp, _vp, _vp]
        L.ref_grid_edges.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
        L.ref_tile_frame.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]
        L.ref_to_local.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]
        L.ref_candidate_tiles.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int]
        L.ref_crop_for_tile.argtypes = [_vp, _vp, C.c_int, _vp]
        L.ref_level_resolution.argtypes = [_vp, C.c_int]
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_hash_combine.restype = C.c_uint64
        L.ref_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int, _vp, _vp]
        L.ref_rng_draws.restype = None
        L.ref_mlp_init.argtypes = [_vp, C.c_int, C.c_uint64, _vp]
        L.ref_mlp_fwd_bwd.argtypes = [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
        L.ref_hash_init.argtypes = [_vp, C.c_uint64, _vp]
        L.ref_hash_init.restype = C.c_uint64
        L.ref_hash_lookup_bwd.argtypes = [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp]
        L.ref_density_activation.argtypes = [C.c_float, C.c_float, _vp]
        L.ref_density_activation.restype = C.c_float
        L.ref_encode_direction.argtypes = [_vp, C.c_int, _vp]
        L.ref_encode_direction.restype = None
        L.ref_chunk_range.argtypes = [C.c_uint64, C.c_int, C.c_int, _vp, _vp]
        L.ref_chunk_range.restype = None

    def project(self, cam, xyz):
        out = np.zeros(2)
        st = self.L.ref_project(C.byref(cam), ptr(_d(xyz)), ptr(out))
        return None if st else out

    def localize(self, cam, px, h):
        xy = np.zeros(2)
        r, it = C.c_double(), C.c_int()
        st = self.L.ref_localize(C.byref(cam), ptr(_d(px)), h, ptr(xy), C.byref(r), C.byref(it))
        return (st, xy, r.value, it.value)

    def ray_from_pixel(self, cam, row, col, zmin, zmax):
        o, d = np.zeros(3), np.zeros(3)
        st = self.L.ref_ray_from_pixel(C.byref(cam), row, col, zmin, zmax, ptr(o), ptr(d))
        return None if st else (o, d)

    def intersect(self, o, d, box):
        t0, t1 = C.c_double(), C.c_double()
        st = self.L.ref_intersect(ptr(_d(o)), ptr(_d(d)), ptr(_d(box)), C.byref(t0), C.byref(t1))
        return None if st else (t0.value, t1.value)

    def segments(self, o, d, boxes):
        b = _d(boxes).reshape(-1, 6)
        n = b.shape[0]
        sl = np.zeros(max(n, 1), np.int32)
        tn, tf = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        m = self.L.ref_segments(ptr(_d(o)), ptr(_d(d)), ptr(b), n, ptr(sl), ptr(tn), ptr(tf))
        if m < 0:
            raise ValueError("TileBoxSet: overlapping tile boxes")
        return [(int(sl[k]), float(tn[k]), float(tf[k])) for k in range(m)]

    def grid_edges(self, roi, rows, cols):
        e, n = np.zeros(cols + 1), np.zeros(rows + 1)
        if self.L.ref_grid_edges(C.byref(roi), rows, cols, ptr(e), ptr(n)):
            raise ValueError("TileGrid::build rejected the grid")
        return e, n

    def tile_frame(self, roi, rows, cols, r, c):
        box, inv = np.zeros(6), np.zeros(3)
        self.L.ref_tile_frame(C.byref(roi), rows, cols, r, c, ptr(box), ptr(inv))
        return box, inv

    def to_local(self, roi, rows, cols, r, c, p):
        out = np.zeros(3)
        self.L.ref_to_local(C.byref(roi), rows, cols, r, c, ptr(_d(p)), ptr(out))
        return out

    def candidate_tiles(self, roi, rows, cols, o, d):
        out = np.zeros(128, np.int32)
        m = self.L.ref_candidate_tiles(C.byref(roi), rows, cols, ptr(_d(o)), ptr(_d(d)), ptr(out), 64)
        return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(min(m, 64))]

    def crop_for_tile(self, cam, box, margin):
        r = np.zeros(4, np.int32)
        st = self.L.ref_crop_for_tile(C.byref(cam), ptr(_d(box)), margin, ptr(r))
        return None if st else tuple(int(v) for v in r)

    def rng_draws(self, seed, kind, n, arg=0):
        u = np.zeros(n, np.uint64)
        f = np.zeros(n, np.float64)
        self.L.ref_rng_draws(seed, kind, arg, n, ptr(u), ptr(f))
        return u if kind in (0, 3) else f

    def mlp_init(self, widths, seed):
        w = np.array(widths, np.int32)
        n = sum(widths[i + 1] * widths[i] + widths[i + 1] for i in range(len(widths) - 1))
        p = np.zeros(n, np.float32)
        self.L.ref_mlp_init(ptr(w), len(widths), seed, ptr(p))
        return p

    def mlp_fwd_bwd(self, widths, params, x, d_out=None):
        w = np.array(widths, np.int32)
        out = np.zeros(widths[-1], np.float32)
        grad = np.zeros_like(params)
        d_in = np.zeros(widths[0], np.float32)
        do = None if d_out is None else np.ascontiguousarray(d_out, np.float32)
        self.L.ref_mlp_fwd_bwd(ptr(w), len(widths), ptr(params), ptr(np.ascontiguousarray(x, np.float32)),
                               ptr(out), ptr(do), ptr(grad), ptr(d_in))
        return out, grad, d_in

    def hash_init(self, cfg, seed):
        n = self.L.ref_hash_init(C.byref(cfg), seed, None)
        t = np.zeros(n, np.float32)
        self.L.ref_hash_init(C.byref(cfg), seed, ptr(t))
        return t

    def hash_lookup_bwd(self, cfg, tables, pts, d_out=None):
        pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 3)
        n = pts.shape[0]
        out = np.zeros((n, cfg.levels * cfg.features), np.float32)
        grad = np.zeros_like(tables) if d_out is not None else None
        do = None if d_out is None else np.ascontiguousarray(d_out, np.float32)
        self.L.ref_hash_lookup_bwd(C.byref(cfg), ptr(tables), n, ptr(pts), ptr(out), ptr(do), ptr(grad))
        return out, grad
