"""Checkpoint format (save/load_tile_checkpoint, save/load_color_checkpoint,
field.hpp:202-210; "versioned binary layout ... bit-exact
round-trip required") and the run layout tiles/r{R}_c{C}.ckpt + color_net.ckpt
(SPEC.md:470).  The reference declares these functions but ships no field.cpp,
so the layout is ours (include/tilefield_gpu.h); the CPU tests below parse it
independently with numpy.  The GPU test checks run save/resume: restored
state is bit-identical and the next step's loss matches the uninterrupted run
(SPEC.md:313 — training itself is deterministic only up to fp32 atomic order,
so the comparison is made on the step computed from identical state)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig, field_sizes
from paper_2507_01631_b200.tilefield import (TileFieldError, load_color_checkpoint, load_tile_checkpoint,
                                             save_color_checkpoint, save_tile_checkpoint, tile_init)

KEYS = ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v", "occupancy")


def _state(fc, seed=3):
    a = tile_init(fc, 7, 1, 2)
    rng = np.random.default_rng(seed)
    for k in ("enc_m", "dnet_m"):
        a[k] = rng.normal(0, 1e-3, a[k].shape).astype(np.float32)
    for k in ("enc_v", "dnet_v"):
        a[k] = rng.random(a[k].shape).astype(np.float32) * 1e-6
    a["occupancy"] = rng.random(a["occupancy"].shape).astype(np.float32)
    a["enc"][:5] = [np.float32(-0.0), np.float32(1e-45), np.float32(3.4e38), np.float32(np.nan), 1.0]
    a["enc_step"], a["dnet_step"] = 41, 40
    return a


def _parse(path, fc):
    """Independent reader of the documented layout."""
    raw = open(path, "rb").read()
    assert raw[:8] == b"TFCKPT01"
    ver, kind = np.frombuffer(raw, np.uint32, 2, 8)
    o = 16
    cfg = raw[o:o + C.sizeof(fc)]
    assert cfg == bytes(fc)
    o += C.sizeof(fc)
    row, col = np.frombuffer(raw, np.int32, 2, o)
    o += 8
    n_params, n_occ, s0, s1 = np.frombuffer(raw, np.uint64, 4, o)
    o += 32
    body = np.frombuffer(raw, np.float32, offset=o)
    return dict(version=int(ver), kind=int(kind), row=int(row), col=int(col), n_params=int(n_params),
                n_occ=int(n_occ), steps=(int(s0), int(s1)), body=body)


def test_tile_checkpoint_round_trip_bit_exact(tmp_path):
    fc = FieldConfig.defaults()
    a = _state(fc)
    p = str(tmp_path / "r1_c2.ckpt")
    save_tile_checkpoint(p, fc, 1, 2, a)
    r, c, b = load_tile_checkpoint(p, fc)
    assert (r, c) == (1, 2)
    for k in KEYS:
        assert a[k].tobytes() == b[k].tobytes(), k  # bit-exact, NaN and -0 included
    assert (b["enc_step"], b["dnet_step"]) == (41, 40)


def test_tile_checkpoint_layout(tmp_path):
    fc = FieldConfig.defaults()
    a = _state(fc)
    p = str(tmp_path / "t.ckpt")
    save_tile_checkpoint(p, fc, 1, 2, a)
    h = _parse(p, fc)
    enc_n, dnet_n, _, _ = field_sizes(fc)
    occ = fc.occupancy_resolution ** 3
    assert (h["version"], h["kind"], h["row"], h["col"]) == (1, 1, 1, 2)
    assert (h["n_params"], h["n_occ"], h["steps"]) == (enc_n + dnet_n, occ, (41, 40))
    assert h["body"].size == 3 * (enc_n + dnet_n) + occ  # nothing else in the file
    o = 0
    for k, n in zip(KEYS, (enc_n, dnet_n, enc_n, enc_n, dnet_n, dnet_n, occ)):
        assert h["body"][o:o + n].tobytes() == a[k].tobytes(), k
        o += n


def test_checkpoint_rejects_mismatch_and_corruption(tmp_path):
    fc = FieldConfig.defaults()
    a = _state(fc)
    p = str(tmp_path / "t.ckpt")
    save_tile_checkpoint(p, fc, 0, 0, a)
    other = FieldConfig.defaults()
    other.occupancy_decay = 0.5
    with pytest.raises(TileFieldError, match="FieldConfig mismatch"):
        load_tile_checkpoint(p, other)
    with pytest.raises(TileFieldError, match="version/kind"):
        load_color_checkpoint(p, fc)  # a tile file is not a colour file
    raw = bytearray(open(p, "rb").read())
    open(p, "wb").write(raw[:-4])
    with pytest.raises(TileFieldError, match="payload size"):
        load_tile_checkpoint(p, fc)
    open(p, "wb").write(raw + b"\0" * 64)
    with pytest.raises(TileFieldError, match="payload size"):
        load_tile_checkpoint(p, fc)
    # a header whose occupancy count exceeds res^3 (stored apart
    # from the FieldConfig) must be rejected before anything is read into the
    # caller's res^3 buffer, even when the payload is padded to match it
    o_nocc = 16 + C.sizeof(fc) + 8 + 8
    bad = bytearray(raw)
    n_occ = fc.occupancy_resolution ** 3
    bad[o_nocc:o_nocc + 8] = np.uint64(n_occ + 1024).tobytes()
    open(p, "wb").write(bad + b"\0" * 4096)
    with pytest.raises(TileFieldError, match="occupancy count"):
        load_tile_checkpoint(p, fc)
    raw[0] = ord("X")
    open(p, "wb").write(raw)
    with pytest.raises(TileFieldError, match="bad magic"):
        load_tile_checkpoint(p, fc)
    with pytest.raises(TileFieldError, match="cannot open"):
        load_tile_checkpoint(str(tmp_path / "missing.ckpt"), fc)


def test_color_checkpoint_round_trip(tmp_path):
    from oracle.pyoracle import Oracle

    fc = FieldConfig.defaults()
    p = Oracle().color_create(fc, 5)
    rng = np.random.default_rng(1)
    m = rng.normal(0, 1, p.shape).astype(np.float32)
    v = rng.random(p.shape).astype(np.float32)
    f = str(tmp_path / "color_net.ckpt")
    save_color_checkpoint(f, fc, p, m, v, 123)
    q, m2, v2, st = load_color_checkpoint(f, fc)
    assert st == 123
    for x, y in ((p, q), (m, m2), (v, v2)):
        assert x.tobytes() == y.tobytes()
    h = _parse(f, fc)
    assert (h["kind"], h["row"], h["col"], h["n_params"], h["steps"][0]) == (2, -1, -1, p.size, 123)


@pytest.mark.gpu
@pytest.mark.parametrize("geometry", [{}, {"table_size": 1 << 17, "n_min": 16, "n_max": 1024}],
                         ids=["default", "T2^17_padded"])
def test_run_save_resume(tmp_path, geometry):
    """Save a run mid-snake and resume it bit-exactly; also for a hash-grid
    geometry whose table count is not a multiple of 4 floats (the slot
    records carry alignment padding, the files do not)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01631_b200.tilefield import Context, snake_path

    scene = synth.make_scene(3, 3, tile_side=96.0, n_views=2, gsd=1.5, seed=4)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=2048, seed=2)
    for k, v in geometry.items():
        setattr(fc, k, v)
    a = Context(scene, fc, tc, max_rays=2048)
    path = snake_path(3, 3)
    it = 0
    for pos in path[:3]:  # visit 3 windows, 4 iterations each
        a.set_window(*pos)
        for _ in range(4):
            a.train_step(it, 0, 2048)
            it += 1
    run = str(tmp_path / "run")
    a.save_run(run)
    assert sorted(os.listdir(os.path.join(run, "tiles")))[:2] == ["r0_c0.ckpt", "r0_c1.ckpt"]
    assert len(os.listdir(os.path.join(run, "tiles"))) == 9
    enc_n, dnet_n, _, _ = field_sizes(fc)
    # the file holds the reference's arrays, no alignment padding
    h = _parse(os.path.join(run, "tiles", "r0_c0.ckpt"), fc)
    assert h["n_params"] == enc_n + dnet_n and h["body"].size == 3 * (enc_n + dnet_n) + 32 ** 3
    b = Context(scene, fc, tc, max_rays=2048)
    b.load_run(run)
    b.set_window(*path[2])
    # slots are ordered differently after moves: match states by tile
    sa_by = {t: a.tile_state(k) for k, t in enumerate(a.window_tiles())}
    sb_by = {t: b.tile_state(k) for k, t in enumerate(b.window_tiles())}
    assert sorted(sa_by) == sorted(sb_by)
    for t, sa in sa_by.items():
        sb = sb_by[t]
        for key in KEYS:
            assert sa[key].tobytes() == sb[key].tobytes(), (t, key)
        assert (sa["enc_step"], sa["dnet_step"]) == (sb["enc_step"], sb["dnet_step"])
    ca, cb = a.color(), b.color()
    assert all(x.tobytes() == y.tobytes() for x, y in zip(ca[:3], cb[:3])) and ca[3] == cb[3]
    la, lb = a.train_step(it, 0, 2048), b.train_step(it, 0, 2048)
    assert abs(la - lb) <= 1e-6 * la, (la, lb)
    # tiles evicted before the save (not in the last window) restore too
    last = set(a.window_tiles())
    a.set_window(*path[0])
    b.set_window(*path[0])
    n = 0
    kb = {t: k for k, t in enumerate(b.window_tiles())}
    for k, t in enumerate(a.window_tiles()):
        if t in last:
            continue
        sa, sb = a.tile_state(k), b.tile_state(kb[t])
        assert sa["enc_step"] > 0
        for key in KEYS:
            assert sa[key].tobytes() == sb[key].tobytes(), (t, key)
        n += 1
    assert n > 0
