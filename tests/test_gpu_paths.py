"""More B200 paths against the oracle: config 1 (single tile), the 16-tile
render path (cmd_render), a full snake progression (advance + accept +
sampler at every position, constant HBM footprint), multi-segment rays and
non-finite gradient reporting (field.hpp:45-48)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig


def _need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cmp_batch(ga, gb):
    for f in ("origin", "direction", "target", "image_id", "row", "col"):
        np.testing.assert_array_equal(ga["rays"][f], gb["rays"][f], err_msg=f)
    for f in ("offsets", "t", "delta", "local", "slot", "endpoint"):
        np.testing.assert_array_equal(ga[f], gb[f], err_msg=f)


def test_config1_single_tile():
    """1x1 grid, 4 views of ~256^2 px (BASELINE config 1)."""
    _need_gpu()
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.config_scene(1, seed=5)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=4096, seed=3)
    ctx = Context(scene, fc, tc, max_rays=4096)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    ctx.set_window(0, 0)
    ses.set_window(0, 0)
    assert ctx.window_tiles() == ses.window_tiles() == [(0, 0)]
    np.testing.assert_array_equal(ctx.accept_list(), ses.build_accept())
    assert ctx.sample(0, 0, 4096, True) == ses.sample(0, 0, 4096, True)
    _cmp_batch(ctx.batch(), ses.batch())
    for it in range(3):
        lg, lr = ctx.train_step(it, 0, 4096), ses.train_step(it, 0, 4096)
        assert abs(lg - lr) <= 1e-2 * lr, (it, lg, lr)


def test_multi_segment_rays_bit_exact():
    """Oblique rays crossing 2-3 tile boxes: segment order, shared-face
    duplicates (delta = 0) and slot runs are bit-exact."""
    _need_gpu()
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(3, 3, tile_side=96.0, n_views=3, gsd=1.0, seed=8, max_off_nadir=30.0)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=8192, seed=4)
    ctx = Context(scene, fc, tc, max_rays=8192)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    ctx.set_window(1, 1)
    ses.set_window(1, 1)
    ses.build_accept()
    assert ctx.sample(1, 0, 8192, True) == ses.sample(1, 0, 8192, True)
    b = ctx.batch()
    _cmp_batch(b, ses.batch())
    runs = []
    for i in range(8192):
        sl = b["slot"][b["offsets"][i]:b["offsets"][i + 1]]
        runs.append(1 + int(np.count_nonzero(np.diff(sl.astype(int)))))
    runs = np.array(runs)
    assert runs.max() >= 3 and (runs == 2).sum() > 100, np.bincount(runs)
    # every shared-face duplicate carries delta = 0
    dup = (np.diff(b["t"]) == 0) & (np.diff(b["slot"].astype(int)) != 0)
    assert dup.sum() > 0 and np.all(b["delta"][:-1][dup] == 0)


def test_snake_progression_bit_exact_and_constant_memory():
    """Full snake over a 4x4 grid, one iteration per position (no occupancy
    update happens, so both sides sample the same occupancy): window tiles,
    accepted lists and batches are bit-exact at every position, the device
    footprint never changes, and step counts persist across evictions."""
    _need_gpu()
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context, snake_path

    scene = synth.make_scene(4, 4, tile_side=128.0, n_views=2, gsd=2.0, seed=12)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=1024, seed=6)
    ctx = Context(scene, fc, tc, max_rays=1024)
    ses = Session(Oracle(), scene, fc, tc, workers=8)
    mem = None
    visits = {}
    path = snake_path(4, 4)
    for it, pos in enumerate(path):
        ctx.set_window(*pos)
        ses.set_window(*pos)
        if it % 2 == 0 and it + 1 < len(path):
            ctx.prefetch_window(*path[it + 1])  # every other move uses the staged buffer
        assert ctx.window_tiles() == ses.window_tiles()
        np.testing.assert_array_equal(ctx.accept_list(), ses.build_accept())
        assert ctx.sample(it, 0, 1024, True) == ses.sample(it, 0, 1024, True)
        _cmp_batch(ctx.batch(), ses.batch())
        ctx.train_step(it, 0, 1024)
        for t in ctx.window_tiles():
            visits[t] = visits.get(t, 0) + 1
        m = ctx.memory_report()["total_device"]
        mem = mem or m
        assert m == mem
    # persistent optimizer steps: each tile was stepped once per visit
    assert visits[(1, 1)] == 4 and visits[(0, 0)] == 1 and visits[(0, 1)] == 2
    ctx.set_window(1, 1)
    for k, t in enumerate(ctx.window_tiles()):
        assert ctx.tile_state(k)["enc_step"] == visits[t]


def test_render_16_tiles_matches_oracle():
    """cmd_render over a 4x4-tile ROI (config 4 shape) from random-init tiles vs
    the oracle's ray_from_pixel + segments + midpoint sampling + field + render."""
    _need_gpu()
    from oracle.pyoracle import Oracle
    from paper_2507_01631_b200.abi import Roi
    from paper_2507_01631_b200.synth import Scene, make_camera
    from paper_2507_01631_b200.tilefield import Context, tile_init

    o = Oracle()
    roi = Roi(0.0, 512.0, 0.0, 512.0, 0.0, 40.0)
    cam = make_camera(roi, 1.0, 17.0, 230.0)
    img = np.zeros((cam.image_rows, cam.image_cols, 3), np.uint8)
    scene = Scene(roi, 4, 4, [cam], [img], 1.0)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=4096, seed=1)
    ctx = Context(scene, fc, tc, max_rays=4096)
    tiles = [(r, c) for r in range(4) for c in range(4)]
    states = [tile_init(fc, 7, r, c) for r, c in tiles]
    rng = np.random.default_rng(2)
    for s in states:  # give the fields structure
        s["enc"] += rng.normal(0, 0.4, s["enc"].shape).astype(np.float32)
        s["occupancy"] = np.where(rng.random(s["occupancy"].shape) < 0.3, 0.0, 1.0).astype(np.float32)
    color = o.color_create(fc, 7)
    ctx.render_setup(tiles, states, color)
    px = np.stack([rng.integers(40, cam.image_rows - 40, 300), rng.integers(40, cam.image_cols - 40, 300)], 1)
    rgb, dep, op = ctx.render_pixels(cam, px.astype(np.int32))
    e, n = o.grid_edges(roi, 4, 4)
    boxes = np.array([[e[c], n[r], 0, e[c + 1], n[r + 1], 40] for r, c in tiles])
    frames = np.array([[b[0], b[1], b[2], 1 / (b[3] - b[0]), 1 / (b[4] - b[1]), 1 / (b[5] - b[2])] for b in boxes])
    checked = 0
    for i, (row, col) in enumerate(px):
        ray = o.ray_from_pixel(cam, int(row), int(col), 0.0, 40.0)
        if ray is None:
            continue
        org, d = ray
        segs = o.segments(org, d, boxes)
        s = o.sample_ray(org, d, segs, frames, spm=tc.samples_per_meter, occupancy=[st["occupancy"] for st in states])
        n_s = len(s["t"])
        sig = np.zeros(n_s, np.float32)
        col_ = np.zeros((n_s, 3), np.float32)
        d3 = d.astype(np.float32)
        for k in range(n_s):
            st = states[s["slot"][k]]
            sig[k], col_[k] = o.query_field(fc, st["enc"], st["dnet"], color, s["local"][k], d3)
        ref_rgb, ref_dep, ref_op, _, _ = o.render_ray(sig, col_, s["t"], s["delta"])
        np.testing.assert_allclose(rgb[i], ref_rgb, atol=5e-3)
        assert abs(op[i] - ref_op) < 5e-3
        if ref_op > 0.05:
            assert abs(dep[i] - ref_dep) < 0.05 * max(1.0, ref_dep)
        checked += 1
    assert checked > 250


def test_nonfinite_gradient_names_the_group():
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context, NonFiniteGradient

    scene = synth.make_scene(2, 2, n_views=1, gsd=2.0, seed=1)
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=512), max_rays=512)
    ctx.set_window(0, 0)
    ctx.train_step(0, 0, 512)
    st = ctx.tile_state(2)
    st["dnet"][:] = np.nan
    ctx.set_tile_state(2, st)
    before = ctx.tile_state(0)
    with pytest.raises(NonFiniteGradient, match=r"non-finite gradient in group tile\("):
        ctx.train_step(1, 0, 512)
    after = ctx.tile_state(0)
    # the step was not applied and the step counters were rolled back
    np.testing.assert_array_equal(after["enc"], before["enc"])
    assert after["enc_step"] == before["enc_step"]
    # the record is consumed once: a second read neither raises nor rolls back again
    ctx.read_loss()
    assert ctx.tile_state(0)["enc_step"] == before["enc_step"]
    _, _, _, cstep = ctx.color()
    # callers that never read the status (bench-style
    # forward_backward + optimizer_step) keep no inflated counts either, and
    # the occupancy update due at iteration 15 is skipped with the step
    occ0 = ctx.tile_state(1)["occupancy"]
    for it in (14, 15):
        ctx.forward_backward(it, 0, 512)
        ctx.optimizer_step(it)
    st1 = ctx.tile_state(0)  # settles the unverified steps
    assert st1["enc_step"] == before["enc_step"]
    np.testing.assert_array_equal(st1["enc"], before["enc"])
    np.testing.assert_array_equal(ctx.tile_state(1)["occupancy"], occ0)
    assert ctx.color()[3] == cstep
    with pytest.raises(NonFiniteGradient, match=r"non-finite gradient in group tile\("):
        ctx.read_loss()
    # a healthy tile state lets training continue with the right counts
    st["dnet"] = ctx.tile_state(0)["dnet"]
    ctx.set_tile_state(2, st)
    ctx.train_step(16, 0, 512)
    assert ctx.tile_state(0)["enc_step"] == before["enc_step"] + 1


def test_pixel_memo_matches_resolving():
    """The per-window pixel memo, with pixels of the previous position copied
    (rays + hit-tile bbox), gives the same accepted lists and batches as
    re-solving every pixel per window (reuse disabled via TFG_NO_MEMO_REUSE in
    a subprocess), along a snake that revisits pixels, with and without the
    prefetched (side-stream) staging of the next position."""
    _need_gpu()
    import json
    import os
    import subprocess
    import sys

    code = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig
from paper_2507_01631_b200.tilefield import Context, snake_path
scene = synth.make_scene(3, 3, tile_side=96.0, n_views=3, gsd=1.0, seed=21, max_off_nadir=30.0)
ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=2048, seed=5), max_rays=2048)
import os
pre = os.environ.get("TFG_TEST_PREFETCH") == "1"
path = snake_path(3, 3) + [(0, 0), (1, 1)]
out = []
for it, pos in enumerate(path):
    ctx.set_window(*pos)
    if pre and it + 1 < len(path):
        ctx.prefetch_window(*path[it + 1])
    acc = ctx.accept_list()
    ctx.sample(it, 0, 2048, True)
    b = ctx.batch()
    out.append([int(acc.size), int(np.bitwise_xor.reduce(acc)) if acc.size else 0,
                float(b["rays"]["origin"].sum()), float(b["t"].sum()), int(b["offsets"][-1])])
print(json.dumps(out))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode, memo, pre in (("memo", "0", "0"), ("solve", "1", "0"), ("pre", "0", "1")):
        env = dict(os.environ, TFG_NO_MEMO_REUSE=memo, TFG_TEST_PREFETCH=pre)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["memo"] == res["solve"]
    assert res["pre"] == res["memo"]
    assert all(r[0] > 0 for r in res["memo"])


def test_prefetched_slide_round_trips_state_bit_exactly():
    """A prefetched move stages the entering tiles' records ahead and moves
    them in by D2D; the evicted state reaches its host record asynchronously.
    Tiles that leave and come back (without training elsewhere) return
    bit-identically, with their Adam step counts."""
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(3, 3, tile_side=96.0, n_views=2, gsd=1.5, seed=14)
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=1024, seed=8), max_rays=1024)
    ctx.set_window(0, 0)
    for it in range(3):
        ctx.train_step(it, 0, 1024)
    before = {t: ctx.tile_state(k) for k, t in enumerate(ctx.window_tiles())}
    ctx.prefetch_window(0, 1)
    ctx.set_window(0, 1)  # (0,0) and (1,0) leave via the staged path
    ctx.train_step(3, 0, 1024)
    ctx.prefetch_window(1, 1)
    ctx.set_window(1, 1)  # (0,1)... leave; (0,0) and (1,0) stay out
    ctx.prefetch_window(0, 0)
    ctx.set_window(0, 0)  # (0,0), (1,0) come back from their host records
    after = {t: ctx.tile_state(k) for k, t in enumerate(ctx.window_tiles())}
    for t in ((0, 0), (1, 0)):
        for key in ("enc", "dnet", "enc_m", "enc_v", "dnet_m", "dnet_v", "occupancy"):
            assert before[t][key].tobytes() == after[t][key].tobytes(), (t, key)
        assert after[t]["enc_step"] == before[t]["enc_step"] == 3
    # the tiles trained at (0,1) carry that step too
    assert after[(0, 1)]["enc_step"] == 4 and after[(1, 1)]["enc_step"] == 4


def test_config3_full_snake_constant_memory_linear_time():
    """Config 3 shape (8x8 grid of 128 m tiles, 49 window positions; 4 of the
    16 views to bound the CPU oracle): the whole snake runs with a constant
    HBM footprint, every tile's Adam steps match its visit count, each move
    costs about the same (time linear in positions), and the accepted list
    and batch are bit-exact against the oracle at the first, a middle and the
    last position."""
    _need_gpu()
    import time

    import torch

    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context, snake_path

    c3 = synth.CONFIGS[3]
    scene = synth.make_scene(8, 8, c3["tile_side"], 40.0, 4, 1.0, seed=3)
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=2048, seed=2)
    ctx = Context(scene, fc, tc, max_rays=2048)
    path = snake_path(8, 8)
    assert len(path) == 49
    check = {0, 24, 48}
    ses = Session(Oracle(), scene, fc, tc, workers=16)
    visits, mem, dt = {}, None, []
    for it, pos in enumerate(path):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.set_window(*pos)
        if it + 1 < len(path):
            ctx.prefetch_window(*path[it + 1])
        torch.cuda.synchronize()
        dt.append(time.perf_counter() - t0)
        if it in check:
            # the oracle jumps here directly, so its slot numbering differs
            # from the GPU's (slots keep their tiles across moves): compare
            # samples by tile
            ses.set_window(*pos)
            np.testing.assert_array_equal(ctx.accept_list(), ses.build_accept())
            assert ctx.sample(it, 0, 2048, True) == ses.sample(it, 0, 2048, True)
            ga, gb = ctx.batch(), ses.batch()
            ta, tb = np.array(ctx.window_tiles()), np.array(ses.window_tiles())
            np.testing.assert_array_equal(ta[ga["slot"]], tb[gb["slot"]])
            ga["slot"] = gb["slot"]
            _cmp_batch(ga, gb)
        ctx.train_step(it, 0, 2048)
        for t in ctx.window_tiles():
            visits[t] = visits.get(t, 0) + 1
        m = ctx.memory_report()["total_device"]
        mem = mem or m
        assert m == mem
    # persistent optimizer state: steps == visits for every resident tile
    for k, t in enumerate(ctx.window_tiles()):
        assert ctx.tile_state(k)["enc_step"] == visits[t]
    assert len(visits) == 64
    # moves (after the first, which builds the initial state) cost about the same
    steady = sorted(dt[1:])
    assert steady[len(steady) * 9 // 10] < 4 * steady[len(steady) // 2] + 0.02


def test_config2_all_positions_bit_exact():
    """BASELINE config 2 (3x3 grid, 8 views at 0.5 m, 16,384 rays; seam
    correctness): at every one of its 4 window positions the accepted list and
    the full batch are bit-exact, and a training step's loss matches."""
    _need_gpu()
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context, snake_path

    scene = synth.config_scene(2, seed=2)
    c2 = synth.CONFIGS[2]
    fc, tc = FieldConfig.defaults(), TrainConfig.defaults(batch_rays=c2["batch"], seed=7)
    ctx = Context(scene, fc, tc, max_rays=c2["batch"])
    ses = Session(Oracle(), scene, fc, tc, workers=16)
    for it, pos in enumerate(snake_path(3, 3)):
        ctx.set_window(*pos)
        ses.set_window(*pos)
        np.testing.assert_array_equal(ctx.accept_list(), ses.build_accept())
        assert ctx.sample(it, 0, c2["batch"], True) == ses.sample(it, 0, c2["batch"], True)
        _cmp_batch(ctx.batch(), ses.batch())
        lg, lr = ctx.train_step(it, 0, c2["batch"]), ses.train_step(it, 0, c2["batch"])
        assert abs(lg - lr) <= 1e-2 * lr, (pos, lg, lr)


def test_pipelined_loss_reads():
    """tfg_loss_request / tfg_loss_poll: the loss of step i read after step i+1
    is enqueued equals the synchronous read; a non-finite step is reported
    once, with the step counts of it and of the later (skipped) steps rolled
    back exactly once."""
    _need_gpu()
    from paper_2507_01631_b200.tilefield import Context, NonFiniteGradient

    scene = synth.make_scene(2, 2, n_views=2, gsd=2.0, seed=6)
    tc = TrainConfig.defaults(batch_rays=1024, seed=3)
    a = Context(scene, FieldConfig.defaults(), tc, max_rays=1024)
    b = Context(scene, FieldConfig.defaults(), tc, max_rays=1024)
    a.set_window(0, 0)
    b.set_window(0, 0)
    sync = [a.train_step(it, 0, 1024) for it in range(6)]
    piped = []
    for it in range(6):
        b.forward_backward(it, 0, 1024)
        b.optimizer_step(it)
        b.request_loss()
        if it > 0:
            piped.append(b.poll_loss())
    piped.append(b.poll_loss())
    np.testing.assert_allclose(piped, sync, rtol=2e-3)
    before = b.tile_state(0)
    good = b.tile_state(2)
    bad = dict(good)
    bad["dnet"] = np.full_like(good["dnet"], np.nan)
    b.set_tile_state(2, bad)
    raised = 0
    for it in range(6, 9):
        b.forward_backward(it, 0, 1024)
        b.optimizer_step(it)
        b.request_loss()
        if it > 6:
            try:
                b.poll_loss()
            except NonFiniteGradient:
                raised += 1
                # steps 6 and 7 (the failing one and the one skipped behind
                # it) are rolled back; repair the tile so step 8 applies
                b.set_tile_state(2, good)
    b.poll_loss()
    assert raised == 1
    after = b.tile_state(0)
    assert after["enc_step"] == before["enc_step"] + 1  # only step 8 was applied
