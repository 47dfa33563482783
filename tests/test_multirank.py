"""Ray-sharded data parallelism on CPU with gloo, world_size 2.

Rank r draws rays [r*B/N, (r+1)*B/N) of the SAME global counter-RNG stream
(rng.hpp; the pixel draw of ray g depends only on (seed, iter, g)), the loss is
normalised by the global B, and the flat gradient is sum-allreduced — so the
reduced gradient equals the single-process gradient of the whole batch (up to
fp32 summation order) and every rank applies the identical Adam step.  This is
exactly what bench.py does over NCCL (ray_begin = rank * B).
"""
import os
import socket

import numpy as np
import pytest

B = 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(ses):
    parts = []
    for k in range(len(ses.window_tiles())):
        e, d, c = ses.grads(k)
        parts += [e, d]
    parts.append(ses.grads(0)[2])
    return np.concatenate(parts)


def _make(workers=2):
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200 import synth
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

    scene = synth.make_scene(2, 2, tile_side=128.0, n_views=2, gsd=2.0, seed=4)
    ses = Session(Oracle(), scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=B, seed=9), workers=workers)
    ses.set_window(0, 0)
    ses.build_accept()
    return ses


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ses = _make()
    share = B // world
    it = 3
    ses.sample(it, rank * share, share, True)
    ses.forward()
    comp = ses.composite()
    ses.backward()
    g = torch.from_numpy(_grads(ses))
    dist.all_reduce(g)
    loss = torch.tensor([comp["loss"]], dtype=torch.float64)
    dist.all_reduce(loss)
    np.save(os.path.join(out_dir, f"g{rank}.npy"), g.numpy())
    np.save(os.path.join(out_dir, f"l{rank}.npy"), loss.numpy())
    dist.destroy_process_group()


def test_sharded_gradient_equals_full_batch(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g0 = np.load(tmp_path / "g0.npy")
    g1 = np.load(tmp_path / "g1.npy")
    np.testing.assert_array_equal(g0, g1)  # every rank holds the same reduced bits
    ses = _make()
    ses.sample(3, 0, B, True)
    ses.forward()
    full = ses.composite()
    ses.backward()
    gf = _grads(ses)
    rel = np.linalg.norm(g0 - gf) / np.linalg.norm(gf)
    assert rel < 1e-5, rel
    l0 = float(np.load(tmp_path / "l0.npy")[0])
    assert abs(l0 - full["loss"]) <= 1e-9 * max(1.0, abs(full["loss"]))


def test_shards_partition_the_global_draw():
    """The union of the shards' rays is the 1-rank batch, ray for ray."""
    ses = _make()
    ses.sample(5, 0, B, True)
    full = ses.batch()["rays"]
    parts = []
    for r in range(4):
        ses.sample(5, r * (B // 4), B // 4, True)
        parts.append(ses.batch()["rays"])
    cat = np.concatenate(parts)
    for f in ("image_id", "row", "col", "origin", "direction"):
        np.testing.assert_array_equal(cat[f], full[f])
