"""Ray-sharded data parallelism through the CUDA library with two ranks
(VERDICT r1 item 5).  The round's GPU boxes have one B200, so both ranks run
their contexts on cuda:0 and the exchange is a gloo allreduce of the flat
gradient on the host: the ranks' kernels never wait on each other, only the
sharding / normalisation / replica logic of bench.py's NCCL path is under test.

Rank r takes rays [r B/2, (r+1) B/2) of the global counter-RNG stream with
batch_rays = B, so the summed gradient is the full-batch gradient (up to the
fp32 order of the hash-table atomics), and after the Adam step both replicas
hold bit-identical parameters."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B = 4096


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ctx():
    from paper_2507_01631_b200 import synth
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_scene(3, 3, tile_side=128.0, n_views=3, gsd=1.0, seed=17)
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=B, seed=9), max_rays=B)
    ctx.set_window(1, 0)
    return ctx


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = _ctx()
    share = B // world
    ctx.forward_backward(3, rank * share, share)
    g = ctx.grad_tensor()
    torch.cuda.synchronize()
    h = g.cpu()
    dist.all_reduce(h)
    g.copy_(h.cuda())
    torch.cuda.synchronize()
    loss = torch.tensor([ctx.read_loss()], dtype=torch.float64)
    dist.all_reduce(loss)
    ctx.optimizer_step(3)
    np.save(os.path.join(out, f"g{rank}.npy"), h.numpy())
    np.save(os.path.join(out, f"l{rank}.npy"), loss.numpy())
    np.save(os.path.join(out, f"p{rank}.npy"), np.concatenate([ctx.tile_state(k)["enc"] for k in range(4)]
                                                             + [ctx.color()[0]]))
    ctx.close()
    dist.destroy_process_group()


def test_two_ranks_equal_full_batch_and_stay_replicas(tmp_path):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    g0, g1 = np.load(tmp_path / "g0.npy"), np.load(tmp_path / "g1.npy")
    assert g0.tobytes() == g1.tobytes()  # every rank holds the same reduced bits
    p0, p1 = np.load(tmp_path / "p0.npy"), np.load(tmp_path / "p1.npy")
    assert p0.tobytes() == p1.tobytes()  # replicas stay identical after Adam
    ctx = _ctx()
    ctx.forward_backward(3, 0, B)
    torch.cuda.synchronize()  # the context's stream is not torch's
    full = ctx.grad_tensor().cpu().numpy()
    full_loss = ctx.read_loss()
    rel = np.linalg.norm(g0 - full) / np.linalg.norm(full)
    assert rel < 1e-4, rel  # fp32 atomic order of the hash-table scatter
    l0 = float(np.load(tmp_path / "l0.npy")[0])
    assert abs(l0 - full_loss) <= 1e-5 * full_loss
