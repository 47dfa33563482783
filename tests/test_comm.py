"""Multi-GPU boundary (SURVEY.md §8b tfg_comm_init, §8e): the library's own
NCCL communicator.  Only one GPU is available per test box, so the
collective is exercised with one rank (the sum over one rank is the
identity); the sharding arithmetic across ranks is covered by
tests/test_multirank.py (gloo, world size 2)."""
import numpy as np
import pytest

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, TrainConfig


def test_unique_id_without_gpu():
    """ncclGetUniqueId needs no device: 128 bytes, fresh per call."""
    from paper_2507_01631_b200.tilefield import Context

    a, b = Context.comm_unique_id(), Context.comm_unique_id()
    assert len(a) == 128 and len(b) == 128
    assert a != b


@pytest.mark.gpu
def test_single_rank_allreduce_is_identity_and_errors_are_named():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01631_b200.tilefield import Context, TileFieldError

    scene = synth.make_scene(2, 2, tile_side=96.0, n_views=2, gsd=1.0, seed=43)
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=512, seed=5), max_rays=512)
    ctx.set_window(0, 0)
    with pytest.raises(TileFieldError, match="comm_init first"):
        ctx.allreduce_grads()
    with pytest.raises(TileFieldError, match="rank outside"):
        ctx.comm_init(Context.comm_unique_id(), 1, 1)
    ctx.comm_init(Context.comm_unique_id(), 0, 1)
    with pytest.raises(TileFieldError, match="already has a communicator"):
        ctx.comm_init(Context.comm_unique_id(), 0, 1)
    ctx.forward_backward(0, 0, 512)
    g = ctx.grad_tensor()
    before = g.clone()
    ctx.allreduce_grads()
    torch.cuda.synchronize()
    assert torch.count_nonzero(before).item() > 0
    assert torch.equal(g, before)
    ctx.optimizer_step(0)
    assert np.isfinite(ctx.read_loss())
    ctx.comm_destroy()
    with pytest.raises(TileFieldError, match="comm_init first"):
        ctx.allreduce_grads()
