"""B200-native Snake-NeRF window hot path (arXiv 2507.01631).

Host-side mirror of the reference's tile-grid / window / sampler / trainer API
(/root/reference/proj/src/core) over the C-ABI in include/tilefield_gpu.h,
implemented by hand-written sm_100a CUDA kernels in csrc/.
"""
__all__ = ["abi", "synth"]
