"""B200-native Neural Parametric Mixtures hot path (arXiv 2504.04315).

The product is the C-ABI library ``libnpm.so`` (include/npm.h, CUDA for
sm_100a in ``csrc/``); ``npm`` is its thin Python binding and ``dp`` the
data-parallel driver (gradient allreduce over torch.distributed / NCCL).
Importing ``paper_2504_04315_b200.npm`` fails loudly if the library is not
built: there is no CPU fallback.
"""
__all__ = ["npm", "dp", "configs"]
