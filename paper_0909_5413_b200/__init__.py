"""B200-native hot path of PetRBF (arXiv 0909.5413): Gaussian RBF interpolation by
GMRES + restricted additive Schwarz over a cell list, in hand-written sm_100a CUDA
kernels behind the C ABI of include/rbf.h (librbf.so).  See DESIGN.md."""
from .rbf import (Context, RbfError, get_nccl_id, interpolate_host, launch_count, lib,  # noqa: F401
                  plan_halo, plan_strips, poison_shared, EXPORTS, LIB_PATH)
