"""B200-native hot path of PetRBF (arXiv 0909.5413): Gaussian RBF interpolation by
GMRES + restricted additive Schwarz over a cell list, in hand-written sm_100a CUDA
kernels behind the C ABI of include/rbf.h (librbf.so).  See DESIGN.md."""
from .rbf import (Context, RbfError, get_nccl_id, get_option, interpolate_host, launch_count,  # noqa: F401
                  lib, options, plan_halo, plan_strips, poison_shared, set_option, trim_memory,
                  EXPORTS, LIB_PATH)
