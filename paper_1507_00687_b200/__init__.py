"""B200-native recursive fast matrix multiplication (hot path of arXiv 1507.00687).

The product is the C-ABI library libfmm_b200.so (include/fmm.h) built from csrc/ for sm_100a;
`fmm` is its thin ctypes binding.  Nothing here imports the test oracle."""
from . import fmm  # noqa: F401
from .fmm import (FmmError, Plan, Rule, choose_variants, comm_unique_id, gemm, lib,  # noqa: F401
                  matmul, node_c, node_st, scale_apply, scale_inside, scale_outside,
                  scale_repeated, unscale)
