"""B200-native GN-CG / ALS CP-decomposition hot path (cpkit drop-in).

The product is the C-ABI library lib/libcpkit_b200.so built from csrc/ for
sm_100a; `cpkit` binds it with ctypes (see include/cpkit.h, cpkit_dev.h).
"""
from . import cpkit  # noqa: F401
from .cpkit import (CpkitError, DeviceProblem, Model, Report, Tensor, decompose,  # noqa: F401
                    generate_low_rank, load, matmul_tensor, probe_dmma_peak)
