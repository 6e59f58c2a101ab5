"""B200-native gPLMM-preconditioned Newton-FGMRES for MAC Navier-Stokes on voxel
images (arXiv 2510.22077).  The compute path is libpmns.so (CUDA sm_100a,
include/pmns.h); this package only marshals arguments.  There is no CPU
fallback: importing without the built library raises."""
from ._lib import (Solver, lib, PmnsError, problem_from_config, default_opts,  # noqa: F401
                   STATUS_NAMES, LIB_PATH, release_cache)
