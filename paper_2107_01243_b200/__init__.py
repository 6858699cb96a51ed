"""paper_2107_01243_b200 -- B200-native matrix-free SEM pressure-Poisson hot path
(Neko, arxiv 2107.01243): Ax = D^T G D per element, gather-scatter QQ^T,
Jacobi-preconditioned CG.  Every step runs in libsem.so (hand-written CUDA for
sm_100a + NCCL); this module only marshals arguments through the C ABI
declared in include/sem.h.  There is no CPU fallback: without the built
library or a CUDA device every call raises.
"""
from ._binding import (SEM_EBREAKDOWN, SEM_ECUDA, SEM_EGEOM, SEM_EINVAL, SEM_ENCCL,  # noqa: F401
                       SEM_ENOMEM, SEM_NOT_CONVERGED, SEM_OK, Context, Plan, SemError,
                       lib_path, load, loopback_comm, loopback_create, loopback_destroy,
                       nccl_comm_destroy, nccl_comm_init, nccl_unique_id, sem_plan_create,
                       sem_setup)

__all__ = ["sem_setup", "sem_plan_create", "Context", "Plan", "SemError", "load", "lib_path",
           "nccl_unique_id", "nccl_comm_init", "nccl_comm_destroy", "loopback_create",
           "loopback_comm", "loopback_destroy"]
