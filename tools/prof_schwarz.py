"""Short workload for ncu on the NEXT-1 Schwarz kernels: C3 (32^3 elements,
N=7): two preconditioner applications (DMMA local solves, combine, coarse
CG on the N=1 context) and three flexible-PCG iterations."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_tgv  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
only_gmres = len(sys.argv) > 2 and sys.argv[2] == "gmres"   # one Jacobi GMRES(30) cycle
spec, N = CONFIGS[cfg]
torch.cuda.set_device(0)
with sem.sem_setup(spec, N) as c:
    X, Y, Z = c.coords()
    b = c.zeros()
    c.rhs(f_tgv(X, Y, Z, xp=torch), b)
    z = c.zeros()
    if only_gmres:
        x = c.zeros()
        c.gmres_solve(b, x, 0.0, 30, 30)
        torch.cuda.synchronize()
        print("prof_schwarz gmres ok")
        sys.exit(0)
    c.set_coarse_graph(False)   # ncu replays kernels, not graphs
    for _ in range(2):
        c.schwarz_apply(b, z, 3)
    c.set_precond("schwarz")
    x = c.zeros()
    c.pcg_solve(b, x, 0.0, 3)
    c.set_precond("jacobi")
    c.gmres_solve(b, x, 0.0, 16, 30)   # multi-dot / multi-axpy with K up to 16
    torch.cuda.synchronize()
print("prof_schwarz ok")
