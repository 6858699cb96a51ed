"""Short, deterministic workload for ncu: C2 mesh (8192 elements, N=7).
Runs apply (Ax+mask kernel, gs kernel), Ax alone, and a 4-iteration PCG."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec, N = CONFIGS[cfg]
torch.cuda.set_device(0)
with sem.sem_setup(spec, N) as c:
    u = torch.empty(c.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    w = c.zeros()
    for _ in range(3):
        c.apply(u, w)
    for _ in range(3):
        c.ax(u, w)
    x = c.zeros()
    c.pcg_solve(u, x, 0.0, 4)
    torch.cuda.synchronize()
print("prof ok")
