"""Ax-only launches at several N (~16M points each) for a side-by-side ncu capture.
  python tools/prof_n.py 5,6,7"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import tgv_box  # noqa: E402

torch.cuda.set_device(0)
for N in [int(v) for v in sys.argv[1].split(",")]:
    ea = int(round(256.0 / (N + 1)))
    with sem.sem_setup(tgv_box(ea, ea, ea), N) as c:
        u = torch.empty(c.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        w = c.zeros()
        for _ in range(2):
            c.ax(u, w)
        torch.cuda.synchronize()
        print(N, c.n_local, flush=True)
