"""Schwarz local-solve kernel timing on C3 and C4 (N=7): the DMMA kernel and
the CUDA-core kernel, CUDA events per launch (sem_timing class 7)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_tgv  # noqa: E402

st = torch.cuda.current_stream()
for cfg in sys.argv[1].split(",") if len(sys.argv) > 1 else ("C3", "C4"):
    spec, N = CONFIGS[cfg]
    with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
        X, Y, Z = c.coords()
        b = c.zeros()
        c.rhs(f_tgv(X, Y, Z, xp=torch), b)
        del X, Y, Z
        z = c.zeros()
        c.schwarz_apply(b, z, 1)
        out = {"lib": os.environ.get("SEM_LIB", "default").split("/")[-1], "cfg": cfg}
        for v in (1, 0):
            c.set_fdm_tc(v)
            c.timing(True)
            for _ in range(10):
                c.schwarz_apply(b, z, 1)
            t, k = c.timing_read(7)
            c.timing(False)
            ms = t / k
            out[f"fdm{v}_ms"] = round(ms, 4)
            out[f"fdm{v}_frac_copy"] = round(20.38 * c.n_local / (ms * 1e-3) / 1e9 / 6550.7, 3)
        print(json.dumps(out), flush=True)
