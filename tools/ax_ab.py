"""Ax-kernel shape A/B on one GPU (run with SEM_LIB pointing at a build.py
--variant build): Ax alone over 4 rotating (u, w) sets, the operator (Ax+gs),
and the Jacobi-PCG iteration, on C2 (8192 elements) and C3 (32768), N=7.
Prints one JSON line per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_tgv, tgv_box  # noqa: E402


def timeit(fn, reps, st):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for q in range(3):
        fn(q)
    e0.record(st)
    for q in range(reps):
        fn(q)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    tag = os.environ.get("SEM_LIB", "default").split("/")[-1]
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3"]
    st = torch.cuda.current_stream()
    for cfg in cfgs:
        if cfg.startswith("N"):      # ~1.25e8 points (C5-like sweep size)
            N = int(cfg[1:])
            ea = max(2, int(round(500 / (N + 1))))
            spec = tgv_box(ea, ea, max(2, int(round(ea / 8)) * 8))
        elif cfg.startswith("M"):    # ~1.6e7 points
            N = int(cfg[1:])
            ea = max(2, int(round(256 / (N + 1))))
            spec = tgv_box(ea, ea, ea)
        elif cfg.startswith("B"):    # B<ex>x<ey>x<ez>: periodic box at N = 7
            N = 7
            spec = tgv_box(*[int(v) for v in cfg[1:].split("x")])
        else:
            spec, N = CONFIGS[cfg]
        with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
            nl = c.n_local
            sets = [(torch.empty(nl, dtype=torch.float64, device="cuda").uniform_(-1, 1), c.zeros())
                    for _ in range(4 if nl * 8 < 2e8 else 2)]
            ns = len(sets)
            ax = timeit(lambda q: c.ax(*sets[q % ns]), 50, st)
            ap = timeit(lambda q: c.apply(*sets[q % ns]), 50, st)
            if os.environ.get("AX_ONLY"):
                print(json.dumps({"lib": tag, "cfg": cfg, "N": N, "n_p": nl, "ax_us": ax * 1e3,
                                  "ax_frac_copy": nl * 64 / (ax / 1e3) / 1e9 / 6550.7,
                                  "apply_us": ap * 1e3}), flush=True)
                continue
            if os.environ.get("PCG_GRAPH") == "0":
                c.set_pcg_graph(False)
            if os.environ.get("PCG_FUSE") == "0":
                c.set_pcg_fuse(False)
            if os.environ.get("PCG_GSU") == "0":
                c.set_pcg_gsu(False)
            if os.environ.get("PCG_GSU_FORCE") in ("0", "1"):
                c.set_pcg_gsu(os.environ["PCG_GSU_FORCE"] == "1")
            X, Y, Z = c.coords()
            b = c.zeros()
            c.rhs(f_tgv(X, Y, Z, xp=torch), b)
            x = c.zeros()
            c.pcg_solve(b, x, 0.0, 8)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            c.pcg_solve(b, x, 0.0, 64)
            e1.record(st)
            e1.synchronize()
            it = e0.elapsed_time(e1) / 64
            print(json.dumps({"lib": tag, "cfg": cfg, "N": N, "n_p": nl, "ax_us": ax * 1e3,
                              "ax_frac_copy": nl * 64 / (ax / 1e3) / 1e9 / 6550.7,
                              "apply_us": ap * 1e3, "pcg_iter_us": it * 1e3,
                              "pcg_gdofs": nl / (it / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
