"""A/B of the gather-scatter schedules (SEM_OPT_GS_MODE) on one GPU: time per
sem_gs call (w L2-resident after a preceding Ax, as in the PCG iteration: the
Ax writing w runs before each timed gs) and bit-identity of every mode's
result with the first mode's.  Prints one JSON line per (config, mode)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, tgv_box  # noqa: E402


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3"]
    modes = [int(m) for m in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 5]
    reps = 50
    for cfg in cfgs:
        if cfg.startswith("N"):
            N = int(cfg[1:])
            ea = max(2, int(round(500 / (N + 1))))
            spec = tgv_box(ea, ea, max(2, int(round(ea / 8)) * 8))
        else:
            spec, N = CONFIGS[cfg]
        st = torch.cuda.current_stream()
        with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
            nl = c.n_local
            u = torch.empty(nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
            w = c.zeros()
            ref = None
            for mode in modes:
                c.set_gs_mode(mode)
                g = u.clone()
                c.gs(g)
                torch.cuda.synchronize()
                same = True
                if ref is None:
                    ref = g
                else:
                    same = bool(torch.equal(ref, g))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                tot = 0.0
                for q in range(reps + 3):
                    c.ax(u, w)
                    e0.record(st)
                    c.gs(w)
                    e1.record(st)
                    e1.synchronize()
                    if q >= 3:
                        tot += e0.elapsed_time(e1)
                ms = tot / reps
                tot2 = 0.0   # gs right after a gs (w certainly L2-resident)
                for q in range(reps + 3):
                    c.gs(w)
                    e0.record(st)
                    c.gs(w)
                    e1.record(st)
                    e1.synchronize()
                    if q >= 3:
                        tot2 += e0.elapsed_time(e1)
                ms2 = tot2 / reps
                e0.record(st)
                for q in range(reps):
                    c.apply(u, w)
                e1.record(st)
                e1.synchronize()
                ap = e0.elapsed_time(e1) / reps
                fb = 1.0 - ((N - 1) / (N + 1)) ** 3
                print(json.dumps({"cfg": cfg, "N": N, "n_p": nl, "mode": mode, "gs_us": ms * 1e3, "gs_after_gs_us": ms2 * 1e3,
                                  "gs_gbs_alg": nl * 20 * fb / (ms / 1e3) / 1e9,
                                  "apply_us": ap * 1e3, "apply_gdofs": nl / (ap / 1e3) / 1e9,
                                  "bit_identical_to_first": same}), flush=True)


if __name__ == "__main__":
    main()
