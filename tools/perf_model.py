"""The paper's performance model (Eqs. 12-15) instantiated for the
B200 hot path.

  torchrun --nproc-per-node P tools/perf_model.py probe > probe.json
      alpha*: 10,000 device ping-pongs through the NVLink mailboxes (rank 0 <-> each
      peer; P:L373 samples 10,000 ping-pongs); beta*: one-sided peer-write bandwidth
      over message sizes (postal model t(m) = alpha* + beta* m).
  python tools/perf_model.py model probe.json <final_measure dir> [out.md]
      T = T_a + T_c per PCG iteration:
        T_a = sum_k max(W_k / (pi P), Q_k / (beta P))      (Eqs. 12-13, cold cache,
              per kernel k of the iteration as built, §5 of DESIGN.md)
        T_c = 2 t_allreduce + t_gs                          (one gs exchange and two
              allreduces per iteration)
        t_allreduce: Eq. 14, max over PEs of the sum of log2(P) sampled latencies
              (the paper's binary fan-in/fan-out), and "as built": every rank
              publishes to every mailbox directly, one level -> max of P samples;
        t_gs: Eq. 15 with the slab's real shared-point count instead of the cube
              surface: 2 beta* n_s + max over the 2 neighbours of (alpha1 + alpha2).
      beta = the STREAM triad measured in the same run, pi = fp64 peak
      derived from unit counts (148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz).
      Prints predicted vs measured per-iteration times and the 8-GPU projection.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PI_FP64 = 148 * 64 * 2 * 1.965e9   # flop/s, derived (B200 has full-rate fp64 vector units)


def probe():
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2107_01243_b200 as sem
    from sem_inputs import CONFIGS, weak_scaled
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [sem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.nccl_comm_init(uid[0], rank, P)
    spec, N = CONFIGS["C2"]
    res = {"P": P, "pingpong": {}, "write_bw": {}}
    with sem.sem_setup(weak_scaled(spec, P), N, rank=rank, nranks=P, nccl_comm=comm) as c:
        for q in range(1, P):
            dist.barrier()
            if rank in (0, q):
                c.p2p_pingpong(q if rank == 0 else 0, 200)          # warm
                rt = c.p2p_pingpong(q if rank == 0 else 0, 10000)
                if rank == 0:
                    one = rt.astype(np.float64) / 2.0 / 1e3          # one-way us
                    res["pingpong"][str(q)] = {
                        "samples": 10000, "mean_us": float(one.mean()),
                        "p50_us": float(np.percentile(one, 50)), "p99_us": float(np.percentile(one, 99)),
                        "max_us": float(one.max()), "samples_us": [round(float(v), 4) for v in one]}
            dist.barrier()
        if rank == 0 and P > 1:
            for nb in (1 << 13, 1 << 16, 1 << 19, 1 << 22, 1 << 23):
                res["write_bw"][str(nb)] = c.p2p_write_bw(1, nb, reps=50)
        dist.barrier()
    sem.nccl_comm_destroy(comm)
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res))


def last_json(path):
    try:
        lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except FileNotFoundError:
        return None


def kernels_per_point(N, built="r02"):
    """W (flops) and Q (bytes) per local point of one PCG iteration as built.

    r02 (DESIGN.md 5.1/5.3): the operator kernel also forms p = dinv r + beta p_old
    from TMA-staged p_old, r, dinv and the per-CTA p.w partials (88 B/pt); the
    r update also does x += alpha p (57 B/pt: w, dinv, r, p, x, mult read; r, x
    written).  r01: separate p kernel, x updated in it."""
    n = N + 1
    fb = 1.0 - ((N - 1) / (N + 1)) ** 3
    if built == "r01":
        return {"Ax": (12 * n + 15, 64.0), "gs": (fb, 20.0 * fb),
                "cg_update": (8.0, 33.0), "cg_p": (5.0, 48.0)}
    return {
        "Ax+p": (12 * n + 15 + 5, 88.0),
        "gs": (fb, 20.0 * fb),
        "cg_update+x": (10.0, 57.0),
    }


def model(probe_path, mdir, out_path=None, built="r02"):
    import random
    pr = json.loads([l for l in open(probe_path) if l.startswith("{")][-1])
    single = [json.loads(l) for l in open(os.path.join(mdir, "measure_single.jsonl")) if l.startswith("{")]
    triad = [r for r in single if r["what"] == "triad"][0]["GBps"] * 1e9
    samples = []
    for v in pr["pingpong"].values():
        samples.extend(v["samples_us"])   # one-way latencies of every peer
    samples = [s * 1e-6 for s in samples]
    bw = pr["write_bw"]
    big = max(bw, key=lambda k: int(k))
    beta_star = 8.0 / (bw[big] * 1e9)   # s per 64-bit word (postal model)
    rnd = random.Random(0)

    def allreduce(P, levels_paper=True, trials=2000):
        if P == 1:
            return 0.0
        L = int(math.ceil(math.log2(P)))
        tot = 0.0
        for _ in range(trials):
            if levels_paper:   # Eq. 14: max over PEs of sum over log2 P levels
                tot += max(sum(rnd.choice(samples) for _ in range(L)) for _ in range(P))
            else:              # as built: one level, P direct publishes
                tot += max(rnd.choice(samples) for _ in range(P))
        return tot / trials

    def gs(P, n_s):
        if P == 1:
            return 0.0
        nn = 1 if P == 2 else 2
        lat = sum(max(rnd.choice(samples) + rnd.choice(samples) for _ in range(nn)) for _ in range(2000)) / 2000
        return 2 * beta_star * n_s + lat

    def predict(n_per_gpu, N, P, n_s, paper_levels):
        ta = 0.0
        for W, Q in kernels_per_point(N, built).values():
            ta += max(W * n_per_gpu / PI_FP64, Q * n_per_gpu / triad)
        tc = 2 * allreduce(P, paper_levels) + gs(P, n_s)
        return ta, tc

    lines = []
    w = lines.append
    w("# Performance model (paper Eqs. 12-15) instantiated for B200\n")
    w(f"beta (triad, same run) = {triad / 1e9:.0f} GB/s; pi (fp64, derived) = {PI_FP64 / 1e12:.1f} TFLOP/s; "
      f"beta* = {beta_star * 1e12:.2f} ps/word ({bw[big]:.0f} GB/s one-sided NVLink writes, "
      f"{int(big) >> 20} MiB messages); alpha* one-way (device ping-pong, 10,000 samples per peer): " +
      "; ".join(f"peer {q}: mean {v['mean_us']:.2f} us, p50 {v['p50_us']:.2f}, p99 {v['p99_us']:.2f}, max {v['max_us']:.2f}"
                for q, v in pr["pingpong"].items()) + "\n")
    w("Per-point costs of one PCG iteration as built (W flops, Q bytes): " +
      ", ".join(f"{k} ({W:.0f}, {Q:.1f})" for k, (W, Q) in kernels_per_point(7, built).items()) + f" at N=7 (iteration as built in {built}).\n")

    # weak scaling: C2 per GPU (bench.py)
    N = 7
    n1 = 8192 * 512
    n_s = 2 * (32 * 7) * (16 * 7)   # two z-faces of the slab (periodic x, y)
    w("## Weak scaling, C2 per GPU (bench.py step)\n")
    w("| P | T_a us | T_c us (Eq. 14 tree) | T_c us (as built) | model T us | measured T us | model / measured |")
    w("|---|---|---|---|---|---|---|")
    for P in (1, 2, 4, 8, 16, 64):
        ta, tc1 = predict(n1, N, P, n_s, True)
        _, tc2 = predict(n1, N, P, n_s, False)
        b = last_json(os.path.join(mdir, f"bench{P}.log")) if P <= 4 else None
        meas = b["ms_per_step"] * 1e3 if b else None
        w(f"| {P} | {ta * 1e6:.1f} | {tc1 * 1e6:.1f} | {tc2 * 1e6:.1f} | {(ta + tc2) * 1e6:.1f} | "
          f"{meas if meas is None else round(meas, 1)} | {'' if meas is None else round((ta + tc2) * 1e6 / meas, 3)} |")
    w("")
    # strong scaling C3 / C4
    for cfg, E, ex, ey in (("C3", 32 ** 3, 32, 32), ("C4", 64 ** 3, 64, 64)):
        ntot = E * 512
        n_s = 2 * (ex * 7) * (ey * 7)
        rows = {}
        for P in (1, 2, 4):
            for l in (open(os.path.join(mdir, f"measure_strong{P}.jsonl")) if os.path.exists(os.path.join(mdir, f"measure_strong{P}.jsonl")) else []):
                if l.startswith("{"):
                    d = json.loads(l)
                    if d["what"] == f"{cfg}_strong":
                        rows[P] = d
        w(f"## Strong scaling, {cfg} ({E} elements, N=7)\n")
        w("Calibrated: T_a scaled by the measured / modelled time at P = 1 (the kernels' "
          "achieved fraction of the triad), T_c as modelled.\n")
        w("| P | model T us (as built) | model efficiency | calibrated T us | calibrated efficiency | measured T us | measured efficiency |")
        w("|---|---|---|---|---|---|---|")
        t1 = None
        m1 = rows[1]["pcg_ms"] / rows[1]["pcg_iters"] * 1e-3 if 1 in rows else None
        kcal = None
        for P in (1, 2, 4, 8, 16, 32, 64):
            ta, tc = predict(ntot / P, N, P, n_s, False)
            t = ta + tc
            if P == 1:
                t1 = t
                kcal = (m1 / ta) if m1 else 1.0
            tcal = kcal * ta + tc
            tcal1 = kcal * predict(ntot, N, 1, n_s, False)[0]
            d = rows.get(P)
            meas = d["pcg_ms"] / d["pcg_iters"] * 1e3 if d else None
            w(f"| {P} | {t * 1e6:.1f} | {t1 / (P * t):.3f} | {tcal * 1e6:.1f} | {tcal1 / (P * tcal):.3f} | "
              f"{'' if meas is None else round(meas, 1)} | "
              f"{'' if (meas is None or m1 is None) else round(m1 * 1e6 / (P * meas), 3)} |")
        w("")
    text = "\n".join(lines) + "\n"
    if out_path:
        open(out_path, "w").write(text)
    print(text)


if __name__ == "__main__":
    if sys.argv[1] == "probe":
        probe()
    else:
        model(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None,
              os.environ.get("SEM_MODEL_BUILT", "r02"))
