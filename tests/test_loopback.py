"""Multi-rank parity on ONE GPU through the loopback transport.

P rank contexts of one process share cuda:0, one host thread and one CUDA
stream each (ctypes releases the GIL inside every libsem call).  Each rank owns
its z-slab (lexicographic element range) and runs the NCCL
transport's code path -- Ax on the boundary elements, pack of the partials of
the entities shared with other ranks, the neighbour exchange, Ax on the
interior elements and the rank-local gather-scatter meanwhile, then the unpack
that adds the rank partials in ascending rank order (Alg. 1,
reading Q10) -- and the CG / GMRES / Schwarz allreduces summed in
ascending rank order, with device copies in place of NCCL.  The gathered
E-vectors are compared with the oracle run with the same number of ranks
(tools/mgpu_common.py): gs bit-exact, apply / rhs 1e-12, PCG +-1 iteration and
x within 1e-10, GMRES and both Schwarz coarse modes.  P = 3 partitions the
meshes raggedly and runs with the shuffle flag (reversed neighbour order,
random arrival delays): results must not depend on completion order.
"""
import os
import sys
import threading

import numpy as np
import pytest

from conftest import ROOT, cuda_available

sys.path.insert(0, os.path.join(ROOT, "tools"))


def _run_ranks(sem, world, P, spec, N, fun, u, gs_mode):
    import torch
    from mgpu_common import rank_run, rank_slice
    outs, errs = [None] * P, [None] * P

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                lo, hi = rank_slice(spec, N, r, P)
                with sem.sem_setup(spec, N, rank=r, nranks=P, nccl_comm=sem.loopback_comm(world, r),
                                   stream=st.cuda_stream) as c:
                    assert c.n_local == hi - lo
                    c.set_gs_mode(gs_mode)
                    outs[r] = rank_run(c, u[lo:hi], fun)
        except BaseException as e:  # noqa: BLE001 -- reported by the main thread
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "loopback ranks hung"
    for e in errs:
        if e is not None:
            raise e
    return outs


@pytest.mark.gpu
@pytest.mark.parametrize("P,flags", [(2, 0), (3, 1), (4, 0)], ids=["P2", "P3-shuffle", "P4"])
def test_loopback_multirank_parity(P, flags):
    import paper_2107_01243_b200 as sem
    from mgpu_common import CASES, OracleRefs, case_field, check
    fails = []
    world = sem.loopback_create(P, flags)
    try:
        for ci, (spec, N, fun) in enumerate(CASES):
            u = case_field(ci, spec, N)
            ref = OracleRefs(spec, N, fun, u, P)
            for gsm in (1, 2):   # flat and element-ordered gs schedules
                outs = _run_ranks(sem, world, P, spec, N, fun, u, gsm)
                tag = f"case{ci} P={P} loopback flags={flags} gs_mode={gsm}"
                f = check(outs, ref, tag)
                print(f"{tag}: {'FAIL' if f else 'ok'} pcg iters {outs[0]['r']['iters']} "
                      f"(oracle {ref.pcg['iters']})", flush=True)
                fails += f
    finally:
        sem.loopback_destroy(world)
    assert not fails, fails


@pytest.mark.gpu
def test_loopback_bench_configuration():
    """The bench's weak-scaled C2 workload at 2 ranks (8,192 elements of N = 7
    per rank, 8.4 M slots) through the loopback transport: the operator on a
    seeded random field within 1e-12 of the oracle run with 2 ranks (normwise),
    and 3 fixed PCG iterations (tol 0, b = A u) within 1e-10 of its iterate."""
    import threading

    import torch

    import oracle as O
    import paper_2107_01243_b200 as sem
    from mgpu_common import rank_slice
    from sem_inputs import CONFIGS, random_field, weak_scaled
    P = 2
    spec, N = weak_scaled(CONFIGS["C2"][0], P), CONFIGS["C2"][1]
    u = random_field(spec.E * (N + 1) ** 3, seed=2024)
    outs, errs = [None] * P, [None] * P
    world = sem.loopback_create(P, 0)

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                lo, hi = rank_slice(spec, N, r, P)
                with sem.sem_setup(spec, N, rank=r, nranks=P, nccl_comm=sem.loopback_comm(world, r),
                                   stream=st.cuda_stream) as c:
                    du = torch.from_numpy(u[lo:hi]).cuda()
                    w = c.zeros()
                    c.apply(du, w)
                    x = c.zeros()
                    res = c.pcg_solve(w, x, 0.0, 3)
                    st.synchronize()
                    outs[r] = (w.cpu().numpy(), x.cpu().numpy(), res["iters"])
        except BaseException as e:  # noqa: BLE001 -- reported by the main thread
            errs[r] = e

    try:
        th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assert not any(t.is_alive() for t in th), "loopback ranks hung"
    finally:
        sem.loopback_destroy(world)
    for e in errs:
        if e is not None:
            raise e
    o = O.Oracle(spec, N, nranks=P)
    wr = o.apply(u)
    W = np.concatenate([q[0] for q in outs])
    assert np.abs(W - wr).max() / np.abs(wr).max() <= 1e-12
    ref = o.pcg(wr, 0.0, 3)
    X = np.concatenate([q[1] for q in outs])
    assert all(q[2] == 3 for q in outs)
    assert np.abs(X - ref["x"]).max() <= 1e-10


@pytest.mark.gpu
def test_loopback_rank_mismatch_rejected():
    """A loopback handle whose world size differs from the mesh's nranks is
    rejected before any collective."""
    import paper_2107_01243_b200 as sem
    from sem_inputs import tgv_box
    world = sem.loopback_create(2, 0)
    try:
        with pytest.raises(sem.SemError) as e:
            sem.sem_setup(tgv_box(2, 2, 4), 3, rank=0, nranks=3,
                          nccl_comm=sem.loopback_comm(world, 0))
        assert e.value.status == sem.SEM_EINVAL
    finally:
        sem.loopback_destroy(world)


@pytest.mark.gpu
def test_loopback_missing_rank_fails_instead_of_hanging():
    """Failure detection: rank 1 of a 2-rank world never arrives; rank 0's
    collective setup returns SEM_ENCCL after the world's timeout (2 s here,
    flags >> 8) instead of hanging."""
    import time

    import paper_2107_01243_b200 as sem
    from sem_inputs import tgv_box
    world = sem.loopback_create(2, 2 << 8)
    try:
        t0 = time.time()
        with pytest.raises(sem.SemError) as e:
            sem.sem_setup(tgv_box(2, 2, 4), 3, rank=0, nranks=2,
                          nccl_comm=sem.loopback_comm(world, 0))
        assert e.value.status == sem.SEM_ENCCL
        assert 1.5 < time.time() - t0 < 60
    finally:
        sem.loopback_destroy(world)


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure path")
def test_loopback_needs_a_device():
    import paper_2107_01243_b200 as sem
    from paper_2107_01243_b200 import build
    build.build()
    with pytest.raises(sem.SemError) as e:
        sem.loopback_create(2)
    assert e.value.status == sem.SEM_ECUDA
