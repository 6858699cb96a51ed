"""Multi-process tests of the element partition (Alg. 1).

* CPU (gloo, world_size 2): each rank builds its host plan; the ranks exchange
  their per-neighbour shared global-number lists over gloo and check that the
  lists are symmetric (what rank r sends to q is what q expects from r) and
  equal to the oracle's; the union of the local numberings covers the mesh.
* GPU (NCCL, all visible GPUs >= 2): tools/mgpu_worker.py under torchrun --
  gs bit-exact, apply/rhs within 1e-12, PCG within 1e-10 of the oracle run
  with the same rank count.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import oracle as O
    import paper_2107_01243_b200 as sem
    from sem_inputs import tgv_box, unit_box
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    msgs = []
    for spec, N in [(tgv_box(2, 2, 4), 3), (unit_box(3, 2, 5), 2), (tgv_box(3, 2, 3), 4)]:
        p = sem.Plan(spec, N, rank=rank, nranks=world)
        ranks, counts = p.neighbors()
        mine = {int(r): p.shared(int(r)).tolist() for r in ranks}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        gid, mult, mask = p.slots()
        gids = [None] * world
        dist.all_gather_object(gids, gid.tolist())
        if rank == 0:
            o = O.Oracle(spec, N, nranks=world)
            for r in range(world):
                for qq in range(world):
                    if r == qq:
                        continue
                    a = allp[r].get(qq, [])
                    b = allp[qq].get(r, [])
                    if a != b:
                        ok = False
                        msgs.append(f"asymmetric lists {r}->{qq}")
                    if a != o.shared(r, qq).tolist():
                        ok = False
                        msgs.append(f"lists differ from oracle {r}->{qq}")
            allg = np.concatenate([np.array(g) for g in gids])
            if not np.array_equal(allg, o.get_int("gid")):
                ok = False
                msgs.append("numbering union differs")
    dist.destroy_process_group()
    q.put((rank, ok, msgs))


def test_gloo_two_rank_plan_exchange():
    import multiprocessing as mp
    from paper_2107_01243_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, msgs in res:
        assert ok, msgs


@pytest.mark.gpu
def test_multi_gpu_parity():
    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    for P in sorted({2, min(n, 4)}):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={P}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.join(ROOT, "tools", "mgpu_worker.py")]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        print(r.stdout[-4000:], r.stderr[-4000:])
        assert r.returncode == 0 and "RESULT PASS" in r.stdout
