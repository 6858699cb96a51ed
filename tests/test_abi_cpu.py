"""CPU checks of the C-ABI library: it loads, exports every symbol that
include/sem.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import pytest

from conftest import ROOT, cuda_available

HEADER = os.path.join(ROOT, "include", "sem.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sem_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def libsem():
    from paper_2107_01243_b200 import build
    so = build.build()
    return ctypes.CDLL(so)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("sem_setup", "sem_ax", "sem_gs", "sem_apply", "sem_pcg_solve", "sem_destroy",
              "sem_pcg_solve_host", "sem_rhs", "sem_last_error", "sem_plan_create"):
        assert s in syms


def test_library_exports_every_declared_symbol(libsem):
    missing = [s for s in declared_symbols() if not hasattr(libsem, s)]
    assert not missing, missing


def test_library_is_sm100a_cuda(libsem):
    import subprocess
    from paper_2107_01243_b200 import lib_path
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure path")
def test_setup_fails_loudly_without_gpu(libsem):
    import paper_2107_01243_b200 as sem
    from sem_inputs import CONFIGS
    spec, N = CONFIGS["C1"]
    m = sem._binding._mesh(spec)
    h = ctypes.c_void_p()
    st = sem.load().sem_setup(ctypes.byref(m), N, ctypes.byref(h))
    assert st == sem.SEM_ECUDA
    assert b"no CUDA device" in sem.load().sem_last_error()


def test_invalid_arguments_rejected(libsem):
    import paper_2107_01243_b200 as sem
    from sem_inputs import unit_box
    with pytest.raises(sem.SemError) as e:
        sem.Plan(unit_box(1, 2, 2, periodic=(1, 0, 0)), 3)     # periodic axis with 1 element
    assert e.value.status == sem.SEM_EINVAL
    with pytest.raises(sem.SemError):
        sem.Plan(unit_box(2, 2, 2), 12)                       # N > 11
    with pytest.raises(sem.SemError):
        sem.Plan(unit_box(2, 1, 1), 3, rank=0, nranks=3)      # P > E
