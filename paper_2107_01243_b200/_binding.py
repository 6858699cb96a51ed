"""ctypes binding for libsem.so (include/sem.h).  Argument marshalling only.

Device buffers are torch.cuda float64 tensors (PyTorch is used for device
memory, streams and process groups); their data pointers cross the C ABI.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

SEM_OK, SEM_NOT_CONVERGED = 0, 1
SEM_EINVAL, SEM_EGEOM, SEM_ECUDA, SEM_ENCCL, SEM_ENOMEM, SEM_EBREAKDOWN = -1, -2, -3, -4, -5, -6

_HERE = os.path.dirname(os.path.abspath(__file__))
# SEM_LIB: a tuning build from build.py --variant (tools only); default in-tree libsem.so
_SO = os.environ.get("SEM_LIB") or os.path.join(_HERE, "libsem.so")
_lib = None


class SemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libsem status {status}: {msg}")
        self.status = status


class SemMesh(C.Structure):
    _fields_ = [("ex", C.c_int32), ("ey", C.c_int32), ("ez", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double),
                ("y1", C.c_double), ("z0", C.c_double), ("z1", C.c_double),
                ("periodic", C.c_int32 * 3), ("deform", C.c_int32), ("deform_amp", C.c_double),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_comm", C.c_void_p),
                ("stream", C.c_void_p)]


class PcgResult(C.Structure):
    _fields_ = [("iters", C.c_int32), ("res_final", C.c_double), ("res_true", C.c_double),
                ("status", C.c_int32)]


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)

_SIGS = {
    "sem_setup": [C.POINTER(SemMesh), C.c_int, C.POINTER(_P)],
    "sem_destroy": [_P],
    "sem_sizes": [_P, _I64P, _I64P, _I64P],
    "sem_ax": [_P, _P, _P],
    "sem_gs": [_P, _P],
    "sem_apply": [_P, _P, _P],
    "sem_rhs": [_P, _P, _P],
    "sem_coords": [_P, _P, _P, _P],
    "sem_pcg_solve": [_P, _P, _P, C.c_double, C.c_int32, C.POINTER(PcgResult)],
    "sem_pcg_solve_host": [_P, _P, _P, C.c_double, C.c_int32, C.POINTER(PcgResult)],
    "sem_helm_apply": [_P, C.c_double, C.c_double, _P, _P],
    "sem_gmres_solve": [_P, _P, _P, C.c_double, C.c_int32, C.c_int32, C.POINTER(PcgResult)],
    "sem_proj_solve": [_P, _P, _P, C.c_double, C.c_int32, C.c_int32, C.c_int32,
                       C.POINTER(PcgResult)],
    "sem_proj_reset": [_P],
    "sem_schwarz_apply": [_P, _P, _P, C.c_int32],
    "sem_proj_size": [_P, C.POINTER(C.c_int32)],
    "sem_rhs_mass": [_P, _P, _P],
    "sem_helm_pcg_solve": [_P, C.c_double, C.c_double, _P, _P, C.c_double, C.c_int32,
                           C.POINTER(PcgResult)],
    "sem_pcg_history": [_P, _P, C.c_int32, C.POINTER(C.c_int32)],
    "sem_export_field": [_P, C.c_int, _P],
    "sem_export_int": [_P, C.c_int, _P],
    "sem_export_plan": [_P, C.POINTER(_P)],
    "sem_plan_create": [C.POINTER(SemMesh), C.c_int, C.POINTER(_P)],
    "sem_plan_destroy": [_P],
    "sem_plan_sizes": [_P, _I64P, _I64P, _I64P, _I64P, C.POINTER(C.c_int32)],
    "sem_plan_slots": [_P, _P, _P, _P],
    "sem_plan_pairs": [_P, _P, _P, _P],
    "sem_plan_neighbors": [_P, _P, _P],
    "sem_plan_shared": [_P, C.c_int32, _P],
    "sem_plan_space": [_P, _P, _P, _P],
    "sem_nccl_unique_id": [_P],
    "sem_nccl_comm_init": [_P, C.c_int, C.c_int, C.POINTER(_P)],
    "sem_nccl_comm_destroy": [_P],
    "sem_loopback_create": [C.c_int, C.c_int, C.POINTER(_P)],
    "sem_loopback_comm": [_P, C.c_int, C.POINTER(_P)],
    "sem_loopback_destroy": [_P],
    "sem_timing": [_P, C.c_int],
    "sem_timing_read": [_P, C.c_int, C.POINTER(C.c_double), _I64P],
    "sem_launch_count": [_P, _I64P],
    "sem_set_option": [_P, C.c_int, C.c_int],
    "sem_debug_read": [_P, C.c_int, _P, C.c_int],
    "sem_p2p_pingpong": [_P, C.c_int, C.c_int, _P],
    "sem_p2p_write_bw": [_P, C.c_int, C.c_int64, C.c_int, _P],
}


def lib_path() -> str:
    return _SO


def load():
    """Load libsem.so (built by paper_2107_01243_b200/build.py); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise SemError(SEM_ECUDA, f"{_SO} is not built (run __graft_entry__.build()); "
                                      "there is no CPU fallback")
        L = C.CDLL(_SO)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.sem_last_error.argtypes = []
        L.sem_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(st, allow=(SEM_OK,)):
    if st not in allow:
        raise SemError(st, load().sem_last_error().decode(errors="replace"))
    return st


def _mesh(spec, rank=0, nranks=1, nccl_comm=None, stream=None) -> SemMesh:
    return SemMesh(spec.ex, spec.ey, spec.ez, spec.x0, spec.x1, spec.y0, spec.y1, spec.z0,
                   spec.z1, (C.c_int32 * 3)(*spec.periodic), int(spec.deform),
                   float(spec.deform_amp), rank, nranks, nccl_comm, stream)


def _dptr(t, n=None, dtype=None):
    """Device pointer of a contiguous CUDA tensor (checked)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise SemError(SEM_EINVAL, "expected a CUDA tensor")
    if not t.is_contiguous():
        raise SemError(SEM_EINVAL, "expected a contiguous tensor")
    if dtype is not None and t.dtype != dtype:
        raise SemError(SEM_EINVAL, f"expected dtype {dtype}, got {t.dtype}")
    if n is not None and t.numel() < n:
        raise SemError(SEM_EINVAL, f"tensor has {t.numel()} < {n} elements")
    return C.c_void_p(t.data_ptr())


# ------------------------------------------------------------------ context
class Context:
    """sem_ctx: one rank's mesh, space, geometry, gs plan and PCG workspace."""

    def __init__(self, spec, N, rank=0, nranks=1, nccl_comm=None, stream=None):
        import torch
        L = load()
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        self._stream_ptr = stream
        m = _mesh(spec, rank, nranks, nccl_comm, stream)
        h = C.c_void_p()
        _check(L.sem_setup(C.byref(m), N, C.byref(h)))
        self._h = h
        self.spec, self.N, self.n, self.rank, self.nranks = spec, N, N + 1, rank, nranks
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(L.sem_sizes(h, C.byref(a), C.byref(b), C.byref(c)))
        self.n_local, self.e_local, self.n_glob = a.value, b.value, c.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().sem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- tensors
    def empty(self):
        import torch
        return torch.empty(self.n_local, dtype=torch.float64, device="cuda")

    def zeros(self):
        import torch
        return torch.zeros(self.n_local, dtype=torch.float64, device="cuda")

    def _f64(self, t):
        import torch
        return _dptr(t, self.n_local, torch.float64)

    # -- hot path
    def ax(self, u, w):
        _check(load().sem_ax(self._h, self._f64(u), self._f64(w)))
        return w

    def gs(self, u):
        _check(load().sem_gs(self._h, self._f64(u)))
        return u

    def apply(self, u, w):
        _check(load().sem_apply(self._h, self._f64(u), self._f64(w)))
        return w

    def rhs(self, f, b):
        _check(load().sem_rhs(self._h, self._f64(f), self._f64(b)))
        return b

    def coords(self):
        X, Y, Z = self.empty(), self.empty(), self.empty()
        _check(load().sem_coords(self._h, self._f64(X), self._f64(Y), self._f64(Z)))
        return X, Y, Z

    def pcg_solve(self, b, x, tol, maxit):
        r = PcgResult()
        _check(load().sem_pcg_solve(self._h, self._f64(b), self._f64(x), float(tol), int(maxit),
                                    C.byref(r)), allow=(SEM_OK, SEM_NOT_CONVERGED))
        return {"iters": r.iters, "status": r.status, "res_final": r.res_final,
                "res_true": r.res_true}

    # ---- NEXT-2: Helmholtz h1 A + h2 B
    def helm_apply(self, h1, h2, u, w):
        _check(load().sem_helm_apply(self._h, float(h1), float(h2), self._f64(u), self._f64(w)))

    def rhs_mass(self, f, b):
        _check(load().sem_rhs_mass(self._h, self._f64(f), self._f64(b)))

    def helm_pcg_solve(self, h1, h2, b, x, tol, maxit):
        r = PcgResult()
        _check(load().sem_helm_pcg_solve(self._h, float(h1), float(h2), self._f64(b), self._f64(x),
                                         float(tol), int(maxit), C.byref(r)),
               allow=(SEM_OK, SEM_NOT_CONVERGED))
        return {"iters": r.iters, "status": r.status, "res_final": r.res_final,
                "res_true": r.res_true}

    # ---- NEXT-3: GMRES and the solution projection
    def gmres_solve(self, b, x, tol, maxit, restart=30):
        r = PcgResult()
        _check(load().sem_gmres_solve(self._h, self._f64(b), self._f64(x), float(tol), int(maxit),
                                      int(restart), C.byref(r)), allow=(SEM_OK, SEM_NOT_CONVERGED))
        return {"iters": r.iters, "status": r.status, "res_final": r.res_final,
                "res_true": r.res_true}

    def proj_solve(self, b, x, tol, maxit, restart=30, m=20):
        r = PcgResult()
        _check(load().sem_proj_solve(self._h, self._f64(b), self._f64(x), float(tol), int(maxit),
                                     int(restart), int(m), C.byref(r)),
               allow=(SEM_OK, SEM_NOT_CONVERGED))
        return {"iters": r.iters, "status": r.status, "res_final": r.res_final,
                "res_true": r.res_true}

    # ---- NEXT-1: two-level additive Schwarz
    def schwarz_apply(self, r, z, which=3):
        """z = M r (which: 1 local part, 2 coarse part, 3 both); builds M on first use."""
        _check(load().sem_schwarz_apply(self._h, self._f64(r), self._f64(z), int(which)))

    def set_precond(self, kind: str):
        """Preconditioner of pcg_solve / gmres_solve / proj_solve: 'jacobi' or
        'schwarz' (flexible PCG / flexible GMRES).  Collective (builds Schwarz)."""
        _check(load().sem_set_option(self._h, 6, {"jacobi": 0, "schwarz": 1}[kind]))

    def set_coarse_graph(self, on: bool):
        """Replay the one-rank Schwarz coarse solve as a CUDA graph (default on)."""
        _check(load().sem_set_option(self._h, 8, 1 if on else 0))

    def set_pcg_graph(self, on: bool):
        """One rank: replay 8-iteration PCG batches as a CUDA graph (default on)."""
        _check(load().sem_set_option(self._h, 14, 1 if on else 0))

    def set_pcg_fuse(self, on: bool):
        """p update fused into the next Ax kernel, x into the r update (default on)."""
        _check(load().sem_set_option(self._h, 15, 1 if on else 0))

    def set_pcg_gsu(self, mode):
        """One rank, fused PCG: gather-scatter performed on read by the r update
        instead of a separate gs kernel: True, False or -1 (default: auto, on
        when a vector exceeds 64 MiB and a z-layer of elements holds <= 8 MiB of it)."""
        _check(load().sem_set_option(self._h, 16, -1 if mode == -1 else (1 if mode else 0)))

    def set_ax_pdl(self, on: bool):
        """PDL launch of the PCG Ax kernel with G prefetched before the grid wait."""
        _check(load().sem_set_option(self._h, 13, 1 if on else 0))

    def set_pcg_variant(self, kind: str):
        """Jacobi-PCG recurrences: 'standard' or 'single_reduction' (Chronopoulos-Gear)."""
        _check(load().sem_set_option(self._h, 12, {"standard": 0, "single_reduction": 1}[kind]))

    def set_fdm_tc(self, on: bool):
        """N = 7 Schwarz local solves on the fp64 tensor cores (default) or CUDA cores."""
        _check(load().sem_set_option(self._h, 9, 1 if on else 0))

    def set_coarse_replicate(self, mode: int):
        """Schwarz coarse level at nranks > 1: -1 auto, 0 distributed, 1 replicated. Collective."""
        _check(load().sem_set_option(self._h, 11, int(mode)))

    def set_coarse_asm(self, mode):
        """Single-rank Schwarz coarse level: CG on the assembled N = 1 operator
        (True / -1 auto, the default; small problems on one thread-block cluster),
        2 = assembled with the multi-kernel solve, or on the element operator + gs (False)."""
        v = mode if mode in (-1, 2) else (1 if mode else 0)
        _check(load().sem_set_option(self._h, 17, v))

    def set_schwarz_graph(self, on: bool):
        """One rank: replay 8-iteration Schwarz flexible-PCG batches as a CUDA graph (default on)."""
        _check(load().sem_set_option(self._h, 18, 1 if on else 0))

    def set_gmres_graph(self, on: bool):
        """One rank: replay GMRES restart cycles as CUDA graphs (default on)."""
        _check(load().sem_set_option(self._h, 19, 1 if on else 0))

    def set_coarse_iters(self, k: int):
        """Maximum CG iterations of the Schwarz coarse solve (default 10)."""
        _check(load().sem_set_option(self._h, 7, int(k)))

    def proj_reset(self):
        _check(load().sem_proj_reset(self._h))

    def proj_size(self) -> int:
        k = C.c_int32()
        _check(load().sem_proj_size(self._h, C.byref(k)))
        return k.value

    def pcg_solve_host(self, b_host: np.ndarray, x_host: np.ndarray, tol, maxit):
        """End-to-end entry point: HOST b in, HOST x out (copies inside libsem)."""
        assert b_host.dtype == np.float64 and x_host.dtype == np.float64
        assert b_host.size >= self.n_local and x_host.size >= self.n_local
        assert b_host.flags.c_contiguous and x_host.flags.c_contiguous
        r = PcgResult()
        _check(load().sem_pcg_solve_host(self._h, C.c_void_p(b_host.ctypes.data),
                                         C.c_void_p(x_host.ctypes.data), float(tol), int(maxit),
                                         C.byref(r)), allow=(SEM_OK, SEM_NOT_CONVERGED))
        return {"iters": r.iters, "status": r.status, "res_final": r.res_final,
                "res_true": r.res_true}

    def pcg_history(self, max_entries=100000):
        buf = np.zeros(max_entries)
        n = C.c_int32()
        _check(load().sem_pcg_history(self._h, C.c_void_p(buf.ctypes.data), max_entries,
                                      C.byref(n)))
        return buf[: n.value]

    # -- exports (host numpy)
    def export_field(self, name):
        which = {"xi": 0, "w": 1, "D": 2, "G": 3, "B": 4, "dinv": 5}[name]
        size = {"xi": self.n, "w": self.n, "D": self.n * self.n, "G": 6 * self.n_local}.get(
            name, self.n_local)
        out = np.zeros(size)
        _check(load().sem_export_field(self._h, which, C.c_void_p(out.ctypes.data)))
        return out.reshape(self.n, self.n) if name == "D" else out

    def export_plan(self):
        """The gather-scatter plan the kernels use, read back from the device (a Plan)."""
        h = C.c_void_p()
        _check(load().sem_export_plan(self._h, C.byref(h)))
        return Plan._from_handle(h, self.N)

    def export_int(self, name):
        which = {"mult": 0, "mask": 1}[name]
        out = np.zeros(self.n_local, dtype=np.int64)
        _check(load().sem_export_int(self._h, which, C.c_void_p(out.ctypes.data)))
        return out

    # -- instrumentation
    def timing(self, enable: bool):
        _check(load().sem_timing(self._h, 1 if enable else 0))

    def timing_read(self, which: int):
        ms, cnt = C.c_double(), C.c_int64()
        _check(load().sem_timing_read(self._h, which, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def _set_option(self, option: int, value: int):
        _check(load().sem_set_option(self._h, int(option), int(value)))

    def set_overlap(self, on: bool):
        """Alg. 1 boundary/interior split of the operator at nranks > 1. Collective."""
        _check(load().sem_set_option(self._h, 3, 1 if on else 0))

    def set_gs_mode(self, mode: int):
        """Gather-scatter schedule: 0 auto, 1 flat, 2 element-ordered chunks."""
        _check(load().sem_set_option(self._h, 4, int(mode)))

    def set_p2p(self, on: bool):
        """Multi-GPU transport: NVLink peer memory (default) or NCCL. Collective."""
        _check(load().sem_set_option(self._h, 2, 1 if on else 0))

    def debug_read(self, which=0, n=16):
        out = np.zeros(n, dtype=np.int64)
        _check(load().sem_debug_read(self._h, which, C.c_void_p(out.ctypes.data), n))
        return out

    def p2p_pingpong(self, peer: int, iters: int) -> np.ndarray:
        """Collective with `peer`: round-trip ns samples (returned on the lower rank)."""
        out = np.zeros(iters, dtype=np.int64)
        _check(load().sem_p2p_pingpong(self._h, peer, iters, C.c_void_p(out.ctypes.data)))
        return out

    def p2p_write_bw(self, peer: int, nbytes: int, reps: int = 20) -> float:
        g = C.c_double()
        _check(load().sem_p2p_write_bw(self._h, peer, int(nbytes), reps, C.byref(g)))
        return g.value

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(load().sem_launch_count(self._h, C.byref(n)))
        return n.value


def sem_setup(spec, N, rank=0, nranks=1, nccl_comm=None, stream=None) -> Context:
    return Context(spec, N, rank, nranks, nccl_comm, stream)


# ------------------------------------------------------------------ host planner
class Plan:
    """sem_plan: the host-only planner (no device)."""

    def __init__(self, spec, N, rank=0, nranks=1):
        L = load()
        m = _mesh(spec, rank, nranks)
        h = C.c_void_p()
        _check(L.sem_plan_create(C.byref(m), N, C.byref(h)))
        self._init(h, N)

    @classmethod
    def _from_handle(cls, h, N):
        self = cls.__new__(cls)
        self._init(h, N)
        return self

    def _init(self, h, N):
        L = load()
        self._h = h
        self.N = N
        a, b, c, d, e = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _check(L.sem_plan_sizes(h, C.byref(a), C.byref(b), C.byref(c), C.byref(d), C.byref(e)))
        self.n_local, self.npairs, self.nseg, self.nsegslots, self.n_nbr = (
            a.value, b.value, c.value, d.value, e.value)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.sem_plan_destroy(self._h)
            self._h = None

    def slots(self):
        gid = np.zeros(self.n_local, dtype=np.int64)
        mult = np.zeros(self.n_local, dtype=np.int64)
        mask = np.zeros(self.n_local, dtype=np.int64)
        _check(load().sem_plan_slots(self._h, C.c_void_p(gid.ctypes.data),
                                     C.c_void_p(mult.ctypes.data), C.c_void_p(mask.ctypes.data)))
        return gid, mult, mask

    def pairs(self):
        pairs = np.zeros(2 * self.npairs, dtype=np.int64)
        off = np.zeros(self.nseg + 1, dtype=np.int64)
        slots = np.zeros(self.nsegslots, dtype=np.int64)
        _check(load().sem_plan_pairs(self._h, C.c_void_p(pairs.ctypes.data),
                                     C.c_void_p(off.ctypes.data), C.c_void_p(slots.ctypes.data)))
        return pairs.reshape(-1, 2), off, slots

    def space(self):
        n = self.N + 1
        xi, w, D = np.zeros(n), np.zeros(n), np.zeros(n * n)
        _check(load().sem_plan_space(self._h, C.c_void_p(xi.ctypes.data), C.c_void_p(w.ctypes.data),
                                     C.c_void_p(D.ctypes.data)))
        return xi, w, D.reshape(n, n)

    def neighbors(self):
        ranks = np.zeros(self.n_nbr, dtype=np.int32)
        counts = np.zeros(self.n_nbr, dtype=np.int64)
        if self.n_nbr:
            _check(load().sem_plan_neighbors(self._h, C.c_void_p(ranks.ctypes.data),
                                             C.c_void_p(counts.ctypes.data)))
        return ranks, counts

    def shared(self, q):
        ranks, counts = self.neighbors()
        idx = np.flatnonzero(ranks == q)
        if len(idx) == 0:
            return np.zeros(0, dtype=np.int64)
        out = np.zeros(counts[idx[0]], dtype=np.int64)
        _check(load().sem_plan_shared(self._h, q, C.c_void_p(out.ctypes.data)))
        return out


def sem_plan_create(spec, N, rank=0, nranks=1) -> Plan:
    return Plan(spec, N, rank, nranks)


# ------------------------------------------------------------------ NCCL
def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load().sem_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def nccl_comm_init(uid: bytes, rank: int, nranks: int):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    _check(load().sem_nccl_comm_init(C.cast(buf, C.c_void_p), rank, nranks, C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm):
    _check(load().sem_nccl_comm_destroy(C.c_void_p(comm)))


# ------------------------------------------------------------------ loopback (tests)
def loopback_create(nranks: int, flags: int = 0):
    """A loopback world: nranks rank contexts on ONE device, one host thread each
    (ctypes releases the GIL inside every libsem call).  flags & 1 shuffles the
    neighbour order and the ranks' arrival times."""
    w = C.c_void_p()
    _check(load().sem_loopback_create(int(nranks), int(flags), C.byref(w)))
    return w.value


def loopback_comm(world, rank: int):
    """Rank `rank`'s handle, passed as nccl_comm to sem_setup."""
    c = C.c_void_p()
    _check(load().sem_loopback_comm(C.c_void_p(world), int(rank), C.byref(c)))
    return c.value


def loopback_destroy(world):
    _check(load().sem_loopback_destroy(C.c_void_p(world)))
