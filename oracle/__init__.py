"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around oracle/liboracle.so (plain C, fp64, -ffp-contract=off;
see oracle.h / oracle.c for the paper citations).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs
may import this package.  It shares no code with paper_2107_01243_b200.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_lib = None

_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
            "-Wall", "-o", _SO, _SRC, "-lm"])
    return _SO


class OMesh(C.Structure):
    _fields_ = [("ex", C.c_int32), ("ey", C.c_int32), ("ez", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double),
                ("y1", C.c_double), ("z0", C.c_double), ("z1", C.c_double),
                ("periodic", C.c_int32 * 3), ("deform", C.c_int32),
                ("deform_amp", C.c_double)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.oracle_legendre.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
        L.oracle_gll.argtypes = [C.c_int, _D, _D]
        L.oracle_deriv.argtypes = [C.c_int, _D, _D]
        L.oracle_ax_raw.argtypes = [C.c_int64, C.c_int, _D, _D, _D, _D]
        L.oracle_diag_raw.argtypes = [C.c_int64, C.c_int, _D, _D, _D]
        L.oracle_setup.argtypes = [C.POINTER(OMesh), C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_free.argtypes = [C.c_void_p]
        L.oracle_free.restype = None
        L.oracle_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3
        L.oracle_get.argtypes = [C.c_void_p, C.c_int, _D]
        L.oracle_get_int.argtypes = [C.c_void_p, C.c_int, _I]
        L.oracle_ax.argtypes = [C.c_void_p, _D, _D]
        L.oracle_gs.argtypes = [C.c_void_p, _D]
        L.oracle_mask_apply.argtypes = [C.c_void_p, _D]
        L.oracle_apply.argtypes = [C.c_void_p, _D, _D]
        L.oracle_rhs.argtypes = [C.c_void_p, _D, _D]
        L.oracle_dot_c.argtypes = [C.c_void_p, _D, _D]
        L.oracle_dot_c.restype = C.c_double
        L.oracle_pcg.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int,
                                 C.POINTER(C.c_int), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.c_void_p]
        L.oracle_helm_apply.argtypes = [C.c_void_p, C.c_double, C.c_double, _D, _D]
        L.oracle_rhs_mass.argtypes = [C.c_void_p, _D, _D]
        L.oracle_helm_dinv.argtypes = [C.c_void_p, C.c_double, C.c_double, _D]
        L.oracle_helm_pcg.argtypes = [C.c_void_p, C.c_double, C.c_double, _D, _D, C.c_double,
                                      C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.c_void_p]
        L.oracle_arnoldi.argtypes = [C.c_void_p, _D, C.c_int, _D, _D]
        L.oracle_gmres.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int, C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.c_void_p]
        L.oracle_proj_create.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_proj_free.argtypes = [C.c_void_p]
        L.oracle_proj_free.restype = None
        L.oracle_proj_size.argtypes = [C.c_void_p]
        L.oracle_proj_project.argtypes = [C.c_void_p, _D, _D, _D]
        L.oracle_proj_update.argtypes = [C.c_void_p, _D]
        L.oracle_proj_solve.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int, C.c_int,
                                        C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.oracle_proj_gram.argtypes = [C.c_void_p, _D]
        L.oracle_cgcg.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int,
                                  C.POINTER(C.c_int), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.c_void_p]
        L.oracle_proj_set_schwarz.argtypes = [C.c_void_p, C.c_void_p]
        L.oracle_schwarz_create.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_schwarz_free.argtypes = [C.c_void_p]
        L.oracle_schwarz_free.restype = None
        L.oracle_schwarz_local_matrix.argtypes = [C.c_void_p, C.c_int64, _D]
        L.oracle_schwarz_apply.argtypes = [C.c_void_p, _D, _D, C.c_int]
        L.oracle_schwarz_pcg.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int,
                                         C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.c_void_p]
        L.oracle_schwarz_gmres.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int, C.c_int,
                                           C.POINTER(C.c_int), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.c_void_p]
        L.oracle_plan.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3 + [C.c_void_p] * 3
        L.oracle_shared.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                    C.c_void_p]
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- 1-D rules
def legendre(N: int, x: float):
    L, dL = C.c_double(), C.c_double()
    lib().oracle_legendre(N, x, C.byref(L), C.byref(dL))
    return L.value, dL.value


def gll(N: int):
    xi, w = np.zeros(N + 1), np.zeros(N + 1)
    assert lib().oracle_gll(N, xi, w) == 0
    return xi, w


def deriv(N: int, xi=None):
    if xi is None:
        xi, _ = gll(N)
    D = np.zeros((N + 1) * (N + 1))
    assert lib().oracle_deriv(N, _f64(xi), D) == 0
    return D.reshape(N + 1, N + 1)


def ax_raw(E: int, N: int, D, G, u):
    w = np.zeros(E * (N + 1) ** 3)
    assert lib().oracle_ax_raw(E, N, _f64(D).ravel(), _f64(G).ravel(), _f64(u).ravel(), w) == 0
    return w


def diag_raw(E: int, N: int, D, G):
    d = np.zeros(E * (N + 1) ** 3)
    assert lib().oracle_diag_raw(E, N, _f64(D).ravel(), _f64(G).ravel(), d) == 0
    return d


# ---------------------------------------------------------------- context
class OracleError(RuntimeError):
    pass


_FIELDS = {"xi": 0, "w": 1, "D": 2, "X": 3, "Y": 4, "Z": 5, "G": 6, "B": 7, "dinv": 8, "c": 9}
_INTS = {"gid": 0, "mult": 1, "mask": 2, "rank": 3}


class Oracle:
    """Mesh + GLL space + geometry + numbering + gs lists, all on the host."""

    def __init__(self, spec, N: int, nranks: int = 1):
        m = OMesh(spec.ex, spec.ey, spec.ez, spec.x0, spec.x1, spec.y0, spec.y1,
                  spec.z0, spec.z1, (C.c_int32 * 3)(*spec.periodic), spec.deform,
                  spec.deform_amp)
        h = C.c_void_p()
        st = lib().oracle_setup(C.byref(m), N, nranks, C.byref(h))
        if st != 0:
            raise OracleError(f"oracle_setup failed with status {st}")
        self._h = h
        self.spec, self.N, self.n, self.nranks = spec, N, N + 1, nranks
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        lib().oracle_sizes(h, C.byref(a), C.byref(b), C.byref(c))
        self.nslots, self.E, self.nglob = a.value, b.value, c.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.oracle_free(h)
            self._h = None

    def get(self, name: str) -> np.ndarray:
        n = self.n
        size = {"xi": n, "w": n, "D": n * n, "G": 6 * self.nslots}.get(name, self.nslots)
        out = np.zeros(size)
        assert lib().oracle_get(self._h, _FIELDS[name], out) == 0
        if name == "D":
            out = out.reshape(n, n)
        return out

    def get_int(self, name: str) -> np.ndarray:
        out = np.zeros(self.nslots, dtype=np.int64)
        assert lib().oracle_get_int(self._h, _INTS[name], out) == 0
        return out

    def ax(self, u):
        w = np.zeros(self.nslots)
        assert lib().oracle_ax(self._h, _f64(u), w) == 0
        return w

    def gs(self, u):
        v = np.array(u, dtype=np.float64, copy=True)
        assert lib().oracle_gs(self._h, v) == 0
        return v

    def mask_apply(self, u):
        v = np.array(u, dtype=np.float64, copy=True)
        lib().oracle_mask_apply(self._h, v)
        return v

    def apply(self, u):
        w = np.zeros(self.nslots)
        assert lib().oracle_apply(self._h, _f64(u), w) == 0
        return w

    def rhs(self, f):
        b = np.zeros(self.nslots)
        assert lib().oracle_rhs(self._h, _f64(f), b) == 0
        return b

    def dot_c(self, a, b) -> float:
        return lib().oracle_dot_c(self._h, _f64(a), _f64(b))

    def pcg(self, b, tol: float, maxit: int):
        x = np.zeros(self.nslots)
        it, rf, rt = C.c_int(), C.c_double(), C.c_double()
        hist = np.zeros(maxit + 1)
        st = lib().oracle_pcg(self._h, _f64(b), x, tol, maxit, C.byref(it), C.byref(rf),
                              C.byref(rt), hist.ctypes.data_as(C.c_void_p))
        if st < 0:
            raise OracleError(f"oracle_pcg failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "res_true": rt.value,
                "status": st, "hist": hist[: it.value + 1]}

    def cgcg(self, b, tol: float, maxit: int):
        """Single-reduction (Chronopoulos-Gear) Jacobi PCG (reading Q34)."""
        x = np.zeros(self.nslots)
        it, rf, rt = C.c_int(), C.c_double(), C.c_double()
        hist = np.zeros(maxit + 1)
        st = lib().oracle_cgcg(self._h, _f64(b), x, tol, maxit, C.byref(it), C.byref(rf),
                               C.byref(rt), hist.ctypes.data_as(C.c_void_p))
        if st < 0:
            raise OracleError(f"oracle_cgcg failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "res_true": rt.value,
                "status": st, "hist": hist[: it.value + 1]}

    # ---- NEXT-2: Helmholtz h1 A + h2 B
    def helm_apply(self, h1: float, h2: float, u):
        w = np.zeros(self.nslots)
        assert lib().oracle_helm_apply(self._h, h1, h2, _f64(u), w) == 0
        return w

    def rhs_mass(self, f):
        b = np.zeros(self.nslots)
        assert lib().oracle_rhs_mass(self._h, _f64(f), b) == 0
        return b

    def helm_dinv(self, h1: float, h2: float):
        d = np.zeros(self.nslots)
        assert lib().oracle_helm_dinv(self._h, h1, h2, d) == 0
        return d

    def helm_pcg(self, h1: float, h2: float, b, tol: float, maxit: int):
        x = np.zeros(self.nslots)
        it, rf, rt = C.c_int(), C.c_double(), C.c_double()
        hist = np.zeros(maxit + 1)
        st = lib().oracle_helm_pcg(self._h, h1, h2, _f64(b), x, tol, maxit, C.byref(it),
                                   C.byref(rf), C.byref(rt), hist.ctypes.data_as(C.c_void_p))
        if st < 0:
            raise OracleError(f"oracle_helm_pcg failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "res_true": rt.value,
                "status": st, "hist": hist[: it.value + 1]}

    # ---- NEXT-3: restarted GMRES and the solution projection
    def gmres(self, b, tol: float, maxit: int, restart: int = 30, x0=None):
        x = np.zeros(self.nslots) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
        it, rf, rt = C.c_int(), C.c_double(), C.c_double()
        hist = np.zeros(maxit + 1)
        st = lib().oracle_gmres(self._h, _f64(b), x, tol, maxit, restart, C.byref(it),
                                C.byref(rf), C.byref(rt), hist.ctypes.data_as(C.c_void_p))
        if st < 0:
            raise OracleError(f"oracle_gmres failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "res_true": rt.value,
                "status": st, "hist": hist[: it.value + 1]}

    def arnoldi(self, b, m: int):
        """Test access: m Arnoldi steps of the GMRES above from b; returns (V, H),
        V [(m+1), nslots], H [(m+1), m]."""
        V = np.zeros((m + 1, self.nslots))
        H = np.zeros((m + 1, m))
        st = lib().oracle_arnoldi(self._h, _f64(b), m, V, H)
        if st < 0:
            raise OracleError(f"oracle_arnoldi failed with status {st}")
        return V, H

    def proj(self, m: int = 20):
        return Proj(self, m)

    def schwarz(self, coarse_iters: int = 10):
        return Schwarz(self, coarse_iters)

    def plan(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        lib().oracle_plan(self._h, C.byref(a), C.byref(b), C.byref(c), None, None, None)
        pairs = np.zeros(2 * a.value, dtype=np.int64)
        off = np.zeros(b.value + 1, dtype=np.int64)
        slots = np.zeros(c.value, dtype=np.int64)
        assert lib().oracle_plan(self._h, C.byref(a), C.byref(b), C.byref(c),
                                 pairs.ctypes.data_as(C.c_void_p),
                                 off.ctypes.data_as(C.c_void_p),
                                 slots.ctypes.data_as(C.c_void_p)) == 0
        return pairs.reshape(-1, 2), off, slots

    def shared(self, r: int, q: int) -> np.ndarray:
        cnt = C.c_int64()
        assert lib().oracle_shared(self._h, r, q, C.byref(cnt), None) == 0
        g = np.zeros(cnt.value, dtype=np.int64)
        assert lib().oracle_shared(self._h, r, q, C.byref(cnt),
                                   g.ctypes.data_as(C.c_void_p)) == 0
        return g


class Proj:
    """Solution-projection space of the oracle (Fischer 1998)."""

    def __init__(self, o: "Oracle", m: int):
        self.o = o
        h = C.c_void_p()
        assert lib().oracle_proj_create(o._h, m, C.byref(h)) == 0
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().oracle_proj_free(self._h)
            self._h = None

    @property
    def size(self) -> int:
        return lib().oracle_proj_size(self._h)

    def project(self, b):
        xb, bd = np.zeros(self.o.nslots), np.zeros(self.o.nslots)
        assert lib().oracle_proj_project(self._h, _f64(b), xb, bd) == 0
        return xb, bd

    def update(self, x) -> bool:
        """True if x was appended, False if skipped (negligible new direction)."""
        return lib().oracle_proj_update(self._h, _f64(x)) == 0

    def set_schwarz(self, s: "Schwarz | None"):
        """NEXT-1 pipeline: projection + flexible GMRES + Schwarz (None: Jacobi)."""
        self._schw = s   # keep it alive
        assert lib().oracle_proj_set_schwarz(self._h, s._h if s is not None else None) == 0

    def solve(self, b, tol: float, maxit: int, restart: int = 30):
        x = np.zeros(self.o.nslots)
        it, rf = C.c_int(), C.c_double()
        st = lib().oracle_proj_solve(self._h, _f64(b), x, tol, maxit, restart, C.byref(it),
                                     C.byref(rf))
        if st < 0:
            raise OracleError(f"oracle_proj_solve failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "status": st}

    def gram(self):
        k = self.size
        G = np.zeros(k * k)
        assert lib().oracle_proj_gram(self._h, G) == 0
        return G.reshape(k, k)


class Schwarz:
    """Two-level additive overlapping Schwarz of the oracle (NEXT-1; P:L257-261;
    readings Q28-Q32 in DESIGN.md)."""

    def __init__(self, o: "Oracle", coarse_iters: int = 10):
        self.o = o
        h = C.c_void_p()
        st = lib().oracle_schwarz_create(o._h, coarse_iters, C.byref(h))
        if st != 0:
            raise OracleError(f"oracle_schwarz_create failed with status {st}")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.oracle_schwarz_free(self._h)
            self._h = None

    def local_matrix(self, e: int):
        n3 = self.o.n ** 3
        A = np.zeros(n3 * n3)
        assert lib().oracle_schwarz_local_matrix(self._h, e, A) == 0
        return A.reshape(n3, n3)

    def apply(self, r, which: int = 3):
        z = np.zeros(self.o.nslots)
        assert lib().oracle_schwarz_apply(self._h, _f64(r), z, which) == 0
        return z

    def pcg(self, b, tol: float, maxit: int):
        x = np.zeros(self.o.nslots)
        it, rf, rt = C.c_int(), C.c_double(), C.c_double()
        hist = np.zeros(maxit + 1)
        st = lib().oracle_schwarz_pcg(self._h, _f64(b), x, tol, maxit, C.byref(it), C.byref(rf),
                                      C.byref(rt), hist.ctypes.data_as(C.c_void_p))
        if st < 0:
            raise OracleError(f"oracle_schwarz_pcg failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "res_true": rt.value,
                "status": st, "hist": hist[: it.value + 1]}

    def gmres(self, b, tol: float, maxit: int, restart: int = 30):
        x = np.zeros(self.o.nslots)
        it, rf, rt = C.c_int(), C.c_double(), C.c_double()
        hist = np.zeros(maxit + 1)
        st = lib().oracle_schwarz_gmres(self._h, _f64(b), x, tol, maxit, restart, C.byref(it),
                                        C.byref(rf), C.byref(rt),
                                        hist.ctypes.data_as(C.c_void_p))
        if st < 0:
            raise OracleError(f"oracle_schwarz_gmres failed with status {st}")
        return {"x": x, "iters": it.value, "res_final": rf.value, "res_true": rt.value,
                "status": st, "hist": hist[: it.value + 1]}
