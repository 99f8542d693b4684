"""ctypes loader of the CPU oracle (oracle/liboracle.so).  TEST INFRASTRUCTURE:
imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "liboracle.so")

from paper_2605_08793_b200._lib import GradientInfoC, ResultC, SinkhornConfigC, SplrConfigC  # noqa: E402

_vp = C.c_void_p


def build() -> None:
    subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so", "selfcheck"], check=True, capture_output=True)


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


class Oracle:
    def __init__(self, lib):
        self.lib = lib
        lib.rgo_last_error.restype = C.c_char_p
        lib.rgo_topk_budget.restype = C.c_long
        lib.rgo_time_gradient.restype = C.c_double
        if hasattr(lib, "rgo_rng_uniform_nth"):
            lib.rgo_rng_uniform_nth.restype = C.c_double

    def _ck(self, st):
        if st != 0:
            raise RuntimeError(f"oracle status {st}: {self.lib.rgo_last_error().decode()}")

    # problems are dicts: n, m, M (F-ordered n x m), a, b, eta
    def gen_problem(self, kind, n, m, eta, d=2, seed=0):
        M = np.zeros((n, m), order="F")
        a = np.zeros(n)
        b = np.zeros(m)
        self._ck(self.lib.rgo_gen_problem(kind.encode(), C.c_long(n), C.c_long(m), C.c_long(d),
                                          C.c_ulonglong(seed), C.c_double(eta), _p(M), _p(a), _p(b)))
        return dict(n=n, m=m, M=M, a=a, b=b, eta=eta)

    def rand_dual(self, n, m, scale, seed):
        al, be = np.zeros(n), np.zeros(m)
        self._ck(self.lib.rgo_rand_dual(C.c_long(n), C.c_long(m), C.c_double(scale), C.c_ulonglong(seed), _p(al), _p(be)))
        return al, be

    def _pargs(self, p):
        M = np.asfortranarray(p["M"])
        return (C.c_long(p["n"]), C.c_long(p["m"]), _p(M), _p(p["a"]), _p(p["b"]), C.c_double(p["eta"])), M

    def gradient(self, p, alpha, beta, naive=False, tr=8, tc=32):
        args, keep = self._pargs(p)
        info = GradientInfoC()
        grad = np.zeros(p["n"] + p["m"] - 1)
        row, col = np.zeros(p["n"]), np.zeros(p["m"])
        self._ck(self.lib.rgo_gradient(1 if naive else 0, *args, _p(alpha), _p(beta), tr, tc, C.byref(info),
                                       _p(grad), _p(row), _p(col)))
        return dict(f=info.f, marginal_error=info.marginal_error, duality_gap=info.duality_gap,
                    grad_norm2=info.grad_norm2, total_mass=info.total_mass, grad=grad, row=row, col=col)

    def plan(self, p, alpha, beta):
        args, keep = self._pargs(p)
        T = np.zeros((p["n"], p["m"]), order="F")
        self._ck(self.lib.rgo_plan(*args, _p(alpha), _p(beta), _p(T)))
        return T

    def optimal_alpha(self, p, alpha, beta):
        args, keep = self._pargs(p)
        out = np.zeros(p["n"])
        self._ck(self.lib.rgo_optimal_alpha(*args, _p(alpha), _p(beta), _p(out)))
        return out

    def optimal_beta(self, p, alpha):
        args, keep = self._pargs(p)
        out = np.zeros(p["m"])
        self._ck(self.lib.rgo_optimal_beta(*args, _p(alpha), _p(out)))
        return out

    def sinkhorn_step(self, p, alpha, beta):
        args, keep = self._pargs(p)
        al, be = alpha.copy(), beta.copy()
        self._ck(self.lib.rgo_sinkhorn_step(*args, _p(al), _p(be)))
        return al, be

    def select_topk(self, T, k):
        T = np.asfortranarray(T, dtype=np.float64)
        n, m = T.shape
        cnt = C.c_long(0)
        self._ck(self.lib.rgo_select_topk(C.c_long(n), C.c_long(m), _p(T), C.c_long(k), None, C.c_long(0), C.byref(cnt)))
        coords = np.zeros((max(cnt.value, 1), 2), dtype=np.int32)
        self._ck(self.lib.rgo_select_topk(C.c_long(n), C.c_long(m), _p(T), C.c_long(k), _p(coords), cnt, C.byref(cnt)))
        return coords[: cnt.value]

    def topk_budget(self, n, m, density):
        return int(self.lib.rgo_topk_budget(C.c_long(n), C.c_long(m), C.c_double(density)))

    def assemble(self, p, alpha, beta, coords, tau):
        args, keep = self._pargs(p)
        coords = np.ascontiguousarray(coords, dtype=np.int32)
        h = _vp()
        self._ck(self.lib.rgo_assemble(*args, _p(alpha), _p(beta), _p(coords), C.c_long(coords.shape[0]),
                                       C.c_double(tau), C.byref(h)))
        return OracleSparse(self, h)

    def _result(self, res, steps):
        rows = [(res.trace[r].iter, res.trace[r].wall_ms, res.trace[r].f, res.trace[r].marginal_error,
                 res.trace[r].duality_gap) for r in range(res.n_trace)]
        out = dict(status=res.status, message=res.message.decode(), trace=rows)
        if steps:
            names = [f[0] for f in res.steps._type_._fields_]
            out["steps"] = [{k: getattr(res.steps[s], k) for k in names} for s in range(res.n_steps)]
        if res.alpha:
            out["alpha"] = np.ctypeslib.as_array(res.alpha, (res.n,)).copy()
            out["beta"] = np.ctypeslib.as_array(res.beta, (res.m,)).copy()
        self.lib.rgo_result_free(C.byref(res))
        return out

    def run_splr(self, p, alpha0, beta0, cfg: SplrConfigC, direction_solver=0):
        args, keep = self._pargs(p)
        res = ResultC()
        self._ck(self.lib.rgo_run_splr(*args, _p(alpha0), _p(beta0), C.byref(cfg), direction_solver, C.byref(res)))
        return self._result(res, True)

    def run_sinkhorn(self, p, alpha0, beta0, cfg: SinkhornConfigC):
        args, keep = self._pargs(p)
        res = ResultC()
        self._ck(self.lib.rgo_run_sinkhorn(*args, _p(alpha0), _p(beta0), C.byref(cfg), C.byref(res)))
        return self._result(res, False)

    def time_gradient(self, p, alpha, beta, reps):
        args, keep = self._pargs(p)
        return float(self.lib.rgo_time_gradient(*args, _p(alpha), _p(beta), reps))


class OracleSparse:
    def __init__(self, o, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.lib.rgo_sparse_free(self.h)
        except Exception:
            pass

    def info(self):
        dim, nnz, nc, pid = C.c_int(), C.c_long(), C.c_long(), C.c_ulonglong()
        self.o.lib.rgo_sparse_info(self.h, C.byref(dim), C.byref(nnz), C.byref(nc), C.byref(pid))
        return dim.value, nnz.value, nc.value, pid.value

    def export(self):
        dim, nnz, _, _ = self.info()
        colptr, rowidx, values = np.zeros(dim + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
        self.o.lib.rgo_sparse_export(self.h, _p(colptr), _p(rowidx), _p(values))
        return colptr, rowidx, values

    def update_values(self, alpha, beta, tau):
        self.o._ck(self.o.lib.rgo_update_values(self.h, _p(alpha), _p(beta), C.c_double(tau)))

    def matvec(self, v):
        y = np.zeros(self.info()[0])
        self.o._ck(self.o.lib.rgo_matvec(self.h, _p(v), _p(y)))
        return y

    def compute_direction(self, g, u=None, v=None, xi=0.0, zeta=0.0, solver=0, cg_rtol=1e-12, cg_max_iter=100000):
        d = np.zeros(self.info()[0])
        its = C.c_int(0)
        self.o._ck(self.o.lib.rgo_compute_direction(self.h, _p(g), _p(u), _p(v), C.c_double(xi), C.c_double(zeta),
                                                    solver, C.c_double(cg_rtol), cg_max_iter, _p(d), C.byref(its)))
        return d, its.value


_oracle = None


def load() -> Oracle:
    global _oracle
    if _oracle is None:
        if not os.path.exists(LIB):
            build()
        _oracle = Oracle(C.CDLL(LIB))
    return _oracle


REF_LIB = os.path.join(ORACLE_DIR, "_ref", "libregot_ref.so")
_ref = None


def load_ref():
    """The reference's OWN code (its headers compiled over oracle/eigen_shim into oracle/_ref), or
    None where it has not been built (it is built only where /root/reference is mounted)."""
    global _ref
    if _ref is None and os.path.exists(REF_LIB):
        _ref = Oracle(C.CDLL(REF_LIB))
    return _ref
