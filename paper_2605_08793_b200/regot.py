"""Host-side mirror of the reference's solver interface over the C ABI.

Same names, argument meaning and error behaviour as the reference's
`namespace regot` (proj/include/regot/*.h): ProblemInstance, DualPoint,
GradientResult, SplrConfig, SinkhornConfig, SolverTrace, run_splr,
run_sinkhorn, fused_gradient, sinkhorn_step, select_topk, assemble,
update_values, compute_direction.  Every call goes through
libregot_b200.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import GradientInfoC, ResultC, SinkhornConfigC, SplrConfigC, StepRecordC

LAYOUT_COLMAJOR = 0
LAYOUT_ROWMAJOR = 1


# ---- errors: one class per reference exception (core.h:21-37) ----------------
class RegotError(RuntimeError):
    status = -1


class DegenerateCostError(RegotError):
    status = 1


class FormatError(RegotError):
    status = 2


class TruncationError(RegotError):
    status = 3


class ValidationError(RegotError):
    status = 4


class IoError(RegotError):
    status = 5


class OracleSizeError(RegotError):
    status = 6


class StructureError(RegotError):
    status = 7


class NotPositiveDefiniteError(RegotError):
    status = 8


class DirectionError(RegotError):
    status = 9


class LineSearchError(RegotError):
    status = 10


class PlotError(RegotError):
    status = 11


class StepError(RegotError):
    """splr.h:315-324: carries the trace collected before the failing step."""

    status = 12

    def __init__(self, msg: str, trace: "SolverTrace"):
        super().__init__(msg)
        self.trace = trace


class CudaError(RegotError):
    status = 100


class NcclError(RegotError):
    status = 101


class DeviceMemoryError(RegotError):
    status = 102


class UnsupportedError(RegotError):
    status = 103


_ERRORS = {
    cls.status: cls
    for cls in (
        DegenerateCostError, FormatError, TruncationError, ValidationError, IoError, OracleSizeError,
        StructureError, NotPositiveDefiniteError, DirectionError, LineSearchError, PlotError,
        CudaError, NcclError, DeviceMemoryError, UnsupportedError,
    )
}


def _raise(status: int, msg: str):
    raise _ERRORS.get(status, RegotError)(msg)


# ---- value types -------------------------------------------------------------------
def _vec(x, n: Optional[int] = None, what: str = "vector") -> np.ndarray:
    v = np.ascontiguousarray(x, dtype=np.float64)
    if v.ndim != 1 or (n is not None and v.shape[0] != n):
        raise ValidationError(f"{what}: length mismatch")
    return v


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class ProblemInstance:
    """problem.h:20-28.  M is n x m; C- or F-contiguous arrays are uploaded as is."""

    n: int
    m: int
    M: np.ndarray
    a: np.ndarray
    b: np.ndarray
    eta: float


@dataclass
class DualPoint:
    """dual.h:14-47: (alpha, beta) with the gauge beta[m-1] == 0."""

    alpha: np.ndarray
    beta: np.ndarray

    @staticmethod
    def zeros(n: int, m: int) -> "DualPoint":
        return DualPoint(np.zeros(n), np.zeros(m))

    @staticmethod
    def from_free(xf, n: int, m: int) -> "DualPoint":
        xf = np.asarray(xf, dtype=np.float64)
        if xf.shape != (n + m - 1,):
            raise ValidationError("DualPoint::from_free: length mismatch")
        beta = np.zeros(m)
        beta[: m - 1] = xf[n:]
        return DualPoint(xf[:n].copy(), beta)

    def to_free(self) -> np.ndarray:
        return np.concatenate([self.alpha, self.beta[:-1]])


@dataclass
class GradientResult:
    """dual.h:50-56 (+ the scalars the device epilogue produces in the same pass)."""

    f: float
    grad: np.ndarray
    row_sums: np.ndarray
    col_sums: np.ndarray
    marginal_error: float = 0.0
    duality_gap: float = 0.0
    grad_norm2: float = 0.0
    total_mass: float = 0.0


@dataclass
class FusedTiling:
    rows: int = 8
    cols: int = 32


@dataclass
class SplrConfig:
    """splr.h:22-60."""

    tau_max: float = 1.0
    S: int = 10
    J: int = 5
    density: float = 0.01
    c1: float = 1e-4
    c2: float = 0.9
    max_iter: int = 1000
    tol: float = 1e-8
    max_ls_trials: int = 30
    record_every: int = 1
    overlap: bool = False
    tiling: FusedTiling = field(default_factory=FusedTiling)
    cg_max_iter: int = 0  # extension: 0 -> library default
    cg_rtol: float = 0.0  # extension: 0 -> library default

    def _c(self) -> SplrConfigC:
        return SplrConfigC(
            self.tau_max, self.S, self.J, self.density, self.c1, self.c2, self.max_iter, self.tol,
            self.max_ls_trials, self.record_every, int(self.overlap), self.tiling.rows, self.tiling.cols,
            self.cg_max_iter, self.cg_rtol,
        )

    def validate(self) -> None:
        c = self._c()
        st = _lib.load().regot_b200_splr_config_validate(C.byref(c))
        if st != 0:
            _raise(st, _lib.load().regot_b200_last_error(None).decode())


@dataclass
class SinkhornConfig:
    """sinkhorn.h:16-31."""

    max_iter: int = 1000
    record_every: int = 1
    tol: float = 0.0

    def _c(self) -> SinkhornConfigC:
        return SinkhornConfigC(self.max_iter, self.record_every, self.tol)

    def validate(self) -> None:
        c = self._c()
        st = _lib.load().regot_b200_sinkhorn_config_validate(C.byref(c))
        if st != 0:
            _raise(st, _lib.load().regot_b200_last_error(None).decode())


def splr_config_hash(cfg: SplrConfig) -> str:
    """splr.h:62-70."""
    buf = C.create_string_buffer(17)
    c = cfg._c()
    _lib.load().regot_b200_splr_config_hash(C.byref(c), buf)
    return buf.value.decode()


def sinkhorn_config_hash(cfg: SinkhornConfig) -> str:
    """sinkhorn.h:33-39."""
    buf = C.create_string_buffer(17)
    c = cfg._c()
    _lib.load().regot_b200_sinkhorn_config_hash(C.byref(c), buf)
    return buf.value.decode()


@dataclass
class TraceRow:
    """trace.h:11-18."""

    iter: int = 0
    wall_ms: float = 0.0
    f: float = 0.0
    marginal_error: float = 0.0
    duality_gap: float = 0.0


@dataclass
class SolverTrace:
    """trace.h:22-41."""

    algo: str = ""
    problem: str = ""
    eta: float = 0.0
    config_hash: str = ""
    rows: List[TraceRow] = field(default_factory=list)

    def append(self, r: TraceRow) -> None:
        if self.rows:
            if r.iter <= self.rows[-1].iter:
                raise ValidationError("SolverTrace: iter must be strictly increasing")
            if r.wall_ms < self.rows[-1].wall_ms:
                raise ValidationError("SolverTrace: wall_ms must be nondecreasing")
        self.rows.append(r)


@dataclass
class SplrStepRecord:
    """splr.h:294-312 (+ cg_iters)."""

    iter: int = 0
    refresh: bool = False
    sinkhorn_selected: bool = False
    f_before: float = 0.0
    f_after: float = 0.0
    f_cand_sinkhorn: float = math.nan
    f_cand_qn: float = 0.0
    gamma: float = 0.0
    g_dot_d: float = 0.0
    gnew_dot_d: float = 0.0
    curvature_ok: bool = False
    ls_failed: bool = False
    lowrank_active: bool = False
    tau: float = 0.0
    factor_retries: int = 0
    ls_evals: int = 0
    cg_iters: int = 0


@dataclass
class SolveStats:
    """Measurement extras of regot_result (no reference counterpart)."""

    device_ms: float = 0.0
    gradient_passes: int = 0
    lse_passes: int = 0
    kernel_launches: int = 0


@dataclass
class SplrResult:
    """splr.h:480-485."""

    x: DualPoint
    trace: SolverTrace
    steps: List[SplrStepRecord]
    stats: SolveStats = field(default_factory=SolveStats)


@dataclass
class SinkhornResult:
    """sinkhorn.h:117-121."""

    x: DualPoint
    trace: SolverTrace
    stats: SolveStats = field(default_factory=SolveStats)


@dataclass
class SparsityPattern:
    """sparsity.h:19-40."""

    n: int
    mm1: int
    coords: np.ndarray  # (k, 2) int32, sorted lexicographically
    k_requested: int = 0

    def contains_minimum_set(self) -> bool:
        c = self.coords
        row0 = np.zeros(self.mm1, bool)
        col0 = np.zeros(self.n, bool)
        row0[c[c[:, 0] == 0, 1]] = True
        col0[c[c[:, 1] == 0, 0]] = True
        return bool(row0.all() and col0.all())


def _fingerprint(p: ProblemInstance) -> bytes:
    """Cheap content hash of a ProblemInstance: both marginals and a strided sample of M (<= 64k entries), so
    in-place edits of a resident instance are seen by Solver.ensure_problem."""
    import hashlib

    h = hashlib.blake2b(digest_size=16)
    M = np.asarray(p.M)
    h.update(repr((M.shape, M.strides, str(M.dtype))).encode())
    h.update(np.ascontiguousarray(p.a, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(p.b, dtype=np.float64).tobytes())
    flat = M.reshape(-1, order="A") if (M.flags.c_contiguous or M.flags.f_contiguous) else M.ravel()
    step = max(1, flat.shape[0] // 65536)
    h.update(np.ascontiguousarray(flat[::step]).tobytes())
    if flat.shape[0]:
        h.update(np.ascontiguousarray(flat[-1:]).tobytes())
    return h.digest()


def topk_budget(p: ProblemInstance, density: float) -> int:
    """splr.h:336-340."""
    return int(_lib.load().regot_b200_topk_budget(p.n, p.m, density))


# ---- device handle -----------------------------------------------------------------------
class Solver:
    """Owns one regot_ctx (one CUDA device, one resident problem)."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        h = C.c_void_p()
        st = self._lib.regot_b200_create(device, C.byref(h))
        if st != 0:
            _raise(st, self._lib.regot_b200_last_error(None).decode())
        self._h = h
        self.device = device
        self._problem_key = None
        self.n = self.m = 0
        self.row_begin = 0
        self.row_count = 0
        self.rank, self.world = 0, 1
        self._sparse = weakref.WeakSet()  # live SparseSym handles: released before the context goes

    def close(self) -> None:
        if getattr(self, "_h", None):
            for A in list(getattr(self, "_sparse", ())):
                A.free()
            for sv in (getattr(self, "_bench_pool", None) or {}).get("all", []):
                sv.close()
            self._lib.regot_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int) -> None:
        if st != 0:
            _raise(st, self._lib.regot_b200_last_error(self._h).decode())

    @property
    def launch_count(self) -> int:
        return int(self._lib.regot_b200_launch_count(self._h))

    def set_pattern_reuse(self, drift_tol: float, max_skips: int = 4) -> None:
        """north_star item (2): at k % S == 0 rebuild the top-k pattern only when the share of the Hessian block's mass
        it holds fell below (1 - drift_tol) x its share at the last rebuild (or after max_skips kept refreshes in a row).
        drift_tol = 0 restores the reference's fixed-S rule (splr.h:352, 359-364)."""
        self._check(self._lib.regot_b200_set_pattern_reuse(self._h, float(drift_tol), int(max_skips)))

    def pattern_counts(self):
        """(rebuilds, reuses) of the top-k pattern since this context was created."""
        a, b = C.c_int64(0), C.c_int64(0)
        self._lib.regot_b200_pattern_counts(self._h, C.byref(a), C.byref(b))
        return int(a.value), int(b.value)

    # -- multi-GPU ---------------------------------------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(256)
        st = _lib.load().regot_b200_comm_unique_id(buf)
        if st != 0:
            _raise(st, _lib.load().regot_b200_last_error(None).decode())
        return buf.raw

    def comm_init(self, rank: int, world: int, unique_ids: Optional[bytes]) -> None:
        buf = C.create_string_buffer(unique_ids, 256) if unique_ids is not None else None
        self._check(self._lib.regot_b200_comm_init(self._h, rank, world, buf))
        self.rank, self.world = rank, world

    # -- problem ------------------------------------------------------------------
    def set_problem(self, p: ProblemInstance, rows: Optional[Tuple[int, int]] = None) -> None:
        """Upload a ProblemInstance; `rows=(begin, count)` uploads one row block of it."""
        M = np.asarray(p.M, dtype=np.float64)
        if M.ndim != 2 or M.shape != (p.n, p.m):
            raise ValidationError("problem: cost matrix shape mismatch")
        a = _vec(p.a, p.n, "problem: marginal")
        b = _vec(p.b, p.m, "problem: marginal")
        if M.flags.f_contiguous and not M.flags.c_contiguous:
            layout, ld = LAYOUT_COLMAJOR, p.n
        else:
            M = np.ascontiguousarray(M)
            layout, ld = LAYOUT_ROWMAJOR, p.m
        begin, count = rows if rows is not None else (0, p.n)
        if rows is None and self.world == 1:
            st = self._lib.regot_b200_set_problem(self._h, p.n, p.m, _ptr(M), layout, ld, _ptr(a), _ptr(b), p.eta)
        else:
            base = M if layout == LAYOUT_COLMAJOR else M[begin:]
            st = self._lib.regot_b200_set_problem_rows(
                self._h, p.n, p.m, begin, count, _ptr(base), layout, ld, _ptr(a), _ptr(b), p.eta
            )
        self._check(st)
        self.n, self.m, self.row_begin, self.row_count = p.n, p.m, begin, count
        # the uploaded instance is held (a freed object's id() can be reused) together with a content fingerprint
        self._problem_key = (p, p.n, p.m, p.eta, begin, count, _fingerprint(p))

    def set_pointcloud(self, X: np.ndarray, Y: np.ndarray, a, b, eta: float, on_the_fly: bool = False,
                       rows: Optional[Tuple[int, int]] = None) -> None:
        """Squared-Euclidean cost of the clouds X (n x d), Y (m x d) divided by its maximum, formed on the
        device (bit-identical to problems.problem_from_points).  on_the_fly=True never stores the matrix."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        if X.ndim != 2 or Y.ndim != 2 or X.shape[1] != Y.shape[1]:
            raise ValidationError("set_pointcloud: X and Y must be (n x d) and (m x d)")
        n, m, d = X.shape[0], Y.shape[0], X.shape[1]
        a = _vec(a, n, "problem: marginal")
        b = _vec(b, m, "problem: marginal")
        begin, count = rows if rows is not None else (0, n)
        if rows is None and self.world == 1:
            st = self._lib.regot_b200_set_pointcloud(self._h, n, m, d, _ptr(X), _ptr(Y), _ptr(a), _ptr(b), eta, int(on_the_fly))
        else:
            st = self._lib.regot_b200_set_pointcloud_rows(
                self._h, n, m, begin, count, d, _ptr(X), _ptr(Y), _ptr(a), _ptr(b), eta, int(on_the_fly))
        self._check(st)
        self.n, self.m, self.row_begin, self.row_count = n, m, begin, count
        self._problem_key = None

    def get_cost(self) -> np.ndarray:
        """This context's cost block (row_count x m), as the kernels see it."""
        out = np.empty((self.row_count, self.m))
        self._check(self._lib.regot_b200_get_cost(self._h, _ptr(out)))
        return out

    def set_problem_block(self, p: ProblemInstance, M_block: np.ndarray, row_begin: int, row_count: int) -> None:
        """Upload rows [row_begin, row_begin + row_count) given as a C-contiguous (row_count x m) array
        (e.g. a view of pinned memory); p supplies n, m, the global marginals and eta (p.M is not read)."""
        if M_block.shape != (row_count, p.m) or not M_block.flags.c_contiguous or M_block.dtype != np.float64:
            raise ValidationError("problem: cost matrix shape mismatch")
        a = _vec(p.a, p.n, "problem: marginal")
        b = _vec(p.b, p.m, "problem: marginal")
        self._check(self._lib.regot_b200_set_problem_rows(
            self._h, p.n, p.m, row_begin, row_count, _ptr(M_block), LAYOUT_ROWMAJOR, p.m, _ptr(a), _ptr(b), p.eta))
        self.n, self.m, self.row_begin, self.row_count = p.n, p.m, row_begin, row_count
        self._problem_key = None

    def set_problem_device(self, n: int, m: int, M_ptr: int, ld: int, a_ptr: int, b_ptr: int, eta: float,
                           rows: Optional[Tuple[int, int]] = None) -> None:
        """Borrow a row-major block already resident in HBM (raw device pointers)."""
        begin, count = rows if rows is not None else (0, n)
        self._check(self._lib.regot_b200_set_problem_device(
            self._h, n, m, begin, count, C.c_void_p(M_ptr), ld, C.c_void_p(a_ptr), C.c_void_p(b_ptr), eta))
        self.n, self.m, self.row_begin, self.row_count = n, m, begin, count
        self._problem_key = None

    def ensure_problem(self, p: ProblemInstance) -> None:
        """Upload p unless this very instance, unchanged, is the resident problem (the free functions below
        call this on every invocation, like the reference passes `const ProblemInstance&`)."""
        k = self._problem_key
        if (k is None or k[0] is not p or k[1:6] != (p.n, p.m, p.eta, self.row_begin, self.row_count)
                or k[6] != _fingerprint(p)):
            self.set_problem(p)

    def validate_problem(self) -> None:
        self._check(self._lib.regot_b200_validate_problem(self._h))

    def _dual(self, x: DualPoint, who: str):
        if x.alpha.shape != (self.n,) or x.beta.shape != (self.m,):
            raise ValidationError(f"{who}: dual point/problem dimension mismatch")
        return _vec(x.alpha), _vec(x.beta)

    # -- dual kernels ---------------------------------------------------------------
    def fused_gradient(self, x: DualPoint) -> GradientResult:
        al, be = self._dual(x, "fused_gradient")
        info = GradientInfoC()
        grad = np.zeros(self.n + self.m - 1)
        row = np.zeros(self.n)
        col = np.zeros(self.m)
        self._check(self._lib.regot_b200_fused_gradient(
            self._h, _ptr(al), _ptr(be), C.byref(info), _ptr(grad), _ptr(row), _ptr(col)))
        return GradientResult(info.f, grad, row, col, info.marginal_error, info.duality_gap, info.grad_norm2,
                              info.total_mass)

    def plan(self, x: DualPoint) -> np.ndarray:
        al, be = self._dual(x, "plan")
        T = np.zeros((self.n, self.m))
        self._check(self._lib.regot_b200_plan(self._h, _ptr(al), _ptr(be), _ptr(T), LAYOUT_ROWMAJOR))
        return T

    # -- Sinkhorn -------------------------------------------------------------------
    def optimal_alpha(self, x: DualPoint) -> np.ndarray:
        al, be = self._dual(x, "optimal_alpha")
        out = np.zeros(self.n)
        self._check(self._lib.regot_b200_optimal_alpha(self._h, _ptr(al), _ptr(be), _ptr(out)))
        return out

    def optimal_beta(self, alpha) -> np.ndarray:
        al = _vec(alpha, self.n, "optimal_beta: alpha")
        out = np.zeros(self.m)
        self._check(self._lib.regot_b200_optimal_beta(self._h, _ptr(al), _ptr(out)))
        return out

    def sinkhorn_step(self, x: DualPoint) -> DualPoint:
        al, be = self._dual(x, "sinkhorn_step")
        al, be = al.copy(), be.copy()
        self._check(self._lib.regot_b200_sinkhorn_step(self._h, _ptr(al), _ptr(be)))
        return DualPoint(al, be)

    @staticmethod
    def _step_record(q) -> SplrStepRecord:
        return SplrStepRecord(
            q.iter, bool(q.refresh), bool(q.sinkhorn_selected), q.f_before, q.f_after, q.f_cand_sinkhorn,
            q.f_cand_qn, q.gamma, q.g_dot_d, q.gnew_dot_d, bool(q.curvature_ok), bool(q.ls_failed),
            bool(q.lowrank_active), q.tau, q.factor_retries, q.ls_evals, q.cg_iters)

    def _unpack(self, res: ResultC, want_steps: bool):
        trace = SolverTrace(res.algo.decode(), "", res.eta, res.config_hash.decode())
        for r in range(res.n_trace):
            t = res.trace[r]
            trace.rows.append(TraceRow(t.iter, t.wall_ms, t.f, t.marginal_error, t.duality_gap))
        steps = []
        if want_steps:
            for s in range(res.n_steps):
                steps.append(self._step_record(res.steps[s]))
        x = None
        if res.alpha and res.beta:
            x = DualPoint(np.ctypeslib.as_array(res.alpha, (res.n,)).copy(),
                          np.ctypeslib.as_array(res.beta, (res.m,)).copy())
        stats = SolveStats(res.device_ms, res.gradient_passes, res.lse_passes, res.kernel_launches)
        return x, trace, steps, stats

    def run_sinkhorn(self, x0: DualPoint, cfg: SinkhornConfig) -> SinkhornResult:
        al, be = self._dual(x0, "run_sinkhorn")
        c = cfg._c()
        res = ResultC()
        st = self._lib.regot_b200_run_sinkhorn(self._h, _ptr(al), _ptr(be), C.byref(c), C.byref(res))
        try:
            self._check(st)
            x, trace, _, stats = self._unpack(res, False)
            return SinkhornResult(x, trace, stats)
        finally:
            self._lib.regot_b200_result_free(C.byref(res))

    def run_splr(self, x0: DualPoint, cfg: SplrConfig) -> SplrResult:
        al, be = self._dual(x0, "run_splr")
        c = cfg._c()
        res = ResultC()
        st = self._lib.regot_b200_run_splr(self._h, _ptr(al), _ptr(be), C.byref(c), C.byref(res))
        try:
            if st == StepError.status:
                _, trace, _, _ = self._unpack(res, False)
                raise StepError(res.message.decode(), trace)
            self._check(st)
            x, trace, steps, stats = self._unpack(res, True)
            return SplrResult(x, trace, steps, stats)
        finally:
            self._lib.regot_b200_result_free(C.byref(res))

    def splr_init(self, x0: DualPoint, cfg: SplrConfig) -> "SplrState":
        """splr.h:326-334."""
        al, be = self._dual(x0, "splr_init")
        c = cfg._c()
        h = C.c_void_p()
        self._check(self._lib.regot_b200_splr_init(self._h, _ptr(al), _ptr(be), C.byref(c), C.byref(h)))
        return SplrState(self, h)

    def splr_step(self, st: "SplrState", cfg: SplrConfig) -> SplrStepRecord:
        """splr.h:348-478: advances `st` in place (the reference moves the state through) and returns the record."""
        st._live()
        c = cfg._c()
        rec = StepRecordC()
        self._check(self._lib.regot_b200_splr_step(self._h, st._h, C.byref(c), C.byref(rec)))
        return self._step_record(rec)

    # -- sparsification ---------------------------------------------------------------
    def select_topk(self, T: np.ndarray, k: int) -> SparsityPattern:
        T = np.asarray(T, dtype=np.float64)
        if T.ndim != 2:
            raise ValidationError("select_topk: T must be a matrix")
        n, m = T.shape
        if T.flags.f_contiguous and not T.flags.c_contiguous:
            layout = LAYOUT_COLMAJOR
        else:
            T = np.ascontiguousarray(T)
            layout = LAYOUT_ROWMAJOR
        cnt = C.c_int64(0)
        self._check(self._lib.regot_b200_select_topk_dense(self._h, n, m, _ptr(T), layout, k, None, 0, C.byref(cnt)))
        coords = np.zeros((max(cnt.value, 1), 2), dtype=np.int32)
        self._check(self._lib.regot_b200_select_topk_dense(
            self._h, n, m, _ptr(T), layout, k, _ptr(coords), cnt.value, C.byref(cnt)))
        return SparsityPattern(n, m - 1, coords[: cnt.value], k)

    def assemble(self, x: DualPoint, omega: SparsityPattern, tau: float,
                 gr: Optional[GradientResult] = None) -> "SparseSym":
        al, be = self._dual(x, "assemble")
        if gr is None:
            gr = self.fused_gradient(x)
        coords = np.ascontiguousarray(omega.coords, dtype=np.int32)
        h = C.c_void_p()
        self._check(self._lib.regot_b200_assemble(
            self._h, _ptr(al), _ptr(be), _ptr(coords), coords.shape[0], tau, _ptr(_vec(gr.row_sums)),
            _ptr(_vec(gr.col_sums)), C.byref(h)))
        return SparseSym(self, h)

    def assemble_topk(self, x: DualPoint, k: int, tau: float, gr: Optional[GradientResult] = None) -> "SparseSym":
        """plan + select_topk + assemble without materialising T (splr.h:361-363)."""
        al, be = self._dual(x, "assemble")
        if gr is None:
            gr = self.fused_gradient(x)
        h = C.c_void_p()
        self._check(self._lib.regot_b200_assemble_topk(
            self._h, _ptr(al), _ptr(be), k, tau, _ptr(_vec(gr.row_sums)), _ptr(_vec(gr.col_sums)), C.byref(h)))
        return SparseSym(self, h)

    def compute_direction(self, A: "SparseSym", g, u=None, v=None, xi: float = 0.0, zeta: float = 0.0,
                          cg_rtol: float = 0.0, cg_max_iter: int = 0) -> Tuple[np.ndarray, int]:
        """splr.h:128-167 with device PCG in place of the sparse Cholesky solve."""
        dim = self.n + self.m - 1
        g = _vec(g, dim, "compute_direction: g")
        uu = None if u is None else _vec(u, dim, "compute_direction: u")
        vv = None if v is None else _vec(v, dim, "compute_direction: v")
        d = np.zeros(dim)
        its = C.c_int32(0)
        self._check(self._lib.regot_b200_compute_direction(
            self._h, A._h, _ptr(g), _ptr(uu), _ptr(vv), xi, zeta, cg_rtol, cg_max_iter, _ptr(d), C.byref(its)))
        return d, int(its.value)

    # -- measurement ----------------------------------------------------------------------
    def set_profiling(self, enabled: bool) -> None:
        self._check(self._lib.regot_b200_set_profiling(self._h, int(enabled)))

    def get_profile(self, kind: int) -> Tuple[int, float]:
        """(launches, total device ms) of kernel class `kind` since set_profiling(True)."""
        n, ms = C.c_int64(0), C.c_double(0.0)
        self._check(self._lib.regot_b200_get_profile(self._h, kind, C.byref(n), C.byref(ms)))
        return int(n.value), float(ms.value)

    def time_kernel(self, which: int, x: DualPoint, iters: int) -> np.ndarray:
        al, be = self._dual(x, "time_kernel")
        ms = np.zeros(iters, dtype=np.float32)
        self._check(self._lib.regot_b200_time_kernel(
            self._h, which, _ptr(al), _ptr(be), iters, ms.ctypes.data_as(_lib.c_float_p)))
        return ms


class SparseSym:
    """Device-resident H_Omega + tau I (sparsity.h:97-195)."""

    def __init__(self, solver: Solver, handle):
        self._s = solver
        self._h = handle
        solver._sparse.add(self)

    def free(self) -> None:
        if self._h:
            self._s._lib.regot_b200_sparse_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def _live(self):
        if not self._h or not self._s._h:
            raise ValidationError("SparseSym: the matrix or its solver was released")

    def info(self):
        self._live()
        dim, nnz, nc, pid = C.c_int32(), C.c_int64(), C.c_int64(), C.c_uint64()
        self._s._check(self._s._lib.regot_b200_sparse_info(self._h, C.byref(dim), C.byref(nnz), C.byref(nc), C.byref(pid)))
        return dim.value, nnz.value, nc.value, pid.value

    def export(self):
        """(colptr, rowidx, values, coords) in the reference's CSC layout (sparsity.h:249-289)."""
        dim, nnz, nc, _ = self.info()
        colptr = np.zeros(dim + 1, np.int32)
        rowidx = np.zeros(nnz, np.int32)
        values = np.zeros(nnz)
        coords = np.zeros((nc, 2), np.int32)
        self._s._check(self._s._lib.regot_b200_sparse_export(
            self._s._h, self._h, _ptr(colptr), _ptr(rowidx), _ptr(values), _ptr(coords)))
        return colptr, rowidx, values, coords

    def export_local(self):
        """(coords, values) of this context's rows of the pattern: global (i, j) pairs in row-major order and
        B_ij = T_ij / eta.  Works on row-sharded contexts (the ranks' pieces concatenate to the global pattern)."""
        self._live()
        cnt = C.c_int64(0)
        self._s._check(self._s._lib.regot_b200_sparse_export_local(self._s._h, self._h, None, None, 0, C.byref(cnt)))
        coords = np.zeros((cnt.value, 2), np.int32)
        values = np.zeros(cnt.value)
        if cnt.value:
            self._s._check(self._s._lib.regot_b200_sparse_export_local(
                self._s._h, self._h, _ptr(coords), _ptr(values), cnt.value, C.byref(cnt)))
        return coords, values

    def update_values(self, x: DualPoint, tau: float, gr: Optional[GradientResult] = None) -> None:
        self._live()
        al, be = self._s._dual(x, "update_values")
        if gr is None:
            gr = self._s.fused_gradient(x)
        self._s._check(self._s._lib.regot_b200_update_values(
            self._s._h, self._h, _ptr(al), _ptr(be), tau, _ptr(_vec(gr.row_sums)), _ptr(_vec(gr.col_sums))))

    def matvec(self, v) -> np.ndarray:
        dim = self.info()[0]
        v = _vec(v, dim, "SparseSym::matvec")
        y = np.zeros(dim)
        self._s._check(self._s._lib.regot_b200_matvec(self._s._h, self._h, _ptr(v), _ptr(y)))
        return y


class SplrState:
    """SplrState (splr.h:82-97), resident on the device."""

    def __init__(self, solver: Solver, handle):
        self._s = solver
        self._h = handle
        solver._sparse.add(self)  # released with the solver, like the matrices

    def free(self) -> None:
        if self._h:
            self._s._lib.regot_b200_splr_state_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def _live(self):
        if not self._h or not self._s._h:
            raise ValidationError("SplrState: the state or its solver was released")

    def _info(self):
        self._live()
        it, hp, info = C.c_int64(), C.c_int32(), GradientInfoC()
        self._s._check(self._s._lib.regot_b200_splr_state_info(self._s._h, self._h, C.byref(it), C.byref(hp), C.byref(info)))
        return it.value, bool(hp.value), info

    @property
    def iter(self) -> int:
        return self._info()[0]

    @property
    def has_prev(self) -> bool:
        return self._info()[1]

    @property
    def x(self) -> DualPoint:
        self._live()
        al, be = np.zeros(self._s.n), np.zeros(self._s.m)
        self._s._check(self._s._lib.regot_b200_splr_state_point(self._s._h, self._h, _ptr(al), _ptr(be), None, None, None))
        return DualPoint(al, be)

    @property
    def cur(self) -> GradientResult:
        """GradientResult at st.x (on a sharded context: this rank's slice of the n-long arrays)."""
        _, _, info = self._info()
        s = self._s
        grad, row, col = np.zeros(s.n + s.m - 1), np.zeros(s.n), np.zeros(s.m)
        s._check(s._lib.regot_b200_splr_state_point(s._h, self._h, None, None, _ptr(grad), _ptr(row), _ptr(col)))
        return GradientResult(info.f, grad, row, col, info.marginal_error, info.duality_gap, info.grad_norm2, info.total_mass)

    @property
    def A(self) -> Optional["SparseSym"]:
        """st.A, borrowed: valid until the next refresh step."""
        self._live()
        h = self._s._lib.regot_b200_splr_state_matrix(self._h)
        return _BorrowedSparse(self._s, C.c_void_p(h)) if h else None


class _BorrowedSparse(SparseSym):
    """A SparseSym owned by an SplrState: never freed from here."""

    def free(self) -> None:
        self._h = None


# ---- free functions with the reference's signatures ------------------------------------------------
_default: Optional[Solver] = None


def default_solver() -> Solver:
    global _default
    if _default is None:
        _default = Solver(0)
    return _default


def _bound(p: ProblemInstance) -> Solver:
    s = default_solver()
    s.ensure_problem(p)
    return s


def fused_gradient(x: DualPoint, p: ProblemInstance, tile: Optional[FusedTiling] = None) -> GradientResult:
    """dual.h:106-164.  `tile` is advisory on the device but validated like the reference."""
    if tile is not None and (tile.rows < 1 or tile.cols < 1):
        raise ValidationError("fused_gradient: invalid tile shape")
    return _bound(p).fused_gradient(x)


def plan(x: DualPoint, p: ProblemInstance) -> np.ndarray:
    """dual.h:83-94."""
    return _bound(p).plan(x)


def objective(x: DualPoint, p: ProblemInstance) -> float:
    """dual.h:184-187."""
    return fused_gradient(x, p).f


def marginal_error(gr: GradientResult, p: ProblemInstance) -> float:
    """dual.h:219-222 (computed by the device epilogue of the same pass)."""
    return gr.marginal_error


def duality_gap(x: DualPoint, gr: GradientResult, p: ProblemInstance) -> float:
    """dual.h:225-229."""
    return gr.duality_gap


def optimal_alpha(x: DualPoint, p: ProblemInstance) -> np.ndarray:
    """sinkhorn.h:44-74."""
    return _bound(p).optimal_alpha(x)


def optimal_beta(alpha, p: ProblemInstance) -> np.ndarray:
    """sinkhorn.h:77-101."""
    return _bound(p).optimal_beta(alpha)


def sinkhorn_step(x: DualPoint, p: ProblemInstance) -> DualPoint:
    """sinkhorn.h:105-115."""
    return _bound(p).sinkhorn_step(x)


def run_sinkhorn(x0: DualPoint, p: ProblemInstance, cfg: SinkhornConfig) -> SinkhornResult:
    """sinkhorn.h:123-171."""
    return _bound(p).run_sinkhorn(x0, cfg)


def run_splr(x0: DualPoint, p: ProblemInstance, cfg: SplrConfig) -> SplrResult:
    """splr.h:487-534."""
    return _bound(p).run_splr(x0, cfg)


def splr_init(x0: DualPoint, p: ProblemInstance, cfg: SplrConfig) -> SplrState:
    """splr.h:326-334."""
    return _bound(p).splr_init(x0, cfg)


def splr_step(st: SplrState, p: ProblemInstance, cfg: SplrConfig) -> Tuple[SplrState, SplrStepRecord]:
    """splr.h:348-478: `st = splr_step(std::move(st), p, cfg, &rec)` -- the state comes back with the record."""
    s = _bound(p)
    if st._s is not s:
        raise ValidationError("splr_step: the state belongs to another solver")
    return st, s.splr_step(st, cfg)


def select_topk(T: np.ndarray, k: int) -> SparsityPattern:
    """sparsity.h:44-91."""
    if k < 0:
        raise ValidationError("select_topk: k must be >= 0")
    return default_solver().select_topk(T, k)


def assemble(x: DualPoint, p: ProblemInstance, omega: SparsityPattern, tau: float,
             gr: Optional[GradientResult] = None) -> SparseSym:
    """sparsity.h:226-300."""
    return _bound(p).assemble(x, omega, tau, gr)


def update_values(A: SparseSym, x: DualPoint, p: ProblemInstance, tau: float,
                  gr: Optional[GradientResult] = None) -> None:
    """sparsity.h:305-323."""
    _bound(p)
    A.update_values(x, tau, gr)
