"""Problem generators: host-side mirror of problem.h plus the BASELINE workloads.

`Rng`, `gen_synthetic1`, `gen_synthetic2`, `normalize_cost`, `validate_problem`
follow the reference (proj/include/regot/problem.h:30-180) draw for draw:
mt19937_64, 53-bit uniforms, Box-Muller with a cached spare, source drawn
before target, row by row, coordinate inner.  `gen_image`, `gen_gmm`,
`gen_uniform` define BASELINE.json configs B, D, E, which have no generator in
the reference.  Plain numpy; the cost matrices are built row-major
(C order), the layout the device wants.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

from .regot import DegenerateCostError, ProblemInstance, ValidationError

_MASK = (1 << 64) - 1


class Rng:
    """problem.h:65-96: std::mt19937_64 + uniform()/normal()."""

    _NN, _MM = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self._NN
        mt[0] = seed & _MASK
        for i in range(1, self._NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self._mt = mt
        self._i = self._NN
        self._spare = 0.0
        self._have_spare = False

    def _twist(self) -> None:
        mt, nn, mm = self._mt, self._NN, self._MM
        for i in range(nn):
            x = (mt[i] & self._UM) | (mt[(i + 1) % nn] & self._LM)
            mt[i] = mt[(i + mm) % nn] ^ (x >> 1) ^ (self._MATRIX_A if (x & 1) else 0)
        self._i = 0

    def next_u64(self) -> int:
        if self._i >= self._NN:
            self._twist()
        x = self._mt[self._i]
        self._i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _MASK

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0**-53

    def normal(self) -> float:
        if self._have_spare:
            self._have_spare = False
            return self._spare
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 2.0 * math.pi * u2
        self._spare = r * math.sin(th)
        self._have_spare = True
        return r * math.cos(th)


def normalize_cost(M: np.ndarray) -> np.ndarray:
    """problem.h:53-61."""
    if M.size == 0:
        raise DegenerateCostError("normalize_cost: empty cost matrix")
    mx = M.max()
    if not (mx > 0.0):
        raise DegenerateCostError("normalize_cost: no strictly positive entry")
    return M / mx


def validate_problem(p: ProblemInstance) -> None:
    """problem.h:30-50."""
    if p.n < 1 or p.m < 1:
        raise ValidationError("problem: n and m must be at least 1")
    if p.M.shape != (p.n, p.m):
        raise ValidationError("problem: cost matrix shape mismatch")
    if p.a.shape != (p.n,) or p.b.shape != (p.m,):
        raise ValidationError("problem: marginal length mismatch")
    if not (p.eta > 0.0) or not math.isfinite(p.eta):
        raise ValidationError("problem: eta must be positive and finite")
    if not (np.isfinite(p.M).all() and np.isfinite(p.a).all() and np.isfinite(p.b).all()):
        raise ValidationError("problem: non-finite entries")
    if not (p.a.min() > 0.0):
        raise ValidationError("problem: a must be elementwise positive")
    if not (p.b.min() > 0.0):
        raise ValidationError("problem: b must be elementwise positive")
    if abs(float(np.sum(p.a)) - 1.0) > 1e-12:
        raise ValidationError("problem: a must sum to 1 within 1e-12")
    if abs(float(np.sum(p.b)) - 1.0) > 1e-12:
        raise ValidationError("problem: b must sum to 1 within 1e-12")


def _seq_sum(v: np.ndarray) -> float:
    s = 0.0
    for x in v.tolist():
        s += x
    return s


def sqeuclid_cost(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """M_ij = sum_k (X_ik - Y_jk)^2, coordinates accumulated in order (problem.h:124-127)."""
    n, d = X.shape
    M = np.zeros((n, Y.shape[0]))
    for k in range(d):
        df = X[:, k][:, None] - Y[:, k][None, :]
        M += df * df
    return M


def gen_synthetic1(n: int, m: int, variant: str, d: int, seed: int, eta: float = 0.001) -> ProblemInstance:
    """problem.h:103-138; variant is "iid" or "diff"."""
    if n < 2 or m < 2:
        raise ValidationError("gen_synthetic1: need n >= 2 and m >= 2")
    if d < 1:
        raise ValidationError("gen_synthetic1: need d >= 1")
    rng = Rng(seed)
    X = np.array([rng.normal() for _ in range(n * d)]).reshape(n, d)
    if variant == "iid":
        Y = np.array([rng.normal() for _ in range(m * d)]).reshape(m, d)
    else:
        Y = np.array([1.0 + 0.5 * rng.normal() for _ in range(m * d)]).reshape(m, d)
    p = ProblemInstance(n, m, normalize_cost(sqeuclid_cost(X, Y)), np.full(n, 1.0 / n), np.full(m, 1.0 / m), eta)
    validate_problem(p)
    return p


def gen_synthetic2(n: int, m: int, eta: float = 0.001) -> ProblemInstance:
    """problem.h:142-180: exponential source vs two-Gaussian mixture on [0, 5]."""
    if n < 2 or m < 2:
        raise ValidationError("gen_synthetic2: need n >= 2 and m >= 2")
    x = 5.0 * np.arange(n, dtype=np.float64) / float(n - 1)
    y = 5.0 * np.arange(m, dtype=np.float64) / float(m - 1)

    def gauss(t, mu, var):
        return np.array([math.exp(-(v - mu) * (v - mu) / (2.0 * var)) for v in t.tolist()]) / math.sqrt(2.0 * math.pi * var)

    a = np.array([math.exp(-v) for v in x.tolist()])
    b = 0.2 * gauss(y, 1.0, 0.04) + 0.8 * gauss(y, 3.0, 0.25)
    a = a / _seq_sum(a)
    b = b / _seq_sum(b)
    df = x[:, None] - y[None, :]
    p = ProblemInstance(n, m, normalize_cost(df * df), a, b, eta)
    validate_problem(p)
    return p


# ---- BASELINE workloads without a reference generator --------------------------
def _blob_histogram(side: int, seed: int) -> np.ndarray:
    rng = Rng(seed)
    blobs = []
    for _ in range(3):
        cx = 0.15 + 0.7 * rng.uniform()
        cy = 0.15 + 0.7 * rng.uniform()
        sg = 0.05 + 0.10 * rng.uniform()
        wt = 0.5 + rng.uniform()
        blobs.append((cx, cy, sg, wt))
    g = np.arange(side, dtype=np.float64) / float(side - 1)
    yy, xx = np.meshgrid(g, g, indexing="ij")  # pixel (r, c) -> (y, x)
    v = np.full((side, side), 1e-6)
    for cx, cy, sg, wt in blobs:
        dx, dy = xx - cx, yy - cy
        e = -(dx * dx + dy * dy) / (2.0 * sg * sg)
        v = v + wt * np.array([math.exp(t) for t in e.ravel().tolist()]).reshape(side, side)
    h = v.ravel()
    return h / _seq_sum(h)


def gen_image(side: int, eta: float, seed_a: int = 11, seed_b: int = 12) -> ProblemInstance:
    """Config B: side x side pixel grids on the unit square, cost = squared distance / 2
    (maximum exactly 1), marginals = 3 Gaussian blobs + floor 1e-6.  side = 100 gives n = m = 10,000."""
    if side < 2:
        raise ValidationError("gen_image: need side >= 2")
    n = side * side
    s = 1.0 / float(side - 1)
    idx = np.arange(n)
    ys, xs = (idx // side).astype(np.float64) * s, (idx % side).astype(np.float64) * s
    dx = xs[:, None] - xs[None, :]
    dy = ys[:, None] - ys[None, :]
    M = 0.5 * (dx * dx + dy * dy)
    p = ProblemInstance(n, n, normalize_cost(M), _blob_histogram(side, seed_a), _blob_histogram(side, seed_b), eta)
    validate_problem(p)
    return p


def _gmm_points(n: int, d: int, comps: int, rng: Rng) -> np.ndarray:
    mu = np.array([2.0 * rng.normal() for _ in range(comps * d)]).reshape(comps, d)
    X = np.zeros((n, d))
    for i in range(n):
        c = int(rng.uniform() * comps) % comps
        sg = 0.5 if c % 2 == 0 else 1.0
        for k in range(d):
            X[i, k] = mu[c, k] + sg * rng.normal()
    return X


def gen_gmm_points(n: int, m: int, d: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Config D clouds: 3-component source, 4-component target Gaussian mixtures in R^d."""
    rng = Rng(seed)
    X = _gmm_points(n, d, 3, rng)
    Y = _gmm_points(m, d, 4, rng)
    return X, Y


def gen_uniform_points(n: int, m: int, d: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Config E clouds: uniform in [0, 1)^d."""
    rng = Rng(seed)
    X = np.array([rng.uniform() for _ in range(n * d)]).reshape(n, d)
    Y = np.array([rng.uniform() for _ in range(m * d)]).reshape(m, d)
    return X, Y


def problem_from_points(X: np.ndarray, Y: np.ndarray, eta: float) -> ProblemInstance:
    n, m = X.shape[0], Y.shape[0]
    p = ProblemInstance(n, m, normalize_cost(sqeuclid_cost(X, Y)), np.full(n, 1.0 / n), np.full(m, 1.0 / m), eta)
    validate_problem(p)
    return p


def make_problem(kind: str, n: int, m: int, eta: float, d: int = 2, seed: int = 0) -> ProblemInstance:
    """problem.h:293-310 (+ the BASELINE kinds image / gmm / uniform)."""
    if kind == "synth1-iid":
        return gen_synthetic1(n, m, "iid", d, seed, eta)
    if kind == "synth1-diff":
        return gen_synthetic1(n, m, "diff", d, seed, eta)
    if kind == "synth2":
        return gen_synthetic2(n, m, eta)
    if kind == "image":
        return gen_image(d, eta)
    if kind == "gmm":
        return problem_from_points(*gen_gmm_points(n, m, d, seed), eta)
    if kind == "uniform":
        return problem_from_points(*gen_uniform_points(n, m, d, seed), eta)
    raise ValidationError(f"make_problem: unknown generator kind '{kind}'")
