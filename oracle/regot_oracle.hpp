// regot_oracle.hpp -- CPU restatement of the `regot` reference hot path.
//
// TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may build, link or execute it.  The product path
// (paper_2605_08793_b200/csrc) never includes this header and has no CPU
// fallback.
//
// What it is: a dependency-free (no Eigen) C++17 restatement of the reference
// algorithm, flat std::vector<double> storage, cost matrix COLUMN-MAJOR exactly
// like the reference's Eigen::MatrixXd (core.h:16).  Every function cites the
// reference file:line it follows (paths relative to /root/reference/proj/
// include/regot/).  Loop order and summation order follow the reference for all
// in-tree arithmetic; the Eigen BLAS-1 reductions (dot/norm/sum, whose internal
// association order is unspecified) are restated as plain
// left-to-right loops.
//
// Parity status: PINNED for the small-size path -- oracle/selfcheck.cpp and
// tests/test_oracle_kat.py replay the reference's own known-answer tests
// (7-value golden trajectory test_splr.cpp:380-402, 2x2 hand case
// test_dual.cpp:72-85, clamp test_dual.cpp:44-53, top-k worked example and tie
// rule test_sparsity.cpp:74-99, 2x2 Cholesky test_sparse_chol.cpp:93-108, ...)
// and, when oracle/_ref is built (reference headers compiled over
// oracle/eigen_shim), compare against the reference's own code run here.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace rgo {

using vec = std::vector<double>;
using ivec = std::vector<int>;

// ---- status codes: one per reference exception class (core.h:21-37) --------
enum Status {
    OK = 0,
    E_DEGENERATE_COST = 1,
    E_FORMAT = 2,
    E_TRUNCATION = 3,
    E_VALIDATION = 4,
    E_IO = 5,
    E_ORACLE_SIZE = 6,
    E_STRUCTURE = 7,
    E_NOT_POSITIVE_DEFINITE = 8,
    E_DIRECTION = 9,
    E_LINE_SEARCH = 10,
    E_PLOT = 11,
    E_STEP = 12,
};

struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& what) { throw Failure(code, what); }

// ---- small reductions (Eigen dot/norm/sum restated sequentially) -----------
inline double dot(const double* x, const double* y, long n)
{
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}
inline double dot(const vec& x, const vec& y) { return dot(x.data(), y.data(), (long)x.size()); }
inline double sqnorm(const vec& x) { return dot(x, x); }
inline double norm2(const vec& x) { return std::sqrt(sqnorm(x)); }
inline double norm_inf(const vec& x)
{
    double s = 0.0;
    for (double v : x) s = std::max(s, std::fabs(v));
    return s;
}

// core.h:42-52 FNV-1a 64
inline std::uint64_t fnv1a(const void* data, std::size_t len, std::uint64_t h = 0xcbf29ce484222325ULL)
{
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

// core.h:69-80 recursive-halving sum, linear below 33 terms
inline double pairwise_sum(const double* x, long n)
{
    if (n <= 32) {
        double s = 0.0;
        for (long i = 0; i < n; ++i) s += x[i];
        return s;
    }
    const long h = n / 2;
    return pairwise_sum(x, h) + pairwise_sum(x + h, n - h);
}

// core.h:85-131 binary-counter tree over fixed-width blocks.  slot[L] holds
// the sum of 2^L consecutive blocks; push() carries like a binary increment,
// fold() adds occupied slots low-to-high.
struct BlockTree {
    std::size_t width;
    std::vector<vec> slot;
    std::vector<char> full;
    explicit BlockTree(std::size_t w) : width(w) {}
    void push(const double* blk)
    {
        vec carry(blk, blk + width);
        std::size_t L = 0;
        for (; L < slot.size() && full[L]; ++L) {
            const vec& s = slot[L];
            for (std::size_t i = 0; i < width; ++i) carry[i] += s[i];
            full[L] = 0;
        }
        if (L == slot.size()) {
            slot.push_back(std::move(carry));
            full.push_back(1);
        } else {
            slot[L] = std::move(carry);
            full[L] = 1;
        }
    }
    void fold(double* out) const
    {
        for (std::size_t i = 0; i < width; ++i) out[i] = 0.0;
        for (std::size_t L = 0; L < slot.size(); ++L)
            if (full[L])
                for (std::size_t i = 0; i < width; ++i) out[i] += slot[L][i];
    }
};

// ---- problem (problem.h:20-61) ----------------------------------------------
struct Problem {
    long n = 0, m = 0;
    vec M;  // column-major: M[j*n + i]
    vec a, b;
    double eta = 0.0;
    double cost(long i, long j) const { return M[(std::size_t)(j * n + i)]; }
};

// problem.h:30-50
inline void validate_problem(const Problem& p)
{
    if (p.n < 1 || p.m < 1) fail(E_VALIDATION, "problem: n and m must be at least 1");
    if ((long)p.M.size() != p.n * p.m) fail(E_VALIDATION, "problem: cost matrix shape mismatch");
    if ((long)p.a.size() != p.n || (long)p.b.size() != p.m)
        fail(E_VALIDATION, "problem: marginal length mismatch");
    if (!(p.eta > 0.0) || !std::isfinite(p.eta))
        fail(E_VALIDATION, "problem: eta must be positive and finite");
    for (double v : p.M) if (!std::isfinite(v)) fail(E_VALIDATION, "problem: non-finite entries");
    double sa = 0.0, sb = 0.0, mina = INFINITY, minb = INFINITY;
    for (double v : p.a) { if (!std::isfinite(v)) fail(E_VALIDATION, "problem: non-finite entries"); sa += v; mina = std::min(mina, v); }
    for (double v : p.b) { if (!std::isfinite(v)) fail(E_VALIDATION, "problem: non-finite entries"); sb += v; minb = std::min(minb, v); }
    if (!(mina > 0.0)) fail(E_VALIDATION, "problem: a must be elementwise positive");
    if (!(minb > 0.0)) fail(E_VALIDATION, "problem: b must be elementwise positive");
    if (std::fabs(sa - 1.0) > 1e-12) fail(E_VALIDATION, "problem: a must sum to 1 within 1e-12");
    if (std::fabs(sb - 1.0) > 1e-12) fail(E_VALIDATION, "problem: b must sum to 1 within 1e-12");
}

// problem.h:53-61
inline void normalize_cost(vec& M)
{
    if (M.empty()) fail(E_DEGENERATE_COST, "normalize_cost: empty cost matrix");
    double mx = M[0];
    for (double v : M) mx = std::max(mx, v);
    if (!(mx > 0.0)) fail(E_DEGENERATE_COST, "normalize_cost: no strictly positive entry");
    for (double& v : M) v /= mx;
}

// problem.h:65-96  mt19937_64, 53-bit uniform, Box-Muller with cached spare
struct Rng {
    std::mt19937_64 g;
    double spare = 0.0;
    bool has_spare = false;
    explicit Rng(std::uint64_t seed) : g(seed) {}
    double uniform() { return (double)(g() >> 11) * 0x1.0p-53; }
    double normal()
    {
        if (has_spare) { has_spare = false; return spare; }
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(th);
        has_spare = true;
        return r * std::cos(th);
    }
};

inline void uniform_marginals(Problem& p)
{
    p.a.assign((std::size_t)p.n, 1.0 / (double)p.n);
    p.b.assign((std::size_t)p.m, 1.0 / (double)p.m);
}

// squared-Euclidean cost of two point sets (points stored row-wise, d coords
// each); the per-pair sum runs over coordinates in order like Eigen's
// (row_i - row_j).squaredNorm() does for small d (problem.h:124-127).
inline void sqeuclid_cost(Problem& p, const vec& X, const vec& Y, long d)
{
    p.M.assign((std::size_t)(p.n * p.m), 0.0);
    for (long j = 0; j < p.m; ++j)
        for (long i = 0; i < p.n; ++i) {
            double s = 0.0;
            for (long k = 0; k < d; ++k) {
                const double df = X[(std::size_t)(i * d + k)] - Y[(std::size_t)(j * d + k)];
                s += df * df;
            }
            p.M[(std::size_t)(j * p.n + i)] = s;
        }
}

// problem.h:103-138 ; variant 0 = iid, 1 = diff
inline Problem gen_synthetic1(long n, long m, int variant, long d, std::uint64_t seed, double eta)
{
    if (n < 2 || m < 2) fail(E_VALIDATION, "gen_synthetic1: need n >= 2 and m >= 2");
    if (d < 1) fail(E_VALIDATION, "gen_synthetic1: need d >= 1");
    Rng rng(seed);
    vec X((std::size_t)(n * d)), Y((std::size_t)(m * d));
    for (auto& v : X) v = rng.normal();
    for (auto& v : Y) {
        const double z = rng.normal();
        v = (variant == 0) ? z : 1.0 + 0.5 * z;
    }
    Problem p;
    p.n = n; p.m = m; p.eta = eta;
    sqeuclid_cost(p, X, Y, d);
    normalize_cost(p.M);
    uniform_marginals(p);
    validate_problem(p);
    return p;
}

// problem.h:142-180
inline Problem gen_synthetic2(long n, long m, double eta)
{
    if (n < 2 || m < 2) fail(E_VALIDATION, "gen_synthetic2: need n >= 2 and m >= 2");
    vec x((std::size_t)n), y((std::size_t)m);
    for (long i = 0; i < n; ++i) x[(std::size_t)i] = 5.0 * (double)i / (double)(n - 1);
    for (long j = 0; j < m; ++j) y[(std::size_t)j] = 5.0 * (double)j / (double)(m - 1);
    const double pi = 3.141592653589793238462643383279502884;
    auto gauss = [pi](double t, double mu, double var) {
        return std::exp(-(t - mu) * (t - mu) / (2.0 * var)) / std::sqrt(2.0 * pi * var);
    };
    Problem p;
    p.n = n; p.m = m; p.eta = eta;
    p.a.resize((std::size_t)n);
    p.b.resize((std::size_t)m);
    for (long i = 0; i < n; ++i) p.a[(std::size_t)i] = std::exp(-x[(std::size_t)i]);
    for (long j = 0; j < m; ++j)
        p.b[(std::size_t)j] = 0.2 * gauss(y[(std::size_t)j], 1.0, 0.04) + 0.8 * gauss(y[(std::size_t)j], 3.0, 0.25);
    double sa = 0.0, sb = 0.0;
    for (double v : p.a) sa += v;
    for (double v : p.b) sb += v;
    for (double& v : p.a) v /= sa;
    for (double& v : p.b) v /= sb;
    p.M.resize((std::size_t)(n * m));
    for (long j = 0; j < m; ++j)
        for (long i = 0; i < n; ++i) {
            const double df = x[(std::size_t)i] - y[(std::size_t)j];
            p.M[(std::size_t)(j * n + i)] = df * df;
        }
    normalize_cost(p.M);
    validate_problem(p);
    return p;
}

// tests/oracles.h:22-44  (uniform cost, random positive marginals)
inline Problem rand_instance(long n, long m, double eta, std::uint64_t seed)
{
    Rng rng(seed);
    Problem p;
    p.n = n; p.m = m; p.eta = eta;
    p.M.resize((std::size_t)(n * m));
    for (long j = 0; j < m; ++j)
        for (long i = 0; i < n; ++i) p.M[(std::size_t)(j * n + i)] = rng.uniform();
    normalize_cost(p.M);
    p.a.resize((std::size_t)n);
    p.b.resize((std::size_t)m);
    for (auto& v : p.a) v = 0.2 + rng.uniform();
    for (auto& v : p.b) v = 0.2 + rng.uniform();
    double sa = 0.0, sb = 0.0;
    for (double v : p.a) sa += v;
    for (double v : p.b) sb += v;
    for (double& v : p.a) v /= sa;
    for (double& v : p.b) v /= sb;
    validate_problem(p);
    return p;
}

// ---- dual point (dual.h:14-47) ----------------------------------------------
struct Dual {
    vec alpha, beta;
    static Dual zeros(long n, long m)
    {
        Dual x;
        x.alpha.assign((std::size_t)n, 0.0);
        x.beta.assign((std::size_t)m, 0.0);
        return x;
    }
    static Dual from_free(const vec& xf, long n, long m)
    {
        if ((long)xf.size() != n + m - 1) fail(E_VALIDATION, "DualPoint::from_free: length mismatch");
        Dual x;
        x.alpha.assign(xf.begin(), xf.begin() + n);
        x.beta.assign(xf.begin() + n, xf.end());
        x.beta.push_back(0.0);
        return x;
    }
    vec to_free() const
    {
        vec xf(alpha);
        xf.insert(xf.end(), beta.begin(), beta.end() - 1);
        return xf;
    }
};

// tests/oracles.h:47-56
inline Dual rand_dual(long n, long m, double scale, std::uint64_t seed)
{
    Rng rng(seed);
    Dual x = Dual::zeros(n, m);
    for (long i = 0; i < n; ++i) x.alpha[(std::size_t)i] = scale * (2.0 * rng.uniform() - 1.0);
    for (long j = 0; j + 1 < m; ++j) x.beta[(std::size_t)j] = scale * (2.0 * rng.uniform() - 1.0);
    return x;
}

struct Grad {
    double f = 0.0;
    vec grad, row, col;
};

// dual.h:62-70  division by eta, clamp to +-700, exp
inline double plan_entry(double ai, double bj, double mij, double eta)
{
    double t = (ai + bj - mij) / eta;
    if (t > 700.0) t = 700.0;
    else if (t < -700.0) t = -700.0;
    return std::exp(t);
}

// dual.h:72-78
inline void check_dims(const Dual& x, const Problem& p, const char* who)
{
    if ((long)x.alpha.size() != p.n || (long)x.beta.size() != p.m)
        fail(E_VALIDATION, std::string(who) + ": dual point/problem dimension mismatch");
    if (x.beta[(std::size_t)(p.m - 1)] != 0.0)
        fail(E_VALIDATION, std::string(who) + ": gauge violated, beta[m-1] must be 0");
}

// dual.h:83-94  dense T, column-major
inline vec plan(const Dual& x, const Problem& p)
{
    check_dims(x, p, "plan");
    vec T((std::size_t)(p.n * p.m));
    for (long j = 0; j < p.m; ++j) {
        const double bj = x.beta[(std::size_t)j];
        for (long i = 0; i < p.n; ++i)
            T[(std::size_t)(j * p.n + i)] = plan_entry(x.alpha[(std::size_t)i], bj, p.cost(i, j), p.eta);
    }
    return T;
}

// dual.h:157-162 shared epilogue: objective from the row sums, gradient blocks
inline void finish_gradient(Grad& g, const Dual& x, const Problem& p, double total)
{
    const long n = p.n, m = p.m;
    g.f = p.eta * total - dot(x.alpha.data(), p.a.data(), n) - dot(x.beta.data(), p.b.data(), m - 1);
    g.grad.resize((std::size_t)(n + m - 1));
    for (long i = 0; i < n; ++i) g.grad[(std::size_t)i] = g.row[(std::size_t)i] - p.a[(std::size_t)i];
    for (long j = 0; j + 1 < m; ++j) g.grad[(std::size_t)(n + j)] = g.col[(std::size_t)j] - p.b[(std::size_t)j];
}

// dual.h:106-164  one pass, tr x tc tiles, plain sums inside a tile, binary-
// counter pairwise merge across column tiles (rows) and across row bands (cols)
inline Grad fused_gradient(const Dual& x, const Problem& p, int tr = 8, int tc = 32)
{
    check_dims(x, p, "fused_gradient");
    if (tr < 1 || tc < 1) fail(E_VALIDATION, "fused_gradient: invalid tile shape");
    const long n = p.n, m = p.m;
    Grad g;
    g.row.resize((std::size_t)n);
    g.col.resize((std::size_t)m);
    BlockTree col_tree((std::size_t)m);
    vec band((std::size_t)m), part((std::size_t)tr);
    for (long i0 = 0; i0 < n; i0 += tr) {
        const long h = std::min<long>(tr, n - i0);
        BlockTree row_tree((std::size_t)h);
        std::fill(band.begin(), band.end(), 0.0);
        for (long j0 = 0; j0 < m; j0 += tc) {
            const long w = std::min<long>(tc, m - j0);
            std::fill(part.begin(), part.begin() + h, 0.0);
            for (long j = j0; j < j0 + w; ++j) {
                const double bj = x.beta[(std::size_t)j];
                const double* Mc = p.M.data() + j * n + i0;
                double cs = 0.0;
                for (long di = 0; di < h; ++di) {
                    const double t = plan_entry(x.alpha[(std::size_t)(i0 + di)], bj, Mc[di], p.eta);
                    part[(std::size_t)di] += t;
                    cs += t;
                }
                band[(std::size_t)j] = cs;
            }
            row_tree.push(part.data());
        }
        row_tree.fold(g.row.data() + i0);
        col_tree.push(band.data());
    }
    col_tree.fold(g.col.data());
    finish_gradient(g, x, p, pairwise_sum(g.row.data(), n));
    return g;
}

// dual.h:168-181  two-pass path; Eigen's rowwise/colwise/sum restated as
// sequential sums over the materialised plan
inline Grad naive_gradient(const Dual& x, const Problem& p)
{
    const vec T = plan(x, p);
    const long n = p.n, m = p.m;
    Grad g;
    g.row.assign((std::size_t)n, 0.0);
    g.col.assign((std::size_t)m, 0.0);
    double total = 0.0;
    for (long j = 0; j < m; ++j)
        for (long i = 0; i < n; ++i) {
            const double t = T[(std::size_t)(j * n + i)];
            g.row[(std::size_t)i] += t;
            g.col[(std::size_t)j] += t;
            total += t;
        }
    finish_gradient(g, x, p, total);
    return g;
}

// dual.h:219-222
inline double marginal_error(const Grad& g, const Problem& p)
{
    double r = 0.0, c = 0.0;
    for (long i = 0; i < p.n; ++i) r += std::fabs(g.row[(std::size_t)i] - p.a[(std::size_t)i]);
    for (long j = 0; j < p.m; ++j) c += std::fabs(g.col[(std::size_t)j] - p.b[(std::size_t)j]);
    return r + c;
}

// dual.h:225-229
inline double duality_gap(const Dual& x, const Grad& g, const Problem& p)
{
    double s = 0.0, t = 0.0;
    for (long i = 0; i < p.n; ++i) s += x.alpha[(std::size_t)i] * (g.row[(std::size_t)i] - p.a[(std::size_t)i]);
    for (long j = 0; j < p.m; ++j) t += x.beta[(std::size_t)j] * (g.col[(std::size_t)j] - p.b[(std::size_t)j]);
    return s + t;
}

// dual.h:191-207  dense Hessian (column-major dim x dim); oracle cap 4096
inline vec hessian_dense(const Dual& x, const Problem& p)
{
    check_dims(x, p, "hessian_dense");
    if (p.n + p.m > 4096) fail(E_ORACLE_SIZE, "hessian_dense: n + m exceeds the oracle cap 4096");
    const long n = p.n, m = p.m, dim = n + m - 1;
    const Grad g = fused_gradient(x, p);
    const vec T = plan(x, p);
    vec H((std::size_t)(dim * dim), 0.0);
    for (long i = 0; i < n; ++i) H[(std::size_t)(i * dim + i)] = g.row[(std::size_t)i] / p.eta;
    for (long j = 0; j + 1 < m; ++j) H[(std::size_t)((n + j) * dim + n + j)] = g.col[(std::size_t)j] / p.eta;
    for (long j = 0; j + 1 < m; ++j)
        for (long i = 0; i < n; ++i) {
            const double v = T[(std::size_t)(j * n + i)] / p.eta;
            H[(std::size_t)((n + j) * dim + i)] = v;
            H[(std::size_t)(i * dim + n + j)] = v;
        }
    return H;
}

// ---- Sinkhorn (sinkhorn.h) --------------------------------------------------
// sinkhorn.h:44-74  row log-sum-exp in two column-major sweeps, no clamp
inline vec optimal_alpha(const Dual& x, const Problem& p)
{
    check_dims(x, p, "optimal_alpha");
    const long n = p.n, m = p.m;
    const double eta = p.eta;
    vec top((std::size_t)n, -std::numeric_limits<double>::infinity());
    for (long j = 0; j < m; ++j) {
        const double bj = x.beta[(std::size_t)j];
        const double* Mc = p.M.data() + j * n;
        for (long i = 0; i < n; ++i) {
            const double v = (bj - Mc[i]) / eta;
            if (v > top[(std::size_t)i]) top[(std::size_t)i] = v;
        }
    }
    vec acc((std::size_t)n, 0.0);
    for (long j = 0; j < m; ++j) {
        const double bj = x.beta[(std::size_t)j];
        const double* Mc = p.M.data() + j * n;
        for (long i = 0; i < n; ++i) acc[(std::size_t)i] += std::exp((bj - Mc[i]) / eta - top[(std::size_t)i]);
    }
    vec out((std::size_t)n);
    for (long i = 0; i < n; ++i)
        out[(std::size_t)i] = eta * (std::log(p.a[(std::size_t)i]) - (top[(std::size_t)i] + std::log(acc[(std::size_t)i])));
    return out;
}

// sinkhorn.h:77-101  column log-sum-exp
inline vec optimal_beta(const vec& alpha, const Problem& p)
{
    if ((long)alpha.size() != p.n) fail(E_VALIDATION, "optimal_beta: alpha length mismatch");
    const long n = p.n, m = p.m;
    const double eta = p.eta;
    vec out((std::size_t)m);
    for (long j = 0; j < m; ++j) {
        const double* Mc = p.M.data() + j * n;
        double top = -std::numeric_limits<double>::infinity();
        for (long i = 0; i < n; ++i) {
            const double v = (alpha[(std::size_t)i] - Mc[i]) / eta;
            if (v > top) top = v;
        }
        double s = 0.0;
        for (long i = 0; i < n; ++i) s += std::exp((alpha[(std::size_t)i] - Mc[i]) / eta - top);
        out[(std::size_t)j] = eta * (std::log(p.b[(std::size_t)j]) - (top + std::log(s)));
    }
    return out;
}

// sinkhorn.h:105-115  alpha(old beta) -> beta(new alpha) -> gauge shift
inline Dual sinkhorn_step(const Dual& x, const Problem& p)
{
    Dual nx;
    nx.alpha = optimal_alpha(x, p);
    nx.beta = optimal_beta(nx.alpha, p);
    const double c = nx.beta[(std::size_t)(p.m - 1)];
    for (double& v : nx.alpha) v += c;
    for (double& v : nx.beta) v -= c;
    nx.beta[(std::size_t)(p.m - 1)] = 0.0;
    return nx;
}

struct TraceRow {
    long iter = 0;
    double wall_ms = 0.0, f = 0.0, marginal_error = 0.0, duality_gap = 0.0;
};

// trace.h:26-36 ordering invariants
inline void trace_append(std::vector<TraceRow>& rows, const TraceRow& r)
{
    if (!rows.empty()) {
        if (r.iter <= rows.back().iter) fail(E_VALIDATION, "SolverTrace: iter must be strictly increasing");
        if (r.wall_ms < rows.back().wall_ms) fail(E_VALIDATION, "SolverTrace: wall_ms must be nondecreasing");
    }
    rows.push_back(r);
}

struct SinkhornConfig {
    long max_iter = 1000;
    long record_every = 1;
    double tol = 0.0;
    // sinkhorn.h:22-30
    void validate() const
    {
        if (max_iter < 1) fail(E_VALIDATION, "SinkhornConfig: max_iter must be >= 1");
        if (record_every < 1) fail(E_VALIDATION, "SinkhornConfig: record_every must be >= 1");
        if (tol < 0.0) fail(E_VALIDATION, "SinkhornConfig: tol must be >= 0");
    }
};

struct SinkhornResult {
    Dual x;
    std::vector<TraceRow> trace;
};

struct WallClock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double ms() const
    {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
};

// sinkhorn.h:123-171
inline SinkhornResult run_sinkhorn(const Dual& x0, const Problem& p, const SinkhornConfig& cfg)
{
    cfg.validate();
    check_dims(x0, p, "run_sinkhorn");
    SinkhornResult out;
    WallClock clk;
    Dual x = x0;
    Grad g = fused_gradient(x, p);
    auto record = [&](long it) {
        trace_append(out.trace, {it, clk.ms(), g.f, marginal_error(g, p), duality_gap(x, g, p)});
    };
    record(0);
    long it = 0;
    bool fresh = true;
    while (it < cfg.max_iter) {
        if (cfg.tol > 0.0 && marginal_error(g, p) <= cfg.tol) break;
        x = sinkhorn_step(x, p);
        ++it;
        fresh = false;
        const bool rec = (it % cfg.record_every == 0) || it == cfg.max_iter;
        if (cfg.tol > 0.0 || rec) {
            g = fused_gradient(x, p);
            fresh = true;
            if (rec) record(it);
        }
    }
    if (!fresh) g = fused_gradient(x, p);
    if (out.trace.back().iter != it) record(it);
    out.x = std::move(x);
    return out;
}

// ---- sparsification (sparsity.h) --------------------------------------------
struct Pattern {
    long n = 0, mm1 = 0, k_requested = 0;
    std::vector<std::pair<int, int>> coords;  // sorted lexicographically, unique
};

// sparsity.h:44-91  top-k of T[:, :m-1] under (value desc, row-major index
// asc), united with first row and first column of the block.  T column-major.
inline Pattern select_topk(const vec& T, long n, long m, long k)
{
    if (k < 0) fail(E_VALIDATION, "select_topk: k must be >= 0");
    Pattern out;
    out.n = n;
    out.mm1 = m - 1;
    out.k_requested = k;
    const long mm1 = m - 1;
    if (mm1 <= 0) return out;
    struct Item { double v; long idx; };
    std::vector<Item> items;
    items.reserve((std::size_t)(n * mm1));
    for (long i = 0; i < n; ++i)
        for (long j = 0; j < mm1; ++j) items.push_back({T[(std::size_t)(j * n + i)], i * mm1 + j});
    auto before = [](const Item& x, const Item& y) { return x.v > y.v || (x.v == y.v && x.idx < y.idx); };
    const long total = (long)items.size();
    const long take = std::min(k, total);
    if (take > 0 && take < total) std::nth_element(items.begin(), items.begin() + take, items.end(), before);
    out.coords.reserve((std::size_t)(take + n + mm1));
    for (long t = 0; t < take; ++t)
        out.coords.emplace_back((int)(items[(std::size_t)t].idx / mm1), (int)(items[(std::size_t)t].idx % mm1));
    for (long i = 0; i < n; ++i) out.coords.emplace_back((int)i, 0);
    for (long j = 1; j < mm1; ++j) out.coords.emplace_back(0, (int)j);
    std::sort(out.coords.begin(), out.coords.end());
    out.coords.erase(std::unique(out.coords.begin(), out.coords.end()), out.coords.end());
    return out;
}

// sparsity.h:97-195  symmetric CSC, both triangles
struct SparseSym {
    int dim = 0;
    ivec colptr, rowidx;
    vec values;
    std::uint64_t pattern_id = 0;
    bool is_transport = false;
    long ot_n = 0, ot_m = 0;
    std::vector<std::pair<int, int>> coords;
    ivec slot_a, slot_b;

    // sparsity.h:112-125 column scatter
    vec matvec(const vec& v) const
    {
        if ((int)v.size() != dim) fail(E_VALIDATION, "SparseSym::matvec: length mismatch");
        vec y((std::size_t)dim, 0.0);
        for (int c = 0; c < dim; ++c) {
            const double vc = v[(std::size_t)c];
            for (int q = colptr[(std::size_t)c]; q < colptr[(std::size_t)c + 1]; ++q)
                y[(std::size_t)rowidx[(std::size_t)q]] += values[(std::size_t)q] * vc;
        }
        return y;
    }
    vec to_dense() const  // column-major dim x dim
    {
        vec D((std::size_t)dim * (std::size_t)dim, 0.0);
        for (int c = 0; c < dim; ++c)
            for (int q = colptr[(std::size_t)c]; q < colptr[(std::size_t)c + 1]; ++q)
                D[(std::size_t)c * (std::size_t)dim + (std::size_t)rowidx[(std::size_t)q]] = values[(std::size_t)q];
        return D;
    }
    // sparsity.h:160-166
    void stamp_pattern()
    {
        std::uint64_t h = fnv1a(&dim, sizeof(dim));
        if (!colptr.empty()) h = fnv1a(colptr.data(), colptr.size() * sizeof(int), h);
        if (!rowidx.empty()) h = fnv1a(rowidx.data(), rowidx.size() * sizeof(int), h);
        pattern_id = h;
    }
    // sparsity.h:170-194
    static SparseSym from_dense(const vec& A, int dim, double drop = 0.0)
    {
        SparseSym S;
        S.dim = dim;
        S.colptr.assign((std::size_t)dim + 1, 0);
        for (int c = 0; c < dim; ++c) {
            S.colptr[(std::size_t)c] = (int)S.rowidx.size();
            for (int r = 0; r < dim; ++r) {
                const double v = A[(std::size_t)c * dim + r], w = A[(std::size_t)r * dim + c];
                if (r == c || std::fabs(v) > drop || std::fabs(w) > drop) {
                    S.rowidx.push_back(r);
                    S.values.push_back(v);
                }
            }
        }
        S.colptr[(std::size_t)dim] = (int)S.rowidx.size();
        S.stamp_pattern();
        return S;
    }
};

// sparsity.h:202-220
inline void fill_transport_values(SparseSym& A, const Dual& x, const Problem& p, double tau, const Grad& g)
{
    const long n = p.n;
    for (long i = 0; i < n; ++i) A.values[(std::size_t)A.colptr[(std::size_t)i]] = g.row[(std::size_t)i] / p.eta + tau;
    for (long j = 0; j + 1 < p.m; ++j)
        A.values[(std::size_t)(A.colptr[(std::size_t)(n + j + 1)] - 1)] = g.col[(std::size_t)j] / p.eta + tau;
    for (std::size_t t = 0; t < A.coords.size(); ++t) {
        const int i = A.coords[t].first, j = A.coords[t].second;
        const double v = plan_entry(x.alpha[(std::size_t)i], x.beta[(std::size_t)j], p.cost(i, j), p.eta) / p.eta;
        A.values[(std::size_t)A.slot_a[t]] = v;
        A.values[(std::size_t)A.slot_b[t]] = v;
    }
}

// sparsity.h:226-294  alpha column i = [diag, n+j ascending]; beta column
// n+j = [i ascending, diag]
inline SparseSym assemble(const Dual& x, const Problem& p, const Pattern& om, double tau, const Grad& g)
{
    check_dims(x, p, "assemble");
    if (tau < 0.0) fail(E_VALIDATION, "assemble: tau must be >= 0");
    if (om.n != p.n || om.mm1 != p.m - 1) fail(E_VALIDATION, "assemble: pattern/problem shape mismatch");
    const long n = p.n, m = p.m;
    const int dim = (int)(n + m - 1);
    const std::size_t nz = om.coords.size();
    SparseSym A;
    A.dim = dim;
    A.is_transport = true;
    A.ot_n = n;
    A.ot_m = m;
    A.coords = om.coords;
    A.slot_a.resize(nz);
    A.slot_b.resize(nz);
    ivec cnt((std::size_t)dim, 1);
    for (const auto& c : A.coords) {
        ++cnt[(std::size_t)c.first];
        ++cnt[(std::size_t)(n + c.second)];
    }
    A.colptr.assign((std::size_t)dim + 1, 0);
    for (int c = 0; c < dim; ++c) A.colptr[(std::size_t)c + 1] = A.colptr[(std::size_t)c] + cnt[(std::size_t)c];
    A.rowidx.assign((std::size_t)A.colptr.back(), 0);
    A.values.assign((std::size_t)A.colptr.back(), 0.0);
    ivec na((std::size_t)n), nb((std::size_t)(m - 1));
    for (long i = 0; i < n; ++i) {
        A.rowidx[(std::size_t)A.colptr[(std::size_t)i]] = (int)i;
        na[(std::size_t)i] = A.colptr[(std::size_t)i] + 1;
    }
    for (long j = 0; j + 1 < m; ++j) {
        A.rowidx[(std::size_t)(A.colptr[(std::size_t)(n + j + 1)] - 1)] = (int)(n + j);
        nb[(std::size_t)j] = A.colptr[(std::size_t)(n + j)];
    }
    for (std::size_t t = 0; t < nz; ++t) {
        const int i = A.coords[t].first, j = A.coords[t].second;
        const int pa = na[(std::size_t)i]++;
        A.rowidx[(std::size_t)pa] = (int)n + j;
        A.slot_a[t] = pa;
        const int pb = nb[(std::size_t)j]++;
        A.rowidx[(std::size_t)pb] = i;
        A.slot_b[t] = pb;
    }
    A.stamp_pattern();
    fill_transport_values(A, x, p, tau, g);
    return A;
}

// sparsity.h:305-317
inline void update_values(SparseSym& A, const Dual& x, const Problem& p, double tau, const Grad& g)
{
    if (!A.is_transport) fail(E_VALIDATION, "update_values: matrix was not assembled from a problem");
    if (A.ot_n != p.n || A.ot_m != p.m) fail(E_VALIDATION, "update_values: problem shape mismatch");
    if (tau < 0.0) fail(E_VALIDATION, "update_values: tau must be >= 0");
    check_dims(x, p, "update_values");
    fill_transport_values(A, x, p, tau, g);
}

// ---- sparse Cholesky (sparse_chol.h) -- ORACLE ONLY, not built on the GPU ----
// sparse_chol.h:21-138  quotient-graph minimum degree, exact external degree,
// smallest-index tie-break via an ordered (degree, vertex) queue
inline ivec min_degree_order(int dim, const ivec& Ap, const ivec& Ai)
{
    std::vector<ivec> adj((std::size_t)dim), vel((std::size_t)dim), ebnd;
    for (int c = 0; c < dim; ++c)
        for (int q = Ap[(std::size_t)c]; q < Ap[(std::size_t)c + 1]; ++q)
            if (Ai[(std::size_t)q] != c) adj[(std::size_t)c].push_back(Ai[(std::size_t)q]);
    std::vector<char> edead, gone((std::size_t)dim, 0);
    ivec deg((std::size_t)dim), mark((std::size_t)dim, -1), perm, bnd;
    int stamp = 0;
    std::set<std::pair<int, int>> q;
    for (int v = 0; v < dim; ++v) {
        deg[(std::size_t)v] = (int)adj[(std::size_t)v].size();
        q.insert({deg[(std::size_t)v], v});
    }
    perm.reserve((std::size_t)dim);
    while (!q.empty()) {
        const int pv = q.begin()->second;
        q.erase(q.begin());
        gone[(std::size_t)pv] = 1;
        perm.push_back(pv);
        const int s0 = ++stamp;
        mark[(std::size_t)pv] = s0;
        bnd.clear();
        auto reach = [&](int v) {
            if (!gone[(std::size_t)v] && mark[(std::size_t)v] != s0) {
                mark[(std::size_t)v] = s0;
                bnd.push_back(v);
            }
        };
        for (int v : adj[(std::size_t)pv]) reach(v);
        for (int e : vel[(std::size_t)pv]) {
            if (edead[(std::size_t)e]) continue;
            for (int v : ebnd[(std::size_t)e]) reach(v);
            edead[(std::size_t)e] = 1;
        }
        if (bnd.empty()) continue;
        std::sort(bnd.begin(), bnd.end());
        const int enew = (int)ebnd.size();
        ebnd.push_back(bnd);
        edead.push_back(0);
        for (int v : bnd) {
            ivec& ev = adj[(std::size_t)v];
            ev.erase(std::remove_if(ev.begin(), ev.end(),
                                    [&](int u) { return gone[(std::size_t)u] || mark[(std::size_t)u] == s0; }),
                     ev.end());
            ivec& el = vel[(std::size_t)v];
            el.erase(std::remove_if(el.begin(), el.end(), [&](int e) { return edead[(std::size_t)e] != 0; }), el.end());
            el.push_back(enew);
        }
        for (int v : bnd) {
            const int sv = ++stamp;
            mark[(std::size_t)v] = sv;
            int d = 0;
            auto count = [&](int u) {
                if (!gone[(std::size_t)u] && mark[(std::size_t)u] != sv) {
                    mark[(std::size_t)u] = sv;
                    ++d;
                }
            };
            for (int u : adj[(std::size_t)v]) count(u);
            for (int e : vel[(std::size_t)v])
                for (int u : ebnd[(std::size_t)e]) count(u);
            q.erase({deg[(std::size_t)v], v});
            deg[(std::size_t)v] = d;
            q.insert({d, v});
        }
    }
    return perm;
}

struct Symbolic {
    int dim = 0;
    ivec perm, iperm, etree, Lp, Li, Cp, Ci, Cmap, rp_ptr, rp_idx;
    std::uint64_t source_pattern_id = 0;
    long nnz_L() const { return Lp.empty() ? 0 : (long)Lp.back(); }
};
struct Numeric {
    std::shared_ptr<const Symbolic> sym;
    vec L;
};

// sparse_chol.h:175-325
inline Symbolic symbolic_analyze(const SparseSym& A)
{
    const int dim = A.dim;
    if (dim < 1) fail(E_STRUCTURE, "symbolic_analyze: empty matrix");
    for (int c = 0; c < dim; ++c) {
        bool diag = false;
        for (int q = A.colptr[(std::size_t)c]; q < A.colptr[(std::size_t)c + 1]; ++q) {
            const int r = A.rowidx[(std::size_t)q];
            if (r < 0 || r >= dim) fail(E_STRUCTURE, "symbolic_analyze: row index out of range");
            if (q > A.colptr[(std::size_t)c] && r <= A.rowidx[(std::size_t)q - 1])
                fail(E_STRUCTURE, "symbolic_analyze: column rows not strictly ascending");
            diag |= (r == c);
        }
        if (!diag) fail(E_STRUCTURE, "symbolic_analyze: missing diagonal entry");
    }
    {   // structural symmetry: the transpose must reproduce the arrays
        ivec tp((std::size_t)dim + 1, 0), ti(A.rowidx.size());
        for (int r : A.rowidx) ++tp[(std::size_t)r + 1];
        for (int c = 0; c < dim; ++c) tp[(std::size_t)c + 1] += tp[(std::size_t)c];
        ivec nx(tp.begin(), tp.end() - 1);
        for (int c = 0; c < dim; ++c)
            for (int q = A.colptr[(std::size_t)c]; q < A.colptr[(std::size_t)c + 1]; ++q)
                ti[(std::size_t)nx[(std::size_t)A.rowidx[(std::size_t)q]]++] = c;
        if (tp != A.colptr || ti != A.rowidx)
            fail(E_STRUCTURE, "symbolic_analyze: pattern is not structurally symmetric");
    }
    Symbolic S;
    S.dim = dim;
    S.source_pattern_id = A.pattern_id;
    S.perm = min_degree_order(dim, A.colptr, A.rowidx);
    S.iperm.assign((std::size_t)dim, 0);
    for (int k = 0; k < dim; ++k) S.iperm[(std::size_t)S.perm[(std::size_t)k]] = k;

    S.Cp.assign((std::size_t)dim + 1, 0);
    std::vector<std::pair<int, int>> buf;
    for (int k = 0; k < dim; ++k) {
        const int oc = S.perm[(std::size_t)k];
        buf.clear();
        for (int q = A.colptr[(std::size_t)oc]; q < A.colptr[(std::size_t)oc + 1]; ++q) {
            const int rn = S.iperm[(std::size_t)A.rowidx[(std::size_t)q]];
            if (rn <= k) buf.emplace_back(rn, q);
        }
        std::sort(buf.begin(), buf.end());
        for (const auto& e : buf) {
            S.Ci.push_back(e.first);
            S.Cmap.push_back(e.second);
        }
        S.Cp[(std::size_t)k + 1] = (int)S.Ci.size();
    }
    S.etree.assign((std::size_t)dim, -1);
    {
        ivec anc((std::size_t)dim, -1);
        for (int k = 0; k < dim; ++k)
            for (int q = S.Cp[(std::size_t)k]; q < S.Cp[(std::size_t)k + 1]; ++q) {
                int i = S.Ci[(std::size_t)q];
                while (i != -1 && i < k) {
                    const int nxt = anc[(std::size_t)i];
                    anc[(std::size_t)i] = k;
                    if (nxt == -1) S.etree[(std::size_t)i] = k;
                    i = nxt;
                }
            }
    }
    S.rp_ptr.assign((std::size_t)dim + 1, 0);
    ivec w((std::size_t)dim, -1), sb((std::size_t)dim), stk((std::size_t)dim), cnt((std::size_t)dim, 1);
    for (int k = 0; k < dim; ++k) {
        int top = dim;
        w[(std::size_t)k] = k;
        for (int q = S.Cp[(std::size_t)k]; q < S.Cp[(std::size_t)k + 1]; ++q) {
            int i = S.Ci[(std::size_t)q];
            if (i >= k) continue;
            int len = 0;
            while (i != -1 && w[(std::size_t)i] != k) {
                sb[(std::size_t)len++] = i;
                w[(std::size_t)i] = k;
                i = S.etree[(std::size_t)i];
            }
            while (len > 0) stk[(std::size_t)--top] = sb[(std::size_t)--len];
        }
        for (int t = top; t < dim; ++t) {
            S.rp_idx.push_back(stk[(std::size_t)t]);
            ++cnt[(std::size_t)stk[(std::size_t)t]];
        }
        S.rp_ptr[(std::size_t)k + 1] = (int)S.rp_idx.size();
    }
    S.Lp.assign((std::size_t)dim + 1, 0);
    for (int c = 0; c < dim; ++c) S.Lp[(std::size_t)c + 1] = S.Lp[(std::size_t)c] + cnt[(std::size_t)c];
    S.Li.assign((std::size_t)S.Lp.back(), 0);
    {
        ivec nx(S.Lp.begin(), S.Lp.end() - 1);
        for (int k = 0; k < dim; ++k) {
            S.Li[(std::size_t)nx[(std::size_t)k]++] = k;
            for (int t = S.rp_ptr[(std::size_t)k]; t < S.rp_ptr[(std::size_t)k + 1]; ++t)
                S.Li[(std::size_t)nx[(std::size_t)S.rp_idx[(std::size_t)t]]++] = k;
        }
    }
    return S;
}

// sparse_chol.h:330-390 up-looking LL', pivot tolerance 1e-13 * max diagonal
inline Numeric numeric_factorize(const std::shared_ptr<const Symbolic>& sym, const SparseSym& A)
{
    if (!sym) fail(E_VALIDATION, "numeric_factorize: null symbolic factor");
    const Symbolic& S = *sym;
    if (S.dim != A.dim || S.source_pattern_id != A.pattern_id)
        fail(E_VALIDATION, "numeric_factorize: matrix pattern does not match the symbolic factor");
    const int dim = S.dim;
    vec Cx(S.Cmap.size());
    for (std::size_t q = 0; q < S.Cmap.size(); ++q) Cx[q] = A.values[(std::size_t)S.Cmap[q]];
    double maxdiag = 0.0;
    for (int k = 0; k < dim; ++k) maxdiag = std::max(maxdiag, Cx[(std::size_t)(S.Cp[(std::size_t)k + 1] - 1)]);
    const double ptol = 1e-13 * maxdiag;
    Numeric F;
    F.sym = sym;
    F.L.assign((std::size_t)S.Lp.back(), 0.0);
    vec& L = F.L;
    vec x((std::size_t)dim, 0.0);
    ivec c(S.Lp.begin(), S.Lp.end() - 1);
    for (int k = 0; k < dim; ++k) {
        for (int q = S.Cp[(std::size_t)k]; q < S.Cp[(std::size_t)k + 1]; ++q) x[(std::size_t)S.Ci[(std::size_t)q]] = Cx[(std::size_t)q];
        double d = x[(std::size_t)k];
        x[(std::size_t)k] = 0.0;
        for (int t = S.rp_ptr[(std::size_t)k]; t < S.rp_ptr[(std::size_t)k + 1]; ++t) {
            const int j = S.rp_idx[(std::size_t)t];
            const double lkj = x[(std::size_t)j] / L[(std::size_t)S.Lp[(std::size_t)j]];
            x[(std::size_t)j] = 0.0;
            for (int q = S.Lp[(std::size_t)j] + 1; q < c[(std::size_t)j]; ++q)
                x[(std::size_t)S.Li[(std::size_t)q]] -= L[(std::size_t)q] * lkj;
            d -= lkj * lkj;
            L[(std::size_t)c[(std::size_t)j]++] = lkj;
        }
        if (d <= ptol)
            fail(E_NOT_POSITIVE_DEFINITE, "numeric_factorize: nonpositive pivot at column " + std::to_string(k));
        L[(std::size_t)c[(std::size_t)k]++] = std::sqrt(d);
    }
    return F;
}

// sparse_chol.h:393-427
inline vec chol_solve(const Numeric& F, const vec& rhs)
{
    if (!F.sym) fail(E_VALIDATION, "solve: empty factor");
    const Symbolic& S = *F.sym;
    if ((int)rhs.size() != S.dim) fail(E_VALIDATION, "solve: rhs length mismatch");
    const int dim = S.dim;
    const vec& L = F.L;
    vec w((std::size_t)dim);
    for (int k = 0; k < dim; ++k) w[(std::size_t)k] = rhs[(std::size_t)S.perm[(std::size_t)k]];
    for (int j = 0; j < dim; ++j) {
        w[(std::size_t)j] /= L[(std::size_t)S.Lp[(std::size_t)j]];
        for (int q = S.Lp[(std::size_t)j] + 1; q < S.Lp[(std::size_t)j + 1]; ++q)
            w[(std::size_t)S.Li[(std::size_t)q]] -= L[(std::size_t)q] * w[(std::size_t)j];
    }
    for (int j = dim - 1; j >= 0; --j) {
        double s = w[(std::size_t)j];
        for (int q = S.Lp[(std::size_t)j] + 1; q < S.Lp[(std::size_t)j + 1]; ++q)
            s -= L[(std::size_t)q] * w[(std::size_t)S.Li[(std::size_t)q]];
        w[(std::size_t)j] = s / L[(std::size_t)S.Lp[(std::size_t)j]];
    }
    vec out((std::size_t)dim);
    for (int k = 0; k < dim; ++k) out[(std::size_t)S.perm[(std::size_t)k]] = w[(std::size_t)k];
    return out;
}

// Jacobi-preconditioned CG on A x = rhs.  NOT in the reference: this is the
// CPU model of the device solver (north_star item 3) used for design studies
// and as the checker of the device PCG kernel.  Returns iterations used.
inline int pcg_solve(const SparseSym& A, const vec& rhs, vec& x, double rtol, int max_it)
{
    const int dim = A.dim;
    vec dinv((std::size_t)dim);
    for (int c = 0; c < dim; ++c)
        for (int q = A.colptr[(std::size_t)c]; q < A.colptr[(std::size_t)c + 1]; ++q)
            if (A.rowidx[(std::size_t)q] == c) dinv[(std::size_t)c] = 1.0 / A.values[(std::size_t)q];
    x.assign((std::size_t)dim, 0.0);
    vec r = rhs, z((std::size_t)dim), pd((std::size_t)dim);
    for (int i = 0; i < dim; ++i) z[(std::size_t)i] = r[(std::size_t)i] * dinv[(std::size_t)i];
    pd = z;
    double rz = dot(r, z);
    const double stop = rtol * rtol * rz;
    int it = 0;
    if (rz == 0.0) return 0;
    for (; it < max_it; ++it) {
        const vec Ap = A.matvec(pd);
        const double pAp = dot(pd, Ap);
        if (!(pAp > 0.0)) return -1 - it;  // breakdown: not positive definite
        const double al = rz / pAp;
        for (int i = 0; i < dim; ++i) {
            x[(std::size_t)i] += al * pd[(std::size_t)i];
            r[(std::size_t)i] -= al * Ap[(std::size_t)i];
            z[(std::size_t)i] = r[(std::size_t)i] * dinv[(std::size_t)i];
        }
        const double rz2 = dot(r, z);
        if (rz2 <= stop) { ++it; break; }
        const double be = rz2 / rz;
        rz = rz2;
        for (int i = 0; i < dim; ++i) pd[(std::size_t)i] = z[(std::size_t)i] + be * pd[(std::size_t)i];
    }
    return it;
}

// ---- SPLR (splr.h) ----------------------------------------------------------
struct SplrConfig {
    double tau_max = 1.0;
    long S = 10, J = 5;
    double density = 0.01, c1 = 1e-4, c2 = 0.9;
    long max_iter = 1000;
    double tol = 1e-8;
    long max_ls_trials = 30, record_every = 1;
    bool overlap = false;
    int tile_rows = 8, tile_cols = 32;
    // oracle-only switch (not in the reference): 0 = sparse Cholesky as in the
    // reference, 1 = Jacobi-PCG model of the device direction solver
    int direction_solver = 0;
    double cg_rtol = 1e-12;
    int cg_max_iter = 20000;
    // splr.h:37-59
    void validate() const
    {
        if (!(c1 > 0.0 && c1 < 0.5)) fail(E_VALIDATION, "SplrConfig: need 0 < c1 < 1/2");
        if (!(c2 > c1 && c2 < 1.0)) fail(E_VALIDATION, "SplrConfig: need c1 < c2 < 1");
        if (S < 1) fail(E_VALIDATION, "SplrConfig: need S >= 1");
        if (J < 0) fail(E_VALIDATION, "SplrConfig: need J >= 0");
        if (!(tau_max > 0.0)) fail(E_VALIDATION, "SplrConfig: need tau_max > 0");
        if (!(density > 0.0 && density <= 1.0)) fail(E_VALIDATION, "SplrConfig: need 0 < density <= 1");
        if (max_iter < 1) fail(E_VALIDATION, "SplrConfig: need max_iter >= 1");
        if (tol < 0.0) fail(E_VALIDATION, "SplrConfig: need tol >= 0");
        if (max_ls_trials < 1) fail(E_VALIDATION, "SplrConfig: need max_ls_trials >= 1");
        if (record_every < 1) fail(E_VALIDATION, "SplrConfig: need record_every >= 1");
    }
};

struct LowRank {
    bool active = false;
    vec u, v;
    double xi = 0.0, zeta = 0.0;
};

struct SplrState {
    Dual x_prev, x;
    vec g_prev;
    Grad cur;
    bool has_prev = false;
    Pattern omega;
    SparseSym A;
    std::shared_ptr<const Symbolic> symbolic;
    long iter = 0;
    long cg_iters_total = 0;
};

// splr.h:102-122
inline LowRank build_low_rank(const SplrState& st, const SparseSym& A)
{
    LowRank R;
    if (!st.has_prev) return R;
    const vec xf = st.x.to_free(), xp = st.x_prev.to_free();
    const std::size_t dim = xf.size();
    vec s(dim), y(dim);
    for (std::size_t i = 0; i < dim; ++i) {
        s[i] = xf[i] - xp[i];
        y[i] = st.cur.grad[i] - st.g_prev[i];
    }
    const double ys = dot(y, s);
    if (!(ys > 1e-6 * sqnorm(y))) return R;
    vec v = A.matvec(s);
    const double vs = dot(v, s);
    if (std::fabs(vs) <= 1e-12 * norm2(v) * norm2(s)) return R;
    R.active = true;
    R.u = y;
    R.v = std::move(v);
    R.xi = 1.0 / ys;
    R.zeta = -1.0 / vs;
    return R;
}

// splr.h:128-167, written against an abstract "apply A^{-1}" so the same body
// serves the Cholesky route (reference) and the PCG model.
template <class Solve>
vec compute_direction_with(Solve&& inv, const LowRank& R, const vec& g)
{
    const std::size_t dim = g.size();
    if (norm_inf(g) == 0.0) return vec(dim, 0.0);
    const vec ag = inv(g);
    vec d(dim);
    bool woodbury = false;
    if (R.active) {
        const vec au = inv(R.u), av = inv(R.v);
        const double k11 = 1.0 / R.xi + dot(R.u, au);
        const double k12 = dot(R.u, av);
        const double k22 = 1.0 / R.zeta + dot(R.v, av);
        const double det = k11 * k22 - k12 * k12;
        const double sc = std::max({std::fabs(k11), std::fabs(k12), std::fabs(k22)});
        if (std::fabs(det) > 1e-14 * sc * sc && sc > 0.0) {
            const double t1 = dot(R.u, ag), t2 = dot(R.v, ag);
            const double z1 = (k22 * t1 - k12 * t2) / det;
            const double z2 = (-k12 * t1 + k11 * t2) / det;
            for (std::size_t i = 0; i < dim; ++i) d[i] = -(ag[i] - au[i] * z1 - av[i] * z2);
            woodbury = true;
        }
    }
    if (!woodbury)
        for (std::size_t i = 0; i < dim; ++i) d[i] = -ag[i];
    if (dot(g, d) < 0.0) return d;
    if (woodbury) {
        for (std::size_t i = 0; i < dim; ++i) d[i] = -ag[i];
        if (dot(g, d) < 0.0) return d;
    }
    fail(E_DIRECTION, "compute_direction: no descent direction");
}

inline vec compute_direction(const Numeric& F, const LowRank& R, const vec& g)
{
    return compute_direction_with([&](const vec& r) { return chol_solve(F, r); }, R, g);
}

struct LineSearchResult {
    double gamma = 0.0;
    vec x_new;
    Grad gr_new;
    double g0_dot_d = 0.0, gnew_dot_d = 0.0;
    bool curvature_ok = false;
    int evals = 0;
};

// splr.h:185-290  bracket by doubling from gamma = 1, then bisection zoom
template <class Oracle>
LineSearchResult line_search(Oracle&& oracle, const vec& x0, const vec& d, double f0, const vec& g0,
                             const SplrConfig& cfg)
{
    const double dphi0 = dot(g0, d);
    if (!(dphi0 < 0.0)) fail(E_VALIDATION, "line_search: g'd must be negative");
    const double c1 = cfg.c1, c2 = cfg.c2;
    struct Trial {
        double gamma, f, dphi;
        vec x;
        Grad gr;
    };
    LineSearchResult best;
    bool have_best = false;
    int evals = 0;
    auto probe = [&](double gamma) {
        Trial e;
        e.gamma = gamma;
        e.x.resize(x0.size());
        for (std::size_t i = 0; i < x0.size(); ++i) e.x[i] = x0[i] + gamma * d[i];
        e.gr = oracle(e.x);
        e.f = e.gr.f;
        e.dphi = dot(e.gr.grad, d);
        ++evals;
        return e;
    };
    auto armijo = [&](const Trial& e) { return std::isfinite(e.f) && e.f <= f0 + c1 * e.gamma * dphi0; };
    auto remember = [&](Trial& e) {
        if (!have_best || e.f < best.gr_new.f) {
            best.gamma = e.gamma;
            best.x_new = std::move(e.x);
            best.gr_new = std::move(e.gr);
            best.g0_dot_d = dphi0;
            best.gnew_dot_d = e.dphi;
            best.curvature_ok = false;
            have_best = true;
        }
    };
    auto accept = [&](Trial& e) {
        LineSearchResult r;
        r.gamma = e.gamma;
        r.x_new = std::move(e.x);
        r.gr_new = std::move(e.gr);
        r.g0_dot_d = dphi0;
        r.gnew_dot_d = e.dphi;
        r.curvature_ok = true;
        r.evals = evals;
        return r;
    };
    auto fallback = [&]() {
        if (!have_best)
            fail(E_LINE_SEARCH, "line_search: no sufficient-decrease point in " + std::to_string(evals) + " trials");
        best.evals = evals;
        return best;
    };
    auto zoom = [&](double lo, double f_lo, double hi) {
        while (evals < cfg.max_ls_trials) {
            const double mid = 0.5 * (lo + hi);
            if (mid == lo || mid == hi) break;
            Trial e = probe(mid);
            if (!armijo(e) || e.f >= f_lo) {
                hi = mid;
                continue;
            }
            const double dphi = e.dphi;
            if (dphi >= c2 * dphi0) return accept(e);
            remember(e);
            if (dphi * (hi - lo) >= 0.0) hi = lo;
            lo = mid;
            f_lo = e.f;
        }
        return fallback();
    };
    double g_prev = 0.0, f_prev = f0, gamma = 1.0;
    while (evals < cfg.max_ls_trials) {
        Trial e = probe(gamma);
        if (!armijo(e) || (g_prev > 0.0 && e.f >= f_prev)) return zoom(g_prev, f_prev, gamma);
        const double dphi = e.dphi;
        if (dphi >= c2 * dphi0) return accept(e);
        remember(e);
        g_prev = gamma;
        f_prev = e.f;
        gamma *= 2.0;
    }
    return fallback();
}

struct StepRecord {
    long iter = 0;
    bool refresh = false, sinkhorn_selected = false;
    double f_before = 0.0, f_after = 0.0;
    double f_cand_sinkhorn = std::numeric_limits<double>::quiet_NaN();
    double f_cand_qn = 0.0, gamma = 0.0, g_dot_d = 0.0, gnew_dot_d = 0.0;
    bool curvature_ok = false, ls_failed = false, lowrank_active = false;
    double tau = 0.0;
    int factor_retries = 0, ls_evals = 0;
    int cg_iters = 0;  // oracle extension: PCG iterations when direction_solver == 1
};

// splr.h:326-334
inline SplrState splr_init(const Dual& x0, const Problem& p, const SplrConfig& cfg)
{
    check_dims(x0, p, "splr_init");
    SplrState st;
    st.x = x0;
    st.cur = fused_gradient(x0, p, cfg.tile_rows, cfg.tile_cols);
    return st;
}

// splr.h:336-340
inline long topk_budget(const Problem& p, double density)
{
    return (long)std::ceil(density * ((double)p.n * (double)(p.m - 1)));
}

// splr.h:348-478.  cfg.overlap only changes scheduling in the reference (the
// result is bitwise identical, test_splr.cpp:270-305), so the oracle always
// runs the serial order.
inline SplrState splr_step(SplrState st, const Problem& p, const SplrConfig& cfg, StepRecord* rec = nullptr)
{
    const long k = st.iter;
    const bool refresh = (k % cfg.S == 0);
    double tau = std::min(cfg.tau_max, norm2(st.cur.grad));
    Dual x_s;
    Grad gr_s;
    bool have_s = false;
    const bool use_chol = (cfg.direction_solver == 0);

    if (refresh) {
        const vec T = plan(st.x, p);
        Pattern om = select_topk(T, p.n, p.m, topk_budget(p, cfg.density));
        st.A = assemble(st.x, p, om, tau, st.cur);
        st.omega = std::move(om);
        if (use_chol) st.symbolic = std::make_shared<const Symbolic>(symbolic_analyze(st.A));
        if (cfg.J > 0) {
            x_s = st.x;
            for (long j = 0; j < cfg.J; ++j) x_s = sinkhorn_step(x_s, p);
            gr_s = fused_gradient(x_s, p, cfg.tile_rows, cfg.tile_cols);
            have_s = true;
        }
    } else {
        update_values(st.A, st.x, p, tau, st.cur);
    }

    Numeric F;
    int retries = 0;
    vec d;
    int cg_used = 0;
    if (use_chol) {
        for (;;) {
            try {
                F = numeric_factorize(st.symbolic, st.A);
                break;
            } catch (const Failure& e) {
                if (e.code != E_NOT_POSITIVE_DEFINITE || retries >= 8) throw;
                tau = (tau > 0.0) ? 2.0 * tau : 1e-8;
                update_values(st.A, st.x, p, tau, st.cur);
                ++retries;
            }
        }
        const LowRank R = build_low_rank(st, st.A);
        d = compute_direction(F, R, st.cur.grad);
        if (rec) rec->lowrank_active = R.active;
    } else {
        // device-solver model: CG breakdown (p'Ap <= 0) plays the role of the
        // non-positive pivot and triggers the same tau escalation
        for (;;) {
            bool broke = false;
            const LowRank R = build_low_rank(st, st.A);
            try {
                d = compute_direction_with(
                    [&](const vec& r) {
                        vec sol;
                        const int it = pcg_solve(st.A, r, sol, cfg.cg_rtol, cfg.cg_max_iter);
                        if (it < 0) { broke = true; throw Failure(E_NOT_POSITIVE_DEFINITE, "pcg breakdown"); }
                        cg_used += it;
                        return sol;
                    },
                    R, st.cur.grad);
                if (rec) rec->lowrank_active = R.active;
                break;
            } catch (const Failure& e) {
                if (!broke || retries >= 8) throw;
                tau = (tau > 0.0) ? 2.0 * tau : 1e-8;
                update_values(st.A, st.x, p, tau, st.cur);
                ++retries;
            }
        }
        st.cg_iters_total += cg_used;
    }

    const long n = p.n, m = p.m;
    auto oracle = [&](const vec& xf) {
        return fused_gradient(Dual::from_free(xf, n, m), p, cfg.tile_rows, cfg.tile_cols);
    };
    LineSearchResult ls;
    bool ls_failed = false;
    try {
        ls = line_search(oracle, st.x.to_free(), d, st.cur.f, st.cur.grad, cfg);
    } catch (const Failure& e) {
        if (e.code != E_LINE_SEARCH) throw;
        ls_failed = true;
        ls.gamma = 0.0;
        ls.x_new = st.x.to_free();
        ls.gr_new = st.cur;
        ls.g0_dot_d = dot(st.cur.grad, d);
        ls.gnew_dot_d = ls.g0_dot_d;
        ls.curvature_ok = false;
        ls.evals = (int)cfg.max_ls_trials;
    }
    const bool pick_s = have_s && std::isfinite(gr_s.f) && (ls_failed || gr_s.f <= ls.gr_new.f);
    if (rec) {
        rec->iter = k;
        rec->refresh = refresh;
        rec->sinkhorn_selected = pick_s;
        rec->f_before = st.cur.f;
        rec->f_cand_qn = ls.gr_new.f;
        rec->f_cand_sinkhorn = have_s ? gr_s.f : std::numeric_limits<double>::quiet_NaN();
        rec->gamma = ls.gamma;
        rec->g_dot_d = ls.g0_dot_d;
        rec->gnew_dot_d = ls.gnew_dot_d;
        rec->curvature_ok = ls.curvature_ok;
        rec->ls_failed = ls_failed;
        rec->tau = tau;
        rec->factor_retries = retries;
        rec->ls_evals = ls.evals;
        rec->cg_iters = cg_used;
    }
    st.x_prev = std::move(st.x);
    st.g_prev = std::move(st.cur.grad);
    st.has_prev = true;
    if (pick_s) {
        st.x = std::move(x_s);
        st.cur = std::move(gr_s);
    } else {
        st.x = Dual::from_free(ls.x_new, n, m);
        st.cur = std::move(ls.gr_new);
    }
    if (rec) rec->f_after = st.cur.f;
    st.iter = k + 1;
    return st;
}

struct SplrResult {
    Dual x;
    std::vector<TraceRow> trace;
    std::vector<StepRecord> steps;
    int status = OK;       // E_STEP when a step failed (trace holds rows so far)
    std::string message;   // "run_splr: step <iter> failed: <what>"
};

// splr.h:487-534.  A failing step does not throw here: the partial trace is
// returned with status E_STEP, which is how the C ABI reports StepError.
inline SplrResult run_splr(const Dual& x0, const Problem& p, const SplrConfig& cfg)
{
    cfg.validate();
    check_dims(x0, p, "run_splr");
    SplrResult out;
    WallClock clk;
    SplrState st = splr_init(x0, p, cfg);
    auto record = [&]() {
        trace_append(out.trace, {st.iter, clk.ms(), st.cur.f, marginal_error(st.cur, p), duality_gap(st.x, st.cur, p)});
    };
    record();
    while (st.iter < cfg.max_iter) {
        if (marginal_error(st.cur, p) <= cfg.tol) break;
        StepRecord rec;
        const long at = st.iter;
        try {
            st = splr_step(std::move(st), p, cfg, &rec);
        } catch (const Failure& e) {
            out.status = E_STEP;
            out.message = "run_splr: step " + std::to_string(at) + " failed: " + e.what();
            return out;
        }
        out.steps.push_back(rec);
        if (st.iter % cfg.record_every == 0 || st.iter == cfg.max_iter) record();
    }
    if (out.trace.back().iter != st.iter) record();
    out.x = std::move(st.x);
    return out;
}

// ---- new workload generators (NOT in the reference) -----------
// These define BASELINE.json configs B, D, E.  They are restated bit-for-bit by
// the product's host side (paper_2605_08793_b200/csrc/generators.cpp) and the
// two are compared in tests.

// config B: 100x100-style image histograms on the unit square grid.
// side*side pixels at (r/(side-1), c/(side-1)); cost = squared distance / 2
// (so the maximum is exactly 1 and normalisation is the identity up to
// rounding); marginals = 3 isotropic Gaussian blobs + floor 1e-6.
inline void blob_histogram(vec& h, long side, std::uint64_t seed)
{
    Rng rng(seed);
    double cx[3], cy[3], sg[3], wt[3];
    for (int b = 0; b < 3; ++b) {
        cx[b] = 0.15 + 0.7 * rng.uniform();
        cy[b] = 0.15 + 0.7 * rng.uniform();
        sg[b] = 0.05 + 0.10 * rng.uniform();
        wt[b] = 0.5 + rng.uniform();
    }
    h.assign((std::size_t)(side * side), 0.0);
    double tot = 0.0;
    for (long r = 0; r < side; ++r)
        for (long c = 0; c < side; ++c) {
            const double y = (double)r / (double)(side - 1), x = (double)c / (double)(side - 1);
            double v = 1e-6;
            for (int b = 0; b < 3; ++b) {
                const double dx = x - cx[b], dy = y - cy[b];
                v += wt[b] * std::exp(-(dx * dx + dy * dy) / (2.0 * sg[b] * sg[b]));
            }
            h[(std::size_t)(r * side + c)] = v;
            tot += v;
        }
    for (double& v : h) v /= tot;
}

inline Problem gen_image(long side, double eta, std::uint64_t seed_a = 11, std::uint64_t seed_b = 12)
{
    if (side < 2) fail(E_VALIDATION, "gen_image: need side >= 2");
    Problem p;
    p.n = p.m = side * side;
    p.eta = eta;
    blob_histogram(p.a, side, seed_a);
    blob_histogram(p.b, side, seed_b);
    p.M.resize((std::size_t)(p.n * p.m));
    const double s = 1.0 / (double)(side - 1);
    for (long j = 0; j < p.m; ++j) {
        const double yj = (double)(j / side) * s, xj = (double)(j % side) * s;
        for (long i = 0; i < p.n; ++i) {
            const double yi = (double)(i / side) * s, xi = (double)(i % side) * s;
            const double dx = xi - xj, dy = yi - yj;
            p.M[(std::size_t)(j * p.n + i)] = 0.5 * (dx * dx + dy * dy);
        }
    }
    normalize_cost(p.M);
    validate_problem(p);
    return p;
}

// config D: Gaussian-mixture clouds in R^d (3 source, 4 target components,
// means 2*N(0,1), sigma alternating 0.5 / 1.0, equal weights).
inline void gmm_points(vec& X, long n, long d, int comps, Rng& rng)
{
    vec mu((std::size_t)(comps * d));
    for (auto& v : mu) v = 2.0 * rng.normal();
    X.resize((std::size_t)(n * d));
    for (long i = 0; i < n; ++i) {
        const int c = (int)(rng.uniform() * comps) % comps;
        const double sg = (c % 2 == 0) ? 0.5 : 1.0;
        for (long k = 0; k < d; ++k) X[(std::size_t)(i * d + k)] = mu[(std::size_t)(c * d + k)] + sg * rng.normal();
    }
}
inline void gen_gmm_points(vec& X, vec& Y, long n, long m, long d, std::uint64_t seed)
{
    Rng rng(seed);
    gmm_points(X, n, d, 3, rng);
    gmm_points(Y, m, d, 4, rng);
}
// config E: uniform clouds in [0,1)^d
inline void gen_uniform_points(vec& X, vec& Y, long n, long m, long d, std::uint64_t seed)
{
    Rng rng(seed);
    X.resize((std::size_t)(n * d));
    Y.resize((std::size_t)(m * d));
    for (auto& v : X) v = rng.uniform();
    for (auto& v : Y) v = rng.uniform();
}
inline Problem problem_from_points(const vec& X, const vec& Y, long n, long m, long d, double eta)
{
    Problem p;
    p.n = n; p.m = m; p.eta = eta;
    sqeuclid_cost(p, X, Y, d);
    normalize_cost(p.M);
    uniform_marginals(p);
    validate_problem(p);
    return p;
}

}  // namespace rgo
