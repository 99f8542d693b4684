// selfcheck.cpp -- pins the CPU oracle against the reference's own known-answer
// tests (TEST INFRASTRUCTURE ONLY).  Each check names the reference test it
// replays (paths relative to /root/reference/proj/tests/).  Exit code 0 iff all
// pass; one PASS/FAIL line per check, like the reference's acceptance runner.
#include "regot_oracle.hpp"

#include <cstdio>
#include <functional>
#include <tuple>

using namespace rgo;

static int g_fail = 0;
static void check(bool ok, const char* what)
{
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++g_fail;
}
static bool close_rel(double x, double y, double eps) { return std::fabs(x - y) <= eps * std::max(std::fabs(x), std::fabs(y)); }

static Problem tiny(long n, long m, double eta)
{
    Problem p;
    p.n = n; p.m = m; p.eta = eta;
    p.M.assign((std::size_t)(n * m), 0.0);
    uniform_marginals(p);
    return p;
}

int main()
{
    // test_dual.cpp:28-33
    {
        const vec T = plan(Dual::zeros(3, 4), tiny(3, 4, 1.0));
        bool ok = true;
        for (double t : T) ok &= (t == 1.0);
        check(ok, "plan is all ones at the origin (test_dual.cpp:28-33)");
    }
    // test_dual.cpp:44-53 clamp
    {
        Problem p = tiny(1, 2, 1e-4);
        Dual x = Dual::zeros(1, 2);
        x.alpha[0] = 1.0;
        const bool hi = plan(x, p)[0] == std::exp(700.0);
        x.alpha[0] = -1.0;
        const bool lo = plan(x, p)[0] == std::exp(-700.0);
        check(hi && lo, "plan clamps extreme exponents to exp(+-700) (test_dual.cpp:44-53)");
    }
    // test_dual.cpp:55-59
    check(close_rel(fused_gradient(Dual::zeros(1, 1), tiny(1, 1, 1.0)).f, 1.0, 1e-15),
          "objective at the scalar origin equals one (test_dual.cpp:55-59)");
    // test_dual.cpp:72-85
    {
        const Grad g = fused_gradient(Dual::zeros(2, 2), tiny(2, 2, 1.0));
        check(g.row[0] == 2.0 && g.row[1] == 2.0 && g.col[0] == 2.0 && g.col[1] == 2.0 && g.grad.size() == 3 &&
                  g.grad[0] == 1.5 && g.grad[1] == 1.5 && g.grad[2] == 1.5 && g.f == 4.0,
              "2x2 hand case: sums 2, grad 1.5, f 4.0 exactly (test_dual.cpp:72-85)");
    }
    // test_dual.cpp:87-119 fused vs naive, tile invariance
    {
        const long sizes[][2] = {{5, 7}, {17, 33}, {64, 64}, {33, 128}, {257, 19}};
        bool ok = true;
        int seed = 0;
        for (const auto& sz : sizes) {
            const Problem p = rand_instance(sz[0], sz[1], 0.1, 300 + seed);
            const Dual x = rand_dual(p.n, p.m, 0.2, 400 + seed);
            ++seed;
            const Grad r = naive_gradient(x, p), f = fused_gradient(x, p);
            ok &= close_rel(f.f, r.f, 1e-12);
            for (std::size_t k = 0; k < r.grad.size(); ++k)
                ok &= std::fabs(f.grad[k] - r.grad[k]) <= 1e-13 + 1e-12 * std::fabs(r.grad[k]);
            for (std::size_t i = 0; i < r.row.size(); ++i) ok &= close_rel(f.row[i], r.row[i], 1e-12);
            for (std::size_t j = 0; j < r.col.size(); ++j) ok &= close_rel(f.col[j], r.col[j], 1e-12);
        }
        check(ok, "fused gradient equals the naive path on 5 shapes (test_dual.cpp:87-106)");
        const Problem p = rand_instance(23, 41, 0.1, 7);
        const Dual x = rand_dual(p.n, p.m, 0.2, 8);
        const Grad r = naive_gradient(x, p);
        ok = true;
        const int tiles[][2] = {{1, 1}, {3, 5}, {64, 64}};
        for (const auto& t : tiles) {
            const Grad f = fused_gradient(x, p, t[0], t[1]);
            for (std::size_t k = 0; k < r.grad.size(); ++k)
                ok &= std::fabs(f.grad[k] - r.grad[k]) <= 1e-13 + 1e-12 * std::fabs(r.grad[k]);
        }
        check(ok, "fused gradient is tile-shape invariant (test_dual.cpp:108-119)");
    }
    // test_dual.cpp:121-135 finite differences
    {
        bool ok = true;
        for (double eta : {0.05, 0.1}) {
            const Problem p = rand_instance(8, 7, eta, 17);
            const Dual x = rand_dual(p.n, p.m, 0.05, 18);
            const vec g = fused_gradient(x, p).grad;
            const vec x0 = x.to_free();
            for (std::size_t k = 0; k < x0.size(); ++k) {
                vec xp = x0, xm = x0;
                xp[k] += 1e-6;
                xm[k] -= 1e-6;
                const double fd = (fused_gradient(Dual::from_free(xp, p.n, p.m), p).f -
                                   fused_gradient(Dual::from_free(xm, p.n, p.m), p).f) / 2e-6;
                ok &= std::fabs(fd - g[k]) / std::max(1.0, std::fabs(g[k])) <= 1e-5;
            }
        }
        check(ok, "gradient matches central finite differences (test_dual.cpp:121-135)");
    }
    // test_sinkhorn.cpp:12-32, 46-55
    {
        const Problem p = rand_instance(24, 17, 0.05, 1001);
        Dual x = rand_dual(p.n, p.m, 0.3, 1002);
        x.alpha = optimal_alpha(x, p);
        const Grad g = fused_gradient(x, p);
        double e = 0.0;
        for (long i = 0; i < p.n; ++i) e += std::fabs(g.row[(std::size_t)i] - p.a[(std::size_t)i]);
        check(e <= 1e-12, "alpha update solves the row block to 1e-12 (test_sinkhorn.cpp:12-19)");
        Problem q;
        q.n = 6; q.m = 9; q.eta = 0.5;
        q.M.assign(54, 1.0);
        uniform_marginals(q);
        const Dual y = sinkhorn_step(Dual::zeros(6, 9), q);
        check(marginal_error(fused_gradient(y, q), q) <= 1e-12,
              "one step solves constant-cost problems (test_sinkhorn.cpp:21-32)");
        const Problem r = rand_instance(10, 7, 0.05, 1301);
        Dual z = rand_dual(r.n, r.m, 0.4, 1302);
        bool ok = true;
        for (int k = 0; k < 5; ++k) {
            z = sinkhorn_step(z, r);
            ok &= z.beta[(std::size_t)(r.m - 1)] == 0.0;
        }
        check(ok, "gauge restored after every step (test_sinkhorn.cpp:46-55)");
    }
    // test_sinkhorn.cpp:57-71 small eta, cold start
    {
        bool ok = true;
        for (double eta : {1e-3, 1e-4}) {
            const Problem p = gen_synthetic2(32, 32, eta);
            Dual x = Dual::zeros(p.n, p.m);
            for (int k = 0; k < 50; ++k) x = sinkhorn_step(x, p);
            for (double v : x.alpha) ok &= std::isfinite(v);
            for (double v : x.beta) ok &= std::isfinite(v);
            const double e = marginal_error(fused_gradient(x, p), p);
            ok &= std::isfinite(e) && e < 2.0;
        }
        check(ok, "log-domain iteration survives eta = 1e-3, 1e-4 (test_sinkhorn.cpp:57-71)");
    }
    // test_problem.cpp:122-141 synth2 structure
    {
        const Problem p = gen_synthetic2(101, 101, 0.01);
        bool mono = true;
        for (long i = 1; i < p.n; ++i) mono &= p.a[(std::size_t)i] < p.a[(std::size_t)(i - 1)];
        auto local_max = [&](long j) { return p.b[(std::size_t)j] > p.b[(std::size_t)(j - 1)] && p.b[(std::size_t)j] > p.b[(std::size_t)(j + 1)]; };
        double mx = 0.0;
        for (double v : p.M) mx = std::max(mx, v);
        check(mono && local_max(20) && local_max(60) && mx == 1.0,
              "synth2: a decreasing, b modes at j=20,60 for m=101, max M == 1 (test_problem.cpp:122-141)");
    }
    // test_sparsity.cpp:74-99 worked example and ties (T column-major here)
    {
        // rows: [3 1 9; 2 2 9; 0 5 9]
        const vec T = {3, 2, 0, 1, 2, 5, 9, 9, 9};
        const Pattern om = select_topk(T, 3, 3, 2);
        const std::vector<std::pair<int, int>> want = {{0, 0}, {0, 1}, {1, 0}, {2, 0}, {2, 1}};
        check(om.coords == want, "top-k worked example coordinates (test_sparsity.cpp:74-85)");
        vec Z(12, 0.0);  // 3 x 4
        auto at = [&](int i, int j) -> double& { return Z[(std::size_t)(j * 3 + i)]; };
        at(0, 1) = at(1, 1) = at(1, 2) = at(2, 2) = 1.0;
        const Pattern ot = select_topk(Z, 3, 4, 1);
        auto has = [&](int i, int j) { return std::count(ot.coords.begin(), ot.coords.end(), std::make_pair(i, j)) == 1; };
        check(has(0, 1) && !has(1, 2) && !has(2, 2), "ties break lexicographically (test_sparsity.cpp:87-99)");
    }
    // test_sparsity.cpp:101-122 top-k vs full sort with injected ties
    {
        Rng rng(2024);
        bool ok = true;
        for (int t = 0; t < 12; ++t) {
            const long n = 2 + (long)(rng.uniform() * 62), m = 2 + (long)(rng.uniform() * 62);
            vec T((std::size_t)(n * m));
            for (long j = 0; j < m; ++j)
                for (long i = 0; i < n; ++i) T[(std::size_t)(j * n + i)] = rng.uniform() < 0.3 ? 0.5 : rng.uniform();
            const long k = (long)(rng.uniform() * (double)(n * (m - 1)));
            const Pattern om = select_topk(T, n, m, k);
            std::vector<std::tuple<double, int, int>> all;
            for (long i = 0; i < n; ++i)
                for (long j = 0; j + 1 < m; ++j) all.emplace_back(-T[(std::size_t)(j * n + i)], (int)i, (int)j);
            std::sort(all.begin(), all.end());
            std::set<std::pair<int, int>> ref;
            for (long q = 0; q < std::min<long>(k, (long)all.size()); ++q)
                ref.insert({std::get<1>(all[(std::size_t)q]), std::get<2>(all[(std::size_t)q])});
            for (long i = 0; i < n; ++i) ref.insert({(int)i, 0});
            for (long j = 0; j + 1 < m; ++j) ref.insert({0, (int)j});
            ok &= om.coords.size() == ref.size() && std::is_sorted(om.coords.begin(), om.coords.end());
            for (const auto& c : om.coords) ok &= ref.count(c) == 1;
        }
        check(ok, "top-k agrees with the full-sort reference on 12 random T (test_sparsity.cpp:101-122)");
    }
    // test_sparsity.cpp:124-148, 172-197
    {
        const Problem p = rand_instance(10, 8, 0.1, 3001);
        const Dual x = rand_dual(p.n, p.m, 0.2, 3002);
        const Grad g = fused_gradient(x, p);
        const SparseSym A = assemble(x, p, select_topk(plan(x, p), p.n, p.m, 12), 0.125, g);
        const vec D = A.to_dense();
        bool ok = true;
        for (long i = 0; i < p.n; ++i) ok &= D[(std::size_t)(i * A.dim + i)] == g.row[(std::size_t)i] / p.eta + 0.125;
        for (long j = 0; j + 1 < p.m; ++j)
            ok &= D[(std::size_t)((p.n + j) * A.dim + p.n + j)] == g.col[(std::size_t)j] / p.eta + 0.125;
        check(ok, "assembled diagonal == sums/eta + tau bitwise (test_sparsity.cpp:124-136)");

        const Problem q = rand_instance(9, 7, 0.1, 3101);
        const Dual y = rand_dual(q.n, q.m, 0.2, 3102);
        const SparseSym F = assemble(y, q, select_topk(plan(y, q), q.n, q.m, q.n * (q.m - 1)), 0.03, fused_gradient(y, q));
        vec H = hessian_dense(y, q);
        const long dim = q.n + q.m - 1;
        for (long c = 0; c < dim; ++c) H[(std::size_t)(c * dim + c)] += 0.03;
        const vec FD = F.to_dense();
        double err = 0.0, sc = 0.0;
        for (std::size_t t = 0; t < H.size(); ++t) {
            err = std::max(err, std::fabs(FD[t] - H[t]));
            sc = std::max(sc, std::fabs(H[t]));
        }
        check(err <= 1e-14 * sc, "full-pattern assembly reconstructs the dense Hessian (test_sparsity.cpp:138-148)");

        const Problem r = rand_instance(11, 9, 0.1, 3401);
        const Dual x0 = rand_dual(r.n, r.m, 0.2, 3402), x1 = rand_dual(r.n, r.m, 0.2, 3403);
        const Pattern om = select_topk(plan(x0, r), r.n, r.m, 20);
        SparseSym U = assemble(x0, r, om, 0.5, fused_gradient(x0, r));
        update_values(U, x1, r, 0.25, fused_gradient(x1, r));
        const SparseSym fresh = assemble(x1, r, om, 0.25, fused_gradient(x1, r));
        check(U.pattern_id == fresh.pattern_id && U.values.size() == fresh.values.size() &&
                  std::memcmp(U.values.data(), fresh.values.data(), sizeof(double) * U.values.size()) == 0,
              "update_values == fresh assemble bitwise (test_sparsity.cpp:172-197)");
    }
    // test_sparse_chol.cpp:93-108 2x2 hand factor, :131-157 arrow
    {
        const vec A2 = {4, 2, 2, 3};
        const SparseSym S = SparseSym::from_dense(A2, 2);
        auto sym = std::make_shared<const Symbolic>(symbolic_analyze(S));
        const Numeric F = numeric_factorize(sym, S);
        check(sym->perm == ivec({0, 1}) && F.L.size() == 3 && F.L[0] == 2.0 && F.L[1] == 1.0 &&
                  close_rel(F.L[2], std::sqrt(2.0), 1e-15),
              "2x2 Cholesky: perm {0,1}, L = [[2,0],[1,sqrt2]] (test_sparse_chol.cpp:93-108)");
        const int dim = 9;
        vec Ar((std::size_t)(dim * dim), 0.0);
        for (int i = 0; i < dim; ++i) {
            Ar[(std::size_t)(i * dim + i)] = 10.0 + i;
            Ar[(std::size_t)(0 * dim + i)] = Ar[(std::size_t)(i * dim + 0)] = (i == 0) ? 10.0 : 1.0;
        }
        const SparseSym Sa = SparseSym::from_dense(Ar, dim);
        const Symbolic sa = symbolic_analyze(Sa);
        check(sa.nnz_L() == 2 * dim - 1, "arrow matrix factors with nnz(L) = 2 dim - 1 (test_sparse_chol.cpp:131-157)");
    }
    // test_sparse_chol.cpp:159-211 random SPD reconstruction + solve (dense check)
    {
        bool ok = true;
        for (int t = 0; t < 10; ++t) {
            const Problem p = rand_instance(9 + t, 8 + t % 3, 0.1, 5000 + t);
            const Dual x = rand_dual(p.n, p.m, 0.2, 5100 + t);
            const SparseSym A = assemble(x, p, select_topk(plan(x, p), p.n, p.m, 15 + 2 * t), 0.05, fused_gradient(x, p));
            auto sym = std::make_shared<const Symbolic>(symbolic_analyze(A));
            const Numeric F = numeric_factorize(sym, A);
            Rng rng(77 + t);
            vec rhs((std::size_t)A.dim);
            for (auto& v : rhs) v = 2.0 * rng.uniform() - 1.0;
            const vec sol = chol_solve(F, rhs);
            const vec back = A.matvec(sol);
            double e = 0.0;
            for (int i = 0; i < A.dim; ++i) e = std::max(e, std::fabs(back[(std::size_t)i] - rhs[(std::size_t)i]));
            ok &= e <= 1e-9;
            vec pc;
            const int it = pcg_solve(A, rhs, pc, 1e-13, 10000);
            double e2 = 0.0;
            for (int i = 0; i < A.dim; ++i) e2 = std::max(e2, std::fabs(pc[(std::size_t)i] - sol[(std::size_t)i]));
            ok &= it > 0 && e2 <= 1e-9 * (1.0 + norm_inf(sol));
        }
        check(ok, "sparse Cholesky solve residual <= 1e-9; PCG model agrees (test_sparse_chol.cpp:159-211)");
    }
    // test_splr.cpp:142-167 quadratic line search
    {
        const int dim = 6;
        const double dg[] = {4, 3, 2, 5, 1, 2};
        const vec b = {1, -1, 2, 0.5, -2, 1};
        auto Q = [&](const vec& z) {
            vec y((std::size_t)dim);
            for (int i = 0; i < dim; ++i) y[(std::size_t)i] = dg[i] * z[(std::size_t)i];
            y[0] += 0.8 * z[1];
            y[1] += 0.8 * z[0];
            return y;
        };
        auto oracle = [&](const vec& z) {
            Grad g;
            const vec qz = Q(z);
            g.grad.resize((std::size_t)dim);
            for (int i = 0; i < dim; ++i) g.grad[(std::size_t)i] = qz[(std::size_t)i] - b[(std::size_t)i];
            g.f = 0.5 * dot(z, qz) - dot(b, z);
            return g;
        };
        const vec x0((std::size_t)dim, 1.0);
        const Grad g0 = oracle(x0);
        // Newton direction: solve the 2x2 coupled block and the diagonal rest
        vec d((std::size_t)dim);
        const double det = 4 * 3 - 0.8 * 0.8;
        d[0] = -(3 * g0.grad[0] - 0.8 * g0.grad[1]) / det;
        d[1] = -(-0.8 * g0.grad[0] + 4 * g0.grad[1]) / det;
        for (int i = 2; i < dim; ++i) d[(std::size_t)i] = -g0.grad[(std::size_t)i] / dg[i];
        SplrConfig cfg;
        const LineSearchResult ls = line_search(oracle, x0, d, g0.f, g0.grad, cfg);
        check(ls.gamma == 1.0 && ls.evals == 1 && ls.curvature_ok,
              "quadratic + Newton direction: gamma = 1 in one evaluation (test_splr.cpp:142-167)");
    }
    // test_splr.cpp:89-107 direction equals dense Newton at full pattern, tau = 0
    {
        bool ok = true;
        for (int t = 0; t < 4; ++t) {
            const Problem p = rand_instance(12, 10, 0.1, 6500 + t);
            const Dual x = rand_dual(p.n, p.m, 0.2, 6600 + t);
            const Grad g = fused_gradient(x, p);
            const SparseSym A = assemble(x, p, select_topk(plan(x, p), p.n, p.m, p.n * (p.m - 1)), 0.0, g);
            auto sym = std::make_shared<const Symbolic>(symbolic_analyze(A));
            const vec d = compute_direction(numeric_factorize(sym, A), LowRank{}, g.grad);
            // residual check against the dense Hessian: H d = -g
            const vec H = hessian_dense(x, p);
            const long dim = p.n + p.m - 1;
            double e = 0.0;
            for (long r = 0; r < dim; ++r) {
                double s = 0.0;
                for (long c = 0; c < dim; ++c) s += H[(std::size_t)(c * dim + r)] * d[(std::size_t)c];
                e = std::max(e, std::fabs(s + g.grad[(std::size_t)r]));
            }
            ok &= e <= 1e-8 * norm_inf(g.grad) && dot(g.grad, d) < 0.0;
        }
        check(ok, "direction solves the dense Newton system at full pattern (test_splr.cpp:89-107)");
    }
    // test_splr.cpp:380-402 GOLDEN trajectory
    {
        const Problem p = gen_synthetic2(32, 32, 0.01);
        SplrConfig cfg;
        cfg.S = 1;
        cfg.J = 0;
        cfg.max_iter = 6;
        cfg.tol = 0.0;
        const SplrResult res = run_splr(Dual::zeros(p.n, p.m), p, cfg);
        const double golden[] = {1.6638586759335181,   0.29051373543167602,  0.21054519582141862, 0.095970055531796022,
                                 0.063997930975742745, 0.044099819557298296, 0.026713859915931643};
        bool ok = res.trace.size() == 7;
        for (std::size_t r = 0; ok && r < 7; ++r) {
            ok &= close_rel(res.trace[r].f, golden[r], 1e-12);
            std::printf("  golden[%zu] %.17g  oracle %.17g  rel %.2e\n", r, golden[r], res.trace[r].f,
                        std::fabs(res.trace[r].f - golden[r]) / golden[r]);
        }
        check(ok, "GOLDEN: 7 objective values, S=1 J=0 synth2 32x32 eta=.01, eps 1e-12 (test_splr.cpp:380-402)");
        cfg.direction_solver = 1;
        const SplrResult rp = run_splr(Dual::zeros(p.n, p.m), p, cfg);
        ok = rp.trace.size() == 7;
        for (std::size_t r = 0; ok && r < 7; ++r) ok &= close_rel(rp.trace[r].f, golden[r], 1e-9);
        check(ok, "GOLDEN via the PCG direction model within 1e-9");
    }
    // test_splr.cpp:201-226 selection rule, :228-268 convergence budgets
    {
        const Problem p = gen_synthetic2(32, 32, 0.01);
        SplrConfig cfg;
        cfg.S = 4;
        cfg.J = 3;
        cfg.max_iter = 24;
        cfg.tol = 0.0;
        const SplrResult res = run_splr(Dual::zeros(p.n, p.m), p, cfg);
        bool ok = res.steps.size() == 24;
        for (const StepRecord& r : res.steps) {
            ok &= r.f_after <= r.f_before + 1e-12 * (1.0 + std::fabs(r.f_before)) && !r.ls_failed;
            if (r.refresh)
                ok &= r.iter % cfg.S == 0 && r.f_after == std::min(r.f_cand_sinkhorn, r.f_cand_qn) &&
                      r.sinkhorn_selected == (r.f_cand_sinkhorn <= r.f_cand_qn);
            else
                ok &= std::isnan(r.f_cand_sinkhorn) && r.f_after == r.f_cand_qn;
        }
        check(ok, "per-step decrease and hybrid selection rule (test_splr.cpp:201-226)");
    }
    {
        const Problem p = gen_synthetic2(64, 64, 0.01);
        SplrConfig cfg;
        cfg.max_iter = 200;
        const SplrResult res = run_splr(Dual::zeros(p.n, p.m), p, cfg);
        bool ok = res.status == OK && res.trace.back().marginal_error <= 1e-8 && res.trace.back().iter <= 200;
        for (const StepRecord& r : res.steps)
            ok &= !r.ls_failed && r.curvature_ok && r.f_cand_qn <= r.f_before + 1e-4 * r.gamma * r.g_dot_d &&
                  r.gnew_dot_d >= 0.9 * r.g_dot_d;
        std::printf("  synth2 64x64 eta=.01: %ld iterations, err %.3e\n", res.trace.back().iter, res.trace.back().marginal_error);
        check(ok, "converges on synth2 64x64 eta=.01 within 200 its, Wolfe certificates (test_splr.cpp:228-251)");
        const Problem q = gen_synthetic2(64, 64, 0.001);
        SplrConfig c2;
        c2.max_iter = 400;
        const SplrResult r2 = run_splr(Dual::zeros(q.n, q.m), q, c2);
        std::printf("  synth2 64x64 eta=.001: %ld iterations, err %.3e\n", r2.trace.back().iter, r2.trace.back().marginal_error);
        check(r2.status == OK && r2.trace.back().marginal_error <= 1e-8,
              "eta = .001 cold start converges within 400 its (test_splr.cpp:253-268)");
    }
    // acceptance.cpp:283-299 criterion 6 on the three generators (seed 7, d = 2)
    {
        bool ok = true;
        const Problem ps[] = {gen_synthetic1(64, 64, 0, 2, 7, 0.01), gen_synthetic1(64, 64, 1, 2, 7, 0.01),
                              gen_synthetic2(64, 64, 0.01)};
        for (const Problem& p : ps) {
            SplrConfig cfg;
            cfg.max_iter = 200;
            const SplrResult r = run_splr(Dual::zeros(p.n, p.m), p, cfg);
            ok &= r.status == OK && r.trace.back().iter <= 200 && r.trace.back().marginal_error <= 1e-8;
            for (std::size_t k = 1; k < r.trace.size(); ++k)
                ok &= r.trace[k].f <= r.trace[k - 1].f + 1e-12 * (1.0 + std::fabs(r.trace[k - 1].f));
            std::printf("  acceptance(6): %ld iterations, err %.3e\n", r.trace.back().iter, r.trace.back().marginal_error);
        }
        check(ok, "acceptance criterion 6: <=1e-8 in <=200 its on synth1-iid/diff, synth2 (acceptance.cpp:283-299)");
    }
    std::printf(g_fail == 0 ? "all oracle checks passed\n" : "%d oracle checks FAILED\n", g_fail);
    return g_fail == 0 ? 0 : 1;
}
