// Thin C-ABI shim over the REFERENCE's own C++ internals, compiled together
// with the unmodified reference sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libpclab_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C oracle against the
// reference itself, by tests/golden/make_golden.py to produce fixtures, and
// by bench.py's CPU baseline / --impl reference arm. It contains no
// algorithm of its own: every function converts plain arrays into the
// reference's types and calls the reference (function names cited).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "error.hpp"
#include "features.hpp"
#include "gnn.hpp"
#include "krylov.hpp"
#include "precond.hpp"
#include "sparse.hpp"

using namespace pclab;

namespace {

thread_local std::string g_err;

SparseCsr to_csr(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals) {
    SparseCsr a;
    a.n_rows = a.n_cols = n;
    a.row_ptr.assign(rp, rp + n + 1);
    a.cols.assign(cols, cols + rp[n]);
    a.values.assign(vals, vals + rp[n]);
    return a;
}

SparseCoo to_coo(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals) {
    return csr_to_coo(to_csr(n, rp, cols, vals));  // sparse.cpp:106 (validates)
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// gen_poisson (sparse.cpp:285-305) -> CSR via coo_to_csr.
int64_t ref_gen_poisson_nnz(int dim, int64_t m, int variable, uint64_t seed) {
    const auto a = variable ? gen_poisson(dim, m, seed) : gen_poisson(dim, m);
    return a.nnz();
}
int ref_gen_poisson(int dim, int64_t m, int variable, uint64_t seed, int64_t* rp,
                    int32_t* cols, double* vals) {
    return guarded([&] {
        const auto c = coo_to_csr(variable ? gen_poisson(dim, m, seed) : gen_poisson(dim, m));
        for (int64_t i = 0; i <= c.n_rows; ++i) rp[i] = c.row_ptr[i];
        for (int64_t k = 0; k < c.nnz(); ++k) {
            cols[k] = static_cast<int32_t>(c.cols[k]);
            vals[k] = c.values[k];
        }
    });
}

// GnnModel::init (gnn.cpp:96)
void ref_gnn_init(uint64_t seed, double* params) {
    const auto m = GnnModel::init(seed);
    std::memcpy(params, m.params.data(), m.params.size() * sizeof(double));
}

// node_features (features.cpp:11)
int ref_node_features(int64_t n, const int64_t* rp, const int32_t* cols,
                      const double* vals, double* out) {
    return guarded([&] {
        const auto f = node_features(to_coo(n, rp, cols, vals));
        std::memcpy(out, f.data(), f.size() * sizeof(double));
    });
}

// build_graph + gnn_forward (features.cpp:74, gnn.cpp:127)
int ref_gnn_forward(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
                    const double* params, double* out, double* sigma) {
    return guarded([&] {
        GnnModel m;
        m.params.assign(params, params + param_layout().total);
        const auto g = build_graph(to_coo(n, rp, cols, vals));
        const auto o = gnn_forward(m, g);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
        *sigma = g.sigma;
    });
}

// ic0 / gnn_ic_predict / nic_predict (precond.cpp:109, 155, 145): factor
// values in lower-triangle order. kind: 0 ic0, 1 gnnic, 2 nic.
int ref_factor(int kind, int64_t n, const int64_t* rp, const int32_t* cols,
               const double* vals, const double* params, double* out, double* p_time) {
    return guarded([&] {
        const auto a = to_coo(n, rp, cols, vals);
        GnnModel m;
        if (params) m.params.assign(params, params + param_layout().total);
        const Preconditioner p =
            kind == 0 ? ic0(a) : (kind == 1 ? gnn_ic_predict(m, a) : nic_predict(m, a));
        std::memcpy(out, p.factor.matrix.values.data(),
                    p.factor.matrix.values.size() * sizeof(double));
        if (p_time) *p_time = p.p_time;
    });
}

struct ref_report {
    int64_t iterations;
    int32_t converged;
    int32_t residual_mismatch;
    double final_rel_residual;
    double true_rel_residual;
    double p_time, cg_time, total_time, tri_solve_time_per_iter;
};

static void fill(ref_report* r, const SolveReport& s) {
    r->iterations = s.iterations;
    r->converged = s.converged;
    r->residual_mismatch = s.residual_mismatch;
    r->final_rel_residual = s.final_rel_residual;
    r->true_rel_residual = s.true_rel_residual;
    r->p_time = s.p_time;
    r->cg_time = s.cg_time;
    r->total_time = s.total_time;
    r->tri_solve_time_per_iter = s.tri_solve_time_per_iter;
}

// pcg (krylov.cpp:114) with a preconditioner built by the reference.
// kind: "none", "jacobi", "ic0", "nic", "gnnic".
int ref_pcg(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
            const double* b, const char* kind, const double* params, double rel_tol,
            int64_t max_iters, double* x, ref_report* rep, double* history) {
    return guarded([&] {
        const auto coo = to_coo(n, rp, cols, vals);
        const std::string k = kind;
        GnnModel m;
        if (params) m.params.assign(params, params + param_layout().total);
        Preconditioner p = k == "none"     ? make_none()
                           : k == "jacobi" ? jacobi(coo)
                           : k == "ic0"    ? ic0(coo)
                           : k == "nic"    ? nic_predict(m, coo)
                                           : gnn_ic_predict(m, coo);
        SolveConfig cfg;
        cfg.rel_tol = rel_tol;
        cfg.max_iters = max_iters;
        cfg.record_residuals = history != nullptr;
        auto [xx, r] = pcg(to_csr(n, rp, cols, vals), std::span<const double>(b, n), p, cfg);
        std::memcpy(x, xx.data(), n * sizeof(double));
        fill(rep, r);
        if (history)
            std::memcpy(history, r.residual_history.data(),
                        r.residual_history.size() * sizeof(double));
    });
}

// pcg (krylov.cpp:114) with a caller-supplied factor on A's lower pattern
// (the bench's bounded CPU sample: per-iteration cost does not depend on
// how the factor values were produced).
int ref_pcg_factor(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
                   const double* lvals, const double* b, double rel_tol, int64_t max_iters,
                   double* x, ref_report* rep) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        SparseCsr a = to_csr(n, rp, cols, vals);
        Preconditioner p;
        p.kind = PrecondKind::IC0;
        SparseCoo& l = p.factor.matrix;
        l.n_rows = l.n_cols = n;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
                if (cols[k] <= i) {
                    l.rows.push_back(i);
                    l.cols.push_back(cols[k]);
                }
        l.values.assign(lvals, lvals + l.rows.size());
        const double setup = secs(t0);
        SolveConfig cfg;
        cfg.rel_tol = rel_tol;
        cfg.max_iters = max_iters;
        auto [xx, r] = pcg(a, std::span<const double>(b, n), p, cfg);
        std::memcpy(x, xx.data(), n * sizeof(double));
        fill(rep, r);
        rep->p_time = setup;
    });
}

// A resident PCG session for the bench's reference arm: the system (CSR)
// and an IC(0)-kind preconditioner on a caller-supplied factor are built
// once; each ref_pcg_session_run is one stock pcg() call (krylov.cpp:114,
// Applier construction included, as every pcg() call does).
struct ref_session {
    SparseCsr a;
    Preconditioner p;
};

void* ref_pcg_session_new(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
                          const double* lvals) {
    auto* s = new ref_session;
    if (guarded([&] {
            s->a = to_csr(n, rp, cols, vals);
            s->p.kind = PrecondKind::IC0;
            SparseCoo& l = s->p.factor.matrix;
            l.n_rows = l.n_cols = n;
            for (int64_t i = 0; i < n; ++i)
                for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
                    if (cols[k] <= i) {
                        l.rows.push_back(i);
                        l.cols.push_back(cols[k]);
                    }
            l.values.assign(lvals, lvals + l.rows.size());
        })) {
        delete s;
        return nullptr;
    }
    return s;
}

int ref_pcg_session_run(void* h, const double* b, double rel_tol, int64_t max_iters, double* x,
                        ref_report* rep) {
    auto* s = static_cast<ref_session*>(h);
    return guarded([&] {
        SolveConfig cfg;
        cfg.rel_tol = rel_tol;
        cfg.max_iters = max_iters;
        auto [xx, r] = pcg(s->a, std::span<const double>(b, s->a.n_rows), s->p, cfg);
        std::memcpy(x, xx.data(), static_cast<size_t>(s->a.n_rows) * sizeof(double));
        fill(rep, r);
    });
}

void ref_pcg_session_free(void* h) { delete static_cast<ref_session*>(h); }

}  // extern "C"
