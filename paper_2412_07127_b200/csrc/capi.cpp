// C-ABI of libpclab_b200.so (include/pclab_b200.h). Status mapping and
// messages follow the reference's capi.cpp:33-56; all numerical work is
// dispatched to the device code in this directory -- there is no host
// fallback for any computation on the solve path.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pclab_b200.h"
#include "core.h"

using namespace pclab_b200;

struct pclab_matrix {
    std::unique_ptr<Matrix> m;
};
struct pclab_model {
    Model m;
};
struct pclab_precond {
    std::unique_ptr<Precond> p;
};

namespace pclab_b200 {

static cudaStream_t g_user_stream = nullptr;  // pclab_set_stream (sticky, documented)
static bool g_user_stream_set = false;
// a stream passed to one *_device call: used for that call only
static thread_local cudaStream_t t_call_stream = nullptr;

void* dev_alloc(size_t bytes) {
    static bool pool_ready = [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ULL;  // never hand freed blocks back to the driver
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        return true;
    }();
    (void)pool_ready;
    void* p = nullptr;
    // 64 bytes of slack: bulk copies (TMA) round ranges out to 16 bytes
    const cudaError_t e = cudaMallocAsync(&p, bytes + 64, lib_stream());
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
        CK(e);
    }
    return p;
}

void dev_free(void* p) { cudaFreeAsync(p, lib_stream()); }

// The stream every library call runs on: the one set by pclab_set_stream
// (e.g. the caller's current stream, so its events bracket our work), else
// a private non-blocking stream.
cudaStream_t lib_stream() {
    if (t_call_stream) return t_call_stream;
    if (g_user_stream_set) return g_user_stream;
    static cudaStream_t s = [] {
        cudaStream_t t;
        CK(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
        return t;
    }();
    return s;
}

static void json_num(std::ostringstream& o, double v) {
    if (std::isfinite(v)) {
        char buf[40];
        std::snprintf(buf, sizeof buf, "%.17g", v);
        o << buf;
    } else {
        o << "null";
    }
}

std::string SolveReport::to_json() const {
    std::ostringstream o;
    o << "{\"iterations\":" << iterations << ",\"converged\":" << (converged ? "true" : "false")
      << ",\"final_rel_residual\":";
    json_num(o, final_rel_residual);
    o << ",\"true_rel_residual\":";
    json_num(o, true_rel_residual);
    o << ",\"residual_mismatch\":" << (residual_mismatch ? "true" : "false") << ",\"p_time\":";
    json_num(o, p_time);
    o << ",\"cg_time\":";
    json_num(o, cg_time);
    o << ",\"total_time\":";
    json_num(o, total_time);
    o << ",\"tri_solve_time_per_iter\":";
    json_num(o, tri_solve_time_per_iter);
    o << ",\"analysis_time\":";
    json_num(o, analysis_time);
    o << ",\"ic0_time\":";
    json_num(o, ic0_time);
    o << ",\"gnn_time\":";
    json_num(o, gnn_time);
    o << ",\"residual_history\":[";
    for (size_t k = 0; k < residual_history.size(); ++k) {
        if (k) o << ",";
        json_num(o, residual_history[k]);
    }
    o << "],\"device\":\"cuda\"}";
    return o.str();
}

}  // namespace pclab_b200

namespace {

thread_local std::string t_error;

pclab_status fail(pclab_status s, const std::string& what) {
    t_error = what;
    return s;
}

template <class F>
pclab_status guarded(F&& f) {
    try {
        f();
        return PCLAB_OK;
    } catch (const DimensionError& e) {
        return fail(PCLAB_ERR_ARGUMENT, e.what());
    } catch (const FormatError& e) {
        return fail(PCLAB_ERR_FORMAT, e.what());
    } catch (const NumericError& e) {
        return fail(PCLAB_ERR_NUMERIC, e.what());
    } catch (const IoError& e) {
        return fail(PCLAB_ERR_IO, e.what());
    } catch (const std::bad_alloc&) {
        return fail(PCLAB_ERR_INTERNAL, "out of memory");
    } catch (const std::exception& e) {
        return fail(PCLAB_ERR_INTERNAL, e.what());
    }
}

char* dup_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (!p) throw std::bad_alloc();
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

// A stream passed to a device entry point is the library stream for that
// call only (stream-ordered temporaries and the kernels that use them share
// one order); the previous stream is restored when the call returns.
struct CallStream {
    cudaStream_t prev;
    explicit CallStream(void* s) : prev(t_call_stream) {
        if (s) t_call_stream = static_cast<cudaStream_t>(s);
    }
    ~CallStream() { t_call_stream = prev; }
    CallStream(const CallStream&) = delete;
    CallStream& operator=(const CallStream&) = delete;
};

std::string entry_str(int64_t i, int64_t j) {
    return "(" + std::to_string(i) + ", " + std::to_string(j) + ")";
}

// make_coo (sparse.cpp:55-72) + SparseCoo::validate (sparse.cpp:25-43) on
// the device (coo.cu)
std::unique_ptr<Matrix> coo_upload(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                                   const int64_t* cols, const double* vals) {
    return matrix_from_coo_device(n_rows, n_cols, nnz, rows, cols, vals, lib_stream());
}

// -------------------------------------------------- Matrix Market (host IO)
std::string lower_str(std::string s) {
    for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}

[[noreturn]] void mm_fail(long line, const std::string& what) {
    throw FormatError("matrix market, line " + std::to_string(line) + ": " + what);
}

bool blank_or_comment(const std::string& l) {
    return (!l.empty() && l[0] == '%') || l.find_first_not_of(" \t\r") == std::string::npos;
}

pclab_matrix* mm_read(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    std::string line;
    long no = 0;
    if (!std::getline(in, line)) mm_fail(1, "empty input");
    ++no;
    std::istringstream hdr(line);
    std::string banner, object, format, field, symmetry;
    hdr >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket") mm_fail(no, "missing %%MatrixMarket banner");
    if (lower_str(object) != "matrix") mm_fail(no, "unsupported object '" + object + "'");
    if (lower_str(format) != "coordinate") mm_fail(no, "unsupported format '" + format + "'");
    if (lower_str(field) != "real") mm_fail(no, "unsupported field '" + field + "'");
    const std::string sym = lower_str(symmetry);
    if (sym != "general" && sym != "symmetric") mm_fail(no, "unsupported symmetry '" + symmetry + "'");
    const bool symmetric = sym == "symmetric";
    int64_t nr = 0, nc = 0, nz = 0;
    for (;;) {
        if (!std::getline(in, line)) mm_fail(no + 1, "missing size line");
        ++no;
        if (blank_or_comment(line)) continue;
        std::istringstream s(line);
        if (!(s >> nr >> nc >> nz)) mm_fail(no, "bad size line");
        std::string extra;
        if (s >> extra) mm_fail(no, "trailing tokens on size line");
        break;
    }
    if (nr < 0 || nc < 0 || nz < 0) mm_fail(no, "negative size");
    if (symmetric && nr != nc) mm_fail(no, "symmetric matrix not square");
    std::vector<int64_t> r, c;
    std::vector<double> v;
    int64_t seen = 0;
    while (seen < nz) {
        if (!std::getline(in, line))
            mm_fail(no + 1, "expected " + std::to_string(nz) + " entries, got " + std::to_string(seen));
        ++no;
        if (blank_or_comment(line)) continue;
        std::istringstream s(line);
        int64_t i = 0, j = 0;
        double x = 0.0;
        if (!(s >> i >> j >> x)) mm_fail(no, "bad entry line");
        std::string extra;
        if (s >> extra) mm_fail(no, "trailing tokens on entry line");
        if (i < 1 || i > nr || j < 1 || j > nc) mm_fail(no, "index out of range");
        if (symmetric && j > i) mm_fail(no, "upper triangle entry in symmetric file");
        r.push_back(i - 1);
        c.push_back(j - 1);
        v.push_back(x);
        if (symmetric && i != j) {
            r.push_back(j - 1);
            c.push_back(i - 1);
            v.push_back(x);
        }
        ++seen;
    }
    auto h = std::make_unique<pclab_matrix>();
    try {
        h->m = coo_upload(nr, nc, static_cast<int64_t>(v.size()), r.data(), c.data(), v.data());
    } catch (const FormatError& e) {
        throw FormatError(std::string("matrix market: ") + e.what());
    }
    return h.release();
}

void download_csr(const Matrix& m, std::vector<int64_t>& rp, std::vector<int32_t>& c,
                  std::vector<double>& v) {
    rp.resize(m.a.n + 1);
    c.resize(m.a.nnz);
    v.resize(m.a.nnz);
    cudaStream_t st = lib_stream();
    CK(cudaMemcpyAsync(rp.data(), m.a.rp.p, sizeof(int64_t) * (m.a.n + 1), cudaMemcpyDeviceToHost, st));
    if (m.a.nnz) {
        CK(cudaMemcpyAsync(c.data(), m.a.cols.p, sizeof(int32_t) * m.a.nnz, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(v.data(), m.a.vals.p, sizeof(double) * m.a.nnz, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
}

void mm_write(const pclab_matrix* a, const std::string& path) {
    std::vector<int64_t> rp;
    std::vector<int32_t> c;
    std::vector<double> v;
    download_csr(*a->m, rp, c, v);
    const int64_t n = a->m->a.n;
    const bool symmetric = n == a->m->n_cols && matrix_symmetric(*a->m, lib_stream());
    std::ofstream out(path);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    out << "%%MatrixMarket matrix coordinate real " << (symmetric ? "symmetric" : "general") << "\n";
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) cnt += !symmetric || c[k] <= i;
    out << n << " " << a->m->n_cols << " " << cnt << "\n";
    char buf[64];
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (symmetric && c[k] > i) continue;
            std::snprintf(buf, sizeof buf, "%.17g", v[k]);
            out << (i + 1) << " " << (c[k] + 1) << " " << buf << "\n";
        }
    if (!out) throw IoError("matrix market write failed");
}

// ------------------------------------------- pclab-gnn checkpoint (JSON)
std::string slurp(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

// Minimal reader for the flat checkpoint object written by model_to_json
// (gnn.cpp:226-233): string/number scalars and one number array.
struct Ckpt {
    std::string format;
    long long version = 0, hidden = 0, blocks = 0, node_features = 0;
    std::vector<double> params;
    bool has_params = false;
};

Ckpt parse_ckpt(const std::string& s, const std::string& path) {
    Ckpt c;
    size_t i = 0;
    auto ws = [&] { while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i; };
    auto bad = [&](const std::string& w) -> void { throw FormatError(path + ": " + w); };
    auto str = [&]() {
        if (s[i] != '"') bad("expected string");
        const size_t e = s.find('"', i + 1);
        if (e == std::string::npos) bad("unterminated string");
        std::string r = s.substr(i + 1, e - i - 1);
        i = e + 1;
        return r;
    };
    auto num = [&]() {
        const char* b = s.c_str() + i;
        char* e = nullptr;
        const double v = std::strtod(b, &e);
        if (e == b) bad("expected number");
        i += static_cast<size_t>(e - b);
        return v;
    };
    ws();
    if (i >= s.size() || s[i] != '{') bad("checkpoint is not a JSON object");
    ++i;
    for (;;) {
        ws();
        if (s[i] == '}') break;
        const std::string key = str();
        ws();
        if (s[i] != ':') bad("expected ':'");
        ++i;
        ws();
        if (s[i] == '"') {
            const std::string v = str();
            if (key == "format") c.format = v;
        } else if (s[i] == '[') {
            ++i;
            std::vector<double> arr;
            ws();
            if (s[i] != ']')
                for (;;) {
                    ws();
                    arr.push_back(num());
                    ws();
                    if (s[i] == ',') { ++i; continue; }
                    if (s[i] == ']') break;
                    bad("bad array");
                }
            ++i;
            if (key == "params") {
                c.params = std::move(arr);
                c.has_params = true;
            }
        } else {
            const double v = num();
            if (key == "version") c.version = static_cast<long long>(v);
            if (key == "hidden") c.hidden = static_cast<long long>(v);
            if (key == "blocks") c.blocks = static_cast<long long>(v);
            if (key == "node_features") c.node_features = static_cast<long long>(v);
        }
        ws();
        if (s[i] == ',') { ++i; continue; }
        if (s[i] == '}') break;
        bad("expected ',' or '}'");
    }
    return c;
}

}  // namespace

extern "C" {

const char* pclab_version(void) { return "1.0.0-b200"; }

const char* pclab_status_name(pclab_status status) {
    switch (status) {
        case PCLAB_OK: return "ok";
        case PCLAB_ERR_ARGUMENT: return "argument";
        case PCLAB_ERR_FORMAT: return "format";
        case PCLAB_ERR_NUMERIC: return "numeric";
        case PCLAB_ERR_IO: return "io";
        case PCLAB_ERR_INTERNAL: return "internal";
    }
    return "unknown";
}

const char* pclab_last_error(void) { return t_error.c_str(); }

pclab_status pclab_matrix_from_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                                   const int64_t* cols, const double* values, pclab_matrix** out) {
    if (out == nullptr || (nnz > 0 && (rows == nullptr || cols == nullptr || values == nullptr)))
        return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_from_coo: null argument");
    if (nnz < 0) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_from_coo: negative nnz");
    return guarded([&] {
        auto h = std::make_unique<pclab_matrix>();
        h->m = coo_upload(n_rows, n_cols, nnz, rows, cols, values);
        *out = h.release();
    });
}

pclab_status pclab_matrix_from_csr(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* cols,
                                   const double* vals, pclab_matrix** out) {
    if (out == nullptr || row_ptr == nullptr || (nnz > 0 && (cols == nullptr || vals == nullptr)))
        return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_from_csr: null argument");
    if (n < 0 || nnz < 0) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_from_csr: negative size");
    return guarded([&] {
        auto h = std::make_unique<pclab_matrix>();
        h->m = matrix_from_csr_device(n, nnz, row_ptr, cols, vals, lib_stream());
        *out = h.release();
    });
}

pclab_status pclab_matrix_gen_poisson(int dim, int64_t m, int variable_coeff, uint64_t coeff_seed,
                                      pclab_matrix** out) {
    if (out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_gen_poisson: null output");
    if (variable_coeff) return pclab_matrix_gen_diffusion(dim, m, -1.0, 1.0, coeff_seed, out);
    return guarded([&] {
        auto h = std::make_unique<pclab_matrix>();
        h->m = gen_poisson_device(dim, m, nullptr, lib_stream());
        *out = h.release();
    });
}

pclab_status pclab_matrix_gen_diffusion(int dim, int64_t m, double lo, double hi, uint64_t seed,
                                        pclab_matrix** out) {
    if (out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_gen_diffusion: null output");
    return guarded([&] {
        if (dim != 2 && dim != 3) throw DimensionError("gen_poisson: dim must be 2 or 3");
        if (m < 1) throw DimensionError("gen_poisson: m must be >= 1");
        const int64_t n = dim == 2 ? m * m : m * m * m;
        // per-cell coefficients drawn on the host with the C library's pow,
        // as sparse.cpp:298-303 does (bitwise input parity)
        std::vector<double> k(static_cast<size_t>(n));
        for (int64_t c = 0; c < n; ++c) k[c] = std::pow(10.0, lo + (hi - lo) * uniform_at(seed, c));
        auto h = std::make_unique<pclab_matrix>();
        h->m = gen_poisson_device(dim, m, k.data(), lib_stream());
        *out = h.release();
    });
}

pclab_status pclab_matrix_gen_elasticity(int64_t m, double nu, const double* moduli, pclab_matrix** out) {
    if (out == nullptr || moduli == nullptr)
        return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_gen_elasticity: null argument");
    return guarded([&] {
        auto h = std::make_unique<pclab_matrix>();
        h->m = gen_elasticity_device(m, nu, moduli, lib_stream());
        *out = h.release();
    });
}

pclab_status pclab_matrix_shape(const pclab_matrix* a, int64_t* n_rows, int64_t* n_cols, int64_t* nnz) {
    if (a == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_shape: null matrix");
    if (n_rows) *n_rows = a->m->a.n;
    if (n_cols) *n_cols = a->m->n_cols;
    if (nnz) *nnz = a->m->a.nnz;
    return PCLAB_OK;
}

pclab_status pclab_matrix_csr(const pclab_matrix* a, int64_t* row_ptr, int32_t* cols, double* vals) {
    if (a == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_csr: null matrix");
    return guarded([&] {
        const DevCsr& c = a->m->a;
        cudaStream_t st = lib_stream();
        if (row_ptr)
            CK(cudaMemcpyAsync(row_ptr, c.rp.p, sizeof(int64_t) * (c.n + 1), cudaMemcpyDefault, st));
        if (cols && c.nnz) CK(cudaMemcpyAsync(cols, c.cols.p, sizeof(int32_t) * c.nnz, cudaMemcpyDefault, st));
        if (vals && c.nnz) CK(cudaMemcpyAsync(vals, c.vals.p, sizeof(double) * c.nnz, cudaMemcpyDefault, st));
        CK(cudaStreamSynchronize(st));
    });
}

pclab_status pclab_matrix_device_csr(const pclab_matrix* a, const int64_t** row_ptr, const int32_t** cols,
                                     const double** vals) {
    if (a == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_device_csr: null matrix");
    if (row_ptr) *row_ptr = a->m->a.rp.p;
    if (cols) *cols = a->m->a.cols.p;
    if (vals) *vals = a->m->a.vals.p;
    return PCLAB_OK;
}

void pclab_matrix_free(pclab_matrix* a) { delete a; }

pclab_status pclab_matrix_read(const char* path, pclab_matrix** out) {
    if (path == nullptr || out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_read: null argument");
    return guarded([&] { *out = mm_read(path); });
}

pclab_status pclab_matrix_write(const pclab_matrix* a, const char* path) {
    if (a == nullptr || path == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_write: null argument");
    return guarded([&] { mm_write(a, path); });
}

pclab_status pclab_model_init(uint64_t seed, pclab_model** out) {
    if (out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_model_init: null output");
    return guarded([&] {
        auto h = std::make_unique<pclab_model>();
        h->m.params = gnn_init_params(seed);
        *out = h.release();
    });
}

pclab_status pclab_model_from_params(const double* params, int64_t count, pclab_model** out) {
    if (out == nullptr || params == nullptr)
        return fail(PCLAB_ERR_ARGUMENT, "pclab_model_from_params: null argument");
    if (count != 997) return fail(PCLAB_ERR_ARGUMENT, "gnn: parameter vector has wrong length");
    auto h = std::make_unique<pclab_model>();
    h->m.params.assign(params, params + count);
    *out = h.release();
    return PCLAB_OK;
}

pclab_status pclab_model_params(const pclab_model* model, double* out) {
    if (model == nullptr || out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_model_params: null argument");
    std::memcpy(out, model->m.params.data(), sizeof(double) * model->m.params.size());
    return PCLAB_OK;
}

pclab_status pclab_model_load(const char* path, pclab_model** out) {
    if (path == nullptr || out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_model_load: null argument");
    return guarded([&] {
        const Ckpt c = parse_ckpt(slurp(path), path);
        if (c.format != "pclab-gnn") throw FormatError("model checkpoint: missing pclab-gnn format tag");
        if (c.version != 1) throw FormatError("model checkpoint: unsupported version");
        if (c.hidden != 8 || c.blocks != 3 || c.node_features != 9)
            throw FormatError("model checkpoint: architecture mismatch");
        if (!c.has_params || c.params.size() != 997)
            throw FormatError("model checkpoint: wrong parameter count");
        auto h = std::make_unique<pclab_model>();
        h->m.params = c.params;
        *out = h.release();
    });
}

pclab_status pclab_model_save(const pclab_model* model, const char* path) {
    if (model == nullptr || path == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_model_save: null argument");
    return guarded([&] {
        std::ofstream out(path);
        if (!out) throw IoError(std::string("cannot open ") + path);
        out << "{\n  \"blocks\": 3,\n  \"format\": \"pclab-gnn\",\n  \"hidden\": 8,\n  \"node_features\": 9,\n"
               "  \"params\": [";
        char buf[40];
        for (size_t k = 0; k < model->m.params.size(); ++k) {
            std::snprintf(buf, sizeof buf, "%.17g", model->m.params[k]);
            out << (k ? ",\n    " : "\n    ") << buf;
        }
        out << "\n  ],\n  \"version\": 1\n}\n";
        if (!out) throw IoError(std::string("write failed: ") + path);
    });
}

pclab_status pclab_model_param_count(const pclab_model* model, uint64_t* out) {
    if (model == nullptr || out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_model_param_count: null argument");
    *out = model->m.params.size();
    return PCLAB_OK;
}

void pclab_model_free(pclab_model* model) { delete model; }

pclab_status pclab_precond_build(pclab_matrix* a, const char* kind, const pclab_model* model,
                                 pclab_precond** out) {
    if (a == nullptr || kind == nullptr || out == nullptr)
        return fail(PCLAB_ERR_ARGUMENT, "pclab_precond_build: null argument");
    return guarded([&] {
        auto h = std::make_unique<pclab_precond>();
        h->p = build_precond(*a->m, parse_kind(kind), model ? &model->m : nullptr, lib_stream());
        *out = h.release();
    });
}

void pclab_precond_free(pclab_precond* p) { delete p; }

pclab_status pclab_precond_info(const pclab_precond* p, int64_t* nnz_lower, int32_t* block_size,
                                int32_t* levels_lower, int32_t* levels_upper, double* sigma) {
    if (p == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_precond_info: null argument");
    const Analysis* an = p->p->an.get();
    const bool factor = p->p->kind == Kind::IC0 || p->p->kind == Kind::NIC || p->p->kind == Kind::GnnIC;
    if (nnz_lower) *nnz_lower = factor && an ? an->lower.nnz : 0;
    if (block_size) *block_size = factor && an ? an->bs : 0;
    if (levels_lower) *levels_lower = factor && an ? an->blk_lo.nlevels : 0;
    if (levels_upper) *levels_upper = factor && an ? an->blk_up.nlevels : 0;
    if (sigma) *sigma = p->p->sigma;
    return PCLAB_OK;
}

pclab_status pclab_precond_layout(const pclab_precond* p, int64_t* out8) {
    if (p == nullptr || out8 == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_precond_layout: null argument");
    const Analysis* an = p->p->an.get();
    for (int k = 0; k < 8; ++k) out8[k] = 0;
    if (!an) return PCLAB_OK;
    out8[0] = an->bsr ? 1 : 0;
    out8[1] = an->a_bsr ? 1 : 0;
    out8[2] = an->bsr ? an->lbc.bcol.n : 0;
    out8[3] = an->bsr ? an->ubc.bcol.n : 0;
    out8[4] = an->a_bsr ? an->abc.bcol.n : 0;
    out8[5] = an->blk_lo.nitems * an->blk_lo.per_item;
    out8[6] = an->blk_up.nitems * an->blk_up.per_item;
    out8[7] = an->blk_lo.lanes + (an->blk_lo.rec ? 1000 : 0);  // + 1000: fixed slot records (rec_trsv_kernel)
    return PCLAB_OK;
}

pclab_status pclab_precond_factor(const pclab_precond* p, double* out) {
    if (p == nullptr || out == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_precond_factor: null argument");
    return guarded([&] {
        if (p->p->lvals.n == 0 && p->p->kind != Kind::IC0 && p->p->kind != Kind::NIC &&
            p->p->kind != Kind::GnnIC)
            throw DimensionError("preconditioner has no factor");
        CK(cudaMemcpyAsync(out, p->p->lvals.p, p->p->lvals.bytes(), cudaMemcpyDefault, lib_stream()));
        CK(cudaStreamSynchronize(lib_stream()));
    });
}

pclab_status pclab_precond_levels(const pclab_precond* p, int32_t* lo, int32_t* up, int32_t* nlo,
                                  int32_t* nup) {
    if (p == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_precond_levels: null argument");
    return guarded([&] {
        if (!p->p->an) throw DimensionError("preconditioner has no factor");
        Analysis& an = *p->p->an;
        cudaStream_t st = lib_stream();
        if (an.row_lo.level.n == 0 && an.lower.n > 0)
            compute_levels(an.lower, an.upper, 1, false, an.row_lo, st);
        if (an.rowlev_up.level.n == 0 && an.lower.n > 0)
            compute_levels(an.upper, an.lower, 1, true, an.rowlev_up, st);
        CK(cudaStreamSynchronize(st));
        // level counts = 1 + max level (both sweeps)
        auto count = [&](const DevBuf<int32_t>& lv, int64_t n) {
            std::vector<int32_t> h(static_cast<size_t>(n));
            if (n) CK(cudaMemcpy(h.data(), lv.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
            int32_t mx = -1;
            for (int32_t v : h) mx = std::max(mx, v);
            return mx + 1;
        };
        const int64_t n = an.lower.n;
        if (nlo) *nlo = count(an.row_lo.level, n);
        if (nup) *nup = count(an.rowlev_up.level, n);
        if (lo && n) CK(cudaMemcpy(lo, an.row_lo.level.p, sizeof(int32_t) * n, cudaMemcpyDefault));
        if (up && n) CK(cudaMemcpy(up, an.rowlev_up.level.p, sizeof(int32_t) * n, cudaMemcpyDefault));
    });
}

pclab_status pclab_precond_timings(const pclab_precond* p, double* ms4) {
    if (p == nullptr || ms4 == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_precond_timings: null argument");
    ms4[0] = p->p->ms_analysis;
    ms4[1] = p->p->ms_ic0;
    ms4[2] = p->p->ms_gnn;
    ms4[3] = p->p->ms_total;
    return PCLAB_OK;
}

pclab_status pclab_matrix_drop_analysis(pclab_matrix* a) {
    if (a == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_matrix_drop_analysis: null matrix");
    return guarded([&] {
        CK(cudaStreamSynchronize(lib_stream()));
        a->m->an.reset();
    });
}

void pclab_set_stream(void* stream) {
    g_user_stream = static_cast<cudaStream_t>(stream);
    g_user_stream_set = stream != nullptr;
}

long long pclab_launch_count(void) { return launch_count(); }

pclab_status pclab_pcg_profile(pclab_matrix* a, const pclab_precond* p, const double* b, double* x,
                               int64_t max_iters, double* ms8) {
    if (a == nullptr || p == nullptr || b == nullptr || x == nullptr || ms8 == nullptr)
        return fail(PCLAB_ERR_ARGUMENT, "pclab_pcg_profile: null argument");
    return guarded([&] {
        if (p->p->a != a->m.get()) throw DimensionError("preconditioner built for another matrix");
        pcg_solve(*a->m, *p->p, b, x, 1e-300, max_iters, false, lib_stream(), ms8);
    });
}

pclab_status pclab_pcg_solve_device(pclab_matrix* a, const pclab_precond* p, const double* b, double* x,
                                    double rel_tol, int64_t max_iters, int record_history, void* stream,
                                    char** report_json_out) {
    if (a == nullptr || p == nullptr || b == nullptr || x == nullptr)
        return fail(PCLAB_ERR_ARGUMENT, "pclab_pcg_solve_device: null argument");
    return guarded([&] {
        if (p->p->a != a->m.get()) throw DimensionError("preconditioner built for another matrix");
        CallStream cs(stream);
        const SolveReport r = pcg_solve(*a->m, *p->p, b, x, rel_tol, max_iters, record_history != 0, lib_stream());
        if (report_json_out) *report_json_out = dup_string(r.to_json());
    });
}

pclab_status pclab_pcg_solve(const pclab_matrix* a, const double* b, const char* kind, const pclab_model* model,
                             double rel_tol, int64_t max_iters, double* x_out, char** report_json_out) {
    if (a == nullptr || b == nullptr || kind == nullptr || x_out == nullptr)
        return fail(PCLAB_ERR_ARGUMENT, "pclab_pcg_solve: null argument");
    return guarded([&] {
        Matrix& m = *const_cast<pclab_matrix*>(a)->m;
        cudaStream_t st = lib_stream();
        const Kind k = parse_kind(kind);
        if ((k == Kind::NIC || k == Kind::GnnIC) && model == nullptr)
            throw DimensionError(std::string("kind '") + kind + "' needs a model");
        auto p = build_precond(m, k, model ? &model->m : nullptr, st);
        const int64_t n = m.a.n;
        DevBuf<double> db(n), dx(n);
        if (n) CK(cudaMemcpyAsync(db.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        const SolveReport r =
            pcg_solve(m, *p, db.p, dx.p, rel_tol > 0.0 ? rel_tol : 1e-6, max_iters > 0 ? max_iters : -1, false, st);
        if (n) CK(cudaMemcpyAsync(x_out, dx.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (report_json_out) *report_json_out = dup_string(r.to_json());
    });
}

pclab_status pclab_spmv_device(const pclab_matrix* a, const double* x, double* y, void* stream) {
    if (a == nullptr || x == nullptr || y == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_spmv_device: null argument");
    return guarded([&] {
        CallStream cs(stream);
        spmv(*a->m, x, y, lib_stream());
        CK(cudaStreamSynchronize(lib_stream()));
    });
}

pclab_status pclab_trsv_device(const pclab_precond* p, int upper, const double* b, double* x, void* stream) {
    if (p == nullptr || b == nullptr || x == nullptr) return fail(PCLAB_ERR_ARGUMENT, "pclab_trsv_device: null argument");
    return guarded([&] {
        const Analysis* an = p->p->an.get();
        if (!an || p->p->lvals.n == 0) throw DimensionError("preconditioner has no factor");
        CallStream cs(stream);
        trsv(*an, *p->p, upper != 0, b, x, lib_stream());
    });
}

pclab_status pclab_run(const char* command, const char* config_json, char** summary_json_out) {
    (void)config_json;
    (void)summary_json_out;
    return fail(PCLAB_ERR_ARGUMENT, std::string("pclab_run: command '") + (command ? command : "") +
                                        "' is outside the accelerated solve path (use the reference CLI)");
}

void pclab_string_free(char* s) { std::free(s); }

double pclab_uniform_at(uint64_t seed, uint64_t i) { return uniform_at(seed, i); }
uint64_t pclab_derive_seed(uint64_t seed, uint64_t tag) { return derive_seed(seed, tag); }
void pclab_field_normal(int64_t n, uint64_t seed, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = normal_at(seed, static_cast<uint64_t>(i));
}
void pclab_field_lognormal(int64_t n, uint64_t seed, double sigma, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = std::exp(sigma * normal_at(seed, static_cast<uint64_t>(i)));
}
void pclab_field_uniform_pm1(int64_t n, uint64_t seed, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * uniform_at(seed, static_cast<uint64_t>(i)) - 1.0;
}

}  // extern "C"
