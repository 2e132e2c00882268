/* Drop-in check: a C client written against the reference's public header
 * (pclab.h, /root/reference/proj/include) -- only its entry points, types
 * and status codes -- linked to libpclab_b200.so instead of the reference.
 *
 *   dropin host          host-only entry points (no GPU needed)
 *   dropin gpu <dir>     matrices, pcg_solve through every kind, Matrix
 *                        Market round trip (files under <dir>)
 *
 * Prints one "key value" line per check; exits 0 when every call returned
 * the status the reference documents. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pclab.h"

static int fails = 0;

static void expect(int cond, const char* what) {
    if (!cond) {
        fprintf(stderr, "FAIL %s (last error: %s)\n", what, pclab_last_error());
        ++fails;
    }
}

static long json_int(const char* js, const char* key) {
    const char* p = strstr(js, key);
    if (!p) return -1;
    p = strchr(p, ':');
    return p ? strtol(p + 1, NULL, 10) : -1;
}

static int host_checks(void) {
    printf("version %s\n", pclab_version());
    for (int s = 0; s <= 5; ++s) printf("status_name %d %s\n", s, pclab_status_name((pclab_status)s));
    pclab_model* m = NULL;
    expect(pclab_model_init(1, &m) == PCLAB_OK, "model_init");
    uint64_t cnt = 0;
    expect(pclab_model_param_count(m, &cnt) == PCLAB_OK && cnt == 997, "param_count 997");
    printf("param_count %llu\n", (unsigned long long)cnt);
    const char* path = "dropin_model.json";
    expect(pclab_model_save(m, path) == PCLAB_OK, "model_save");
    pclab_model* m2 = NULL;
    expect(pclab_model_load(path, &m2) == PCLAB_OK, "model_load");
    uint64_t cnt2 = 0;
    expect(pclab_model_param_count(m2, &cnt2) == PCLAB_OK && cnt2 == 997, "reloaded count");
    remove(path);
    pclab_model* bad = NULL;
    const pclab_status st = pclab_model_load("/nonexistent/dir/model.json", &bad);
    printf("load_missing %s %s\n", pclab_status_name(st), pclab_last_error());
    expect(st == PCLAB_ERR_IO && bad == NULL, "missing model is an IO error");
    double x = 0.0, b = 1.0;
    expect(pclab_pcg_solve(NULL, &b, "ic0", NULL, 0.0, 0, &x, NULL) == PCLAB_ERR_ARGUMENT, "null matrix");
    pclab_model_free(m);
    pclab_model_free(m2);
    return fails;
}

static int gpu_checks(const char* dir) {
    /* 1-D Laplacian (tridiagonal 2, -1) from unsorted triplets */
    enum { N = 64 };
    int64_t rows[3 * N], cols[3 * N];
    double vals[3 * N];
    int64_t nnz = 0;
    for (int64_t i = N - 1; i >= 0; --i) {
        rows[nnz] = i; cols[nnz] = i; vals[nnz++] = 2.0;
        if (i > 0) { rows[nnz] = i; cols[nnz] = i - 1; vals[nnz++] = -1.0; }
        if (i + 1 < N) { rows[nnz] = i; cols[nnz] = i + 1; vals[nnz++] = -1.0; }
    }
    pclab_matrix* a = NULL;
    expect(pclab_matrix_from_coo(N, N, nnz, rows, cols, vals, &a) == PCLAB_OK, "from_coo");
    int64_t nr = 0, nc = 0, nz = 0;
    expect(pclab_matrix_shape(a, &nr, &nc, &nz) == PCLAB_OK && nr == N && nc == N && nz == nnz, "shape");
    double b[N], x[N];
    for (int i = 0; i < N; ++i) b[i] = 1.0;
    const char* kinds[3] = {"none", "jacobi", "ic0"};
    for (int k = 0; k < 3; ++k) {
        char* rep = NULL;
        expect(pclab_pcg_solve(a, b, kinds[k], NULL, 1e-10, 0, x, &rep) == PCLAB_OK, kinds[k]);
        /* exact solution of T x = 1: x_i = (i + 1)(N - i) / 2 */
        double err = 0.0;
        for (int i = 0; i < N; ++i) err = fmax(err, fabs(x[i] - 0.5 * (i + 1) * (N - i)));
        printf("laplace1d %s iterations %ld maxerr %.3e\n", kinds[k], rep ? json_int(rep, "\"iterations\"") : -1L,
               err);
        expect(err < 1e-4, "1-D solution");
        pclab_string_free(rep);
    }
    /* duplicates are rejected with the reference's status */
    int64_t r2[2] = {0, 0}, c2[2] = {1, 1};
    double v2[2] = {1.0, 2.0};
    pclab_matrix* d = NULL;
    const pclab_status sd = pclab_matrix_from_coo(2, 2, 2, r2, c2, v2, &d);
    printf("duplicate %s %s\n", pclab_status_name(sd), pclab_last_error());
    expect(sd == PCLAB_ERR_FORMAT && d == NULL, "duplicate rejected");
    /* Poisson 3-D through every kind, then a Matrix Market round trip */
    pclab_matrix* p = NULL;
    expect(pclab_matrix_gen_poisson(3, 10, 1, 5, &p) == PCLAB_OK, "gen_poisson");
    pclab_model* m = NULL;
    expect(pclab_model_init(1, &m) == PCLAB_OK, "model_init");
    pclab_matrix_shape(p, &nr, &nc, &nz);
    double* pb = malloc(sizeof(double) * nr);
    double* px = malloc(sizeof(double) * nr);
    for (int64_t i = 0; i < nr; ++i) pb[i] = 1.0 + 0.001 * (double)(i % 7);
    const char* all[5] = {"none", "jacobi", "ic0", "nic", "gnnic"};
    for (int k = 0; k < 5; ++k) {
        char* rep = NULL;
        const pclab_status s = pclab_pcg_solve(p, pb, all[k], m, 1e-8, 0, px, &rep);
        printf("poisson3d %s status %s iterations %ld\n", all[k], pclab_status_name(s),
               rep ? json_int(rep, "\"iterations\"") : -1L);
        expect(s == PCLAB_OK, all[k]);
        pclab_string_free(rep);
    }
    char path[1024];
    snprintf(path, sizeof path, "%s/dropin.mtx", dir);
    expect(pclab_matrix_write(p, path) == PCLAB_OK, "matrix_write");
    pclab_matrix* q = NULL;
    expect(pclab_matrix_read(path, &q) == PCLAB_OK, "matrix_read");
    int64_t qr = 0, qc = 0, qz = 0;
    pclab_matrix_shape(q, &qr, &qc, &qz);
    expect(qr == nr && qc == nc && qz == nz, "round trip shape");
    char* s1 = NULL;
    expect(pclab_pcg_solve(q, pb, "ic0", NULL, 1e-8, 0, px, &s1) == PCLAB_OK, "solve after round trip");
    printf("roundtrip iterations %ld\n", s1 ? json_int(s1, "\"iterations\"") : -1L);
    pclab_string_free(s1);
    pclab_model_free(m);
    pclab_matrix_free(a);
    pclab_matrix_free(p);
    pclab_matrix_free(q);
    free(pb);
    free(px);
    return fails;
}

int main(int argc, char** argv) {
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_checks(argc > 2 ? argv[2] : ".") ? 1 : 0;
    return host_checks() ? 1 : 0;
}
