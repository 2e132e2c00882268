/* CPU oracle: plain-C restatement of the reference path. TEST
 * INFRASTRUCTURE ONLY -- see pclab_oracle.h for who may load it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/src). Compiled with
 * -ffp-contract=off so that products and sums round exactly like the
 * reference's x86-64 build (no FMA contraction), which makes most
 * results bit-identical to the reference. */
#include "pclab_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL
static const double PI = 3.14159265358979323846;

/* rng.hpp:12-16 */
uint64_t or_mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
/* rng.hpp:21-23 */
uint64_t or_bits_at(uint64_t seed, uint64_t i) { return or_mix64(seed + (i + 1) * GAMMA); }
/* rng.hpp:26-28 */
double or_uniform_at(uint64_t seed, uint64_t i) {
    return (double)(or_bits_at(seed, i) >> 11) * 0x1.0p-53;
}
/* rng.hpp:31-33 */
uint64_t or_derive_seed(uint64_t seed, uint64_t tag) {
    return or_mix64(seed ^ or_mix64(tag + GAMMA));
}
/* Not in the reference (its generators only draw uniforms): Box-Muller on
 * the counter stream, u1 = 1 - U(2i) in (0,1], u2 = U(2i+1). */
double or_normal_at(uint64_t seed, uint64_t i) {
    const double u1 = 1.0 - or_uniform_at(seed, 2 * i);
    const double u2 = or_uniform_at(seed, 2 * i + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * PI * u2);
}

/* ------------------------------------------------------------------ */
/* Poisson / diffusion (sparse.cpp:232-305)                           */
/* ------------------------------------------------------------------ */

int64_t or_poisson_n(int dim, int64_t m) { return dim == 2 ? m * m : m * m * m; }

int64_t or_poisson_nnz(int dim, int64_t m) {
    const int64_t n = or_poisson_n(dim, m);
    const int64_t faces = (int64_t)dim * (m - 1) * (dim == 2 ? m : m * m);
    return n + 2 * faces;
}

/* sparse.cpp:298-303 with the exponent range generalised: the reference
 * draws 10^(2u-1); lo=-1, hi=1 reproduces it bit for bit because
 * (-1) + 2u == 2u - 1 exactly in IEEE arithmetic. */
void or_cell_coeffs(int64_t n, uint64_t seed, double lo, double hi, double* k) {
    for (int64_t c = 0; c < n; ++c) {
        const double u = or_uniform_at(seed, (uint64_t)c);
        k[c] = pow(10.0, lo + (hi - lo) * u);
    }
}

static double face_k(double klo, double khi) { return 2.0 * klo * khi / (klo + khi); }

/* assemble_poisson (sparse.cpp:232-282), emitted row by row in CSR. The
 * diagonal is accumulated in the reference's order: contributions pushed
 * by earlier cells (z-, y-, x-neighbour, in processing order) first, then
 * the cell's own axis loop. */
int or_gen_poisson(int dim, int64_t m, const double* cell_k, int64_t* rp,
                   int32_t* cols, double* vals) {
    if ((dim != 2 && dim != 3) || m < 1) return OR_ERR_ARGUMENT;
    const int64_t n = or_poisson_n(dim, m);
    const int64_t st[3] = {1, m, m * m};
    int64_t pos = 0;
    rp[0] = 0;
    for (int64_t c = 0; c < n; ++c) {
        const int64_t crd[3] = {c % m, (c / m) % m, dim == 3 ? c / (m * m) : 0};
        const double kc = cell_k ? cell_k[c] : 1.0;
        double diag = 0.0;
        for (int ax = dim - 1; ax >= 0; --ax)
            if (crd[ax] > 0) {
                const double kl = cell_k ? cell_k[c - st[ax]] : 1.0;
                diag += face_k(kl, kc);
            }
        for (int ax = 0; ax < dim; ++ax) {
            if (crd[ax] == 0) diag += kc;
            if (crd[ax] + 1 < m) {
                const double kh = cell_k ? cell_k[c + st[ax]] : 1.0;
                diag += face_k(kc, kh);
            } else {
                diag += kc;
            }
        }
        for (int ax = dim - 1; ax >= 0; --ax)
            if (crd[ax] > 0) {
                const double kl = cell_k ? cell_k[c - st[ax]] : 1.0;
                cols[pos] = (int32_t)(c - st[ax]);
                vals[pos++] = -face_k(kl, kc);
            }
        cols[pos] = (int32_t)c;
        vals[pos++] = diag;
        for (int ax = 0; ax < dim; ++ax)
            if (crd[ax] + 1 < m) {
                const double kh = cell_k ? cell_k[c + st[ax]] : 1.0;
                cols[pos] = (int32_t)(c + st[ax]);
                vals[pos++] = -face_k(kc, kh);
            }
        rp[c + 1] = pos;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Q1 hexahedral elasticity (this repo's generator; not in reference) */
/* ------------------------------------------------------------------ */

/* Trilinear brick of edge h, isotropic material E = 1, Poisson ratio nu,
 * 2x2x2 Gauss quadrature. Local node a = ax + 2 ay + 4 az, local dof
 * 3a + component. Voigt order xx, yy, zz, yz, xz, xy. The loop order is
 * part of the specification (the device generator mirrors it). */
void or_element_stiffness(double h, double nu, double* ke) {
    double d[6][6];
    memset(d, 0, sizeof d);
    const double c0 = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) d[i][j] = i == j ? c0 * (1.0 - nu) : c0 * nu;
    for (int i = 3; i < 6; ++i) d[i][i] = c0 * (1.0 - 2.0 * nu) / 2.0;
    const double g = 1.0 / sqrt(3.0);
    const double gp[2] = {-g, g};
    const double dscale = 2.0 / h;
    const double detj = (h / 2.0) * (h / 2.0) * (h / 2.0);
    memset(ke, 0, sizeof(double) * 576);
    for (int qz = 0; qz < 2; ++qz)
        for (int qy = 0; qy < 2; ++qy)
            for (int qx = 0; qx < 2; ++qx) {
                const double xi = gp[qx], eta = gp[qy], zeta = gp[qz];
                double b[6][24];
                memset(b, 0, sizeof b);
                for (int a = 0; a < 8; ++a) {
                    const double sx = (a & 1) ? 1.0 : -1.0;
                    const double sy = (a & 2) ? 1.0 : -1.0;
                    const double sz = (a & 4) ? 1.0 : -1.0;
                    const double dx = 0.125 * sx * (1.0 + sy * eta) * (1.0 + sz * zeta) * dscale;
                    const double dy = 0.125 * sy * (1.0 + sx * xi) * (1.0 + sz * zeta) * dscale;
                    const double dz = 0.125 * sz * (1.0 + sx * xi) * (1.0 + sy * eta) * dscale;
                    b[0][3 * a + 0] = dx;
                    b[1][3 * a + 1] = dy;
                    b[2][3 * a + 2] = dz;
                    b[3][3 * a + 1] = dz;
                    b[3][3 * a + 2] = dy;
                    b[4][3 * a + 0] = dz;
                    b[4][3 * a + 2] = dx;
                    b[5][3 * a + 0] = dy;
                    b[5][3 * a + 1] = dx;
                }
                double db[6][24];
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 24; ++j) {
                        double s = 0.0;
                        for (int k = 0; k < 6; ++k) s += d[i][k] * b[k][j];
                        db[i][j] = s;
                    }
                for (int i = 0; i < 24; ++i)
                    for (int j = i; j < 24; ++j) {
                        double s = 0.0;
                        for (int k = 0; k < 6; ++k) s += b[k][i] * db[k][j];
                        ke[i * 24 + j] += s * detj;
                    }
            }
    /* mirror the upper triangle so Ke (and hence A) is exactly symmetric,
     * as lower_triangle (sparse.cpp:189) demands bitwise symmetry */
    for (int i = 0; i < 24; ++i)
        for (int j = 0; j < i; ++j) ke[i * 24 + j] = ke[j * 24 + i];
}

/* m elements per side on the unit cube, (m+1)^3 nodes, 3 dof/node, the
 * iz == 0 face clamped and its dofs eliminated. */
void or_elasticity_dims(int64_t m, int64_t* n, int64_t* nnz) {
    const int64_t p = m + 1;
    *n = 3 * p * p * m;
    /* per free node: 3 rows x 3 x (#free neighbour nodes incl. itself) */
    int64_t cnt_xy = 0; /* sum over (ix,iy) of in-plane neighbour count */
    for (int64_t i = 0; i < p; ++i) {
        const int64_t cx = (i > 0) + 1 + (i + 1 < p);
        cnt_xy += cx;
    }
    const int64_t plane = cnt_xy * cnt_xy; /* sum over (ix,iy) of cx*cy */
    int64_t total = 0;
    for (int64_t iz = 1; iz < p; ++iz) {
        const int64_t cz = (iz > 1) + 1 + (iz + 1 < p);
        total += plane * cz;
    }
    *nnz = 9 * total;
}

void or_lognormal_field(int64_t n, uint64_t seed, double sigma, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = exp(sigma * or_normal_at(seed, (uint64_t)i));
}
void or_normal_field(int64_t n, uint64_t seed, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = or_normal_at(seed, (uint64_t)i);
}
/* experiment_rhs (experiments.cpp:303-308) without the seed derivation. */
void or_uniform_pm1_field(int64_t n, uint64_t seed, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * or_uniform_at(seed, (uint64_t)i) - 1.0;
}

/* Entry (p,c),(q,d) = sum over elements e containing p and q, in
 * ascending element index, of E_e * Ke[3 a + c][3 b + d]. */
int or_gen_elasticity(int64_t m, double nu, const double* moduli, int64_t* rp,
                      int32_t* cols, double* vals) {
    if (m < 1) return OR_ERR_ARGUMENT;
    const int64_t p1 = m + 1;
    const int64_t off = 3 * p1 * p1;
    double ke[576];
    or_element_stiffness(1.0 / (double)m, nu, ke);
    int64_t pos = 0;
    rp[0] = 0;
    int64_t row = 0;
    for (int64_t iz = 1; iz < p1; ++iz)
        for (int64_t iy = 0; iy < p1; ++iy)
            for (int64_t ix = 0; ix < p1; ++ix)
                for (int c = 0; c < 3; ++c) {
                    for (int dz = -1; dz <= 1; ++dz)
                        for (int dy = -1; dy <= 1; ++dy)
                            for (int dx = -1; dx <= 1; ++dx) {
                                const int64_t qx = ix + dx, qy = iy + dy, qz = iz + dz;
                                if (qx < 0 || qx >= p1 || qy < 0 || qy >= p1 || qz < 1 ||
                                    qz >= p1)
                                    continue;
                                const int64_t q = qx + p1 * qy + p1 * p1 * qz;
                                for (int d = 0; d < 3; ++d) {
                                    double acc = 0.0;
                                    for (int64_t ez = iz - 1; ez <= iz; ++ez) {
                                        if (ez < 0 || ez >= m || ez < qz - 1 || ez > qz) continue;
                                        for (int64_t ey = iy - 1; ey <= iy; ++ey) {
                                            if (ey < 0 || ey >= m || ey < qy - 1 || ey > qy) continue;
                                            for (int64_t ex = ix - 1; ex <= ix; ++ex) {
                                                if (ex < 0 || ex >= m || ex < qx - 1 || ex > qx)
                                                    continue;
                                                const int64_t e = ex + m * ey + m * m * ez;
                                                const int a = (int)((ix - ex) + 2 * (iy - ey) + 4 * (iz - ez));
                                                const int bb = (int)((qx - ex) + 2 * (qy - ey) + 4 * (qz - ez));
                                                acc += moduli[e] * ke[(3 * a + c) * 24 + 3 * bb + d];
                                            }
                                        }
                                    }
                                    cols[pos] = (int32_t)(3 * q + d - off);
                                    vals[pos++] = acc;
                                }
                            }
                    rp[++row] = pos;
                }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* structure                                                          */
/* ------------------------------------------------------------------ */

int64_t or_lower_nnz(int64_t n, const int64_t* rp, const int32_t* cols) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) c += cols[k] <= i;
    return c;
}

/* lower_triangle (sparse.cpp:189-204) on CSR. */
void or_lower(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
              int64_t* lrp, int32_t* lcols, double* lvals) {
    int64_t pos = 0;
    lrp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (cols[k] <= i) {
                lcols[pos] = cols[k];
                if (lvals) lvals[pos] = vals[k];
                ++pos;
            }
        lrp[i + 1] = pos;
    }
}

/* csr_transpose (sparse.cpp:137-157), also recording the source slot. */
void or_transpose(int64_t n, const int64_t* lrp, const int32_t* lcols,
                  const double* lvals, int64_t* urp, int32_t* ucols, double* uvals,
                  int64_t* u2l) {
    memset(urp, 0, sizeof(int64_t) * (size_t)(n + 1));
    const int64_t nnz = lrp[n];
    for (int64_t k = 0; k < nnz; ++k) urp[lcols[k] + 1]++;
    for (int64_t i = 1; i <= n; ++i) urp[i] += urp[i - 1];
    int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(next, urp, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = lrp[i]; k < lrp[i + 1]; ++k) {
            const int64_t slot = next[lcols[k]]++;
            ucols[slot] = (int32_t)i;
            if (uvals) uvals[slot] = lvals[k];
            if (u2l) u2l[slot] = k;
        }
    free(next);
}

/* Level sets of the forward substitution DAG: row i waits for every
 * j < i in its row (krylov.cpp:60-85 visits exactly those). */
int64_t or_levels_lower(int64_t n, const int64_t* lrp, const int32_t* lcols,
                        int32_t* level) {
    int32_t nl = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t lv = 0;
        for (int64_t k = lrp[i]; k < lrp[i + 1]; ++k) {
            const int32_t j = lcols[k];
            if (j < i && level[j] + 1 > lv) lv = level[j] + 1;
        }
        level[i] = lv;
        if (lv + 1 > nl) nl = lv + 1;
    }
    return nl;
}

/* Backward substitution DAG on U = L^T (krylov.cpp:87-112). */
int64_t or_levels_upper(int64_t n, const int64_t* urp, const int32_t* ucols,
                        int32_t* level) {
    int32_t nl = 0;
    for (int64_t i = n - 1; i >= 0; --i) {
        int32_t lv = 0;
        for (int64_t k = urp[i]; k < urp[i + 1]; ++k) {
            const int32_t j = ucols[k];
            if (j > i && level[j] + 1 > lv) lv = level[j] + 1;
        }
        level[i] = lv;
        if (lv + 1 > nl) nl = lv + 1;
    }
    return nl;
}

int64_t or_block_levels_lower(int64_t n, int bs, const int64_t* lrp,
                              const int32_t* lcols, int32_t* level) {
    const int64_t nb = n / bs;
    int32_t nl = 0;
    for (int64_t b = 0; b < nb; ++b) {
        int32_t lv = 0;
        for (int64_t i = b * bs; i < (b + 1) * bs; ++i)
            for (int64_t k = lrp[i]; k < lrp[i + 1]; ++k) {
                const int64_t jb = lcols[k] / bs;
                if (jb < b && level[jb] + 1 > lv) lv = level[jb] + 1;
            }
        level[b] = lv;
        if (lv + 1 > nl) nl = lv + 1;
    }
    return nl;
}

int64_t or_block_levels_upper(int64_t n, int bs, const int64_t* urp,
                              const int32_t* ucols, int32_t* level) {
    const int64_t nb = n / bs;
    int32_t nl = 0;
    for (int64_t b = nb - 1; b >= 0; --b) {
        int32_t lv = 0;
        for (int64_t i = b * bs; i < (b + 1) * bs; ++i)
            for (int64_t k = urp[i]; k < urp[i + 1]; ++k) {
                const int64_t jb = ucols[k] / bs;
                if (jb > b && level[jb] + 1 > lv) lv = level[jb] + 1;
            }
        level[b] = lv;
        if (lv + 1 > nl) nl = lv + 1;
    }
    return nl;
}

/* ------------------------------------------------------------------ */
/* kernels                                                            */
/* ------------------------------------------------------------------ */

/* csr_matvec (sparse.cpp:121-135) */
void or_csr_matvec(int64_t n, const int64_t* rp, const int32_t* cols,
                   const double* vals, const double* x, double* y) {
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc += vals[k] * x[cols[k]];
        y[i] = acc;
    }
}

/* tri_solve_lower (krylov.cpp:60-85) */
int or_trsv_lower(int64_t n, const int64_t* lrp, const int32_t* lcols,
                  const double* lvals, const double* b, double* x, int64_t* bad_row) {
    for (int64_t i = 0; i < n; ++i) {
        double acc = b[i], diag = 0.0;
        for (int64_t k = lrp[i]; k < lrp[i + 1]; ++k) {
            const int64_t j = lcols[k];
            if (j < i)
                acc -= lvals[k] * x[j];
            else if (j == i)
                diag = lvals[k];
            else {
                if (bad_row) *bad_row = i;
                return OR_ERR_FORMAT;
            }
        }
        if (diag == 0.0) {
            if (bad_row) *bad_row = i;
            return OR_ERR_NUMERIC;
        }
        x[i] = acc / diag;
    }
    return OR_OK;
}

/* tri_solve_upper (krylov.cpp:87-112) */
int or_trsv_upper(int64_t n, const int64_t* urp, const int32_t* ucols,
                  const double* uvals, const double* b, double* x, int64_t* bad_row) {
    for (int64_t i = n - 1; i >= 0; --i) {
        double acc = b[i], diag = 0.0;
        for (int64_t k = urp[i]; k < urp[i + 1]; ++k) {
            const int64_t j = ucols[k];
            if (j > i)
                acc -= uvals[k] * x[j];
            else if (j == i)
                diag = uvals[k];
            else {
                if (bad_row) *bad_row = i;
                return OR_ERR_FORMAT;
            }
        }
        if (diag == 0.0) {
            if (bad_row) *bad_row = i;
            return OR_ERR_NUMERIC;
        }
        x[i] = acc / diag;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* IC(0) (precond.cpp:23-75 attempt, 109-143 shift policy)            */
/* ------------------------------------------------------------------ */

static int ic0_attempt(int64_t n, const int64_t* lrp, const int32_t* lcols,
                       const double* a, double shift, double* v, int64_t* fail_row) {
    const int64_t nnz = lrp[n];
    for (int64_t k = 0; k < nnz; ++k) v[k] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t beg = lrp[i], end = lrp[i + 1];
        double diag_acc = 0.0;
        for (int64_t k = beg; k < end; ++k) {
            const int64_t j = lcols[k];
            if (j == i) {
                const double s = a[k] + shift - diag_acc;
                if (!(s > 0.0)) {
                    *fail_row = i;
                    return OR_ERR_NUMERIC;
                }
                v[k] = sqrt(s);
                break;
            }
            double s = a[k];
            int64_t pi = beg, pj = lrp[j];
            const int64_t pj_end = lrp[j + 1] - 1; /* diag_pos[j] */
            while (pi < k && pj < pj_end) {
                const int32_t ci = lcols[pi], cj = lcols[pj];
                if (ci == cj) {
                    s -= v[pi] * v[pj];
                    ++pi;
                    ++pj;
                } else if (ci < cj) {
                    ++pi;
                } else {
                    ++pj;
                }
            }
            const double lij = s / v[pj_end];
            v[k] = lij;
            diag_acc += lij * lij;
        }
    }
    return OR_OK;
}

int or_ic0(int64_t n, const int64_t* lrp, const int32_t* lcols, const double* avals,
           double* out, int64_t* fail_row, int* attempts) {
    double max_diag = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t last = lrp[i + 1] - 1;
        if (lrp[i + 1] == lrp[i] || lcols[last] != i) {
            *fail_row = i;
            return OR_ERR_FORMAT;
        }
        const double d = fabs(avals[last]);
        if (d > max_diag) max_diag = d;
    }
    const double alpha0 = 1e-8 * max_diag;
    for (int attempt = 0;; ++attempt) {
        const double shift = attempt == 0 ? 0.0 : alpha0 * (double)(1 << (attempt - 1));
        *attempts = attempt;
        const int st = ic0_attempt(n, lrp, lcols, avals, shift, out, fail_row);
        if (st == OR_OK) return OR_OK;
        if (attempt == 3) return st;
    }
}

/* ------------------------------------------------------------------ */
/* GNN (features.cpp, sparse.cpp:206-224, gnn.cpp)                    */
/* ------------------------------------------------------------------ */

/* node_features (features.cpp:11-72) */
void or_node_features(int64_t n, const int64_t* rp, const int32_t* cols,
                      const double* vals, double* f) {
    double* deg = (double*)calloc((size_t)(n ? n : 1), sizeof(double));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (cols[k] != i) deg[i] += 1.0;
    for (int64_t i = 0; i < n; ++i) {
        double* row = f + i * OR_NODE_FEATURES;
        double diag = 0.0, osum = 0.0, omax = 0.0;
        double mx = 0.0, mn = 1e300, mean = 0.0, var = 0.0;
        int64_t cnt = 0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const double av = fabs(vals[k]);
            if (cols[k] == i) {
                diag = av;
                continue;
            }
            osum += av;
            if (av > omax) omax = av;
            const double d = deg[cols[k]];
            if (d > mx) mx = d;
            if (d < mn) mn = d;
            mean += d;
            ++cnt;
        }
        row[0] = deg[i];
        row[1] = row[2] = row[3] = row[4] = 0.0;
        if (cnt > 0) {
            mean /= (double)cnt;
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                if (cols[k] == i) continue;
                const double d = deg[cols[k]];
                var += (d - mean) * (d - mean);
            }
            var /= (double)cnt;
            row[1] = mx;
            row[2] = mn;
            row[3] = mean;
            row[4] = var;
        }
        const double denom = diag + osum;
        row[5] = denom > 0.0 ? diag / denom : 0.0;
        if (omax > 0.0) {
            double dd = diag / omax;
            row[6] = dd < 0.0 ? 0.0 : (dd > 100.0 ? 100.0 : dd);
        } else {
            row[6] = 100.0;
        }
        const double angle = 2.0 * PI * (double)i / (double)n;
        row[7] = sin(angle);
        row[8] = cos(angle);
    }
    free(deg);
}

/* scale_by_std (sparse.cpp:206-224) */
double or_scale_by_std(int64_t nnz, const double* v, double* out) {
    if (nnz == 0) return 1.0;
    const double cnt = (double)nnz;
    double mean = 0.0;
    for (int64_t k = 0; k < nnz; ++k) mean += v[k];
    mean /= cnt;
    double var = 0.0, amax = 0.0;
    for (int64_t k = 0; k < nnz; ++k) {
        var += (v[k] - mean) * (v[k] - mean);
        if (fabs(v[k]) > amax) amax = fabs(v[k]);
    }
    const double sd = sqrt(var / cnt);
    if (sd <= 1e-13 * amax) {
        for (int64_t k = 0; k < nnz; ++k) out[k] = v[k];
        return 1.0;
    }
    for (int64_t k = 0; k < nnz; ++k) out[k] = v[k] / sd;
    return sd;
}

/* ParamLayout (gnn.hpp:18-27, gnn.cpp:14-41) */
typedef struct {
    int w1, b1, w2, b2, in, out;
} mlp_t;
static const int kEdgeIn[3] = {19, 18, 18};
static const int kNodeIn[3] = {11, 10, 10};
static void layout(mlp_t* edge, mlp_t* node) {
    int off = 18;
    for (int b = 0; b < 3; ++b) {
        mlp_t* ms[2] = {&edge[b], &node[b]};
        const int ins[2] = {kEdgeIn[b], kNodeIn[b]};
        const int outs[2] = {1, OR_HIDDEN};
        for (int t = 0; t < 2; ++t) {
            ms[t]->in = ins[t];
            ms[t]->out = outs[t];
            ms[t]->w1 = off;
            off += OR_HIDDEN * ins[t];
            ms[t]->b1 = off;
            off += OR_HIDDEN;
            ms[t]->w2 = off;
            off += outs[t] * OR_HIDDEN;
            ms[t]->b2 = off;
            off += outs[t];
        }
    }
}

/* GnnModel::init (gnn.cpp:96-117) */
void or_gnn_init(uint64_t seed, double* p) {
    mlp_t e[3], nd[3];
    layout(e, nd);
    for (int k = 0; k < OR_PARAMS; ++k) p[k] = 0.0;
    for (int c = 0; c < 9; ++c) p[c] = 1.0;
    uint64_t ctr = 0;
    for (int b = 0; b < 3; ++b) {
        const mlp_t* ms[2] = {&e[b], &nd[b]};
        for (int t = 0; t < 2; ++t) {
            const mlp_t* m = ms[t];
            const double s1 = 1.0 / sqrt((double)m->in);
            const int n1 = OR_HIDDEN * m->in + OR_HIDDEN;
            for (int k = 0; k < n1; ++k)
                p[m->w1 + k] = -s1 + (s1 - -s1) * or_uniform_at(seed, ctr++);
            const double s2 = 1.0 / sqrt((double)OR_HIDDEN);
            const int n2 = m->out * OR_HIDDEN + m->out;
            for (int k = 0; k < n2; ++k)
                p[m->w2 + k] = -s2 + (s2 - -s2) * or_uniform_at(seed, ctr++);
        }
    }
}

/* GnnModel::zero (gnn.cpp:119-125) */
void or_gnn_zero(double* p) {
    for (int k = 0; k < OR_PARAMS; ++k) p[k] = 0.0;
    for (int c = 0; c < 9; ++c) p[c] = 1.0;
}

/* mlp_apply (gnn.cpp:43-57) */
static void mlp_apply(const double* p, const mlp_t* m, const double* x, double* y) {
    double hid[OR_HIDDEN];
    for (int h = 0; h < OR_HIDDEN; ++h) {
        double acc = p[m->b1 + h];
        const double* row = p + m->w1 + h * m->in;
        for (int i = 0; i < m->in; ++i) acc += row[i] * x[i];
        hid[h] = tanh(acc);
    }
    for (int o = 0; o < m->out; ++o) {
        double acc = p[m->b2 + o];
        const double* row = p + m->w2 + o * OR_HIDDEN;
        for (int h = 0; h < OR_HIDDEN; ++h) acc += row[h] * hid[h];
        y[o] = acc;
    }
}

static int all_finite(const double* v, int64_t len) {
    for (int64_t i = 0; i < len; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* build_graph (features.cpp:74-84) + gnn_forward (gnn.cpp:127-219) */
int or_gnn_forward(int64_t n, const int64_t* rp, const int32_t* cols,
                   const double* vals, const double* p, double* out, double* sigma,
                   int* bad_block) {
    mlp_t em[3], nm[3];
    layout(em, nm);
    const int64_t ne = or_lower_nnz(n, rp, cols);
    int64_t* lrp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int32_t* lcols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ne ? ne : 1));
    double* lvals = (double*)malloc(sizeof(double) * (size_t)(ne ? ne : 1));
    or_lower(n, rp, cols, vals, lrp, lcols, lvals);
    double* ef = (double*)malloc(sizeof(double) * (size_t)(ne ? ne : 1));
    *sigma = or_scale_by_std(ne, lvals, ef);
    int64_t* erow = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne ? ne : 1));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = lrp[i]; k < lrp[i + 1]; ++k) erow[k] = i;

    double* feat = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1) * 9);
    or_node_features(n, rp, cols, vals, feat);

    double* x = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1) * 9);
    for (int c = 0; c < 9; ++c) {
        double mu = 0.0;
        for (int64_t v = 0; v < n; ++v) mu += feat[v * 9 + c];
        mu /= (double)n;
        double var = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            const double d = feat[v * 9 + c] - mu;
            var += d * d;
        }
        var /= (double)n;
        const double inv = 1.0 / (sqrt(var) + 1e-6);
        for (int64_t v = 0; v < n; ++v) {
            const double xh = (feat[v * 9 + c] - mu) * inv;
            x[v * 9 + c] = p[c] * xh + p[9 + c];
        }
    }
    double* cnt = (double*)calloc((size_t)(n ? n : 1), sizeof(double));
    for (int64_t k = 0; k < ne; ++k) {
        cnt[erow[k]] += 1.0;
        if (erow[k] != lcols[k]) cnt[lcols[k]] += 1.0;
    }
    double* eprev = NULL;
    double* ecur = (double*)malloc(sizeof(double) * (size_t)(ne ? ne : 1));
    double* msum = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* xn = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1) * OR_HIDDEN);
    int st = OR_OK;
    for (int b = 0; b < 3 && st == OR_OK; ++b) {
        const int xw = b == 0 ? 9 : OR_HIDDEN;
        double in[19];
        for (int64_t k = 0; k < ne; ++k) {
            int w = 0;
            if (eprev) in[w++] = eprev[k];
            in[w++] = ef[k];
            const int64_t i = erow[k], j = lcols[k];
            for (int c = 0; c < xw; ++c) in[w++] = x[i * xw + c];
            for (int c = 0; c < xw; ++c) in[w++] = x[j * xw + c];
            mlp_apply(p, &em[b], in, &ecur[k]);
        }
        if (!all_finite(ecur, ne)) {
            st = OR_ERR_NUMERIC;
            *bad_block = b + 1;
            break;
        }
        for (int64_t v = 0; v < n; ++v) msum[v] = 0.0;
        for (int64_t k = 0; k < ne; ++k) {
            msum[erow[k]] += ecur[k];
            if (erow[k] != lcols[k]) msum[lcols[k]] += ecur[k];
        }
        double nin[11];
        for (int64_t v = 0; v < n; ++v) {
            int w = 0;
            for (int c = 0; c < xw; ++c) nin[w++] = x[v * xw + c];
            nin[w++] = msum[v];
            nin[w++] = cnt[v] > 0.0 ? msum[v] / cnt[v] : 0.0;
            mlp_apply(p, &nm[b], nin, &xn[v * OR_HIDDEN]);
        }
        if (!all_finite(xn, n * OR_HIDDEN)) {
            st = OR_ERR_NUMERIC;
            *bad_block = b + 1;
            break;
        }
        memcpy(x, xn, sizeof(double) * (size_t)n * OR_HIDDEN);
        if (!eprev) eprev = (double*)malloc(sizeof(double) * (size_t)(ne ? ne : 1));
        memcpy(eprev, ecur, sizeof(double) * (size_t)ne);
    }
    if (st == OR_OK)
        for (int64_t k = 0; k < ne; ++k)
            out[k] = erow[k] == lcols[k] ? exp(ecur[k] / 2.0) : ecur[k];
    free(lrp);
    free(lcols);
    free(lvals);
    free(ef);
    free(erow);
    free(feat);
    free(x);
    free(cnt);
    free(eprev);
    free(ecur);
    free(msum);
    free(xn);
    return st;
}

/* ------------------------------------------------------------------ */
/* PCG (krylov.cpp:114-190)                                           */
/* ------------------------------------------------------------------ */

static double dot(int64_t n, const double* a, const double* b) {
#ifdef OR_DOT_STRIDED
    /* sensitivity builds only (tests/golden/sensitivity.py): the products
     * summed in OR_DOT_STRIDED interleaved partial sums, then the partials
     * in order -- a parallel reduction's association, same terms */
    double part[OR_DOT_STRIDED];
    for (int t = 0; t < OR_DOT_STRIDED; ++t) part[t] = 0.0;
    for (int64_t i = 0; i < n; ++i) part[i % OR_DOT_STRIDED] += a[i] * b[i];
    double s = 0.0;
    for (int t = 0; t < OR_DOT_STRIDED; ++t) s += part[t];
    return s;
#else
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
#endif
}

int or_pcg(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
           const double* b, int kind, const int64_t* lrp, const int32_t* lcols,
           const double* lvals, double rel_tol, int64_t max_iters, double* x,
           or_report* rep, double* history) {
    if (!(rel_tol > 0.0)) return OR_ERR_ARGUMENT;
    if (max_iters < 0) max_iters = 10 * n;
    memset(rep, 0, sizeof *rep);
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    const double bnorm = sqrt(dot(n, b, b));
    if (bnorm == 0.0) {
        rep->converged = 1;
        if (history) history[0] = 0.0;
        return OR_OK;
    }
    const size_t sz = sizeof(double) * (size_t)n;
    double *r = malloc(sz), *z = malloc(sz), *pv = malloc(sz), *ap = malloc(sz),
           *y = malloc(sz), *d = malloc(sz);
    int64_t *urp = NULL, *u2l = NULL;
    int32_t* ucols = NULL;
    double* uvals = NULL;
    if (kind == OR_PC_FACTOR) {
        const int64_t lnnz = lrp[n];
        urp = malloc(sizeof(int64_t) * (size_t)(n + 1));
        ucols = malloc(sizeof(int32_t) * (size_t)(lnnz ? lnnz : 1));
        uvals = malloc(sizeof(double) * (size_t)(lnnz ? lnnz : 1));
        or_transpose(n, lrp, lcols, lvals, urp, ucols, uvals, NULL);
    }
    if (kind == OR_PC_JACOBI)
        for (int64_t i = 0; i < n; ++i) {
            d[i] = 0.0;
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
                if (cols[k] == i) d[i] = vals[k];
        }
    int st = OR_OK;
    memcpy(r, b, sz);
    double rel = sqrt(dot(n, r, r)) / bnorm;
    if (history) history[0] = rel;
    rep->final_rel_residual = rel;
    rep->converged = rel <= rel_tol;
#define APPLY()                                                                  \
    do {                                                                         \
        if (kind == OR_PC_NONE)                                                  \
            memcpy(z, r, sz);                                                    \
        else if (kind == OR_PC_JACOBI)                                           \
            for (int64_t i = 0; i < n; ++i) z[i] = r[i] / d[i];                  \
        else {                                                                   \
            int64_t bad;                                                         \
            st = or_trsv_lower(n, lrp, lcols, lvals, r, y, &bad);                \
            if (st == OR_OK) st = or_trsv_upper(n, urp, ucols, uvals, y, z, &bad); \
        }                                                                        \
    } while (0)
    if (!rep->converged) {
        APPLY();
        double rz = dot(n, r, z);
        memcpy(pv, z, sz);
        for (int64_t k = 1; k <= max_iters && st == OR_OK; ++k) {
            or_csr_matvec(n, rp, cols, vals, pv, ap);
            const double pap = dot(n, pv, ap);
            if (!(pap > 0.0)) {
                rep->iterations = k;
                st = OR_ERR_CURVATURE;
                break;
            }
            const double alpha = rz / pap;
            for (int64_t i = 0; i < n; ++i) {
                x[i] += alpha * pv[i];
                r[i] -= alpha * ap[i];
            }
            rel = sqrt(dot(n, r, r)) / bnorm;
            rep->iterations = k;
            if (history) history[k] = rel;
            if (rel <= rel_tol) {
                rep->converged = 1;
                break;
            }
            APPLY();
            const double rz_new = dot(n, r, z);
            const double beta = rz_new / rz;
            rz = rz_new;
            for (int64_t i = 0; i < n; ++i) pv[i] = z[i] + beta * pv[i];
        }
        rep->final_rel_residual = rel;
    }
#undef APPLY
    or_csr_matvec(n, rp, cols, vals, x, ap);
    for (int64_t i = 0; i < n; ++i) ap[i] = b[i] - ap[i];
    rep->true_rel_residual = sqrt(dot(n, ap, ap)) / bnorm;
    rep->residual_mismatch =
        fabs(rep->true_rel_residual - rep->final_rel_residual) > 10.0 * rel_tol;
    free(r);
    free(z);
    free(pv);
    free(ap);
    free(y);
    free(d);
    free(urp);
    free(ucols);
    free(uvals);
    free(u2l);
    return st;
}
