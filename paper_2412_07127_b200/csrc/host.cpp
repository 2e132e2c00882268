// Host-side helpers: counter RNG (reference src/rng.hpp), GNN
// initialisation (src/gnn.cpp:96-117), the Q1 element stiffness and the
// seeded input fields. Compiled with -ffp-contract=off so every product
// and sum rounds like the oracle's (no FMA contraction).
#include <cmath>
#include <cstring>

#include "core.h"

namespace pclab_b200 {

namespace {
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
constexpr double kPi = 3.14159265358979323846;
}  // namespace

double uniform_at(uint64_t seed, uint64_t i) {
    return static_cast<double>(mix64(seed + (i + 1) * kGamma) >> 11) * 0x1.0p-53;
}

uint64_t derive_seed(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag + kGamma)); }

double normal_at(uint64_t seed, uint64_t i) {
    const double u1 = 1.0 - uniform_at(seed, 2 * i);
    const double u2 = uniform_at(seed, 2 * i + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}

std::vector<double> gnn_init_params(uint64_t seed) {
    // layout: gain[9] bias[9], then per block: edge MLP (in 19/18/18 -> 8 -> 1)
    // and node MLP (in 11/10/10 -> 8 -> 8); weights row-major out x in.
    std::vector<double> p(997, 0.0);
    for (int c = 0; c < 9; ++c) p[c] = 1.0;
    const int ein[3] = {19, 18, 18}, nin[3] = {11, 10, 10};
    int off = 18;
    uint64_t ctr = 0;
    for (int b = 0; b < 3; ++b) {
        const int ins[2] = {ein[b], nin[b]};
        const int outs[2] = {1, 8};
        for (int t = 0; t < 2; ++t) {
            const double s1 = 1.0 / std::sqrt(static_cast<double>(ins[t]));
            const int n1 = 8 * ins[t] + 8;
            for (int k = 0; k < n1; ++k) p[off + k] = -s1 + (s1 - -s1) * uniform_at(seed, ctr++);
            off += n1;
            const double s2 = 1.0 / std::sqrt(8.0);
            const int n2 = outs[t] * 8 + outs[t];
            for (int k = 0; k < n2; ++k) p[off + k] = -s2 + (s2 - -s2) * uniform_at(seed, ctr++);
            off += n2;
        }
    }
    return p;
}

// Trilinear brick, E = 1, 2x2x2 Gauss; identical operation order to
// oracle/pclab_oracle.c:or_element_stiffness (the specification of the
// elasticity generator), upper triangle mirrored for exact symmetry.
void element_stiffness(double h, double nu, double* ke) {
    double d[6][6];
    std::memset(d, 0, sizeof d);
    const double c0 = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) d[i][j] = i == j ? c0 * (1.0 - nu) : c0 * nu;
    for (int i = 3; i < 6; ++i) d[i][i] = c0 * (1.0 - 2.0 * nu) / 2.0;
    const double g = 1.0 / std::sqrt(3.0);
    const double gp[2] = {-g, g};
    const double dscale = 2.0 / h;
    const double detj = (h / 2.0) * (h / 2.0) * (h / 2.0);
    std::memset(ke, 0, sizeof(double) * 576);
    for (int qz = 0; qz < 2; ++qz)
        for (int qy = 0; qy < 2; ++qy)
            for (int qx = 0; qx < 2; ++qx) {
                const double xi = gp[qx], eta = gp[qy], zeta = gp[qz];
                double b[6][24];
                std::memset(b, 0, sizeof b);
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
    for (int i = 0; i < 24; ++i)
        for (int j = 0; j < i; ++j) ke[i * 24 + j] = ke[j * 24 + i];
}

}  // namespace pclab_b200
