// Device math of the GNN kernels (gnn.cu); also compiled stand-alone by
// tools/tanh_check.cu, which measures it against the library's tanh.
#pragma once

namespace pclab_b200 {

// tanh without branches: 1 - 2 / (1 + e^(2|x|)), sign restored. e^t by
// t = k ln2 + r, |r| <= ln2 / 2, a degree-11 Taylor polynomial (truncation
// 6e-15 relative) scaled by 2^k in the exponent field; the reciprocal from
// the hardware seed and two Newton steps. Absolute error < 1e-14 (tools/tanh_check.cu
// against the library's on the device, run by tests/test_gpu_variants.py) at about
// two thirds of the FP64 instructions of the library routine, whose two
// branches (small / large argument) a warp of mixed arguments both executes:
// the edge MLP is bound by its eight tanh per edge.
#ifndef GNN_LIBM_TANH
__device__ __forceinline__ double tanh_nb(double x) {
    const double t = fmin(fabs(x), 20.0) * 2.0;  // tanh(20) rounds to 1
    const double kf = rint(t * 1.4426950408889634074);
    double r = fma(kf, -6.93147180369123816490e-01, t);
    r = fma(kf, -1.90821492927058770002e-10, r);
    double p = 2.50521083854417187751e-08;  // 1 / 11!
    p = fma(p, r, 2.75573192239858906526e-07);
    p = fma(p, r, 2.75573192239858906526e-06);
    p = fma(p, r, 2.48015873015873015873e-05);
    p = fma(p, r, 1.98412698412698412698e-04);
    p = fma(p, r, 1.38888888888888888889e-03);
    p = fma(p, r, 8.33333333333333333333e-03);
    p = fma(p, r, 4.16666666666666666667e-02);
    p = fma(p, r, 1.66666666666666666667e-01);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const int k = static_cast<int>(kf);  // 0 .. 58
    const double e = __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
    const double d = e + 1.0;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    y = fma(y, fma(-d, y, 1.0), y);
    y = fma(y, fma(-d, y, 1.0), y);
    const double v = copysign(fma(-2.0, y, 1.0), x);
    return x != x ? x : v;  // NaN in, NaN out (the caller's non-finite check)
}
#else
__device__ __forceinline__ double tanh_nb(double x) { return tanh(x); }
#endif


}  // namespace pclab_b200
