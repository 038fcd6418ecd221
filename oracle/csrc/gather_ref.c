/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's periodic
 * point-sampling kernels.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference leg of bench.py may load this library.
 *
 * Follows /root/reference/pkg/src/flowreg/_kernels.py:
 *   nearest  : floor(q + 0.5) with Python floor-mod wrap      (_kernels.py:103-118)
 *   linear   : 2^d corners, weights (1-t, t)                   (_kernels.py:120-160)
 *   cubic    : Lagrange nodes at offsets -1..2 of floor(q)     (_kernels.py:162-219)
 * Arithmetic: weights and accumulation in double for every storage type,
 * result rounded to the storage type at the end (numba promotes f32*f64 to
 * f64; the reference's f32 mode therefore returns the f64 sum rounded).
 * Compiled with -ffp-contract=off so no FMA contraction changes rounding.
 *
 * Grids are 3D (n0, n1, n2), C-order; 2D grids are passed as (1, n0, n1)
 * with q0 == NULL (the size-1 axis then contributes the exact factor 1).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

static inline int64_t pmod(int64_t i, int64_t n) {
    int64_t r = i % n;
    return r < 0 ? r + n : r;
}

static inline void lagrange4(double t, double w[4]) {
    w[0] = -t * (t - 1.0) * (t - 2.0) / 6.0;
    w[1] = (t + 1.0) * (t - 1.0) * (t - 2.0) / 2.0;
    w[2] = -(t + 1.0) * t * (t - 2.0) / 2.0;
    w[3] = (t + 1.0) * t * (t - 1.0) / 6.0;
}

#define DEFINE_GATHER(NAME, T)                                                              \
    void NAME(const T *vals, int64_t n0, int64_t n1, int64_t n2, const double *q0,          \
              const double *q1, const double *q2, int64_t npts, int method, T *out) {       \
        _Pragma("omp parallel for schedule(static)")                                        \
        for (int64_t p = 0; p < npts; ++p) {                                                \
            double a0 = q0 ? q0[p] : 0.0, a1 = q1[p], a2 = q2[p];                           \
            if (method == 0) {                                                              \
                int64_t i = pmod((int64_t)floor(a0 + 0.5), n0);                             \
                int64_t j = pmod((int64_t)floor(a1 + 0.5), n1);                             \
                int64_t k = pmod((int64_t)floor(a2 + 0.5), n2);                             \
                out[p] = vals[(i * n1 + j) * n2 + k];                                       \
            } else if (method == 1) {                                                       \
                double f0 = floor(a0), f1 = floor(a1), f2 = floor(a2);                      \
                double t0 = a0 - f0, t1 = a1 - f1, t2 = a2 - f2;                            \
                int64_t i0 = pmod((int64_t)f0, n0), j0 = pmod((int64_t)f1, n1);             \
                int64_t k0 = pmod((int64_t)f2, n2);                                         \
                int64_t i1 = (i0 + 1) % n0, j1 = (j0 + 1) % n1, k1 = (k0 + 1) % n2;         \
                double r[2][2];                                                             \
                int64_t ii[2] = {i0, i1}, jj[2] = {j0, j1};                                 \
                for (int a = 0; a < 2; ++a)                                                 \
                    for (int b = 0; b < 2; ++b) {                                           \
                        const T *row = vals + (ii[a] * n1 + jj[b]) * n2;                    \
                        r[a][b] = (1.0 - t2) * (double)row[k0] + t2 * (double)row[k1];      \
                    }                                                                       \
                double s0 = (1.0 - t1) * r[0][0] + t1 * r[0][1];                            \
                double s1 = (1.0 - t1) * r[1][0] + t1 * r[1][1];                            \
                out[p] = (T)((1.0 - t0) * s0 + t0 * s1);                                    \
            } else {                                                                        \
                double f0 = floor(a0), f1 = floor(a1), f2 = floor(a2);                      \
                double w0[4], w1[4], w2[4];                                                 \
                lagrange4(a0 - f0, w0);                                                     \
                lagrange4(a1 - f1, w1);                                                     \
                lagrange4(a2 - f2, w2);                                                     \
                int64_t b0 = (int64_t)f0 - 1, b1 = (int64_t)f1 - 1, b2 = (int64_t)f2 - 1;   \
                int64_t kk[4];                                                              \
                for (int c = 0; c < 4; ++c) kk[c] = pmod(b2 + c, n2);                       \
                double acc = 0.0;                                                           \
                for (int a = 0; a < 4; ++a) {                                               \
                    int64_t ia = pmod(b0 + a, n0);                                          \
                    double plane = 0.0;                                                     \
                    for (int b = 0; b < 4; ++b) {                                           \
                        const T *row = vals + (ia * n1 + pmod(b1 + b, n1)) * n2;            \
                        double rsum = 0.0;                                                  \
                        for (int c = 0; c < 4; ++c) rsum += w2[c] * (double)row[kk[c]];     \
                        plane += w1[b] * rsum;                                              \
                    }                                                                       \
                    acc += w0[a] * plane;                                                   \
                }                                                                           \
                out[p] = (T)acc;                                                            \
            }                                                                               \
        }                                                                                   \
    }

DEFINE_GATHER(oracle_gather_f64, double)
DEFINE_GATHER(oracle_gather_f32, float)

/* nearest on int32 label volumes (metrics.transport_labels path) */
void oracle_gather_i32(const int32_t *vals, int64_t n0, int64_t n1, int64_t n2, const double *q0,
                       const double *q1, const double *q2, int64_t npts, int32_t *out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; ++p) {
        double a0 = q0 ? q0[p] : 0.0;
        int64_t i = pmod((int64_t)floor(a0 + 0.5), n0);
        int64_t j = pmod((int64_t)floor(q1[p] + 0.5), n1);
        int64_t k = pmod((int64_t)floor(q2[p] + 0.5), n2);
        out[p] = vals[(i * n1 + j) * n2 + k];
    }
}
