// Shared device/host definitions for libflowreg_b200 (sm_100a).
//
// Layout (fields.py:162,190,237): every field is C-order over
// (n0, n1, n2), last axis fastest.  2D grids are stored as (1, n0, n1): the
// size-1 leading axis is exact under every operator (interp weights (0,1,0,0),
// FD8 differences vanish, DFT frequency 0).  A vector field has d components
// (d = 2 or 3); component c differentiates / displaces along grid axis
// (3 - d) + c.  Time series are (n_t + 1, n0, n1, n2).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace frg {

// Slab decomposition (multi-GPU, dist.py): a rank owns n0 consecutive planes
// of a global grid with n0g planes along axis 0.  SOURCE fields of the SL
// gathers and FD8 stencils are then stored with h0 ghost planes before and
// after the owned planes ((n0 + 2 h0, n1, n2), pointer at the first ghost
// plane) and are not wrapped along axis 0; outputs, displacements and
// epilogue inputs stay (n0, n1, n2).  h0 == 0 / n0g == 0: the periodic
// single-GPU grid.
struct Dims {
    int n0, n1, n2;  // n0 == 1 for 2D grids
    long long N;     // n0 * n1 * n2
    int d;           // vector components (2 or 3)
    int h0 = 0;      // ghost planes of source fields along axis 0 (slab mode)
    int n0g = 0;     // global axis-0 length (slab mode), 0 = n0
    __host__ __device__ int axis_len(int a) const { return a == 0 ? n0 : (a == 1 ? n1 : n2); }
    // length of the full (global) axis: sets the grid spacing 2 pi / n
    __host__ __device__ int axis_glob(int a) const { return (a == 0 && n0g > 0) ? n0g : axis_len(a); }
    __host__ __device__ int comp_axis(int c) const { return (3 - d) + c; }
};

inline Dims make_dims(const int32_t n[3], int d) {
    Dims g;
    g.n0 = n[0];
    g.n1 = n[1];
    g.n2 = n[2];
    g.N = (long long)g.n0 * g.n1 * g.n2;
    g.d = d;
    g.h0 = 0;
    g.n0g = 0;
    return g;
}

// source plane of (unwrapped) plane index b along axis 0
__host__ __device__ __forceinline__ int src_plane(const Dims& g, int b) {
    if (g.h0 > 0) return b + g.h0;
    if ((unsigned)b < (unsigned)g.n0) return b;
    int r = b % g.n0;
    return r < 0 ? r + g.n0 : r;
}

// BSPLINE: cubic B-spline on prefiltered coefficients (the caller's field is
// prefiltered spectrally first, spectral.cu SK_BSPLINE_PREFILTER); same 4-tap
// stencil geometry as CUBIC.
enum Method { NEAREST = 0, LINEAR = 1, CUBIC = 2, BSPLINE = 3 };
enum DType { F32 = 0, F64 = 1, I32 = 2 };

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// status codes of the C-ABI (include/flowreg_b200.h)
constexpr int OK = 0;
constexpr int E_ARG = -1;
constexpr int E_NONFINITE = -2;
constexpr int E_CUDA = -3;
constexpr int E_CUFFT = -4;
constexpr int E_STATE = -5;

#define FRG_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::frg::Error(::frg::E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define FRG_CHECK_LAUNCH() FRG_CUDA(cudaGetLastError())

#define FRG_REQUIRE(cond, msg)                                \
    do {                                                      \
        if (!(cond)) throw ::frg::Error(::frg::E_ARG, (msg)); \
    } while (0)

constexpr double TWO_PI = 6.283185307179586476925286766559;

// number of SMs on B200; grids for grid-stride kernels are multiples of it
constexpr int NUM_SMS = 148;

inline int blocks_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return (int)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------------------
// periodic index helpers
// ---------------------------------------------------------------------------

// floor-mod of an integer (Python semantics, _kernels.py:107-118)
__host__ __device__ __forceinline__ int pmod(long long i, int n) {
    long long r = i % n;
    return (int)(r < 0 ? r + n : r);
}

template <typename T>
struct Real;
template <>
struct Real<float> {
    __device__ __forceinline__ static float floor_(float x) { return floorf(x); }
};
template <>
struct Real<double> {
    __device__ __forceinline__ static double floor_(double x) { return floor(x); }
};

// Lagrange cubic weights for nodes at offsets -1, 0, 1, 2 (_kernels.py:162-167)
// (divisions by 6 and 2 replaced by multiplications: no FCHK/slow-path division
// per weight; the difference is within one rounding of the reference's weights)
template <typename T>
__device__ __forceinline__ void lagrange4(T t, T w[4]) {
    const T one = T(1), two = T(2), sixth = T(1.0 / 6.0), half = T(0.5);
    const T tm1 = t - one, tm2 = t - two, tp1 = t + one;
    w[0] = -t * tm1 * tm2 * sixth;
    w[1] = tp1 * tm1 * tm2 * half;
    w[2] = -tp1 * t * tm2 * half;
    w[3] = tp1 * t * tm1 * sixth;
}

// uniform cubic B-spline weights at offsets -1, 0, 1, 2 (t in [0, 1))
template <typename T>
__device__ __forceinline__ void bspline4(T t, T w[4]) {
    const T sixth = T(1.0 / 6.0), omt = T(1) - t, t2 = t * t, t3 = t2 * t;
    w[0] = omt * omt * omt * sixth;
    w[1] = (T(3) * t3 - T(6) * t2 + T(4)) * sixth;
    w[2] = (T(-3) * t3 + T(3) * t2 + T(3) * t + T(1)) * sixth;
    w[3] = t3 * sixth;
}

template <typename T, int M>
__device__ __forceinline__ void weights4(T t, T w[4]) {
    if (M == BSPLINE)
        bspline4(t, w);
    else
        lagrange4(t, w);
}

// Periodic wrap of an index that is usually inside [0, n) or within a few
// periods of it: one unsigned compare on the common path, % only on wrap.
__device__ __forceinline__ int wrap_near(int b, int n) {
    if ((unsigned)b >= (unsigned)n) {
        b %= n;
        if (b < 0) b += n;
    }
    return b;
}

// Per-axis stencil: wrapped node indices (already multiplied by the axis
// stride, 32-bit: N < 2^31 for every grid up to 1024^3) and weights.
// NT = taps per axis (1 nearest, 2 linear, 4 cubic).
template <typename T, int NT>
struct Axis {
    int off[NT];
    T w[NT];
};

template <int M>
struct Taps {
    static constexpr int value = ((M == CUBIC || M == BSPLINE) ? 4 : (M == LINEAR ? 2 : 1));
};

// Build the axis stencil for node `base` (any integer, wrapped here) and
// fractional offset t in [0, 1).  For NEAREST, base = floor(q + 0.5).
template <typename T, int M>
__device__ __forceinline__ void axis_stencil(int base, T t, int n, int stride, Axis<T, Taps<M>::value>& ax) {
    if (M == NEAREST) {
        ax.off[0] = wrap_near(base, n) * stride;
        ax.w[0] = T(1);
    } else if (M == LINEAR) {
        int i0 = wrap_near(base, n);
        int i1 = i0 + 1;
        if (i1 >= n) i1 -= n;
        ax.off[0] = i0 * stride;
        ax.off[1] = i1 * stride;
        ax.w[0] = T(1) - t;
        ax.w[1] = t;
    } else {
        T w[4];
        weights4<T, M>(t, w);
        if (n == 1) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                ax.off[a] = 0;
                ax.w[a] = w[a];
            }
        } else {
            int b = wrap_near(base - 1, n);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                int x = b + a;
                if (x >= n) x -= n;  // n >= 4 for every axis longer than 1
                ax.off[a] = x * stride;
                ax.w[a] = w[a];
            }
        }
    }
}

// Full tensor-product stencil for one query point.
template <typename T, int M>
struct Stencil {
    Axis<T, Taps<M>::value> a0, a1, a2;
};

// floor(q) of an arbitrary f64 fractional index reduced into [0, n) first,
// so huge coordinates keep Python floor-mod semantics (_kernels.py:107-118).
__device__ __forceinline__ int reduce_index(double fl, int n) { return pmod((long long)fl, n); }

// Query point given as f64 fractional indices (the sample_nd boundary).
template <int M>
__device__ __forceinline__ void make_stencil_q(const Dims& g, double q0, double q1, double q2,
                                               Stencil<double, M>& s) {
    if (M == NEAREST) {
        axis_stencil<double, M>(reduce_index(floor(q0 + 0.5), g.n0), 0.0, g.n0, g.n1 * g.n2, s.a0);
        axis_stencil<double, M>(reduce_index(floor(q1 + 0.5), g.n1), 0.0, g.n1, g.n2, s.a1);
        axis_stencil<double, M>(reduce_index(floor(q2 + 0.5), g.n2), 0.0, g.n2, 1, s.a2);
    } else {
        double f0 = floor(q0), f1 = floor(q1), f2 = floor(q2);
        axis_stencil<double, M>(reduce_index(f0, g.n0), q0 - f0, g.n0, g.n1 * g.n2, s.a0);
        axis_stencil<double, M>(reduce_index(f1, g.n1), q1 - f1, g.n1, g.n2, s.a1);
        axis_stencil<double, M>(reduce_index(f2, g.n2), q2 - f2, g.n2, 1, s.a2);
    }
}

// Query point = grid node (i, j, k) + displacement (index units).  The
// integer part is split off exactly, so precision does not degrade with n.
template <typename T, int M>
__device__ __forceinline__ void make_stencil_disp(const Dims& g, int i, int j, int k, T d0, T d1, T d2,
                                                  Stencil<T, M>& s) {
    if (M == NEAREST) {
        axis_stencil<T, M>(i + (int)Real<T>::floor_(d0 + T(0.5)), T(0), g.n0, g.n1 * g.n2, s.a0);
        axis_stencil<T, M>(j + (int)Real<T>::floor_(d1 + T(0.5)), T(0), g.n1, g.n2, s.a1);
        axis_stencil<T, M>(k + (int)Real<T>::floor_(d2 + T(0.5)), T(0), g.n2, 1, s.a2);
    } else {
        T f0 = Real<T>::floor_(d0), f1 = Real<T>::floor_(d1), f2 = Real<T>::floor_(d2);
        axis_stencil<T, M>(i + (int)f0, d0 - f0, g.n0, g.n1 * g.n2, s.a0);
        axis_stencil<T, M>(j + (int)f1, d1 - f1, g.n1, g.n2, s.a1);
        axis_stencil<T, M>(k + (int)f2, d2 - f2, g.n2, 1, s.a2);
    }
}

// Apply a stencil to one field.  Accumulation order mirrors the reference:
// innermost over the last axis, then axis 1, then axis 0 (_kernels.py:207-219).
template <typename A, typename T, int M, typename V>
__device__ __forceinline__ A apply_stencil(const V* __restrict__ f, const Stencil<T, M>& s) {
    constexpr int NT = Taps<M>::value;
    if (M == NEAREST) {
        return (A)__ldg(f + (s.a0.off[0] + s.a1.off[0] + s.a2.off[0]));
    } else if (M == LINEAR) {
        A c[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const V* row = f + (s.a0.off[a] + s.a1.off[b]);
                c[a][b] = (A(1) - (A)s.a2.w[1]) * (A)__ldg(row + s.a2.off[0]) +
                          (A)s.a2.w[1] * (A)__ldg(row + s.a2.off[1]);
            }
        A t1 = (A)s.a1.w[1], t0 = (A)s.a0.w[1];
        return (A(1) - t0) * ((A(1) - t1) * c[0][0] + t1 * c[0][1]) +
               t0 * ((A(1) - t1) * c[1][0] + t1 * c[1][1]);
    } else {
        A acc = A(0);
#pragma unroll
        for (int a = 0; a < NT; ++a) {
            A plane = A(0);
#pragma unroll
            for (int b = 0; b < NT; ++b) {
                const V* row = f + (s.a0.off[a] + s.a1.off[b]);
                A r = A(0);
#pragma unroll
                for (int c = 0; c < NT; ++c) r += (A)s.a2.w[c] * (A)__ldg(row + s.a2.off[c]);
                plane += (A)s.a1.w[b] * r;
            }
            acc += (A)s.a0.w[a] * plane;
        }
        return acc;
    }
}

// ---------------------------------------------------------------------------
// voxel launch geometry: block (32, 8) over (k, j), grid z over i.  No
// integer division anywhere; the flat index fits in 32 bits.
// ---------------------------------------------------------------------------
#ifndef FRG_BY
#define FRG_BY 8
#endif
constexpr int BX = 32, BY = FRG_BY;

struct Vox {
    int i, j, k, p;
};

inline dim3 vox_grid(const Dims& g) { return dim3((g.n2 + BX - 1) / BX, (g.n1 + BY - 1) / BY, g.n0); }
inline dim3 vox_block() { return dim3(BX, BY, 1); }

__device__ __forceinline__ bool vox(const Dims& g, Vox& v) {
    v.k = blockIdx.x * BX + threadIdx.x;
    v.j = blockIdx.y * BY + threadIdx.y;
    v.i = blockIdx.z;
    if (v.k >= g.n2 || v.j >= g.n1) return false;
    v.p = (v.i * g.n1 + v.j) * g.n2 + v.k;
    return true;
}

// flat index -> (i, j, k)
__device__ __forceinline__ void unflatten(const Dims& g, long long p, int& i, int& j, int& k) {
    k = (int)(p % g.n2);
    long long r = p / g.n2;
    j = (int)(r % g.n1);
    i = (int)(r / g.n1);
}

}  // namespace frg
