// 8th-order centred first derivatives with periodic wrap (diffops.py:76-129).
//
// Coordinates decrease with the index, so u(x - s h) sits at index j + s and
// u(x + s h) at j - s (diffops.py:80-95):
//   du/dx(j) = sum_{s=4..1} w_s (u[j+s] - u[j-s]) / (840 h),
//   w_4 = 3, w_3 = -32, w_2 = 168, w_1 = -672.
// One thread per voxel produces all d derivative components of one slice.
#include "ops.h"

namespace frg {

constexpr int FD_TPB = 256;

template <typename T>
__device__ __forceinline__ T fd8_line(const T* __restrict__ u, long long base, int j, int n, long long stride,
                                      T inv840h) {
    const T w[4] = {T(3), T(-32), T(168), T(-672)};  // s = 4, 3, 2, 1
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int s = 4 - k;
        int jp = j + s;
        if (jp >= n) jp -= n;
        int jm = j - s;
        if (jm < 0) jm += n;
        acc += w[k] * __ldg(u + base + jp * stride);
        acc -= w[k] * __ldg(u + base + jm * stride);
    }
    return acc * inv840h;
}

template <typename T>
__global__ void __launch_bounds__(FD_TPB) k_fd8_grad(Dims g, int nslices, const T* __restrict__ u,
                                                     T* __restrict__ out) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int sl = blockIdx.y;
    if (p >= g.N || sl >= nslices) return;
    int idx[3];
    unflatten(g, p, idx[0], idx[1], idx[2]);
    const T* us = u + (long long)sl * g.N;
    T* os = out + (long long)sl * g.d * g.N;
    const long long strides[3] = {(long long)g.n1 * g.n2, (long long)g.n2, 1};
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        int n = g.axis_len(a);
        long long base = p - (long long)idx[a] * strides[a];
        T inv = T(1) / (T(840) * T(TWO_PI / n));
        // reference divides by 840 h; multiply by the reciprocal is within 1 ulp
        os[(long long)c * g.N + p] = fd8_line<T>(us, base, idx[a], n, strides[a], inv);
    }
}

template <typename T>
__global__ void __launch_bounds__(FD_TPB) k_fd8_div(Dims g, const T* __restrict__ v, T* __restrict__ out) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    int idx[3];
    unflatten(g, p, idx[0], idx[1], idx[2]);
    const long long strides[3] = {(long long)g.n1 * g.n2, (long long)g.n2, 1};
    T acc = T(0);
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        int n = g.axis_len(a);
        long long base = p - (long long)idx[a] * strides[a];
        T inv = T(1) / (T(840) * T(TWO_PI / n));
        acc += fd8_line<T>(v + (long long)c * g.N, base, idx[a], n, strides[a], inv);
    }
    out[p] = acc;
}

void fd8_gradient(const Dims& g, int tdtype, int nslices, const void* u, void* out, cudaStream_t st) {
    for (int c = 0; c < g.d; ++c)
        FRG_REQUIRE(g.axis_len(g.comp_axis(c)) >= 9, "8th-order stencil needs n_i >= 9");
    dim3 grid(blocks_for(g.N, FD_TPB), nslices);
    if (tdtype == F64)
        k_fd8_grad<double><<<grid, FD_TPB, 0, st>>>(g, nslices, (const double*)u, (double*)out);
    else
        k_fd8_grad<float><<<grid, FD_TPB, 0, st>>>(g, nslices, (const float*)u, (float*)out);
    FRG_CHECK_LAUNCH();
}

void fd8_divergence(const Dims& g, int tdtype, const void* v, void* out, cudaStream_t st) {
    for (int c = 0; c < g.d; ++c)
        FRG_REQUIRE(g.axis_len(g.comp_axis(c)) >= 9, "8th-order stencil needs n_i >= 9");
    int nb = blocks_for(g.N, FD_TPB);
    if (tdtype == F64)
        k_fd8_div<double><<<nb, FD_TPB, 0, st>>>(g, (const double*)v, (double*)out);
    else
        k_fd8_div<float><<<nb, FD_TPB, 0, st>>>(g, (const float*)v, (float*)out);
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
