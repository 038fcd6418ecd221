// 8th-order centred first derivatives with periodic wrap (diffops.py:76-129).
//
// Coordinates decrease with the index, so u(x - s h) sits at index j + s and
// u(x + s h) at j - s (diffops.py:80-95):
//   du/dx(j) = sum_{s=4..1} w_s (u[j+s] - u[j-s]) / (840 h),
//   w_4 = 3, w_3 = -32, w_2 = 168, w_1 = -672.
// One thread per voxel produces all d derivative components of one slice;
// the (32, 8) block tile keeps the axis-1/axis-2 neighbours in L1.
#include "ops.h"

namespace frg {

template <typename T>
__device__ __forceinline__ T fd8_line(const T* __restrict__ u, int base, int j, int n, int stride, T inv840h) {
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

// Slab mode (g.h0 >= 4): sources carry h0 ghost planes, so the axis-0
// stencil reads planes i +- s of the taller source grid without wrapping
// (fd8_line with n = a length the offsets never reach).
template <typename T>
__device__ __forceinline__ T fd8_axis(const Dims& g, const T* __restrict__ us, const Vox& v, int a) {
    const int idx[3] = {v.i, v.j, v.k};
    const int strides[3] = {g.n1 * g.n2, g.n2, 1};
    const T inv = T(1) / (T(840) * T(TWO_PI / g.axis_glob(a)));
    const int ps = v.p + g.h0 * strides[0];  // voxel in the source grid
    if (a == 0 && g.h0 > 0)
        return fd8_line<T>(us, ps - (idx[0] + g.h0) * strides[0], idx[0] + g.h0, 1 << 30, strides[0], inv);
    return fd8_line<T>(us, ps - idx[a] * strides[a], idx[a], g.axis_len(a), strides[a], inv);
}

template <typename T>
__global__ void __launch_bounds__(BX * BY) k_fd8_grad(Dims g, int nslices, const T* __restrict__ u,
                                                     T* __restrict__ out) {
    Vox v;
    if (!vox(g, v)) return;
    const size_t Ns = (size_t)(g.n0 + 2 * g.h0) * g.n1 * g.n2;
    for (int sl = 0; sl < nslices; ++sl) {
        const T* us = u + (size_t)sl * Ns;
        T* os = out + (size_t)sl * g.d * g.N;
        for (int c = 0; c < g.d; ++c) os[(size_t)c * g.N + v.p] = fd8_axis<T>(g, us, v, g.comp_axis(c));
    }
}

template <typename T>
__global__ void __launch_bounds__(BX * BY) k_fd8_div(Dims g, const T* __restrict__ vf, T* __restrict__ out) {
    Vox v;
    if (!vox(g, v)) return;
    const size_t Ns = (size_t)(g.n0 + 2 * g.h0) * g.n1 * g.n2;
    T acc = T(0);
    for (int c = 0; c < g.d; ++c) acc += fd8_axis<T>(g, vf + (size_t)c * Ns, v, g.comp_axis(c));
    out[v.p] = acc;
}

void fd8_gradient(const Dims& g, int tdtype, int nslices, const void* u, void* out, cudaStream_t st) {
    FRG_REQUIRE(g.h0 == 0 || g.h0 >= 4, "slab FD8 needs >= 4 ghost planes");
    for (int c = 0; c < g.d; ++c)
        FRG_REQUIRE(g.axis_glob(g.comp_axis(c)) >= 9, "8th-order stencil needs n_i >= 9");
    if (tdtype == F64)
        k_fd8_grad<double><<<vox_grid(g), vox_block(), 0, st>>>(g, nslices, (const double*)u, (double*)out);
    else
        k_fd8_grad<float><<<vox_grid(g), vox_block(), 0, st>>>(g, nslices, (const float*)u, (float*)out);
    FRG_CHECK_LAUNCH();
}

void fd8_divergence(const Dims& g, int tdtype, const void* v, void* out, cudaStream_t st) {
    FRG_REQUIRE(g.h0 == 0 || g.h0 >= 4, "slab FD8 needs >= 4 ghost planes");
    for (int c = 0; c < g.d; ++c)
        FRG_REQUIRE(g.axis_glob(g.comp_axis(c)) >= 9, "8th-order stencil needs n_i >= 9");
    if (tdtype == F64)
        k_fd8_div<double><<<vox_grid(g), vox_block(), 0, st>>>(g, (const double*)v, (double*)out);
    else
        k_fd8_div<float><<<vox_grid(g), vox_block(), 0, st>>>(g, (const float*)v, (float*)out);
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
