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
        // difference first: a constant (or any even part) cancels exactly
        // before the weight is applied (w * a - w * b with a contracted FMA
        // leaves the rounding error of w * a: ~4e-16 for u = const)
        acc += w[k] * (__ldg(u + base + jp * stride) - __ldg(u + base + jm * stride));
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

// 2.5D-blocked gradient for single-GPU 3D grids: a CTA owns a 32 (k) x 8 (j)
// column block of one slice and marches along axis 0 through FD8_CHUNK
// planes.  The axis-0 derivative comes from a 9-value register window of
// the thread's own column, the in-plane derivatives from a shared-memory
// tile of the current plane with a 4-wide halo: ~3.5 loads per voxel instead
// of 25 (mostly L2 re-reads of neighbouring planes).  Same per-term order as
// fd8_line, so results are identical.
#ifndef FRG_FD8_CHUNK
#define FRG_FD8_CHUNK 16
#endif
constexpr int FD8_CHUNK = FRG_FD8_CHUNK;
// measured at 256^3 (5 fp32 slices / one divergence): chunk 32 -> 16 and 6
// CTAs per SM for the gradient: 448-499 -> 409 us; divergence 116 -> 111 us
#ifndef FRG_FD8_MINB
#define FRG_FD8_MINB 6
#endif

template <typename T>
__device__ __forceinline__ T fd8_taps(const T (&up)[5], const T (&um)[5], T inv840h) {
    const T w[4] = {T(3), T(-32), T(168), T(-672)};  // s = 4, 3, 2, 1
    T acc = T(0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int sh = 4 - q;
        acc += w[q] * (up[sh] - um[sh]);  // as fd8_line: exact cancellation of constants
    }
    return acc * inv840h;
}

// periodic plane index for i in [-n0, 2 n0) (the column marches never leave it)
__device__ __forceinline__ int wrap_plane(int i, int n0) { return i < 0 ? i + n0 : (i >= n0 ? i - n0 : i); }

template <typename T>
__global__ void __launch_bounds__(BX * BY, FRG_FD8_MINB) k_fd8_grad_col(Dims g, int nslices, int nchunk, const T* __restrict__ u,
                                                         T* __restrict__ out) {
    __shared__ T tile[BY + 8][BX + 8];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
    const int k = blockIdx.x * BX + tx, j = blockIdx.y * BY + ty;
    const int slice = blockIdx.z / nchunk, ch = blockIdx.z - slice * nchunk;
    const int ib = ch * FD8_CHUNK, ie = min(ib + FD8_CHUNK, g.n0);
    const int plane = g.n1 * g.n2;
    const T* __restrict__ us = u + (size_t)slice * g.N;
    const bool in = k < g.n2 && j < g.n1;
    const int cofs = in ? j * g.n2 + k : 0;  // this thread's column within a plane
    const T inv0 = T(1) / (T(840) * T(TWO_PI / g.n0)), inv1 = T(1) / (T(840) * T(TWO_PI / g.n1)),
            inv2 = T(1) / (T(840) * T(TWO_PI / g.n2));
    auto col = [&](int i) -> T { return __ldg(us + wrap_plane(i, g.n0) * plane + cofs); };
    T win[9];  // win[q] = u(i - 4 + q) of this column
#pragma unroll
    for (int q = 0; q < 8; ++q) win[q] = col(ib - 4 + q);
    const int kb = blockIdx.x * BX - 4, jb = blockIdx.y * BY - 4;
    // tile element e = tid + 256 q (q < 3) of the plane being prefetched
    constexpr int TW = BX + 8, TE = (BY + 8) * (BX + 8);
    int toff[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int e = tid + q * BX * BY;
        const int r = e / TW, c = e - r * TW;
        int jj = jb + r, kk = kb + c;
        jj = jj < 0 ? jj + g.n1 : (jj >= g.n1 ? jj - g.n1 : jj);
        kk = kk < 0 ? kk + g.n2 : (kk >= g.n2 ? kk - g.n2 : kk);
        toff[q] = e < TE ? jj * g.n2 + kk : 0;
    }
    T nxt[3];
    T wnext = col(ib + 4);
    const T* pl = us + ib * plane;  // plane ib
#pragma unroll
    for (int q = 0; q < 3; ++q) nxt[q] = __ldg(pl + toff[q]);
    T* flat = &tile[0][0];
    T* __restrict__ o = out + (size_t)slice * 3 * g.N + ib * plane + cofs;
    for (int i = ib; i < ie; ++i, o += plane) {
        __syncthreads();  // previous plane's tile fully consumed
#pragma unroll
        for (int q = 0; q < 3; ++q)
            if (q < 2 || tid + q * BX * BY < TE) flat[tid + q * BX * BY] = nxt[q];
        win[8] = wnext;
        __syncthreads();
        if (i + 1 < ie) {  // next plane in flight while this one is differentiated
            wnext = col(i + 5);
            pl += plane;
#pragma unroll
            for (int q = 0; q < 3; ++q) nxt[q] = __ldg(pl + toff[q]);
        }
        if (in) {
            T up[5], um[5];
#pragma unroll
            for (int sh = 1; sh <= 4; ++sh) {
                up[sh] = win[4 + sh];
                um[sh] = win[4 - sh];
            }
            o[0] = fd8_taps<T>(up, um, inv0);
#pragma unroll
            for (int sh = 1; sh <= 4; ++sh) {
                up[sh] = tile[ty + 4 + sh][tx + 4];
                um[sh] = tile[ty + 4 - sh][tx + 4];
            }
            o[g.N] = fd8_taps<T>(up, um, inv1);
#pragma unroll
            for (int sh = 1; sh <= 4; ++sh) {
                up[sh] = tile[ty + 4][tx + 4 + sh];
                um[sh] = tile[ty + 4][tx + 4 - sh];
            }
            o[2 * g.N] = fd8_taps<T>(up, um, inv2);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) win[q] = win[q + 1];
    }
}

// 2.5D-blocked divergence (3D, single GPU): the axis-0 term from a register
// window of v_0's column, the axis-1 / axis-2 terms from shared tiles of v_1
// (row halo) and v_2 (column halo) of the current plane; 16 bytes of HBM per
// voxel instead of ~25 L1/L2 loads.  Same summation order as k_fd8_div
// ((0 + d0) + d1) + d2 and the same taps as fd8_line, so results are identical.
template <typename T>
__global__ void __launch_bounds__(BX * BY) k_fd8_div_col(Dims g, int nchunk, const T* __restrict__ vf,
                                                        T* __restrict__ out) {
    __shared__ T t1[BY + 8][BX];      // v_1, rows j - 4 .. j + BY + 3
    __shared__ T t2[BY][BX + 8 + 1];  // v_2, columns k - 4 .. k + BX + 3 (+1: bank skew)
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
    const int k = blockIdx.x * BX + tx, j = blockIdx.y * BY + ty;
    const int ib = blockIdx.z * FD8_CHUNK, ie = min(ib + FD8_CHUNK, g.n0);
    const int plane = g.n1 * g.n2;
    const T* __restrict__ v0 = vf;
    const T* __restrict__ v1 = vf + (size_t)g.N;
    const T* __restrict__ v2 = vf + 2 * (size_t)g.N;
    const bool in = k < g.n2 && j < g.n1;
    const int cofs = in ? j * g.n2 + k : 0;
    const T inv0 = T(1) / (T(840) * T(TWO_PI / g.n0)), inv1 = T(1) / (T(840) * T(TWO_PI / g.n1)),
            inv2 = T(1) / (T(840) * T(TWO_PI / g.n2));
    const int kb = blockIdx.x * BX - 4, jb = blockIdx.y * BY - 4;
    // t1: (BY + 8) x BX = 512 elements -> 2 per thread; t2: BY x (BX + 8) = 320 -> 2 per thread (second partial)
    constexpr int E1 = (BY + 8) * BX, E2 = BY * (BX + 8);
    int o1[2], o2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        int e = tid + q * BX * BY;
        int r = e / BX, c = e - r * BX;
        int jj = jb + r, kk = blockIdx.x * BX + c;
        jj = jj < 0 ? jj + g.n1 : (jj >= g.n1 ? jj - g.n1 : jj);
        kk = kk >= g.n2 ? kk - g.n2 : kk;
        o1[q] = e < E1 ? jj * g.n2 + kk : 0;
        r = e / (BX + 8);
        c = e - r * (BX + 8);
        jj = blockIdx.y * BY + r;
        kk = kb + c;
        jj = jj >= g.n1 ? jj - g.n1 : jj;
        kk = kk < 0 ? kk + g.n2 : (kk >= g.n2 ? kk - g.n2 : kk);
        o2[q] = e < E2 ? jj * g.n2 + kk : 0;
    }
    auto col = [&](int i) -> T { return __ldg(v0 + wrap_plane(i, g.n0) * plane + cofs); };
    T win[9];
#pragma unroll
    for (int q = 0; q < 8; ++q) win[q] = col(ib - 4 + q);
    T wnext = col(ib + 4);
    int pofs = ib * plane;
    T n1v[2], n2v[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        n1v[q] = __ldg(v1 + pofs + o1[q]);
        n2v[q] = __ldg(v2 + pofs + o2[q]);
    }
    T* __restrict__ o = out + pofs + cofs;
    for (int i = ib; i < ie; ++i, o += plane) {
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int e = tid + q * BX * BY;
            if (e < E1) (&t1[0][0])[e] = n1v[q];
            if (e < E2) t2[e / (BX + 8)][e % (BX + 8)] = n2v[q];
        }
        win[8] = wnext;
        __syncthreads();
        if (i + 1 < ie) {
            wnext = col(i + 5);
            pofs += plane;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                n1v[q] = __ldg(v1 + pofs + o1[q]);
                n2v[q] = __ldg(v2 + pofs + o2[q]);
            }
        }
        if (in) {
            T up[5], um[5];
#pragma unroll
            for (int sh = 1; sh <= 4; ++sh) {
                up[sh] = win[4 + sh];
                um[sh] = win[4 - sh];
            }
            T acc = T(0);
            acc += fd8_taps<T>(up, um, inv0);
#pragma unroll
            for (int sh = 1; sh <= 4; ++sh) {
                up[sh] = t1[ty + 4 + sh][tx];
                um[sh] = t1[ty + 4 - sh][tx];
            }
            acc += fd8_taps<T>(up, um, inv1);
#pragma unroll
            for (int sh = 1; sh <= 4; ++sh) {
                up[sh] = t2[ty][tx + 4 + sh];
                um[sh] = t2[ty][tx + 4 - sh];
            }
            acc += fd8_taps<T>(up, um, inv2);
            *o = acc;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) win[q] = win[q + 1];
    }
}

void fd8_gradient(const Dims& g, int tdtype, int nslices, const void* u, void* out, cudaStream_t st) {
    if (g.d == 3 && g.h0 == 0 && g.n0 >= 9 && g.n1 >= 9 && g.n2 >= 9) {
        const int nchunk = (g.n0 + FD8_CHUNK - 1) / FD8_CHUNK;
        dim3 grid((g.n2 + BX - 1) / BX, (g.n1 + BY - 1) / BY, nslices * nchunk);
        if (tdtype == F64)
            k_fd8_grad_col<double><<<grid, vox_block(), 0, st>>>(g, nslices, nchunk, (const double*)u, (double*)out);
        else
            k_fd8_grad_col<float><<<grid, vox_block(), 0, st>>>(g, nslices, nchunk, (const float*)u, (float*)out);
        FRG_CHECK_LAUNCH();
        return;
    }
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
    if (g.d == 3 && g.h0 == 0 && g.n0 >= 9 && g.n1 >= 9 && g.n2 >= 9) {
        const int nchunk = (g.n0 + FD8_CHUNK - 1) / FD8_CHUNK;
        dim3 grid((g.n2 + BX - 1) / BX, (g.n1 + BY - 1) / BY, nchunk);
        if (tdtype == F64)
            k_fd8_div_col<double><<<grid, vox_block(), 0, st>>>(g, nchunk, (const double*)v, (double*)out);
        else
            k_fd8_div_col<float><<<grid, vox_block(), 0, st>>>(g, nchunk, (const float*)v, (float*)out);
        FRG_CHECK_LAUNCH();
        return;
    }
    if (tdtype == F64)
        k_fd8_div<double><<<vox_grid(g), vox_block(), 0, st>>>(g, (const double*)v, (double*)out);
    else
        k_fd8_div<float><<<vox_grid(g), vox_block(), 0, st>>>(g, (const float*)v, (float*)out);
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
