// TMA-staged fp32 semi-Lagrangian gather engine (sm_100a).
//
// Same contract as k_sl (sl_tile.cuh: Op supplies disp / field / done), for
// fp32 fields gathered with LINEAR or CUBIC stencils — every fp32 SL step of
// the state, adjoint, incremental and departure solves.  Differences:
//
//  * the shared-memory box has a FIXED geometry TB_I x TB_J x TB_K (planes x
//    rows x columns), so every tap of a stencil is one LDS at a compile-time
//    immediate offset from a single per-voxel base address (no per-row
//    address arithmetic: 64 LDS + 84 FMA per cubic point);
//  * the box is filled by TMA (cp.async.bulk.tensor.2d over the field viewed
//    as (n0*n1) rows x n2 columns, one TB_J x TB_K load per needed plane,
//    issued by one thread and completed on an mbarrier): no per-element
//    staging instructions in the SM.  Periodic wrap: planes wrap exactly
//    (the plane index is reduced before the load); rows / columns leaving
//    the grid are patched with 4-byte cp.async from their periodic images
//    after the TMA lands.  Grids smaller than the box (tests, 2D) stage the
//    whole box with cp.async instead.  (per-plane 2D loads let the plane index
//    wrap exactly and load only the S0 planes a tile needs);
//  * multi-field gathers reuse the box: the TMA of field f+1 is issued as
//    soon as field f has been consumed;
//  * tiles whose stencil bounding box exceeds the fixed box gather straight
//    from global memory (any displacement field is handled).
#pragma once

#include <cuda.h>

#include <cstdlib>
#include <type_traits>

#include "sl_tile.cuh"

namespace frg {

// box: 64 x 16 x 12 fp32 = 48 KB.  TMA box starts must be 16-byte aligned
// along the contiguous axis (an unaligned start faults with an illegal
// instruction), so the column origin is rounded down to a multiple of 4.
// Row pitch 64 (= 0 mod 32 banks): lanes of a warp whose stencils sit on
// different box rows still hit distinct banks (their columns differ).
#ifndef FRG_SLF_MINB_MF
#define FRG_SLF_MINB_MF 3  // the same for multi-field gathers (single box)
#endif
#ifndef FRG_SLF_MINB_DB
#define FRG_SLF_MINB_DB 2  // the same for double-buffered multi-field gathers (FRG_SL_DB)
#endif
#ifndef FRG_SLF_MINB
#define FRG_SLF_MINB 4  // resident CTAs per SM the single-field engine is register-budgeted for
#endif
#ifndef FRG_TB_J
#define FRG_TB_J 16
#endif
#ifndef FRG_TB_I
#define FRG_TB_I 12
#endif
constexpr int TB_K = 64, TB_J = FRG_TB_J, TB_I = FRG_TB_I;
constexpr int TB_VOL = TB_K * TB_J * TB_I;
constexpr int TB_PLANE = TB_K * TB_J;

template <int NF>
struct alignas(64) TmaMaps {
    CUtensorMap m[NF];
};

// host: 2D tiled tensor map over an fp32 (n0, n1, n2) field viewed as
// (n0*n1, n2), box TB_J rows x TB_K columns
void encode_field_map(CUtensorMap* map, const float* ptr, const Dims& g, int box_k = TB_K, int box_j = TB_J);
// host: whether the TMA engine applies to this grid (every axis >= its box edge)
inline bool tma_grid_ok(const Dims& g) {
    return (g.h0 > 0 || g.n0 >= TB_I) && g.n1 >= TB_J && g.n2 >= TB_K && (g.n2 % 4) == 0;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(float* dst, const CUtensorMap* map, int col, int row, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(dst)),
        "l"((unsigned long long)map), "r"(col), "r"(row), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"((unsigned long long)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// host: 3D tiled map over `planes` stacked fp32 (n1, n2) planes, box 4 planes x BY rows x BX columns
// (the per-voxel streams of one SL tile)
void encode_tile_stream_map(CUtensorMap* map, const float* ptr, int n1, int n2, long long planes);

// issue the S0 plane loads of one field box (one thread)
template <int PLANE = TB_PLANE>
__device__ __forceinline__ void tma_box(float* box, const CUtensorMap* map, const Dims& g, int lo0, int lo1, int lo2,
                                        int S0, uint64_t* bar) {
    mbar_expect_tx(bar, (unsigned)(S0 * PLANE * sizeof(float)));
    for (int a = 0; a < S0; ++a) tma_load_2d(box + a * PLANE, map, lo2, src_plane(g, lo0 + a) * g.n1 + lo1, bar);
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Off-rank planes over NVLink peer memory (slab mode without ghost planes,
// dist.py peer mode).  Each rank exposes its owned planes of a gathered
// source in a window buffer mapped into every other rank (CUDA IPC); a plane
// index b of the local slab that falls outside [0, n0) is read from the rank
// that owns global plane rank * n0 + b — by TMA (one device-resident tensor
// map per rank and field) into the box, or by P2P loads in the per-voxel
// fallback and the periodic patches.  Exactly the stencil planes a tile needs
// cross NVLink, with no ghost-plane exchange and no limit on |disp_0|.
constexpr int PEER_MAX = 8;
struct PeerPlanes {
    int nranks = 0;  // 0: not in peer mode
    int rank = 0;
    const CUtensorMap* maps[3] = {nullptr, nullptr, nullptr};  // per field: nranks maps, rank r's window
    const float* base[3][PEER_MAX] = {};                       // per field, per rank: window base
};
// kernel argument: the peer tables in peer-mode instantiations, nothing in
// the single-GPU / ghost-plane ones (no registers, branches or parameter
// space spent on the common path)
template <bool PEER>
struct PeerArg : PeerPlanes {};
template <>
struct PeerArg<false> {};

// owner rank and its local plane of local plane index b (|b| < n0g)
__device__ __forceinline__ void peer_plane(const Dims& g, const PeerPlanes& pp, int b, int& owner, int& local) {
    int G = pp.rank * g.n0 + b;
    G = G < 0 ? G + g.n0g : (G >= g.n0g ? G - g.n0g : G);
    owner = G / g.n0;
    local = G - owner * g.n0;
}
__device__ __forceinline__ const float* peer_plane_ptr(const Dims& g, const PeerPlanes& pp, int f, int b) {
    int o, l;
    peer_plane(g, pp, b, o, l);
    return pp.base[f][o] + (size_t)l * g.n1 * g.n2;
}
template <int PLANE = TB_PLANE>
__device__ __forceinline__ void tma_box_peer(float* box, const PeerPlanes& pp, int f, const Dims& g, int lo0, int lo1,
                                             int lo2, int S0, uint64_t* bar) {
    mbar_expect_tx(bar, (unsigned)(S0 * PLANE * sizeof(float)));
    for (int a = 0; a < S0; ++a) {
        int o, l;
        peer_plane(g, pp, lo0 + a, o, l);
        tma_load_2d(box + a * PLANE, pp.maps[f] + o, lo2, l * g.n1 + lo1, bar);
    }
}
// per-voxel stencil with axis-0 planes resolved through the peer windows
template <int M>
__device__ __forceinline__ float peer_interp(const Dims& g, const PeerPlanes& pp, int f, int b0, int b1, int b2,
                                             float t0, float t1, float t2) {
    constexpr int NT = Taps<M>::value;
    Axis<float, NT> a0, a1, a2;
    axis_stencil<float, M>(0, t0, 1 << 30, 0, a0);  // weights only (no wrap along axis 0)
    axis_stencil<float, M>(b1, t1, g.n1, g.n2, a1);
    axis_stencil<float, M>(b2, t2, g.n2, 1, a2);
    const int first = b0 - Halo<M>::lo;
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < NT; ++a) {
        const float* __restrict__ pl = peer_plane_ptr(g, pp, f, first + a);
        float plane = 0.f;
#pragma unroll
        for (int b = 0; b < NT; ++b) {
            float row = 0.f;
#pragma unroll
            for (int c = 0; c < NT; ++c) row = fmaf(a2.w[c], __ldg(pl + a1.off[b] + a2.off[c]), row);
            plane = fmaf(a1.w[b], row, plane);
        }
        acc = fmaf(a0.w[a], plane, acc);
    }
    return acc;
}

// Lagrange cubic weights (nodes -1, 0, 1, 2; _kernels.py:162-167) in 3 FADD +
// 10 FMUL: the shared products t(t-1) and (t+1)(t-2) are formed once.
__device__ __forceinline__ void lagrange4f(float t, float (&w)[4]) {
    const float tm1 = t - 1.f, tm2 = t - 2.f, tp1 = t + 1.f;
    const float p = t * tm1, q = tp1 * tm2;
    w[0] = (p * tm2) * (-1.f / 6.f);
    w[1] = (q * tm1) * 0.5f;
    w[2] = (q * t) * -0.5f;
    w[3] = (p * tp1) * (1.f / 6.f);
}

// 64-tap cubic from a fixed-geometry box: every tap an immediate offset from p
template <int K = TB_K, int PLANE = TB_PLANE>
__device__ __forceinline__ float cubic_fixed(const float* __restrict__ p, const float (&w0)[4], const float (&w1)[4],
                                             const float (&w2)[4]) {
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        float plane = 0.f;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float* row = p + a * PLANE + b * K;
            float r = w2[0] * row[0];
            r = fmaf(w2[1], row[1], r);
            r = fmaf(w2[2], row[2], r);
            r = fmaf(w2[3], row[3], r);
            plane = fmaf(w1[b], r, plane);
        }
        acc = fmaf(w0[a], plane, acc);
    }
    return acc;
}

template <int K = TB_K, int PLANE = TB_PLANE>
__device__ __forceinline__ float linear_fixed(const float* __restrict__ b, float t0, float t1, float t2) {
    // same expression order as box_interp<LINEAR> / apply_stencil<LINEAR>
    float c00 = (1.f - t2) * b[0] + t2 * b[1];
    float c01 = (1.f - t2) * b[K] + t2 * b[K + 1];
    float c10 = (1.f - t2) * b[PLANE] + t2 * b[PLANE + 1];
    float c11 = (1.f - t2) * b[PLANE + K] + t2 * b[PLANE + K + 1];
    return (1.f - t0) * ((1.f - t1) * c00 + t1 * c01) + t0 * ((1.f - t1) * c10 + t1 * c11);
}

// copy the box elements whose coordinate along `axis` leaves [0, n) from their
// periodic images (after the TMA zero-filled them); 4-byte cp.async
template <int J = TB_J, int K = TB_K, class PlaneOf>
__device__ __forceinline__ void patch_axis_f(float* __restrict__ box, const PlaneOf& plane_of, const Dims& g,
                                             int lo0, int lo1, int lo2, int S0, int S1, int S2, int axis, int tid,
                                             int nthreads) {
    const int lo = axis == 0 ? lo0 : (axis == 1 ? lo1 : lo2);
    const int S = axis == 0 ? S0 : (axis == 1 ? S1 : S2);
    const int n = g.axis_len(axis);
    // out-of-range index ranges along the axis: [0, a_end) and [b_beg, S)
    const int a_end = lo < 0 ? min(-lo, S) : 0;
    const int b_beg = lo + S > n ? max(n - lo, 0) : S;
    const int cnt = a_end + (S - b_beg);
    if (cnt == 0) return;
    // the two other extents; the column patch (axis 2, after axis 1) skips the
    // rows the row patch already wrote (no duplicate writes of the corners)
    const int E1 = axis == 0 ? S1 : S0;           // outer of the remaining pair
    int E2 = axis == 2 ? S1 : S2;                 // inner of the remaining pair
    int r0 = 0;
    if (axis == 2) {
        r0 = lo1 < 0 ? min(-lo1, S1) : 0;
        E2 = (lo1 + S1 > g.n1 ? max(g.n1 - lo1, 0) : S1) - r0;
        if (E2 <= 0) return;
    }
    const int total = cnt * E1 * E2;
    // multiply-high division (exact below 2^16: every TB box; the pipe engine's larger boxes divide)
    const bool magic = total < 65536;
    const unsigned m2 = div_magic((unsigned)E2), m1 = div_magic((unsigned)E1);
    for (int e = tid; e < total; e += nthreads) {
        int r = magic ? (int)fast_div((unsigned)e, m2) : e / E2;
        const int in2 = e - r * E2;
        const int q = magic ? (int)fast_div((unsigned)r, m1) : r / E1;
        const int in1 = r - q * E1;
        const int x = q < a_end ? q : b_beg + (q - a_end);
        int a, b, c;
        if (axis == 0) {
            a = x; b = in1; c = in2;
        } else if (axis == 1) {
            a = in1; b = x; c = in2;
        } else {
            a = in1; b = r0 + in2; c = x;
        }
        const int gj = wrap_near(lo1 + b, g.n1), gk = wrap_near(lo2 + c, g.n2);
        cp_async_elem<4>(box + (a * J + b) * K + c, plane_of(lo0 + a) + (gj * g.n2 + gk));
    }
}
template <int J = TB_J, int K = TB_K>
__device__ __forceinline__ void patch_axis(float* __restrict__ box, const float* __restrict__ src, const Dims& g,
                                           int lo0, int lo1, int lo2, int S0, int S1, int S2, int axis, int tid,
                                           int nthreads = BX * BY) {
    const int lo = axis == 0 ? lo0 : (axis == 1 ? lo1 : lo2);
    const int S = axis == 0 ? S0 : (axis == 1 ? S1 : S2);
    const int n = g.axis_len(axis);
    const int a_end = lo < 0 ? min(-lo, S) : 0;
    const int b_beg = lo + S > n ? max(n - lo, 0) : S;
    const int cnt = a_end + (S - b_beg);
    if (cnt == 0) return;
    const int E1 = axis == 0 ? S1 : S0;
    int E2 = axis == 2 ? S1 : S2;
    int r0 = 0;
    if (axis == 2) {  // rows outside [0, n1) were written by the axis-1 patch
        r0 = lo1 < 0 ? min(-lo1, S1) : 0;
        E2 = (lo1 + S1 > g.n1 ? max(g.n1 - lo1, 0) : S1) - r0;
        if (E2 <= 0) return;
    }
    const int total = cnt * E1 * E2;
    // multiply-high division (exact below 2^16: every TB box; the pipe engine's larger boxes divide)
    const bool magic = total < 65536;
    const unsigned m2 = div_magic((unsigned)E2), m1 = div_magic((unsigned)E1);
    for (int e = tid; e < total; e += nthreads) {
        int r = magic ? (int)fast_div((unsigned)e, m2) : e / E2;
        const int in2 = e - r * E2;
        const int q = magic ? (int)fast_div((unsigned)r, m1) : r / E1;
        const int in1 = r - q * E1;
        const int x = q < a_end ? q : b_beg + (q - a_end);
        int a, b, c;
        if (axis == 0) {
            a = x; b = in1; c = in2;
        } else if (axis == 1) {
            a = in1; b = x; c = in2;
        } else {
            a = in1; b = r0 + in2; c = x;
        }
        const int gi = src_plane(g, lo0 + a), gj = wrap_near(lo1 + b, g.n1), gk = wrap_near(lo2 + c, g.n2);
        cp_async_elem<4>(box + (a * J + b) * K + c, src + ((gi * g.n1 + gj) * g.n2 + gk));
    }
}

// whole-box cp.async staging with wrap (grids smaller than the TMA box)
__device__ __forceinline__ void stage_fixed(float* __restrict__ box, const float* __restrict__ src, const Dims& g,
                                            int lo0, int lo1, int lo2, int S0, int S1, int S2, int tid) {
    const int total = S0 * S1 * S2;
    for (int e = tid; e < total; e += BX * BY) {
        int r = e / S2;
        const int c = e - r * S2;
        const int a = r / S1;
        const int b = r - a * S1;
        const int gi = src_plane(g, lo0 + a), gj = wrap_near(lo1 + b, g.n1), gk = wrap_near(lo2 + c, g.n2);
        cp_async_elem<4>(box + (a * TB_J + b) * TB_K + c, src + ((gi * g.n1 + gj) * g.n2 + gk));
    }
}

#ifndef FRG_SL_DB
#define FRG_SL_DB 0  // measured: 2 CTAs/SM with two 48 KB boxes lose more than the overlap gains
#endif
// Ops whose TMA-fed tile epilogue is prefetched into a second box-sized
// buffer while the gathers run (Op::kEarlyEpilogue, IncFirstOp)
template <class Op, class = void>
struct EarlyEpi : std::false_type {};
template <class Op>
struct EarlyEpi<Op, std::void_t<decltype(Op::kEarlyEpilogue)>> : std::bool_constant<Op::kEarlyEpilogue> {};

template <int NF, bool EARLY = false>
struct SlfSmem {
    // one 48 KB box per CTA for single-field steps (4 CTAs / SM); multi-field
    // gathers double-buffer (the next field's TMA overlaps this field's taps)
    static constexpr int NB = (NF > 1 && FRG_SL_DB) ? 2 : 1;
    // + 1 KB: the dynamic window is re-aligned to 1024 B in the kernel (the
    // compiler-placed start after the static shared variables is not)
    static constexpr size_t bytes = (size_t)(NB + (EARLY ? 1 : 0)) * TB_VOL * sizeof(float) + 1024;
};

// Ops may take the whole per-thread tile in one epilogue call (done_tile)
template <class Op, class = void>
struct HasTile : std::false_type {};
template <class Op>
struct HasTile<Op, std::void_t<decltype(&Op::template done_tile<SL_TI>)>> : std::true_type {};

template <class Op, class = void>
struct HasTileSmem : std::false_type {};
template <class Op>
struct HasTileSmem<Op, std::void_t<decltype(&Op::template done_tile_smem<SL_TI>)>> : std::true_type {};

template <class Op, class = void>
struct PreOf {
    struct type {};
};
template <class Op>
struct PreOf<Op, std::void_t<typename Op::Pre>> {
    using type = typename Op::Pre;
};

template <class Op, class = void>
struct HasDs : std::false_type {};
template <class Op>
struct HasDs<Op, std::void_t<decltype(std::declval<const Op&>().ds.plan)>> : std::true_type {};

__device__ __forceinline__ int4 encode_plan(int lo0, int lo1, int lo2, int S0, int S1, int S2) {
    return make_int4(lo0, lo1, lo2, min(S0, 1023) | (min(S1, 1023) << 10) | (min(S2, 1023) << 20));
}

// One CTA per SL tile (same decomposition as k_slf): the stencil bounding box
// of the tile's departure points -> plan[tile].
template <typename T, int M>
__global__ void __launch_bounds__(BX* BY) k_tile_plan(Dims g, DispSrc<T> ds, int4* __restrict__ plan) {
    __shared__ int bb[6];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
    const int k = blockIdx.x * BX + tx, j = blockIdx.y * BY + ty, i_base = blockIdx.z * SL_TI;
    if (tid < 6) bb[tid] = INT_MAX;
    int mn0 = INT_MAX, mn1 = INT_MAX, mn2 = INT_MAX, mx0 = INT_MIN, mx1 = INT_MIN, mx2 = INT_MIN;
    if (k < g.n2 && j < g.n1) {
#pragma unroll
        for (int u = 0; u < SL_TI; ++u) {
            const int i = i_base + u;
            if (i >= g.n0) continue;
            T d0, d1, d2;
            ds.get((i * g.n1 + j) * g.n2 + k, d0, d1, d2);
            const int b0 = i + (int)Real<T>::floor_(d0), b1 = j + (int)Real<T>::floor_(d1),
                      b2 = k + (int)Real<T>::floor_(d2);
            mn0 = min(mn0, b0);
            mx0 = max(mx0, b0);
            mn1 = min(mn1, b1);
            mx1 = max(mx1, b1);
            mn2 = min(mn2, b2);
            mx2 = max(mx2, b2);
        }
    }
    mn0 = warp_min_i(mn0);
    mn1 = warp_min_i(mn1);
    mn2 = warp_min_i(mn2);
    mx0 = warp_max_i(mx0);
    mx1 = warp_max_i(mx1);
    mx2 = warp_max_i(mx2);
    __syncthreads();
    if (tx == 0 && mn0 != INT_MAX) {
        atomicMin(&bb[0], mn0);
        atomicMin(&bb[1], mn1);
        atomicMin(&bb[2], mn2);
        atomicMin(&bb[3], -mx0);
        atomicMin(&bb[4], -mx1);
        atomicMin(&bb[5], -mx2);
    }
    __syncthreads();
    if (tid == 0) {
        const int t = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        if (bb[0] == INT_MAX) {
            plan[t] = make_int4(0, 0, 0, -1);
        } else {
            const int lo0 = bb[0] - Halo<M>::lo, lo1 = bb[1] - Halo<M>::lo, lo2 = (bb[2] - Halo<M>::lo) & ~3;
            plan[t] = encode_plan(lo0, lo1, lo2, -bb[3] + Halo<M>::hi - lo0 + 1, -bb[4] + Halo<M>::hi - lo1 + 1,
                                  -bb[5] + Halo<M>::hi - lo2 + 1);
        }
    }
}

// Lagrange weights for two points at once (Blackwell paired fp32: FADD2/FMUL2),
// lane-for-lane identical to lagrange4f
__device__ __forceinline__ void lagrange4f_x2(float2 t, float2 (&w)[4]) {
    const float2 tm1 = __fadd2_rn(t, make_float2(-1.f, -1.f)), tm2 = __fadd2_rn(t, make_float2(-2.f, -2.f));
    const float2 tp1 = __fadd2_rn(t, make_float2(1.f, 1.f));
    const float2 p = __fmul2_rn(t, tm1), q = __fmul2_rn(tp1, tm2);
    w[0] = __fmul2_rn(__fmul2_rn(p, tm2), make_float2(-1.f / 6.f, -1.f / 6.f));
    w[1] = __fmul2_rn(__fmul2_rn(q, tm1), make_float2(0.5f, 0.5f));
    w[2] = __fmul2_rn(__fmul2_rn(q, t), make_float2(-0.5f, -0.5f));
    w[3] = __fmul2_rn(__fmul2_rn(p, tp1), make_float2(1.f / 6.f, 1.f / 6.f));
}

// cubic B-spline weights for two points (paired fp32), lane-for-lane equal to bspline4<float>
__device__ __forceinline__ void bspline4f_x2(float2 t, float2 (&w)[4]) {
    const float2 sixth = make_float2(1.f / 6.f, 1.f / 6.f);
    const float2 omt = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-t.x, -t.y));
    const float2 t2 = __fmul2_rn(t, t), t3 = __fmul2_rn(t2, t);
    w[0] = __fmul2_rn(__fmul2_rn(__fmul2_rn(omt, omt), omt), sixth);
    float2 a = __fmul2_rn(make_float2(3.f, 3.f), t3);
    a = __fadd2_rn(a, __fmul2_rn(make_float2(-6.f, -6.f), t2));
    w[1] = __fmul2_rn(__fadd2_rn(a, make_float2(4.f, 4.f)), sixth);
    float2 b = __fmul2_rn(make_float2(-3.f, -3.f), t3);
    b = __fadd2_rn(b, __fmul2_rn(make_float2(3.f, 3.f), t2));
    b = __fadd2_rn(b, __fmul2_rn(make_float2(3.f, 3.f), t));
    w[2] = __fmul2_rn(__fadd2_rn(b, make_float2(1.f, 1.f)), sixth);
    w[3] = __fmul2_rn(t3, sixth);
}

template <int M>
__device__ __forceinline__ void weights4f_x2(float2 t, float2 (&w)[4]) {
    if (M == BSPLINE)
        bspline4f_x2(t, w);
    else
        lagrange4f_x2(t, w);
}

// two cubic stencils with paired FMAs: the taps of point A and point B load
// into the two halves of one register pair; lane-for-lane identical to
// cubic_fixed
template <int K = TB_K, int PLANE = TB_PLANE>
__device__ __forceinline__ float2 cubic_fixed_x2(const float* __restrict__ pA, const float* __restrict__ pB,
                                                 const float2 (&w0)[4], const float2 (&w1)[4],
                                                 const float2 (&w2)[4]) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        float2 plane = make_float2(0.f, 0.f);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float* rA = pA + a * PLANE + b * K;
            const float* rB = pB + a * PLANE + b * K;
            float2 r = __fmul2_rn(w2[0], make_float2(rA[0], rB[0]));
            r = __ffma2_rn(w2[1], make_float2(rA[1], rB[1]), r);
            r = __ffma2_rn(w2[2], make_float2(rA[2], rB[2]), r);
            r = __ffma2_rn(w2[3], make_float2(rA[3], rB[3]), r);
            plane = __ffma2_rn(w1[b], r, plane);
        }
        acc = __ffma2_rn(w0[a], plane, acc);
    }
    return acc;
}

// mbarrier wait with a suspend-time hint: the warp sleeps in hardware until
// the phase completes instead of spinning on try_wait (issue slots stay free)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 1000000;\n"
        "@!P1 bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Programmatic dependent launch (PDL): every SL step lets the next launch
// start as soon as all of its CTAs are resident, and waits for its
// predecessor's results only where it reads them — the plan / displacement
// loads and the stencil bases of step j+1 overlap the tail of step j (the
// displacement maps and plans of a solve are built long before its steps).
// Ops whose displacement is produced by the preceding SL launch (ComposeOp,
// DepartureOp's velocity) declare kLateDisp and wait before any load.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
template <class Op, class = void>
struct LateDisp : std::false_type {};
template <class Op>
struct LateDisp<Op, std::void_t<decltype(Op::kLateDisp)>> : std::bool_constant<Op::kLateDisp> {};

template <int M, int NF, class Op, bool PEER>
__global__ void __launch_bounds__(BX* BY, NF == 1 ? FRG_SLF_MINB
                                                   : (EarlyEpi<Op>::value     ? 2
                                                      : SlfSmem<NF>::NB == 2 ? FRG_SLF_MINB_DB
                                                                             : FRG_SLF_MINB_MF))
    k_slf(Dims g, const __grid_constant__ Op op, const __grid_constant__ TmaMaps<NF> maps, int use_tma,
          const __grid_constant__ PeerArg<PEER> pp) {
    static_assert(M == LINEAR || M == CUBIC || M == BSPLINE, "k_slf: linear / cubic / B-spline only");
    static_assert(SL_TI % 2 == 0, "k_slf pairs the voxels of a thread");
    extern __shared__ __align__(16) unsigned char sdyn[];
    // offset arithmetic on the shared array itself (not through uintptr_t) so
    // that the taps compile to LDS, not generic LD
    float* sbox = reinterpret_cast<float*>(sdyn + ((1024u - (smem_u32(sdyn) & 1023u)) & 1023u));
    constexpr int NB = SlfSmem<NF>::NB;
    __shared__ __align__(8) uint64_t bars[NB + 1];  // + the epilogue's (done_tile_smem TMA rounds)
    __shared__ int bb[6];  // min0, min1, min2, -max0, -max1, -max2 of the stencil bases
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
    const int k = blockIdx.x * BX + tx;
    const int j = blockIdx.y * BY + ty;
    const int i_base = blockIdx.z * SL_TI;
    const bool in_kj = (k < g.n2) && (j < g.n1);
    if (tid == 0) {
        for (int b = 0; b <= NB; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (tid < 6) bb[tid] = INT_MAX;
    __syncthreads();  // barrier + bb initialised before anyone uses them (nothing is in flight yet)
    griddep_launch_dependents();
    if constexpr (LateDisp<Op>::value) griddep_wait();

    const int4* plan = nullptr;
    if constexpr (HasDs<Op>::value) plan = op.ds.plan;
    int4 pe = make_int4(0, 0, 0, 0);
    if (plan) pe = __ldg(plan + (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);

    // every independent global load first (displacements, epilogue inputs,
    // plan entry), so the CTA pays one memory latency, not three in a row
    bool ok[SL_TI];
    float dsp[SL_TI][3];
    if constexpr (HasDs<Op>::value) {
        // the map's component pointers and the column offset once per thread
        // (DispSrc::get per voxel re-derived them under each voxel's predicate)
        const int plane = g.n1 * g.n2, p0 = (i_base * g.n1 + j) * g.n2 + k;
        const float* __restrict__ a0 = op.ds.a[0];
        const float* __restrict__ a1 = op.ds.a[1] + p0;
        const float* __restrict__ a2 = op.ds.a[2] + p0;
#pragma unroll
        for (int u = 0; u < SL_TI; ++u) {
            ok[u] = in_kj && i_base + u < g.n0;
            dsp[u][0] = dsp[u][1] = dsp[u][2] = 0.f;
            if (ok[u]) {
                dsp[u][0] = a0 ? __ldg(a0 + p0 + u * plane) : 0.f;
                dsp[u][1] = __ldg(a1 + u * plane);
                dsp[u][2] = __ldg(a2 + u * plane);
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < SL_TI; ++u) {
            const int i = i_base + u;
            ok[u] = in_kj && i < g.n0;
            dsp[u][0] = dsp[u][1] = dsp[u][2] = 0.f;
            if (ok[u]) op.disp((i * g.n1 + j) * g.n2 + k, dsp[u][0], dsp[u][1], dsp[u][2]);
        }
    }
    // the gathered sources and epilogue inputs may be the predecessor's outputs
    if constexpr (!LateDisp<Op>::value) griddep_wait();
    using PreT = typename PreOf<Op>::type;
    PreT pre[SL_TI];
    if constexpr (HasPre<Op>::value) {
#pragma unroll
        for (int u = 0; u < SL_TI; ++u)
            if (ok[u]) pre[u] = op.pre(((i_base + u) * g.n1 + j) * g.n2 + k);
    }

    int lo0, lo1, lo2, S0, S1, S2;
    if (plan) {
        // precomputed box: issue the TMA as soon as the plan entry arrives
        if (pe.w < 0) return;  // empty tile
        lo0 = pe.x;
        lo1 = pe.y;
        lo2 = pe.z;
        S0 = pe.w & 1023;
        S1 = (pe.w >> 10) & 1023;
        S2 = (pe.w >> 20) & 1023;
        if (tid == 0 && use_tma && S0 <= TB_I && S1 <= TB_J && S2 <= TB_K) {
            for (int b = 0; b < NB; ++b) {
                if constexpr (PEER)
                    tma_box_peer(sbox + b * TB_VOL, pp, b, g, lo0, lo1, lo2, S0, &bars[b]);
                else
                    tma_box(sbox + b * TB_VOL, &maps.m[b], g, lo0, lo1, lo2, S0, &bars[b]);
            }
            if constexpr (EarlyEpi<Op>::value)
                op.prefetch_epilogue(sbox + NB * TB_VOL, &bars[NB], make_int3(blockIdx.x * BX, blockIdx.y * BY, i_base));
        }
        // no CTA barrier here: the other warps go on with their displacement
        // arithmetic while thread 0 waits for the plan entry and issues the TMA
    }
    int base0[SL_TI], base1[SL_TI], base2[SL_TI];
    float fr0[SL_TI], fr1[SL_TI], fr2[SL_TI];
    int mn0 = INT_MAX, mn1 = INT_MAX, mn2 = INT_MAX, mx0 = INT_MIN, mx1 = INT_MIN, mx2 = INT_MIN;
#pragma unroll
    for (int u = 0; u < SL_TI; ++u) {
        const int i = i_base + u;
        const float d0 = dsp[u][0], d1 = dsp[u][1], d2 = dsp[u][2];
        const float f0 = floorf(d0), f1 = floorf(d1), f2 = floorf(d2);
        base0[u] = i + (int)f0;
        base1[u] = j + (int)f1;
        base2[u] = k + (int)f2;
        fr0[u] = d0 - f0;
        fr1[u] = d1 - f1;
        fr2[u] = d2 - f2;
        if (ok[u]) {
            mn0 = min(mn0, base0[u]);
            mx0 = max(mx0, base0[u]);
            mn1 = min(mn1, base1[u]);
            mx1 = max(mx1, base1[u]);
            mn2 = min(mn2, base2[u]);
            mx2 = max(mx2, base2[u]);
        }
    }
    if (!plan) {
    // CTA bounding box: warp REDUX, then 6 shared atomics per warp
    mn0 = warp_min_i(mn0);
    mn1 = warp_min_i(mn1);
    mn2 = warp_min_i(mn2);
    mx0 = warp_max_i(mx0);
    mx1 = warp_max_i(mx1);
    mx2 = warp_max_i(mx2);
    if (tx == 0 && mn0 != INT_MAX) {
        atomicMin(&bb[0], mn0);
        atomicMin(&bb[1], mn1);
        atomicMin(&bb[2], mn2);
        atomicMin(&bb[3], -mx0);
        atomicMin(&bb[4], -mx1);
        atomicMin(&bb[5], -mx2);
    }
    __syncthreads();
    mn0 = bb[0];
    if (mn0 == INT_MAX) return;  // empty tile (uniform across the CTA)
    mn1 = bb[1];
    mn2 = bb[2];
    mx0 = -bb[3];
    mx1 = -bb[4];
    mx2 = -bb[5];
    lo0 = mn0 - Halo<M>::lo;
    lo1 = mn1 - Halo<M>::lo;
    lo2 = (mn2 - Halo<M>::lo) & ~3;
    S0 = mx0 + Halo<M>::hi - lo0 + 1;
    S1 = mx1 + Halo<M>::hi - lo1 + 1;
    S2 = mx2 + Halo<M>::hi - lo2 + 1;
    if (tid == 0 && use_tma && S0 <= TB_I && S1 <= TB_J && S2 <= TB_K) {
        for (int b = 0; b < NB; ++b) {
            if constexpr (PEER)
                tma_box_peer(sbox + b * TB_VOL, pp, b, g, lo0, lo1, lo2, S0, &bars[b]);
            else
                tma_box(sbox + b * TB_VOL, &maps.m[b], g, lo0, lo1, lo2, S0, &bars[b]);
        }
        if constexpr (EarlyEpi<Op>::value)
            op.prefetch_epilogue(sbox + NB * TB_VOL, &bars[NB], make_int3(blockIdx.x * BX, blockIdx.y * BY, i_base));
    }
    }
    const bool fits = S0 <= TB_I && S1 <= TB_J && S2 <= TB_K;


    float vals[SL_TI][NF];
    if (fits) {
        // (planes never need a patch: tma_box / stage_fixed resolve them)
        const bool wrap = lo1 < 0 || lo1 + S1 > g.n1 || lo2 < 0 || lo2 + S2 > g.n2;
        // per-voxel smem offset of the first tap (same for every field)
        int off[SL_TI];
#pragma unroll
        for (int u = 0; u < SL_TI; ++u)  // inactive voxels read tap 0 (result discarded)
            off[u] = ok[u] ? ((base0[u] - Halo<M>::lo - lo0) * TB_J + (base1[u] - Halo<M>::lo - lo1)) * TB_K +
                                 (base2[u] - Halo<M>::lo - lo2)
                           : 0;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const float* src = op.field(f);
            float* box = sbox + (f % NB) * TB_VOL;
            if (use_tma) {
                mbar_wait_sleep(&bars[f % NB], (unsigned)((f / NB) & 1));
                if (wrap) {  // planes already wrapped by tma_box
                    if constexpr (PEER) {
                        auto of = [&](int b) { return peer_plane_ptr(g, pp, f, b); };
                        patch_axis_f<TB_J, TB_K>(box, of, g, lo0, lo1, lo2, S0, S1, S2, 1, tid, BX * BY);
                        patch_axis_f<TB_J, TB_K>(box, of, g, lo0, lo1, lo2, S0, S1, S2, 2, tid, BX * BY);
                    } else {
                        patch_axis(box, src, g, lo0, lo1, lo2, S0, S1, S2, 1, tid);
                        patch_axis(box, src, g, lo0, lo1, lo2, S0, S1, S2, 2, tid);
                    }
                    cp_async_wait_all();
                    __syncthreads();
                }
            } else {
                if (f > 0) __syncthreads();
                stage_fixed(box, src, g, lo0, lo1, lo2, S0, S1, S2, tid);
                cp_async_wait_all();
                __syncthreads();
            }
            if (M == CUBIC || M == BSPLINE) {
#pragma unroll
                for (int u = 0; u < SL_TI; u += 2) {
                    float2 w0[4], w1[4], w2[4];
                    weights4f_x2<M>(make_float2(fr0[u], fr0[u + 1]), w0);
                    weights4f_x2<M>(make_float2(fr1[u], fr1[u + 1]), w1);
                    weights4f_x2<M>(make_float2(fr2[u], fr2[u + 1]), w2);
                    const float2 r = cubic_fixed_x2(box + off[u], box + off[u + 1], w0, w1, w2);
                    vals[u][f] = r.x;
                    vals[u + 1][f] = r.y;
                }
            } else {
#pragma unroll
                for (int u = 0; u < SL_TI; ++u) vals[u][f] = linear_fixed(box + off[u], fr0[u], fr1[u], fr2[u]);
            }
            if (use_tma && f + NB < NF) {
                __syncthreads();  // every thread is done reading this buffer
                if (tid == 0) {
                    fence_proxy_async();
                    if constexpr (PEER)
                        tma_box_peer(box, pp, f + NB, g, lo0, lo1, lo2, S0, &bars[f % NB]);
                    else
                        tma_box(box, &maps.m[f + NB], g, lo0, lo1, lo2, S0, &bars[f % NB]);
                }
            }
        }
    } else {
        // source-grid view: ghost planes are ordinary planes of a taller grid
        Dims gsrc = g;
        gsrc.n0 = g.n0 + 2 * g.h0;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const float* src = op.field(f);
#pragma unroll
            for (int u = 0; u < SL_TI; ++u) {
                if constexpr (PEER)
                    vals[u][f] = ok[u] ? peer_interp<M>(g, pp, f, base0[u], base1[u], base2[u], fr0[u], fr1[u], fr2[u])
                                       : 0.f;
                else
                    vals[u][f] = ok[u] ? global_interp<float, M, float>(gsrc, src, base0[u] + g.h0, base1[u],
                                                                        base2[u], fr0[u], fr1[u], fr2[u])
                                       : 0.f;
            }
        }
    }
    if constexpr (HasTileSmem<Op>::value) {
        if (fits && 12 * SL_TI * BX * BY <= TB_VOL) {
            __syncthreads();  // the box is free once every thread is done with the last gather
            op.template done_tile_smem<SL_TI>((i_base * g.n1 + j) * g.n2 + k, g.n1 * g.n2, ok, vals, sbox, tid,
                                              BX * BY, &bars[NB], use_tma,
                                              make_int3(blockIdx.x * BX, blockIdx.y * BY, i_base),
                                              EarlyEpi<Op>::value && use_tma ? sbox + NB * TB_VOL : nullptr);
            return;
        }
    }
    if constexpr (HasTile<Op>::value) {
        op.template done_tile<SL_TI>((i_base * g.n1 + j) * g.n2 + k, g.n1 * g.n2, ok, vals);
        return;
    }
#pragma unroll
    for (int u = 0; u < SL_TI; ++u)
        if (ok[u]) {
            const int p = ((i_base + u) * g.n1 + j) * g.n2 + k;
            if constexpr (HasPre<Op>::value)
                op.done(p, vals[u], pre[u]);
            else
                op.done(p, vals[u]);
        }
}

// host: build the tile plan of an fp32 displacement map for `method`
// (plan: sl_grid(g) tiles of int4)
void build_tile_plan(const Dims& g, int method, const float* disp, int4* plan, cudaStream_t st);
inline size_t tile_plan_count(const Dims& g) {
    const dim3 gr = sl_grid(g);
    return (size_t)gr.x * gr.y * gr.z;
}

// host: peer windows registered by frg_peer_register (tma.cu); fills pp for
// the launch's source fields, false when field 0 is not a registered window
bool peer_planes_of(const Dims& g, const float* const* fields, int nf, PeerPlanes& pp);

template <int M, int NF, class Op>
void launch_slf(const Dims& g, const Op& op_in, cudaStream_t st) {
    Op op = op_in;
    if constexpr (HasDs<Op>::value)
        if (op.ds.plan && plan_method(op.ds.plan) != M) op.ds.plan = nullptr;
    TmaMaps<NF> maps;
    PeerPlanes pp;
    const float* fields[NF];
    for (int f = 0; f < NF; ++f) fields[f] = op.field(f);
    const bool peer = g.n0g > 0 && g.h0 == 0 && peer_planes_of(g, fields, NF, pp);
    FRG_REQUIRE(peer || g.n0g == 0 || g.h0 > 0, "slab gathers without ghost planes need registered peer windows");
    const int use_tma = (peer || tma_grid_ok(g)) ? 1 : 0;
    for (int f = 0; f < NF; ++f) {
        if (use_tma && !peer)
            encode_field_map(&maps.m[f], op.field(f), g);
        else
            memset(&maps.m[f], 0, sizeof(CUtensorMap));
    }
    constexpr size_t smem = SlfSmem<NF, EarlyEpi<Op>::value>::bytes;
    static bool attr_set[2] = {false, false};  // per instantiation
    if (!attr_set[peer]) {
        if (peer)
            FRG_CUDA(cudaFuncSetAttribute(k_slf<M, NF, Op, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        else
            FRG_CUDA(cudaFuncSetAttribute(k_slf<M, NF, Op, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        attr_set[peer] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = sl_grid(g);
    cfg.blockDim = vox_block();
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    // not inside CUDA-graph capture (the small-grid matvec graph measured
    // 151 -> 160 us at 64^3 with programmatic edges; eager launches gain)
    static const bool pdl = getenv("FRG_NO_PDL") == nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (pdl) FRG_CUDA(cudaStreamIsCapturing(st, &cs));
    cfg.attrs = at;
    cfg.numAttrs = (pdl && cs == cudaStreamCaptureStatusNone) ? 1 : 0;
    if (peer) {
        PeerArg<true> pa;
        static_cast<PeerPlanes&>(pa) = pp;
        FRG_CUDA(cudaLaunchKernelEx(&cfg, k_slf<M, NF, Op, true>, g, op, maps, use_tma, pa));
    } else {
        FRG_CUDA(cudaLaunchKernelEx(&cfg, k_slf<M, NF, Op, false>, g, op, maps, use_tma, PeerArg<false>()));
    }
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
