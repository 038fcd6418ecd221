// Shared-memory tiled semi-Lagrangian gather engine (sm_100a).
//
// One CTA owns an output tile of BX x BY x TI voxels (k fastest).  Each
// thread reads the displacement of its TI voxels, the CTA reduces the
// bounding box of every interpolation stencil in the tile (for the synthetic
// velocities a tile's departure points move coherently, so the box is the
// tile plus the intra-tile displacement spread plus 3 halo planes), stages
// each gathered field's box into shared memory with coalesced row loads
// (periodic wrap applied on load, optional f64->f32 conversion), and then
// evaluates the 64-tap cubic (8-tap linear, 1-tap nearest) stencils from
// shared memory.  Tiles whose box exceeds the shared-memory budget fall back
// to direct (L1/L2) gathers, so any displacement field is handled.
//
// The Op functor supplies: the displacement of a voxel (disp), the NF field
// pointers (field), and the pointwise epilogue (done) that consumes the NF
// gathered values — so every SL time step of the state, adjoint,
// incremental state / adjoint, RK2 departure, deformation-tensor and
// composition solves is ONE kernel.
#pragma once

#include <climits>
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace frg {

#ifndef SL_TI_OVERRIDE
#define SL_TI_OVERRIDE 4
#endif
constexpr int SL_TI = SL_TI_OVERRIDE;  // voxels per thread along axis 0

// box budget per CTA: 24 KB for fp32 (several CTAs per SM), 44 KB for the
// f64 parity path (static shared memory is limited to 48 KB)
template <typename T>
struct BoxCap {
    static constexpr int value = (sizeof(T) == 4 ? 32 * 1024 : 44 * 1024) / (int)sizeof(T);
};

// asynchronous global -> shared copy of one element (LDGSTS), no register staging
template <int BYTES>
__device__ __forceinline__ void cp_async_elem(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Stage box rows [lo0.., lo1.., lo2..] of field src into smem.  One warp per
// box row, lanes along the contiguous axis; every copy is issued before any
// is waited on, so the whole box is in flight at once.
// floor(e / d) for e, d < 2^16 with one IMAD.HI: m = floor(2^32 / d) + 1
__device__ __forceinline__ unsigned fast_div(unsigned e, unsigned m) { return __umulhi(e, m); }
__host__ __device__ __forceinline__ unsigned div_magic(unsigned d) {
    // floor((2^32 - 1) / d) + 1: exact floor(e / d) for e, d < 2^16 (32-bit division only)
    return 0xFFFFFFFFu / d + 1u;
}

// The box is flattened over all CTA threads (e = tid + 256 r), row / column
// recovered with multiply-high magic division — no integer division, every
// lane busy whatever the row length.
template <typename T, typename V>
__device__ __forceinline__ void stage_box(T* __restrict__ box, const V* __restrict__ src, const Dims& g, int lo0,
                                          int lo1, int lo2, int S1, int S2, int S2p, int vol, int tid) {
    const unsigned m2 = div_magic((unsigned)S2), m1 = div_magic((unsigned)S1);
    const bool inner_k = lo2 >= 0 && lo2 + S2 <= g.n2;
    auto addr = [&](int e, const V*& s, T*& d) {
        const int r = (int)fast_div((unsigned)e, m2);
        const int c = e - r * S2;
        const int a = (int)fast_div((unsigned)r, m1);
        const int b = r - a * S1;
        const int gi = wrap_near(lo0 + a, g.n0), gj = wrap_near(lo1 + b, g.n1);
        const int gk = inner_k ? lo2 + c : wrap_near(lo2 + c, g.n2);
        s = src + ((gi * g.n1 + gj) * g.n2 + gk);
        d = box + (r * S2p + c);
    };
    if constexpr (sizeof(T) == sizeof(V)) {
        for (int e = tid; e < vol; e += BX * BY) {
            const V* s;
            T* d;
            addr(e, s, d);
            cp_async_elem<sizeof(T)>(d, s);
        }
        cp_async_wait_all();
    } else {
        // converting copy through registers: batches of 8 independent loads in flight
        constexpr int B = 8;
        for (int e0 = tid; e0 < vol; e0 += B * BX * BY) {
            V v[B];
            T* d[B];
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const int e = e0 + q * BX * BY;
                const V* s;
                d[q] = nullptr;
                if (e < vol) {
                    addr(e, s, d[q]);
                    v[q] = __ldg(s);
                }
            }
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (d[q]) *d[q] = (T)v[q];
        }
    }
}

// 16-byte chunked staging (cp.async.cg 16 B): rows of the box are whole
// aligned chunks inside the period along k; one (row, chunk) per thread.
template <typename T>
__device__ __forceinline__ void stage_box_vec(T* __restrict__ box, const T* __restrict__ src, const Dims& g, int lo0,
                                              int lo1, int lo2, int S0, int S1, int S2c, int S2p, int tid) {
    constexpr int VEC = 16 / (int)sizeof(T);
    const unsigned mc = div_magic((unsigned)S2c), m1 = div_magic((unsigned)S1);
    const int total = S0 * S1 * S2c;
    for (int q = tid; q < total; q += BX * BY) {
        const int r = (int)fast_div((unsigned)q, mc);
        const int ch = q - r * S2c;
        const int a = (int)fast_div((unsigned)r, m1);
        const int b = r - a * S1;
        const int gi = wrap_near(lo0 + a, g.n0), gj = wrap_near(lo1 + b, g.n1);
        const T* s = src + ((gi * g.n1 + gj) * g.n2 + lo2 + ch * VEC);
        unsigned d = (unsigned)__cvta_generic_to_shared(box + (r * S2p + ch * VEC));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(s));
    }
    cp_async_wait_all();
}

// Ops may split their epilogue into a load phase (pre(p) -> Op::Pre, issued
// before the stencils are evaluated, so its latency hides behind them) and a
// compute/store phase (done(p, vals, pre)).  Ops without pre() get done(p, vals).
template <class Op, class = void>
struct HasPre : std::false_type {};
template <class Op>
struct HasPre<Op, std::void_t<decltype(std::declval<const Op&>().pre(0))>> : std::true_type {};

template <class Op, typename T, int NF>
__device__ __forceinline__ void op_done(const Op& op, int p, const T (&vals)[NF]) {
    if constexpr (HasPre<Op>::value)
        op.done(p, vals, op.pre(p));
    else
        op.done(p, vals);
}

template <int M>
struct Halo {
    static constexpr int lo = ((M == CUBIC || M == BSPLINE) ? 1 : 0);
    static constexpr int hi = ((M == CUBIC || M == BSPLINE) ? 2 : (M == LINEAR ? 1 : 0));
};

__device__ __forceinline__ int warp_min_i(int v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_max_i(int v) { return __reduce_max_sync(0xffffffffu, v); }

// evaluate one stencil from the staged box (no wrap needed inside the box)
template <typename T, int M>
__device__ __forceinline__ T box_interp(const T* __restrict__ box, int S1, int S2, int r0, int r1, int r2, T t0,
                                        T t1, T t2) {
    // r_a = (base_a - lo_a): box coordinate of the first tap
    if (M == NEAREST) {
        return box[(r0 * S1 + r1) * S2 + r2];
    } else if (M == LINEAR) {
        const T* b = box + (r0 * S1 + r1) * S2 + r2;
        T c00 = (T(1) - t2) * b[0] + t2 * b[1];
        T c01 = (T(1) - t2) * b[S2] + t2 * b[S2 + 1];
        T c10 = (T(1) - t2) * b[S1 * S2] + t2 * b[S1 * S2 + 1];
        T c11 = (T(1) - t2) * b[S1 * S2 + S2] + t2 * b[S1 * S2 + S2 + 1];
        return (T(1) - t0) * ((T(1) - t1) * c00 + t1 * c01) + t0 * ((T(1) - t1) * c10 + t1 * c11);
    } else {
        T w0[4], w1[4], w2[4];
        weights4<T, M>(t0, w0);
        weights4<T, M>(t1, w1);
        weights4<T, M>(t2, w2);
        const int sa = S1 * S2;
        const T* p0 = box + ((r0 * S1 + r1) * S2 + r2);
        T acc = T(0);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const T* row = p0;
            T plane = T(0);
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                T r = w2[0] * row[0];
                r += w2[1] * row[1];
                r += w2[2] * row[2];
                r += w2[3] * row[3];
                plane += w1[bb] * r;
                row += S2;
            }
            acc += w0[a] * plane;
            p0 += sa;
        }
        return acc;
    }
}

// stencil from a (wrapped) node base and fractional part, evaluated in global memory
template <typename T, int M, typename V>
__device__ __forceinline__ T global_interp(const Dims& g, const V* __restrict__ f, int b0, int b1, int b2, T t0, T t1,
                                           T t2) {
    Stencil<T, M> s;
    axis_stencil<T, M>(b0, t0, g.n0, g.n1 * g.n2, s.a0);
    axis_stencil<T, M>(b1, t1, g.n1, g.n2, s.a1);
    axis_stencil<T, M>(b2, t2, g.n2, 1, s.a2);
    return apply_stencil<T, T, M, V>(f, s);
}

// Generic tiled SL kernel.  T: arithmetic / box type; Op::V: source type of
// the gathered fields (may be wider than T: converted on staging).
template <typename T, int M, int NF, class Op>
__global__ void __launch_bounds__(BX * BY, (sizeof(T) == 4 && NF == 1) ? 4 : 2) k_sl(Dims g, Op op) {
    __shared__ __align__(16) T box[BoxCap<T>::value];
    __shared__ int red[6][BY];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int k = blockIdx.x * BX + tx;
    const int j = blockIdx.y * BY + ty;
    const int i_base = blockIdx.z * SL_TI;
    const bool in_kj = (k < g.n2) && (j < g.n1);

    int base0[SL_TI], base1[SL_TI], base2[SL_TI];
    T fr0[SL_TI], fr1[SL_TI], fr2[SL_TI];
    int mn0 = INT_MAX, mn1 = INT_MAX, mn2 = INT_MAX, mx0 = INT_MIN, mx1 = INT_MIN, mx2 = INT_MIN;
#pragma unroll
    for (int u = 0; u < SL_TI; ++u) {
        const int i = i_base + u;
        base0[u] = base1[u] = base2[u] = 0;
        fr0[u] = fr1[u] = fr2[u] = T(0);
        if (in_kj && i < g.n0) {
            const int p = (i * g.n1 + j) * g.n2 + k;
            T d0, d1, d2;
            op.disp(p, d0, d1, d2);
            if (M == NEAREST) {
                d0 += T(0.5);
                d1 += T(0.5);
                d2 += T(0.5);
            }
            T f0 = Real<T>::floor_(d0), f1 = Real<T>::floor_(d1), f2 = Real<T>::floor_(d2);
            base0[u] = i + (int)f0;
            base1[u] = j + (int)f1;
            base2[u] = k + (int)f2;
            fr0[u] = d0 - f0;
            fr1[u] = d1 - f1;
            fr2[u] = d2 - f2;
            mn0 = min(mn0, base0[u]);
            mx0 = max(mx0, base0[u]);
            mn1 = min(mn1, base1[u]);
            mx1 = max(mx1, base1[u]);
            mn2 = min(mn2, base2[u]);
            mx2 = max(mx2, base2[u]);
        }
    }
    // CTA-wide bounding box of the stencil bases
    mn0 = warp_min_i(mn0);
    mn1 = warp_min_i(mn1);
    mn2 = warp_min_i(mn2);
    mx0 = warp_max_i(mx0);
    mx1 = warp_max_i(mx1);
    mx2 = warp_max_i(mx2);
    if (tx == 0) {
        red[0][ty] = mn0;
        red[1][ty] = mn1;
        red[2][ty] = mn2;
        red[3][ty] = mx0;
        red[4][ty] = mx1;
        red[5][ty] = mx2;
    }
    __syncthreads();
    mn0 = red[0][0];
    mn1 = red[1][0];
    mn2 = red[2][0];
    mx0 = red[3][0];
    mx1 = red[4][0];
    mx2 = red[5][0];
#pragma unroll
    for (int w = 1; w < BY; ++w) {
        mn0 = min(mn0, red[0][w]);
        mn1 = min(mn1, red[1][w]);
        mn2 = min(mn2, red[2][w]);
        mx0 = max(mx0, red[3][w]);
        mx1 = max(mx1, red[4][w]);
        mx2 = max(mx2, red[5][w]);
    }
    if (mn0 == INT_MAX) return;  // empty tile (uniform across the CTA)
    const int lo0 = mn0 - Halo<M>::lo, lo1 = mn1 - Halo<M>::lo;
    int lo2 = mn2 - Halo<M>::lo;
    const int S0 = mx0 + Halo<M>::hi - lo0 + 1;
    const int S1 = mx1 + Halo<M>::hi - lo1 + 1;
    int S2 = mx2 + Halo<M>::hi - lo2 + 1;
    // 16-byte staging: widen the k-range to whole 16-byte chunks when the rows
    // need no periodic wrap along k (the common case)
    constexpr int VEC = 16 / (int)sizeof(T);
    bool vec = sizeof(T) == sizeof(typename Op::V) && (g.n2 % VEC) == 0 && lo2 >= 0;
    if (vec) {
        const int a2 = lo2 - lo2 % VEC;
        const int w = ((S2 + (lo2 - a2) + VEC - 1) / VEC) * VEC;
        if (a2 + w <= g.n2) {
            lo2 = a2;
            S2 = w;
        } else {
            vec = false;
        }
    }
    // rows padded to 32 elements: lanes of a warp on different box rows then
    // never hit the same shared-memory bank (their columns differ by < 32)
    const int S2p = (S2 + 31) & ~31;
    const long long vol = (long long)S0 * S1 * S2;
    const bool fits = (long long)S0 * S1 * S2p <= BoxCap<T>::value;

    T vals[SL_TI][NF];
    if (fits) {
        const int tid = ty * BX + tx;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            if (f > 0) __syncthreads();
            const typename Op::V* src = op.field(f);
            if (vec && (((uintptr_t)src & 15) == 0))
                stage_box_vec<T>(box, (const T*)src, g, lo0, lo1, lo2, S0, S1, S2 / VEC, S2p, tid);
            else
                stage_box<T, typename Op::V>(box, src, g, lo0, lo1, lo2, S1, S2, S2p, (int)vol, tid);
            __syncthreads();
#pragma unroll
            for (int u = 0; u < SL_TI; ++u)
                vals[u][f] = (in_kj && i_base + u < g.n0)
                                 ? box_interp<T, M>(box, S1, S2p, base0[u] - Halo<M>::lo - lo0,
                                                    base1[u] - Halo<M>::lo - lo1, base2[u] - Halo<M>::lo - lo2,
                                                    fr0[u], fr1[u], fr2[u])
                                 : T(0);
        }
    } else {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const typename Op::V* src = op.field(f);
#pragma unroll
            for (int u = 0; u < SL_TI; ++u)
                vals[u][f] = (in_kj && i_base + u < g.n0)
                                 ? global_interp<T, M, typename Op::V>(g, src, base0[u], base1[u], base2[u], fr0[u],
                                                                       fr1[u], fr2[u])
                                 : T(0);
        }
    }
#pragma unroll
    for (int u = 0; u < SL_TI; ++u) {
        const int i = i_base + u;
        if (in_kj && i < g.n0) op_done(op, (i * g.n1 + j) * g.n2 + k, vals[u]);
    }
}

// ---------------------------------------------------------------------------
// displacement sources (per grid axis; axis 0 is absent in 2D)
// ---------------------------------------------------------------------------
// A displacement map may carry a TILE PLAN: per SL tile, the stencil bounding
// box (lo0, lo1, lo2 aligned down to 4, S0 | S1 << 10 | S2 << 20; w = -1 for an
// empty tile), computed once per map (k_tile_plan) and reused by every SL step
// on that map, so the SL kernels issue their box TMA as soon as the plan entry
// arrives instead of after a displacement load + block reduction.
template <typename T>
struct DispSrc {
    const T* a[3];
    const int4* plan;
    __device__ __forceinline__ void get(int p, T& d0, T& d1, T& d2) const {
        d0 = a[0] ? a[0][p] : T(0);
        d1 = a[1][p];
        d2 = a[2][p];
    }
};

// Host-side, thread-local binding of a displacement buffer to its plan for the
// duration of a scope (the context binds disp_f / disp_b around its solves);
// disp_src() attaches the plan when the map pointer and method match.
struct PlanBinding {
    const void* disp = nullptr;
    const int4* plan = nullptr;
    int method = -1;
};
inline thread_local PlanBinding g_plan_bind[2];
struct PlanScope {
    int slot;
    PlanScope(int s, const void* disp, const int4* plan, int method) : slot(s) {
        g_plan_bind[s].disp = disp;
        g_plan_bind[s].plan = plan;
        g_plan_bind[s].method = method;
    }
    ~PlanScope() { g_plan_bind[slot] = PlanBinding(); }
};
inline int plan_method(const int4* plan) {
    for (const PlanBinding& b : g_plan_bind)
        if (b.plan == plan) return b.method;
    return -1;
}

template <typename T>
inline DispSrc<T> disp_src(const Dims& g, const T* disp) {
    DispSrc<T> s;
    s.a[0] = s.a[1] = s.a[2] = nullptr;
    s.plan = nullptr;
    for (int c = 0; c < g.d; ++c) s.a[g.comp_axis(c)] = disp + (size_t)c * g.N;
    for (const PlanBinding& b : g_plan_bind)
        if (b.disp == (const void*)disp && b.plan) s.plan = b.plan;
    return s;
}

inline int tcode(float) { return F32; }
inline int tcode(double) { return F64; }


inline dim3 sl_grid(const Dims& g) {
    return dim3((g.n2 + BX - 1) / BX, (g.n1 + BY - 1) / BY, (g.n0 + SL_TI - 1) / SL_TI);
}

template <typename T, int NF, class Op>
void launch_sl_generic(const Dims& g, int method, const Op& op, cudaStream_t st) {
    FRG_REQUIRE(g.h0 == 0, "slab (ghost-plane) SL steps need fp32 linear / cubic transport");
    switch (method) {
        case NEAREST: k_sl<T, NEAREST, NF, Op><<<sl_grid(g), vox_block(), 0, st>>>(g, op); break;
        case LINEAR: k_sl<T, LINEAR, NF, Op><<<sl_grid(g), vox_block(), 0, st>>>(g, op); break;
        case CUBIC: k_sl<T, CUBIC, NF, Op><<<sl_grid(g), vox_block(), 0, st>>>(g, op); break;
        case BSPLINE: k_sl<T, BSPLINE, NF, Op><<<sl_grid(g), vox_block(), 0, st>>>(g, op); break;
        default: throw Error(E_ARG, "unknown interpolation method");
    }
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
