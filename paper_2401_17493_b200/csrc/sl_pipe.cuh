// Persistent, double-buffered TMA pipeline for the fp32 SL gather steps
// (sm_100a).  Same tiles (32 x 8 x 4 voxels, 4 per thread along axis 0), tile
// plans, TMA boxes and stencils as k_slf (sl_fast.cuh); different execution
// model:
//
//  * one CTA of PIPE_GROUPS x 256 threads per SM, looping over the tiles; group
//    g takes tiles blockIdx.x + (g + GROUPS * n) * gridDim.x (tiles running at
//    the same time are neighbours, so the boxes they share stay in L2);
//  * each group owns two box slots: while it computes tile n from one, the TMA
//    of the next box is already in flight into the other, and the displacement
//    / epilogue loads of tile n + 1 are issued before tile n is computed —
//    k_slf pays the box and the per-voxel latencies once per CTA with only 4
//    CTAs per SM to cover them;
//  * no producer warp (it would cost the consumers registers: 17 warps per SM
//    cap them at 96): thread 0 of the group re-arms a slot (waits for the
//    group's 8 warps on the slot's `empty` mbarrier, issues the TMA that
//    completes its `full` mbarrier) right after the group consumed it.
//
// Tiles whose stencil box does not fit the fixed box gather from global memory;
// tiles touching the periodic boundary patch box rows / columns from their
// images (4-byte cp.async by the group + the group's named barrier), as k_slf.
#pragma once

#include "sl_fast.cuh"

namespace frg {

#ifndef FRG_PIPE_GROUPS
#define FRG_PIPE_GROUPS 2
#endif
// consumer groups of BX x BY threads (one tile each, 4 voxels per thread along
// axis 0 as k_slf); group g takes the CTA's tiles it = g, g + GROUPS, ...
constexpr int PIPE_GROUPS = FRG_PIPE_GROUPS;
constexpr int PIPE_GTHREADS = BX * BY;
constexpr int PIPE_GWARPS = PIPE_GTHREADS / 32;
constexpr int PIPE_THREADS = PIPE_GROUPS * PIPE_GTHREADS;
#ifndef FRG_PIPE_GSLOTS
#define FRG_PIPE_GSLOTS 3
#endif
constexpr int PIPE_GSLOTS = FRG_PIPE_GSLOTS;  // box slots per group
constexpr int PIPE_SLOTS = PIPE_GSLOTS * PIPE_GROUPS;
// box geometry of the pipeline (planes x rows x columns): sized to the tile's
// stencil box with a few cells of displacement spread (tile 4 x 8 x 32 +
// 3-cell stencil: <= 4 + 3 + 3 planes, 8 + 3 + 3 rows), row pitch 64 (= 0 mod
// 32 banks), so that 3 boxes per group fit in shared memory
#ifndef FRG_PB_I
#define FRG_PB_I 10
#endif
#ifndef FRG_PB_J
#define FRG_PB_J 14
#endif
#ifndef FRG_PB_K
#define FRG_PB_K 64
#endif
constexpr int PB_I = FRG_PB_I, PB_J = FRG_PB_J, PB_K = FRG_PB_K;
constexpr int PB_PLANE = PB_J * PB_K, PB_VOL = PB_I * PB_PLANE;
static_assert(PB_PLANE % 32 == 0, "TMA destinations (box planes) must be 128-byte aligned");
static_assert(PB_K % 4 == 0 && PB_K <= 256 && PB_J <= 256, "pipeline box within the TMA box limits");

struct SlpSmem {
    static constexpr size_t bytes = (size_t)PIPE_SLOTS * PB_VOL * sizeof(float) + 1024;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier of one consumer group (id 1 + g; 0 is __syncthreads)
__device__ __forceinline__ void group_sync(int g) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "n"(PIPE_GTHREADS) : "memory");
}
__device__ __forceinline__ bool plan_fits(const int4& pe) {
    return (pe.w & 1023) <= PB_I && ((pe.w >> 10) & 1023) <= PB_J && ((pe.w >> 20) & 1023) <= PB_K;
}

// tile index -> (bx, by, bz), advanced by a fixed stride without divisions
struct TileWalk {
    int bx, by, bz, sx, sy, sz, gx, gy;
    __device__ __forceinline__ void init(int t, int stride, int gx_, int gy_) {
        gx = gx_;
        gy = gy_;
        bx = t % gx;
        by = (t / gx) % gy;
        bz = t / (gx * gy);
        sx = stride % gx;
        sy = (stride / gx) % gy;
        sz = stride / (gx * gy);
    }
    __device__ __forceinline__ void next() {
        bx += sx;
        int cy = 0;
        if (bx >= gx) {
            bx -= gx;
            cy = 1;
        }
        by += sy + cy;
        int cz = 0;
        if (by >= gy) {
            by -= gy;
            cz = 1;
        }
        bz += sz + cz;
    }
};

// per-tile consumer inputs (loaded one tile ahead)
template <class Op>
struct SlpIn {
    int4 pe;
    bool ok[SL_TI];
    float d[SL_TI][3];
    typename PreOf<Op>::type pre[SL_TI];
};

template <class Op>
__device__ __forceinline__ void slp_load(const Op& op, const Dims& g, int t, const TileWalk& w, int k, int j,
                                         SlpIn<Op>& in) {
    in.pe = __ldg(op.ds.plan + t);
    const int plane = g.n1 * g.n2;
    const int p0 = (w.bz * SL_TI * g.n1 + j) * g.n2 + k;
#pragma unroll
    for (int u = 0; u < SL_TI; ++u) {
        in.ok[u] = k < g.n2 && j < g.n1 && w.bz * SL_TI + u < g.n0;
        in.d[u][0] = in.d[u][1] = in.d[u][2] = 0.f;
        if (in.ok[u]) op.disp(p0 + u * plane, in.d[u][0], in.d[u][1], in.d[u][2]);
    }
    if constexpr (HasPre<Op>::value) {
#pragma unroll
        for (int u = 0; u < SL_TI; ++u)
            if (in.ok[u]) in.pre[u] = op.pre(p0 + u * plane);
    }
}

template <int M, int NF, class Op>
__global__ void __launch_bounds__(PIPE_THREADS, 1)
    k_slp(Dims g, Op op, const __grid_constant__ TmaMaps<NF> maps, int ntiles, int gx, int gy) {
    static_assert(M == LINEAR || M == CUBIC || M == BSPLINE, "k_slp: linear / cubic / B-spline only");
    static_assert(SL_TI % 2 == 0, "k_slp pairs the voxels of a thread");
    extern __shared__ __align__(16) unsigned char sdyn[];
    float* sbox = reinterpret_cast<float*>(sdyn + ((1024u - (smem_u32(sdyn) & 1023u)) & 1023u));
    __shared__ __align__(8) uint64_t full[PIPE_SLOTS], empty[PIPE_SLOTS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < PIPE_SLOTS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], PIPE_GWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // group-local position q = n * NF + f (tile n of the group, field f) lives
    // in slot GSLOTS g + q % GSLOTS, phase (q / GSLOTS) & 1; every position takes a slot
    // (tiles that are empty or do not fit get a plain arrive instead of a TMA)
    const int grp = warp / PIPE_GWARPS, gtid = tid - grp * PIPE_GTHREADS;
    const int tx = gtid & (BX - 1), ty = gtid / BX;
    const int stride = PIPE_GROUPS * gridDim.x;
    const int t0 = blockIdx.x + grp * gridDim.x;
    if (t0 >= ntiles) return;
    auto arm = [&](int q, const int4& pe) {  // thread gtid == 0: load position q into its slot
        const int slot = PIPE_GSLOTS * grp + q % PIPE_GSLOTS;
        const int f = q % NF;
        if (pe.w >= 0 && plan_fits(pe)) {
            fence_proxy_async();
            tma_box<PB_PLANE>(sbox + slot * PB_VOL, &maps.m[f], g, pe.x, pe.y, pe.z, pe.w & 1023, &full[slot]);
        } else {
            mbar_arrive(&full[slot]);
        }
    };
    int t = t0;
    TileWalk w;
    w.init(t, stride, gx, gy);
    SlpIn<Op> nxt;
    slp_load(op, g, t, w, w.bx * BX + tx, w.by * BY + ty, nxt);
    auto plan_of = [&](int m) {  // plan entry of the group's tile m (empty past the end)
        const int tm = t0 + m * stride;
        return tm < ntiles ? __ldg(op.ds.plan + tm) : make_int4(0, 0, 0, -1);
    };
    if (gtid == 0)
        for (int q = 0; q < PIPE_GSLOTS; ++q)
            if (t0 + (q / NF) * stride < ntiles) arm(q, plan_of(q / NF));
    // tiles whose boxes are armed while tile n is computed: positions
    // n NF + f + GSLOTS, f < NF, i.e. tiles n + A .. n + B
    constexpr int A = PIPE_GSLOTS / NF, B = (NF - 1 + PIPE_GSLOTS) / NF;
    static_assert(B - A <= 1, "at most two tiles re-armed per tile");
    const int plane = g.n1 * g.n2;
    for (int n = 0; t < ntiles; t += stride, ++n) {
        const SlpIn<Op> cur = nxt;
        const int k = w.bx * BX + tx, j = w.by * BY + ty, ib = w.bz * SL_TI;
        w.next();
        if (t + stride < ntiles) slp_load(op, g, t + stride, w, w.bx * BX + tx, w.by * BY + ty, nxt);
        int4 peA = make_int4(0, 0, 0, -1), peB = peA;  // issuer: plans of tiles n + A, n + B (in flight meanwhile)
        if (gtid == 0) {
            peA = A == 1 ? nxt.pe : plan_of(n + A);
            peB = B == A ? peA : plan_of(n + B);
        }
        const bool live = cur.pe.w >= 0;
        const bool fits = live && plan_fits(cur.pe);
        const int lo0 = cur.pe.x, lo1 = cur.pe.y, lo2 = cur.pe.z;
        const int S0 = cur.pe.w & 1023, S1 = (cur.pe.w >> 10) & 1023, S2 = (cur.pe.w >> 20) & 1023;
        int b0[SL_TI], b1[SL_TI], b2[SL_TI];
        float fr0[SL_TI], fr1[SL_TI], fr2[SL_TI];
#pragma unroll
        for (int u = 0; u < SL_TI; ++u) {
            const float f0 = floorf(cur.d[u][0]), f1 = floorf(cur.d[u][1]), f2 = floorf(cur.d[u][2]);
            b0[u] = ib + u + (int)f0;
            b1[u] = j + (int)f1;
            b2[u] = k + (int)f2;
            fr0[u] = cur.d[u][0] - f0;
            fr1[u] = cur.d[u][1] - f1;
            fr2[u] = cur.d[u][2] - f2;
        }
        float vals[SL_TI][NF];
        const bool wrap = lo1 < 0 || lo1 + S1 > g.n1 || lo2 < 0 || lo2 + S2 > g.n2;
        int off[SL_TI];
#pragma unroll
        for (int u = 0; u < SL_TI; ++u)
            off[u] = cur.ok[u] ? ((b0[u] - Halo<M>::lo - lo0) * PB_J + (b1[u] - Halo<M>::lo - lo1)) * PB_K +
                                     (b2[u] - Halo<M>::lo - lo2)
                               : 0;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const int q = n * NF + f, slot = PIPE_GSLOTS * grp + q % PIPE_GSLOTS;
            const unsigned par = (unsigned)(q / PIPE_GSLOTS) & 1u;
            float* box = sbox + slot * PB_VOL;
            mbar_wait_sleep(&full[slot], par);
            if (fits) {
                if (wrap) {
                    const float* src = op.field(f);
                    patch_axis<PB_J, PB_K>(box, src, g, lo0, lo1, lo2, S0, S1, S2, 1, gtid, PIPE_GTHREADS);
                    patch_axis<PB_J, PB_K>(box, src, g, lo0, lo1, lo2, S0, S1, S2, 2, gtid, PIPE_GTHREADS);
                    cp_async_wait_all();
                    group_sync(grp);
                }
                if (M == CUBIC || M == BSPLINE) {
#pragma unroll
                    for (int u = 0; u < SL_TI; u += 2) {
                        float2 w0[4], w1[4], w2[4];
                        weights4f_x2<M>(make_float2(fr0[u], fr0[u + 1]), w0);
                        weights4f_x2<M>(make_float2(fr1[u], fr1[u + 1]), w1);
                        weights4f_x2<M>(make_float2(fr2[u], fr2[u + 1]), w2);
                        const float2 r = cubic_fixed_x2<PB_K, PB_PLANE>(box + off[u], box + off[u + 1], w0, w1, w2);
                        vals[u][f] = r.x;
                        vals[u + 1][f] = r.y;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < SL_TI; ++u) vals[u][f] = linear_fixed<PB_K, PB_PLANE>(box + off[u], fr0[u], fr1[u], fr2[u]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (gtid == 0) {
                // re-arm this slot with position q + GSLOTS once the whole group is done with it
                const int q2 = q + PIPE_GSLOTS, n2 = q2 / NF;
                if (t + (n2 - n) * stride < ntiles) {
                    mbar_wait(&empty[slot], par);
                    arm(q2, n2 == n + A ? peA : peB);
                }
            }
        }
        if (!live) continue;
        if (!fits) {
            Dims gsrc = g;
            gsrc.n0 = g.n0 + 2 * g.h0;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const float* src = op.field(f);
#pragma unroll
                for (int u = 0; u < SL_TI; ++u)
                    vals[u][f] = cur.ok[u] ? global_interp<float, M, float>(gsrc, src, b0[u] + g.h0, b1[u], b2[u],
                                                                            fr0[u], fr1[u], fr2[u])
                                           : 0.f;
            }
        }
        const int p0 = (ib * g.n1 + j) * g.n2 + k;
        if constexpr (HasTile<Op>::value) {
            op.template done_tile<SL_TI>(p0, plane, cur.ok, vals);
        } else {
#pragma unroll
            for (int u = 0; u < SL_TI; ++u)
                if (cur.ok[u]) {
                    if constexpr (HasPre<Op>::value)
                        op.done(p0 + u * plane, vals[u], cur.pre[u]);
                    else
                        op.done(p0 + u * plane, vals[u]);
                }
        }
    }
}

// Measured slower than k_slf and therefore off by default (256^3 planned cubic
// gather, CUDA events, L2 flushed): k_slf 175 us; this engine 246-263 us with 2
// groups (16 warps, 128 registers, 2 or 4 slots), 249 us with 3 slots of
// 64-column boxes, 302 / 327 us with 3 / 4 groups (80 / 64 registers, spills).
// ncu: issue 46-50 %, shared-pipe 50-57 %, only 16 warps per SM to hide the LDS
// and FMA latencies of the stencils, and the next tile's displacement /
// epilogue registers carried through the stencil cost occupancy; 48-column
// boxes (pitch 16 mod 32 banks) add bank conflicts.  Kept as a build option
// (-DFRG_USE_PIPE=1) with its parity tests passing.
#ifndef FRG_USE_PIPE
#define FRG_USE_PIPE 0
#endif

// host: runs the pipelined engine when it applies (fp32 field on a TMA-sized
// grid, the map has a tile plan for this method); false -> caller uses k_slf
template <int M, int NF, class Op>
bool launch_slp(const Dims& g, const Op& op, cudaStream_t st) {
    if constexpr (!FRG_USE_PIPE || !HasDs<Op>::value || HasTileSmem<Op>::value) {
        return false;
    } else {
        if (getenv("FRG_NO_PIPE")) return false;
        if (!op.ds.plan || plan_method(op.ds.plan) != M || !tma_grid_ok(g)) return false;
        TmaMaps<NF> maps;
        for (int f = 0; f < NF; ++f) encode_field_map(&maps.m[f], op.field(f), g, PB_K, PB_J);
        static int nsm = 0;
        static bool attr = false;  // per instantiation
        if (!attr) {
            FRG_CUDA(cudaFuncSetAttribute(k_slp<M, NF, Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)SlpSmem::bytes));
            int dev = 0;
            FRG_CUDA(cudaGetDevice(&dev));
            FRG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            attr = true;
        }
        const dim3 tg = sl_grid(g);
        const int ntiles = (int)(tg.x * tg.y * tg.z);
        const int grid = ntiles < nsm ? ntiles : nsm;
        k_slp<M, NF, Op><<<grid, PIPE_THREADS, SlpSmem::bytes, st>>>(g, op, maps, ntiles, (int)tg.x, (int)tg.y);
        FRG_CHECK_LAUNCH();
        return true;
    }
}

}  // namespace frg
