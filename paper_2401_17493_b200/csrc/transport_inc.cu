// Incremental state transport (transport.py:147-176): fused SL step kernels.
#include "ops.h"
#include "sl_half.cuh"

#include <type_traits>
#include <utility>
#include <vector>

namespace frg {

// Launch probe for bench.py: while armed, CUDA events bracket every IncFirstOp
// launch (the GN matvec's dominant kernel) on its own stream; frg_probe_read
// sums their durations.  Off (two branches per matvec) unless armed.
namespace {
struct Probe {
    bool armed = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
};
Probe& probe() {
    static Probe p;
    return p;
}
}  // namespace

void probe_arm(bool on) { probe().armed = on; }

void probe_read(double* total_ms, long long* count) {
    Probe& p = probe();
    double t = 0.0;
    for (auto& e : p.ev) {
        FRG_CUDA(cudaEventSynchronize(e.second));
        float ms = 0.f;
        FRG_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
        t += ms;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    *total_ms = t;
    *count = (long long)p.ev.size();
    p.ev.clear();
}

template <class F>
static void probed(cudaStream_t st, F&& launch) {
    Probe& p = probe();
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (p.armed) cudaStreamIsCapturing(st, &cs);
    if (!p.armed || cs != cudaStreamCaptureStatusNone) {
        launch();
        return;
    }
    cudaEvent_t a, b;
    FRG_CUDA(cudaEventCreate(&a));
    FRG_CUDA(cudaEventCreate(&b));
    FRG_CUDA(cudaEventRecord(a, st));
    launch();
    FRG_CUDA(cudaEventRecord(b, st));
    p.ev.emplace_back(a, b);
}

// ---------------------------------------------------------------------------
// incremental state (transport.py:147-176)
//   m~_{j+1} = m~_j(y) + S_j,   S_j = h/2 (f0 + f1),
//   f0 = -grad m_j(y) . v~(y),  f1 = -grad m_{j+1}(x) . v~(x);   m~_0 = 0.
// S_j does not depend on m~, so ONE kernel gathers v~(y) (3 fields) and forms
// every S_j from the per-velocity caches grad m_j(y) (grads_y) and grad m_j
// (grads); m~_1 = S_0 exactly (m~_0(y) = 0).  Each later step is then a
// single-field SL gather plus one add: m~_{j+1} = m~_j(y) + S_j.
// ---------------------------------------------------------------------------
template <typename T, int D>
struct IncFirstOp {
    using V = T;
    DispSrc<T> ds;
    const T* vtT[D];  // gathered source (slab: with ghost planes)
    const T* vl[D];   // v~ at the output voxels
    const T* gy;  // n_t x D x N, grad m_j at y
    const T* gx;  // (n_t + 1) x D x N, grad m_j at x
    size_t N;
    int n_t;
    T* m1;
    T* fin;
    T* S;  // (n_t - 1) x N: S_1 .. S_{n_t-1}
    T fsign, hh;
    // TMA-fed epilogue (fp32, 3D): the gradient slices of a tile arrive as
    // 4 KB boxes (4 planes x 8 rows x 32 columns, the tile's own voxels) issued
    // by one thread, instead of 24 per-element cp.async per voxel and their
    // address arithmetic (ncu: 264 integer instructions per voxel)
    alignas(64) CUtensorMap tm_gy;  // gy as n_t D n0 stacked planes
    alignas(64) CUtensorMap tm_gx;  // gx as (n_t + 1) D n0 stacked planes
    int tma_epi = 0, n0 = 0;
#ifndef FRG_INC_PREFETCH
#define FRG_INC_PREFETCH 0
#endif
    // round 0 of the TMA epilogue issued with the gather boxes into a second
    // 48 KB buffer (k_slf, EarlyEpi): 2 CTAs / SM instead of 3.  Measured
    // slower (matvec 3630 vs 3544 us at 256^3): build option, off
    static constexpr bool kEarlyEpilogue = FRG_INC_PREFETCH && std::is_same<T, float>::value && D == 3;
    __device__ __forceinline__ void issue_round(T* buf, uint64_t* ebar, int3 org, int j0, int nj, int nthreads) const {
        mbar_expect_tx(ebar, (unsigned)(nj * 2 * D * SL_TI * nthreads * sizeof(T)));
        for (int jj = 0; jj < nj; ++jj) {
            const int j = j0 + jj;
            for (int c = 0; c < D; ++c) {
                tma_load_3d(buf + (size_t)((jj * 2 * D + c) * SL_TI) * nthreads, &tm_gy, org.x, org.y,
                            (j * D + c) * n0 + org.z, ebar);
                tma_load_3d(buf + (size_t)((jj * 2 * D + D + c) * SL_TI) * nthreads, &tm_gx, org.x, org.y,
                            ((j + 1) * D + c) * n0 + org.z, ebar);
            }
        }
    }
    __device__ __forceinline__ void prefetch_epilogue(T* buf, uint64_t* ebar, int3 org) const {
        if (tma_epi) issue_round(buf, ebar, org, 0, n_t > 1 ? 2 : 1, BX * BY);
    }
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const { ds.get(p, d0, d1, d2); }
    __host__ __device__ __forceinline__ const T* field(int f) const { return vtT[f]; }
    void set_field(int f, const T* p) { vtT[f] = p; }
    // Tile epilogue (the TI voxels of one thread, p0 + u * pstride): the
    // gradient loads of all voxels for one j are independent read-only loads
    // in flight together, instead of one dependent round trip per voxel and j.
    template <int TI>
    __device__ __forceinline__ void done_tile(int p0, int pstride, const bool (&ok)[TI],
                                              const T (&vals)[TI][D]) const {
        T vx[TI][D];
#pragma unroll
        for (int u = 0; u < TI; ++u)
#pragma unroll
            for (int c = 0; c < D; ++c) vx[u][c] = ok[u] ? __ldg(vl[c] + p0 + u * pstride) : T(0);
        for (int j = 0; j < n_t; ++j) {
            const T* __restrict__ gyj = gy + (size_t)j * D * N + p0;
            const T* __restrict__ gxj = gx + (size_t)(j + 1) * D * N + p0;
            T sj[TI];
#pragma unroll
            for (int u = 0; u < TI; ++u) {
                T f0 = T(0), f1 = T(0);
                if (ok[u]) {
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        f0 -= __ldg(gyj + c * N + u * pstride) * vals[u][c];
                        f1 -= __ldg(gxj + c * N + u * pstride) * vx[u][c];
                    }
                }
                sj[u] = hh * (f0 + f1);
            }
#pragma unroll
            for (int u = 0; u < TI; ++u) {
                if (!ok[u]) continue;
                const int p = p0 + u * pstride;
                if (j == 0) {
                    if (m1) m1[p] = sj[u];
                    if (fin) fin[p] = fsign * sj[u];
                } else {
                    S[(size_t)(j - 1) * N + p] = sj[u];
                }
            }
        }
    }
    // Shared-memory-staged tile epilogue (fp32, after the last gather, when
    // the 48 KB box is free): the gradient slices of two time steps
    // (grad m_j(y) and grad m_{j+1}, 12 fields x TI voxels per thread) are
    // copied with cp.async all at once, so the epilogue pays ceil(n_t / 2)
    // memory round trips with 48 loads in flight per thread instead of n_t
    // round trips with 24.  Each thread reads back only what it copied: no
    // CTA barrier between the stages.
    template <int TI>
    __device__ __forceinline__ void done_tile_smem(int p0, int pstride, const bool (&ok)[TI],
                                                   const T (&vals)[TI][D], T* smem, int tid, int nthreads,
                                                   uint64_t* ebar, int use_tma, int3 org, T* pre_smem = nullptr) const {
        static_assert(sizeof(T) == 4, "smem-staged epilogue is the fp32 path");
        T vx[TI][D];
#pragma unroll
        for (int u = 0; u < TI; ++u)
#pragma unroll
            for (int c = 0; c < D; ++c) vx[u][c] = ok[u] ? __ldg(vl[c] + p0 + u * pstride) : T(0);
        auto slot = [&](int q, int u) -> T* { return smem + ((size_t)(q * TI + u) * nthreads + tid); };
        if constexpr (D == 3 && TI == SL_TI) {
            if (use_tma && tma_epi) {
                // box q of a round holds field q's (TI, BY, BX) tile: voxel (u, ty, tx) at
                // u * 256 + tid == slot(q, u), the layout the cp.async path writes
                const bool pre = pre_smem != nullptr && tma_epi;
                for (int j0 = 0, r = 0; j0 < n_t; j0 += 2, ++r) {
                    const int nj = (j0 + 1 < n_t) ? 2 : 1;
                    // round 0 may already be in flight in pre_smem (issued with the gather boxes)
                    T* buf = (pre && r == 0) ? pre_smem : smem;
                    if (!(pre && r == 0)) {
                        if (r > 0 && !(pre && r == 1)) __syncthreads();  // the previous round's boxes are consumed
                        if (tid == 0) {
                            fence_proxy_async();
                            issue_round(buf, ebar, org, j0, nj, nthreads);
                        }
                    }
                    mbar_wait_sleep(ebar, (unsigned)(r & 1));
                    auto slot = [&](int q, int u) -> T* { return buf + ((size_t)(q * TI + u) * nthreads + tid); };
                    for (int jj = 0; jj < nj; ++jj) {
                        const int j = j0 + jj;
#pragma unroll
                        for (int u = 0; u < TI; ++u) {
                            if (!ok[u]) continue;
                            T f0 = T(0), f1 = T(0);
#pragma unroll
                            for (int c = 0; c < D; ++c) {
                                f0 -= *slot(jj * 2 * D + c, u) * vals[u][c];
                                f1 -= *slot(jj * 2 * D + D + c, u) * vx[u][c];
                            }
                            const T sj = hh * (f0 + f1);
                            const int p = p0 + u * pstride;
                            if (j == 0) {
                                if (m1) m1[p] = sj;
                                if (fin) fin[p] = fsign * sj;
                            } else {
                                S[(size_t)(j - 1) * N + p] = sj;
                            }
                        }
                    }
                }
                return;
            }
        }
        for (int j0 = 0; j0 < n_t; j0 += 2) {
            const int nj = (j0 + 1 < n_t) ? 2 : 1;
            for (int jj = 0; jj < nj; ++jj) {
                const int j = j0 + jj;
#pragma unroll
                for (int c = 0; c < D; ++c)
#pragma unroll
                    for (int u = 0; u < TI; ++u)
                        if (ok[u]) {
                            const size_t p = (size_t)p0 + u * pstride;
                            cp_async_elem<4>(slot(jj * 2 * D + c, u), gy + ((size_t)j * D + c) * N + p);
                            cp_async_elem<4>(slot(jj * 2 * D + D + c, u), gx + ((size_t)(j + 1) * D + c) * N + p);
                        }
            }
            cp_async_wait_all();
            for (int jj = 0; jj < nj; ++jj) {
                const int j = j0 + jj;
#pragma unroll
                for (int u = 0; u < TI; ++u) {
                    if (!ok[u]) continue;
                    T f0 = T(0), f1 = T(0);
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        f0 -= *slot(jj * 2 * D + c, u) * vals[u][c];
                        f1 -= *slot(jj * 2 * D + D + c, u) * vx[u][c];
                    }
                    const T sj = hh * (f0 + f1);
                    const int p = p0 + u * pstride;
                    if (j == 0) {
                        if (m1) m1[p] = sj;
                        if (fin) fin[p] = fsign * sj;
                    } else {
                        S[(size_t)(j - 1) * N + p] = sj;
                    }
                }
            }
        }
    }
    __device__ __forceinline__ void done(int p, const T (&vals)[D]) const {
        T vx[D];
#pragma unroll
        for (int c = 0; c < D; ++c) vx[c] = vl[c][p];
        for (int j = 0; j < n_t; ++j) {
            T f0 = T(0), f1 = T(0);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                f0 -= gy[((size_t)j * D + c) * N + p] * vals[c];
                f1 -= gx[((size_t)(j + 1) * D + c) * N + p] * vx[c];
            }
            const T sj = hh * (f0 + f1);
            if (j == 0) {
                if (m1) m1[p] = sj;
                if (fin) fin[p] = fsign * sj;
            } else {
                S[(size_t)(j - 1) * N + p] = sj;
            }
        }
    }
};

template <typename T>
struct IncStepOp {
    using V = T;
    DispSrc<T> ds;
    const T* mj;
    const T* Sj;
    T* mnext;
    T* fin;
    T fsign;
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const { ds.get(p, d0, d1, d2); }
    __host__ __device__ __forceinline__ const T* field(int) const { return mj; }
    void set_field(int, const T* p) { mj = p; }
    using Pre = T;
    __device__ __forceinline__ T pre(int p) const { return Sj[p]; }
    __device__ __forceinline__ void done(int p, const T (&vals)[1], T s) const {
        const T m = vals[0] + s;
        if (mnext) mnext[p] = m;
        if (fin) fin[p] = fsign * m;
    }
};

// the TMA-fed epilogue's maps (fp32, 3D grids the TMA engine takes)
static void set_tile_streams(IncFirstOp<float, 3>& op, const Dims& g, int n_t) {
    op.tma_epi = 0;
    if (g.n2 % 4 != 0 || g.n2 < BX || g.n1 < BY || getenv("FRG_NO_TMA_EPILOGUE")) return;
    op.n0 = g.n0;
    encode_tile_stream_map(&op.tm_gy, op.gy, g.n1, g.n2, (long long)n_t * 3 * g.n0);
    encode_tile_stream_map(&op.tm_gx, op.gx, g.n1, g.n2, (long long)(n_t + 1) * 3 * g.n0);
    op.tma_epi = 1;
}

template <typename T, typename CV, int D>
static void inc_state_d(const Dims& g, int method, int n_t, const T* disp, const T* grads, const T* grads_y,
                        const CV* vt, T* vtT, T* S, T* series, T* fin, T fsign, bool keep, cudaStream_t st) {
    const size_t N = g.N;
    T ht = (T)(1.0 / n_t);
    // slice buffers: keep == full series, else ping-pong in series[0..1]
    auto slice = [&](int j) -> T* { return keep ? series + (size_t)j * N : series + (size_t)(j & 1) * N; };
    if (keep) FRG_CUDA(cudaMemsetAsync(series, 0, sizeof(T) * N, st));
    // v~ in transport precision once (the SL gathers stage it from HBM)
    const T* vsrc;
    if constexpr (std::is_same<T, CV>::value) {
        vsrc = vt;
    } else {
        convert(tcode(CV(0)), vt, tcode(T(0)), vtT, (long long)D * N, st);
        vsrc = vtT;
    }
    {
        IncFirstOp<T, D> op;
        op.ds = disp_src(g, disp);
        for (int c = 0; c < D; ++c) {
            op.vtT[c] = vsrc + c * N;
            op.vl[c] = vsrc + c * N;
        }
        op.gy = grads_y;
        op.gx = grads;
        op.N = N;
        op.n_t = n_t;
        op.m1 = (n_t == 1 && !keep) ? nullptr : slice(1);
        op.fin = (n_t == 1) ? fin : nullptr;
        op.S = S;
        op.fsign = fsign;
        op.hh = T(0.5) * ht;
        if constexpr (std::is_same<T, float>::value && D == 3) set_tile_streams(op, g, n_t);
        probed(st, [&] { launch_sl<T, D>(g, method, op, st); });
    }
    for (int j = 1; j < n_t; ++j) {
        bool last = (j == n_t - 1);
        IncStepOp<T> op;
        op.ds = disp_src(g, disp);
        op.mj = slice(j);
        op.Sj = S + (size_t)(j - 1) * N;
        op.mnext = (last && !keep) ? nullptr : slice(j + 1);
        op.fin = last ? fin : nullptr;
        op.fsign = fsign;
        launch_sl<T, 1>(g, method, op, st);
    }
}

void inc_first(const Dims& g, int method, int n_t, const float* disp, const float* grads, const float* grads_y,
               const float* vt_src, const float* vt_loc, float* m1, float* S, cudaStream_t st) {
    FRG_REQUIRE(g.d == 3, "slab transport is 3D");
    const size_t Ns = (size_t)(g.n0 + 2 * g.h0) * g.n1 * g.n2;
    IncFirstOp<float, 3> op;
    op.ds = disp_src(g, disp);
    for (int c = 0; c < 3; ++c) {  // vt_loc == nullptr: the owned planes of vt_src
        op.vtT[c] = vt_src + c * Ns;
        op.vl[c] = vt_loc ? vt_loc + c * g.N : vt_src + c * Ns + (size_t)g.h0 * g.n1 * g.n2;
    }
    op.gy = grads_y;
    op.gx = grads;
    op.N = g.N;
    op.n_t = n_t;
    op.m1 = m1;
    op.fin = nullptr;
    op.S = S;
    op.fsign = 0.f;
    op.hh = 0.5f * (float)(1.0 / n_t);
    set_tile_streams(op, g, n_t);
    probed(st, [&] { launch_sl<float, 3>(g, method, op, st); });
}

void inc_step(const Dims& g, int method, const float* disp, const float* m_src, const float* Sj, float* m_next,
              cudaStream_t st, float* fin, float fsign) {
    IncStepOp<float> op;
    op.ds = disp_src(g, disp);
    op.mj = m_src;
    op.Sj = Sj;
    op.mnext = m_next;
    op.fin = fin;
    op.fsign = fsign;
    launch_sl<float, 1>(g, method, op, st);
}

template <typename T, typename CV>
static void inc_state_t(const Dims& g, int method, int n_t, const T* disp, const T* grads, const T* grads_y,
                        const CV* vt, T* vtT, T* S, T* series, T* fin, T fsign, bool keep, cudaStream_t st) {
    if (g.d == 3)
        inc_state_d<T, CV, 3>(g, method, n_t, disp, grads, grads_y, vt, vtT, S, series, fin, fsign, keep, st);
    else
        inc_state_d<T, CV, 2>(g, method, n_t, disp, grads, grads_y, vt, vtT, S, series, fin, fsign, keep, st);
}

void inc_state(const Dims& g, int tdtype, int cdtype, int method, int n_t, const void* disp, const void* grads,
               const void* grads_y, const void* vt, void* vtT, void* S, void* series, void* final_out,
               double final_sign, bool keep_series, cudaStream_t st) {
    if (tdtype == F64 && cdtype == F64)
        inc_state_t<double, double>(g, method, n_t, (const double*)disp, (const double*)grads,
                                    (const double*)grads_y, (const double*)vt, (double*)vtT, (double*)S,
                                    (double*)series, (double*)final_out, final_sign, keep_series, st);
    else if (tdtype == F32 && cdtype == F32)
        inc_state_t<float, float>(g, method, n_t, (const float*)disp, (const float*)grads, (const float*)grads_y,
                                  (const float*)vt, (float*)vtT, (float*)S, (float*)series, (float*)final_out,
                                  (float)final_sign, keep_series, st);
    else if (tdtype == F32 && cdtype == F64)
        inc_state_t<float, double>(g, method, n_t, (const float*)disp, (const float*)grads, (const float*)grads_y,
                                   (const double*)vt, (float*)vtT, (float*)S, (float*)series, (float*)final_out,
                                   (float)final_sign, keep_series, st);
    else
        throw Error(E_ARG, "inc_state: unsupported dtype combination");
}

}  // namespace frg
