// Periodic cubic B-spline prefilter as three separable passes (sm_100a).
//
// The coefficients c of the periodic cubic B-spline interpolant of f solve,
// along every axis, (c[i-1] + 4 c[i] + c[i+1]) / 6 = f[i] (the spectral symbol
// (4 + 2 cos(2 pi m / n)) / 6 of oracle/flowreg_oracle.py bspline_prefilter;
// the reference has no B-spline).  The inverse of that circulant
// is the symmetric kernel
//     h[m] = sqrt(3) (z^|m| + z^(n - |m|)) / (1 - z^n),   z = sqrt(3) - 2,
// whose taps fall by |z| = 0.268 per cell: |m| <= K with K = 16 (fp32) / 32
// (f64) leaves a truncation of 2 sqrt(3) |z|^(K+1) / (1 - |z|) < 1e-9 / 1e-19
// of the signal, far below the storage rounding.  Each pass reads and writes
// the field once (HBM-bound, 8 B / voxel fp32), replacing the R2C + scale +
// C2R cuFFT round trip the spectral path needs per prefiltered field.
//
//  * k_fir_row: the contiguous axis — one warp per row segment of 32 Q
//    outputs, staged with its +-K wrap halo in shared memory (one pad word per
//    Q elements: the lanes' windows sit on distinct banks); each lane produces
//    Q consecutive outputs from a register window of Q + 2K values.
//    Results go back through shared memory so the row stores coalesce.
//  * k_fir_col: a strided axis — a CTA stages an (8 Q R + 2K) x 32 tile
//    (rows of 32 contiguous columns, coalesced, every load in flight at
//    once), each thread produces R runs of Q consecutive outputs of one
//    column from register windows (a warp reads one smem row: 32 banks).
#include <cstdlib>

#include "ops.h"
#include "spectral.h"

namespace frg {

namespace {

// K: taps each side; Q: consecutive outputs per thread (register window Q + 2K)
template <typename T>
struct FirK;
template <>
struct FirK<float> {
    static constexpr int K = 16, Q = 8;
};
template <>
struct FirK<double> {
    static constexpr int K = 32, Q = 4;
};

template <typename T>
struct FirTaps {
    T z, c;  // pole, gain sqrt(3) / (1 - z^n)
};

template <typename T>
FirTaps<T> fir_taps(int n) {
    const double z = std::sqrt(3.0) - 2.0;
    FirTaps<T> t;
    t.z = (T)z;
    t.c = (T)(std::sqrt(3.0) / (1.0 - std::pow(z, n)));
    return t;
}

// The Q outputs of one thread from its window win[e] = x[o0 - K + e]:
//   out[q] = c (sum_{m >= 0} z^m x[q - m] + sum_{m >= 1} z^m x[q + m]),
// the kernel h[m] = c z^|m| of the periodic inverse (its z^(n - |m|) images
// are below 1e-10 of the signal for n >= 2K + 2).  Each one-sided sum is a
// first-order recursion seeded from the K window cells beyond the thread's
// outputs: 2K + 4 Q FMA-class operations for Q outputs instead of (2K + 1) Q
// for the direct FIR (the kernels were instruction-bound); the sums reach
// further than K taps inside the window, so the truncation is <= |z|^(K+1).
template <typename T, int Q, int K, class Win>
__device__ __forceinline__ void fir_rec(const Win& win, T z, T c, T (&res)[Q]) {
    // causal: P[q] = x[q] + z P[q - 1], seeded by Horner over x[-K] .. x[0]
    T P = win(0);
#pragma unroll
    for (int e = 1; e <= K; ++e) P = fma(z, P, win(e));
    res[0] = P;
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        P = fma(z, P, win(K + q));
        res[q] = P;
    }
    // anticausal: A[q] = z B[q], B[q] = x[q + 1] + z B[q + 1], seeded by
    // Horner over x[Q - 1 + K] .. x[Q]
    T B = win(Q - 1 + 2 * K);
#pragma unroll
    for (int e = Q - 2 + 2 * K; e >= Q + K; --e) B = fma(z, B, win(e));
#pragma unroll
    for (int q = Q - 1; q >= 0; --q) {
        res[q] = c * fma(z, B, res[q]);
        B = fma(z, B, win(K + q));
    }
}

// periodic index: one compare in range, a division only for indices outside
// [0, n) (a column tile of 8 Q R + 2K rows can exceed a short axis)
__device__ __forceinline__ int wrapi(int i, int n) {
    if ((unsigned)i >= (unsigned)n) {
        i %= n;
        i = i < 0 ? i + n : i;
    }
    return i;
}
// the same for i in [-n, 2n) (every axis at least as long as the tile + halo)
__device__ __forceinline__ int wrap1(int i, int n) {
    i = i < 0 ? i + n : i;
    return i >= n ? i - n : i;
}

constexpr int ROW_WARPS = 8;
#ifndef FRG_FIR_ROW_BLOCKS_PER_SM
#define FRG_FIR_ROW_BLOCKS_PER_SM 16
#endif
// shared index of row element e: one pad word per Q elements, so the lanes'
// windows (lane * Q + j) fall on 32 distinct banks (Q + 1 odd)
template <int Q>
__device__ __forceinline__ int rpad(int e) { return e + e / Q; }

// contiguous axis: rows of length n2, nrows = n0 * n1
template <typename T>
__global__ void __launch_bounds__(32 * ROW_WARPS) k_fir_row(const T* __restrict__ in, T* __restrict__ out, int n2,
                                                             long long nrows, FirTaps<T> taps) {
    constexpr int K = FirK<T>::K, Q = FirK<T>::Q, W = Q + 2 * K, ROW_SEG = 32 * Q;
    constexpr int SMN = ROW_SEG + 2 * K + (ROW_SEG + 2 * K) / Q + 1;
    __shared__ T sm[ROW_WARPS][SMN];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // PDL: let the next pass / SL step start its prologue, read only after the
    // predecessor (the producing step or the previous pass) has completed
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int nseg = (n2 + ROW_SEG - 1) / ROW_SEG;
    const int nwork = (int)(nrows * nseg);  // < 2^31 for every grid the engine takes (<= 1024^3)
    for (int item = blockIdx.x * ROW_WARPS + w; item < nwork; item += gridDim.x * ROW_WARPS) {
        const int row = nseg == 1 ? item : item / nseg;
        const int s0 = (item - row * nseg) * ROW_SEG;
        const T* __restrict__ src = in + (size_t)row * n2;
        T* s = sm[w];
        __syncwarp();
        // every load of the segment in flight at once (one latency per segment)
        constexpr int LPL = (ROW_SEG + 2 * K) / 32;
        static_assert((ROW_SEG + 2 * K) % 32 == 0, "row segment + halo must be whole warps");
        T ld[LPL];
#pragma unroll
        for (int r = 0; r < LPL; ++r) {
            const int e = s0 - K + lane + 32 * r;
            ld[r] = __ldg(src + (n2 >= ROW_SEG + K ? wrap1(e, n2) : wrapi(e, n2)));
        }
#pragma unroll
        for (int r = 0; r < LPL; ++r) s[rpad<Q>(lane + 32 * r)] = ld[r];
        __syncwarp();
        const int o0 = lane * Q;  // this lane's Q outputs: s0 + o0 ..
        T res[Q];
        fir_rec<T, Q, K>([&](int e) { return s[rpad<Q>(o0 + e)]; }, taps.z, taps.c, res);
        // outputs back through shared memory so the global stores coalesce
        __syncwarp();
#pragma unroll
        for (int q = 0; q < Q; ++q) s[rpad<Q>(o0 + q)] = res[q];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < Q; ++r) {
            const int o = s0 + lane + 32 * r;
            if (o < n2) out[(size_t)row * n2 + o] = s[rpad<Q>(lane + 32 * r)];
        }
    }
}

// strided axis: point (outer, line, c) at outer * ostride + line * lstride + c,
// line in [0, nl) along the filtered axis, c in [0, n2) contiguous.  A CTA
// covers COL_SEG = 8 Q R outputs of 32 columns (each thread R windows of Q).
#ifndef FRG_FIR_COL_R
#define FRG_FIR_COL_R 4
#endif
constexpr int COL_R = FRG_FIR_COL_R;
template <typename T>
__global__ void __launch_bounds__(256) k_fir_col(const T* __restrict__ in, T* __restrict__ out, int nl,
                                                 long long lstride, long long ostride, int n2, FirTaps<T> taps) {
    constexpr int K = FirK<T>::K, Q = FirK<T>::Q, W = Q + 2 * K, COL_SEG = 8 * Q * COL_R, ROWS = COL_SEG + 2 * K;
    __shared__ T sm[ROWS][32];
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int c = blockIdx.x * 32 + tx;
    const int l0 = blockIdx.y * COL_SEG;
    const long long base = (long long)blockIdx.z * ostride;
    static_assert(ROWS % 8 == 0, "tile rows must split over the 8 thread rows");
    const int ls = (int)lstride;  // line offsets fit 32 bits (<= 1024^3 grids)
    if (c < n2) {
        const T* __restrict__ src = in + base + c;
        T ld[ROWS / 8];
#pragma unroll
        for (int r = 0; r < ROWS / 8; ++r) {
            const int e = l0 - K + ty + 8 * r;
            ld[r] = __ldg(src + (nl >= COL_SEG + K ? wrap1(e, nl) : wrapi(e, nl)) * ls);
        }
#pragma unroll
        for (int r = 0; r < ROWS / 8; ++r) sm[ty + 8 * r][tx] = ld[r];
    }
    __syncthreads();
    if (c >= n2) return;
#pragma unroll
    for (int rep = 0; rep < COL_R; ++rep) {
        const int o0 = (ty + 8 * rep) * Q;
        T res[Q];
        fir_rec<T, Q, K>([&](int e) { return sm[o0 + e][tx]; }, taps.z, taps.c, res);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int l = l0 + o0 + q;
            if (l < nl) out[base + c + l * ls] = res[q];
        }
    }
}

// programmatic dependent launch (as the SL steps, sl_fast.cuh), off inside graph capture
template <typename K, typename... Args>
void pdl_launch(K kern, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool pdl = getenv("FRG_NO_PDL") == nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (pdl) FRG_CUDA(cudaStreamIsCapturing(st, &cs));
    cfg.attrs = at;
    cfg.numAttrs = (pdl && cs == cudaStreamCaptureStatusNone) ? 1 : 0;
    FRG_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

struct FirScratch {
    void* p = nullptr;
    size_t cap = 0;
};
thread_local FirScratch g_fir_tmp;

void* fir_tmp(size_t bytes) {
    if (bytes > g_fir_tmp.cap) {
        if (g_fir_tmp.p) FRG_CUDA(cudaFree(g_fir_tmp.p));
        g_fir_tmp.p = nullptr;
        FRG_CUDA(cudaMalloc(&g_fir_tmp.p, bytes));
        g_fir_tmp.cap = bytes;
    }
    return g_fir_tmp.p;
}

template <typename T>
void fir_pass(const Dims& g, int axis, const T* in, T* out, cudaStream_t st) {
    const int n = g.axis_len(axis);
    const FirTaps<T> taps = fir_taps<T>(n);
    constexpr int Q = FirK<T>::Q, ROW_SEG = 32 * Q, COL_SEG = 8 * Q * COL_R;
    if (axis == 2) {
        const long long nrows = (long long)g.n0 * g.n1;
        const long long work = nrows * ((g.n2 + ROW_SEG - 1) / ROW_SEG);
        const int blocks = (int)std::min<long long>((work + ROW_WARPS - 1) / ROW_WARPS, 148LL * FRG_FIR_ROW_BLOCKS_PER_SM);
        pdl_launch(k_fir_row<T>, dim3(blocks), dim3(32 * ROW_WARPS), st, in, out, g.n2, nrows, taps);
    } else {
        const long long lstride = axis == 1 ? g.n2 : (long long)g.n1 * g.n2;
        const long long ostride = axis == 1 ? (long long)g.n1 * g.n2 : g.n2;
        const int nouter = axis == 1 ? g.n0 : g.n1;
        dim3 grid((g.n2 + 31) / 32, (n + COL_SEG - 1) / COL_SEG, nouter);
        pdl_launch(k_fir_col<T>, grid, dim3(32, 8), st, in, out, n, lstride, ostride, g.n2, taps);
    }
    FRG_CHECK_LAUNCH();
}

template <typename T>
void fir_prefilter(const Dims& g, const T* in, T* out, cudaStream_t st) {
    int axes[3], P = 0;
    for (int a = 2; a >= 0; --a)
        if (g.axis_len(a) > 1) axes[P++] = a;
    if (P == 0) {
        FRG_CUDA(cudaMemcpyAsync(out, in, sizeof(T) * g.N, cudaMemcpyDeviceToDevice, st));
        return;
    }
    T* tmp = (T*)fir_tmp(sizeof(T) * g.N);
    // (measured: a kernel fusing the axis-2 and axis-1 passes through a
    // shared-memory slab of 32 + 2K rows ran 128 us vs 108 us for the three
    // separate passes at 256^3 fp32 — fewer resident CTAs, exposed staging)
    // alternate out / tmp so that the last pass lands in out
    const T* src = in;
    for (int q = 0; q < P; ++q) {
        T* dst = ((P - 1 - q) % 2 == 0) ? out : tmp;
        fir_pass<T>(g, axes[q], src, dst, st);
        src = dst;
    }
}

}  // namespace

bool bspline_fir_applies(const Dims& g, int dtype) {
    if (g.h0 > 0 || (dtype != F32 && dtype != F64)) return false;
    const int K = dtype == F64 ? FirK<double>::K : FirK<float>::K;
    for (int a = 0; a < 3; ++a) {
        const int n = g.axis_len(a);
        if (n > 1 && n < 2 * K + 2) return false;  // short axes: the spectral path
    }
    return true;
}

void bspline_prefilter_fir(const Dims& g, int dtype, const void* in, void* out, cudaStream_t st) {
    FRG_REQUIRE(in != out, "bspline prefilter: in and out must differ");
    if (dtype == F64)
        fir_prefilter<double>(g, (const double*)in, (double*)out, st);
    else
        fir_prefilter<float>(g, (const float*)in, (float*)out, st);
}

}  // namespace frg
