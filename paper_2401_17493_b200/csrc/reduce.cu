// Deterministic reductions and fused pointwise updates for control-space
// vectors (fields.py:320-344; optimizer.py:92-140).
//
// Reductions are two-pass with a fixed grid (a multiple of the 148 SMs):
// warp shuffles + a block tree in pass 1, one block over the partials in a
// fixed order in pass 2, f64 accumulation throughout, no atomics, so the
// result is bitwise reproducible run to run.
#include <mutex>

#include "ops.h"

namespace frg {

constexpr int R_TPB = 256;
constexpr int R_MAX_BLOCKS = NUM_SMS * 8;

enum RedOp { R_DOT = 0, R_ABSMAX = 1, R_MINMAXSUM = 2, R_NONFINITE = 3 };

struct Scratch {
    double* partials = nullptr;  // 3 * R_MAX_BLOCKS
    double* result = nullptr;    // device, 3
    double* host = nullptr;      // pinned, 3
    std::mutex mu;
};
static Scratch g_scratch;

static void ensure_scratch() {
    if (!g_scratch.partials) {
        FRG_CUDA(cudaMalloc(&g_scratch.partials, sizeof(double) * 3 * R_MAX_BLOCKS));
        FRG_CUDA(cudaMalloc(&g_scratch.result, sizeof(double) * 3));
        FRG_CUDA(cudaMallocHost(&g_scratch.host, sizeof(double) * 3));
    }
}

// max / min that propagate NaN (np.max / np.min semantics; fmax / fmin drop
// NaN operands, which would let a blown-up field report finite bounds)
__device__ __forceinline__ double nmax(double a, double b) { return (a != a || b != b) ? a + b : fmax(a, b); }
__device__ __forceinline__ double nmin(double a, double b) { return (a != a || b != b) ? a + b : fmin(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = nmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// block-reduce three lanes of values: (sum-or-max, min, sum)
template <int OP>
__device__ void block_reduce3(double& a, double& b, double& c) {
    __shared__ double sa[R_TPB / 32], sb[R_TPB / 32], sc[R_TPB / 32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (OP == R_DOT || OP == R_NONFINITE) {
        a = warp_sum(a);
    } else if (OP == R_ABSMAX) {
        a = warp_max(a);
    } else {
        a = warp_max(a);
        b = warp_min(b);
        c = warp_sum(c);
    }
    if (lane == 0) {
        sa[wid] = a;
        sb[wid] = b;
        sc[wid] = c;
    }
    __syncthreads();
    if (wid == 0) {
        int nw = blockDim.x >> 5;
        a = lane < nw ? sa[lane] : (OP == R_ABSMAX || OP == R_MINMAXSUM ? -INFINITY : 0.0);
        b = lane < nw ? sb[lane] : INFINITY;
        c = lane < nw ? sc[lane] : 0.0;
        if (OP == R_DOT || OP == R_NONFINITE) {
            a = warp_sum(a);
        } else if (OP == R_ABSMAX) {
            a = warp_max(a);
        } else {
            a = warp_max(a);
            b = warp_min(b);
            c = warp_sum(c);
        }
    }
}

template <typename TA, typename TB, int OP>
__global__ void __launch_bounds__(R_TPB) k_reduce_pass1(const TA* __restrict__ x, const TB* __restrict__ y,
                                                        long long n, double* __restrict__ partials) {
    double a = (OP == R_ABSMAX || OP == R_MINMAXSUM) ? -INFINITY : 0.0;
    double b = INFINITY, c = 0.0;
    if (OP == R_ABSMAX) a = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double xv = (double)x[i];
        if (OP == R_DOT) {
            a += xv * (double)y[i];
        } else if (OP == R_ABSMAX) {
            a = nmax(a, fabs(xv));
        } else if (OP == R_MINMAXSUM) {
            a = nmax(a, xv);
            b = nmin(b, xv);
            c += xv;
        } else {
            a += isfinite(xv) ? 0.0 : 1.0;
        }
    }
    block_reduce3<OP>(a, b, c);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = a;
        partials[R_MAX_BLOCKS + blockIdx.x] = b;
        partials[2 * R_MAX_BLOCKS + blockIdx.x] = c;
    }
}

template <int OP>
__global__ void __launch_bounds__(R_TPB) k_reduce_pass2(const double* __restrict__ partials, int nblocks,
                                                        double* __restrict__ result) {
    double a = (OP == R_ABSMAX) ? 0.0 : ((OP == R_MINMAXSUM) ? -INFINITY : 0.0);
    double b = INFINITY, c = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
        if (OP == R_DOT || OP == R_NONFINITE) {
            a += partials[i];
        } else if (OP == R_ABSMAX) {
            a = nmax(a, partials[i]);
        } else {
            a = nmax(a, partials[i]);
            b = nmin(b, partials[R_MAX_BLOCKS + i]);
            c += partials[2 * R_MAX_BLOCKS + i];
        }
    }
    block_reduce3<OP>(a, b, c);
    if (threadIdx.x == 0) {
        result[0] = a;
        result[1] = b;
        result[2] = c;
    }
}

template <typename TA, typename TB, int OP>
static void reduce_t(const TA* x, const TB* y, long long n, double out[3], cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_scratch.mu);
    ensure_scratch();
    int nb = (int)std::min<long long>(blocks_for(n, R_TPB * 4), R_MAX_BLOCKS);
    k_reduce_pass1<TA, TB, OP><<<nb, R_TPB, 0, st>>>(x, y, n, g_scratch.partials);
    FRG_CHECK_LAUNCH();
    k_reduce_pass2<OP><<<1, R_TPB, 0, st>>>(g_scratch.partials, nb, g_scratch.result);
    FRG_CHECK_LAUNCH();
    FRG_CUDA(cudaMemcpyAsync(g_scratch.host, g_scratch.result, sizeof(double) * 3, cudaMemcpyDeviceToHost, st));
    FRG_CUDA(cudaStreamSynchronize(st));
    out[0] = g_scratch.host[0];
    out[1] = g_scratch.host[1];
    out[2] = g_scratch.host[2];
}

double dot(int dtype, const void* a, const void* b, long long n, cudaStream_t st) {
    double r[3];
    if (dtype == F64)
        reduce_t<double, double, R_DOT>((const double*)a, (const double*)b, n, r, st);
    else
        reduce_t<float, float, R_DOT>((const float*)a, (const float*)b, n, r, st);
    return r[0];
}

double abs_max(int dtype, const void* a, long long n, cudaStream_t st) {
    double r[3];
    if (dtype == F64)
        reduce_t<double, double, R_ABSMAX>((const double*)a, (const double*)a, n, r, st);
    else
        reduce_t<float, float, R_ABSMAX>((const float*)a, (const float*)a, n, r, st);
    return r[0];
}

void min_max_sum(int dtype, const void* a, long long n, double out[3], cudaStream_t st) {
    double r[3];
    if (dtype == F64)
        reduce_t<double, double, R_MINMAXSUM>((const double*)a, (const double*)a, n, r, st);
    else
        reduce_t<float, float, R_MINMAXSUM>((const float*)a, (const float*)a, n, r, st);
    out[0] = r[1];  // min
    out[1] = r[0];  // max
    out[2] = r[2];  // sum
}

bool all_finite(int dtype, const void* a, long long n, cudaStream_t st) {
    double r[3];
    if (dtype == F64)
        reduce_t<double, double, R_NONFINITE>((const double*)a, (const double*)a, n, r, st);
    else
        reduce_t<float, float, R_NONFINITE>((const float*)a, (const float*)a, n, r, st);
    return r[0] == 0.0;
}

// ---------------------------------------------------------------------------
// pointwise
// ---------------------------------------------------------------------------
constexpr int P_TPB = 256;

template <typename S, typename D>
__global__ void k_convert_scalar(const S* __restrict__ s, D* __restrict__ d, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = (D)s[i];
}

// 4 elements per thread, 16/32-byte vector loads and stores (both pointers
// 32-byte aligned: torch / cudaMalloc allocations and whole-field offsets)
template <typename S, typename D>
__global__ void k_convert(const S* __restrict__ s, D* __restrict__ d, long long n) {
    long long i = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
    if (i + 3 < n) {
        S a[4];
        if constexpr (sizeof(S) == 8) {
            const double2 x = reinterpret_cast<const double2*>(s + i)[0], y = reinterpret_cast<const double2*>(s + i)[1];
            a[0] = x.x; a[1] = x.y; a[2] = y.x; a[3] = y.y;
        } else {
            const float4 x = *reinterpret_cast<const float4*>(s + i);
            a[0] = x.x; a[1] = x.y; a[2] = x.z; a[3] = x.w;
        }
        if constexpr (sizeof(D) == 8) {
            reinterpret_cast<double2*>(d + i)[0] = make_double2((double)a[0], (double)a[1]);
            reinterpret_cast<double2*>(d + i)[1] = make_double2((double)a[2], (double)a[3]);
        } else {
            *reinterpret_cast<float4*>(d + i) = make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]);
        }
    } else {
        for (; i < n; ++i) d[i] = (D)s[i];
    }
}

void convert(int sdtype, const void* src, int ddtype, void* dst, long long n, cudaStream_t st) {
    const bool aligned = (((uintptr_t)src | (uintptr_t)dst) & 31) == 0;
    if (!aligned && sdtype != ddtype) {
        // rare: unaligned views; scalar path through the same kernel (n <= 3 per thread never vectorised)
        int nb = blocks_for(n, P_TPB);
        if (sdtype == F64 && ddtype == F32)
            k_convert_scalar<double, float><<<nb, P_TPB, 0, st>>>((const double*)src, (float*)dst, n);
        else
            k_convert_scalar<float, double><<<nb, P_TPB, 0, st>>>((const float*)src, (double*)dst, n);
        FRG_CHECK_LAUNCH();
        return;
    }
    int nb = blocks_for((n + 3) / 4, P_TPB);
    if (sdtype == F64 && ddtype == F32)
        k_convert<double, float><<<nb, P_TPB, 0, st>>>((const double*)src, (float*)dst, n);
    else if (sdtype == F32 && ddtype == F64)
        k_convert<float, double><<<nb, P_TPB, 0, st>>>((const float*)src, (double*)dst, n);
    else if (sdtype == ddtype) {
        FRG_CUDA(cudaMemcpyAsync(dst, src, n * (sdtype == F64 ? 8 : 4), cudaMemcpyDeviceToDevice, st));
        return;
    } else
        throw Error(E_ARG, "convert: unsupported dtypes");
    FRG_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_axpby(T a, const T* __restrict__ x, T b, T* __restrict__ y, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // b == 0 must not read y (it may be uninitialised, 0 * NaN = NaN)
    if (i < n) y[i] = (b == T(0)) ? a * x[i] : a * x[i] + b * y[i];
}

void axpby(int dtype, double a, const void* x, double b, void* y, long long n, cudaStream_t st) {
    int nb = blocks_for(n, P_TPB);
    if (dtype == F64)
        k_axpby<double><<<nb, P_TPB, 0, st>>>(a, (const double*)x, b, (double*)y, n);
    else
        k_axpby<float><<<nb, P_TPB, 0, st>>>((float)a, (const float*)x, (float)b, (float*)y, n);
    FRG_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_xpay(const T* __restrict__ x, T a, const T* __restrict__ y, T* __restrict__ z, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[i] = x[i] + a * y[i];
}

void xpay_to(int dtype, const void* x, double a, const void* y, void* z, long long n, cudaStream_t st) {
    int nb = blocks_for(n, P_TPB);
    if (dtype == F64)
        k_xpay<double><<<nb, P_TPB, 0, st>>>((const double*)x, a, (const double*)y, (double*)z, n);
    else
        k_xpay<float><<<nb, P_TPB, 0, st>>>((const float*)x, (float)a, (const float*)y, (float*)z, n);
    FRG_CHECK_LAUNCH();
}

// x += k s ; r -= k hs ; partial sums of r*r  (optimizer.py:129-132)
template <typename T>
__global__ void __launch_bounds__(R_TPB) k_pcg_update(T k, const T* __restrict__ s, const T* __restrict__ hs,
                                                      T* __restrict__ x, T* __restrict__ r, long long n,
                                                      double* __restrict__ partials) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        x[i] = x[i] + k * s[i];
        T rn = r[i] - k * hs[i];
        r[i] = rn;
        a += (double)rn * (double)rn;
    }
    block_reduce3<R_DOT>(a, b, c);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = a;
        partials[R_MAX_BLOCKS + blockIdx.x] = 0.0;
        partials[2 * R_MAX_BLOCKS + blockIdx.x] = 0.0;
    }
}

double pcg_update(int dtype, double k, const void* s, const void* hs, void* x, void* r, long long n,
                  cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_scratch.mu);
    ensure_scratch();
    int nb = (int)std::min<long long>(blocks_for(n, R_TPB * 4), R_MAX_BLOCKS);
    if (dtype == F64)
        k_pcg_update<double><<<nb, R_TPB, 0, st>>>(k, (const double*)s, (const double*)hs, (double*)x, (double*)r, n,
                                                   g_scratch.partials);
    else
        k_pcg_update<float><<<nb, R_TPB, 0, st>>>((float)k, (const float*)s, (const float*)hs, (float*)x, (float*)r,
                                                  n, g_scratch.partials);
    FRG_CHECK_LAUNCH();
    k_reduce_pass2<R_DOT><<<1, R_TPB, 0, st>>>(g_scratch.partials, nb, g_scratch.result);
    FRG_CHECK_LAUNCH();
    FRG_CUDA(cudaMemcpyAsync(g_scratch.host, g_scratch.result, sizeof(double), cudaMemcpyDeviceToHost, st));
    FRG_CUDA(cudaStreamSynchronize(st));
    return g_scratch.host[0];
}

template <typename O, typename S>
__global__ void k_add_into(O* __restrict__ out, const S* __restrict__ src, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = out[i] + (O)src[i];
}

void add_into(int odtype, void* out, int sdtype, const void* src, long long n, cudaStream_t st) {
    int nb = blocks_for(n, P_TPB);
    if (odtype == F64 && sdtype == F64)
        k_add_into<double, double><<<nb, P_TPB, 0, st>>>((double*)out, (const double*)src, n);
    else if (odtype == F64 && sdtype == F32)
        k_add_into<double, float><<<nb, P_TPB, 0, st>>>((double*)out, (const float*)src, n);
    else if (odtype == F32 && sdtype == F32)
        k_add_into<float, float><<<nb, P_TPB, 0, st>>>((float*)out, (const float*)src, n);
    else
        throw Error(E_ARG, "add_into: unsupported dtypes");
    FRG_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_fill(T* a, T v, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

void fill(int dtype, void* a, double value, long long n, cudaStream_t st) {
    int nb = blocks_for(n, P_TPB);
    if (dtype == F64)
        k_fill<double><<<nb, P_TPB, 0, st>>>((double*)a, value, n);
    else
        k_fill<float><<<nb, P_TPB, 0, st>>>((float*)a, (float)value, n);
    FRG_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_scale_diff(const T* __restrict__ a, const T* __restrict__ b, T sa, T* __restrict__ out,
                             long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = sa * (a[i] - b[i]);
}

void scale_diff(int dtype, const void* a, const void* b, double sa, void* out, long long n, cudaStream_t st) {
    int nb = blocks_for(n, P_TPB);
    if (dtype == F64)
        k_scale_diff<double><<<nb, P_TPB, 0, st>>>((const double*)a, (const double*)b, sa, (double*)out, n);
    else
        k_scale_diff<float><<<nb, P_TPB, 0, st>>>((const float*)a, (const float*)b, (float)sa, (float*)out, n);
    FRG_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_lincomb3(T c1, const T* __restrict__ a, T c2, const T* __restrict__ b, T c3,
                           const T* __restrict__ c, T* __restrict__ out, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T v = c1 * a[i];
    if (b) v += c2 * b[i];
    if (c) v += c3 * c[i];
    out[i] = v;
}

void lincomb3(int dtype, double c1, const void* a, double c2, const void* b, double c3, const void* c, void* out,
              long long n, cudaStream_t st) {
    int nb = blocks_for(n, P_TPB);
    if (dtype == F64)
        k_lincomb3<double><<<nb, P_TPB, 0, st>>>(c1, (const double*)a, c2, (const double*)b, c3, (const double*)c,
                                                 (double*)out, n);
    else
        k_lincomb3<float><<<nb, P_TPB, 0, st>>>((float)c1, (const float*)a, (float)c2, (const float*)b, (float)c3,
                                                (const float*)c, (float*)out, n);
    FRG_CHECK_LAUNCH();
}

// out (+)= (sum_c gm_c s_c) gm   (kkt.py:288, 302)
template <typename T>
__global__ void k_rank_one(Dims g, const T* __restrict__ gm, const T* __restrict__ s, T* __restrict__ out, bool acc) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    T dotv = T(0);
    for (int c = 0; c < g.d; ++c) dotv += gm[(long long)c * g.N + p] * s[(long long)c * g.N + p];
    for (int c = 0; c < g.d; ++c) {
        long long o = (long long)c * g.N + p;
        T v = dotv * gm[o];
        out[o] = acc ? out[o] + v : v;
    }
}

void rank_one(const Dims& g, int dtype, const void* gm, const void* s, void* out, bool acc, cudaStream_t st) {
    int nb = blocks_for(g.N, P_TPB);
    if (dtype == F64)
        k_rank_one<double><<<nb, P_TPB, 0, st>>>(g, (const double*)gm, (const double*)s, (double*)out, acc);
    else
        k_rank_one<float><<<nb, P_TPB, 0, st>>>(g, (const float*)gm, (const float*)s, (float*)out, acc);
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
