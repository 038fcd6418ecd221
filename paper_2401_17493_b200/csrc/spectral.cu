// Spectral operators: cuFFT R2C/C2R (D2Z/Z2D) bracketed by fused pointwise
// kernels on the half spectrum (diffops.py:44-366).
//
// The reference uses complex fftn/ifftn(...).real; every multiplier it
// applies is Hermitian (real even symbols, -i m with the Nyquist bin zeroed,
// the Nyquist-zeroed projection), so the real-to-complex pair computes the
// same result with half the traffic.  Normalisation 1/N is folded into the
// pointwise kernel.  Half-spectrum index (i0, i1, i2), i2 in [0, n2/2].
#include <cufft.h>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "ops.h"
#include <cstdlib>

#include "spectral.h"

#include <type_traits>

namespace frg {

#define FRG_CUFFT(call)                                                                   \
    do {                                                                                  \
        cufftResult _r = (call);                                                          \
        if (_r != CUFFT_SUCCESS)                                                          \
            throw ::frg::Error(::frg::E_CUFFT, std::string(#call) + " failed: " + std::to_string((int)_r)); \
    } while (0)

// ---------------------------------------------------------------------------
// plan cache
// ---------------------------------------------------------------------------
cufftHandle PlanCache::get(const Dims& g, int type, int batch) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(g.n0, g.n1, g.n2, type, batch);
    auto it = plans.find(key);
    if (it != plans.end()) return it->second;
    cufftHandle h;
    int dims3[3] = {g.n0, g.n1, g.n2};
    int dims2[2] = {g.n1, g.n2};
    int rank = g.n0 == 1 ? 2 : 3;
    int* dims = rank == 3 ? dims3 : dims2;
    FRG_CUFFT(cufftPlanMany(&h, rank, dims, nullptr, 1, 0, nullptr, 1, 0, (cufftType)type, batch));
    plans[key] = h;
    return h;
}

void PlanCache::clear() {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : plans) cufftDestroy(kv.second);
    plans.clear();
}

PlanCache::~PlanCache() {
    // plans are intentionally leaked at process exit (the CUDA context may be gone)
}

static PlanCache g_plans;

PlanCache& shared_plans() { return g_plans; }

Workspace::~Workspace() {}
// Spectral workspaces come from the context buffer pool (kkt.cu): a plain
// cudaFree of these 0.1-0.4 GB buffers at context teardown measured 0.1-1.5 s
// on the GPU box, inside every registration's wall time.
void* Workspace::get(size_t bytes) {
    if (bytes > cap) {
        if (ptr) {
            FRG_CUDA(cudaDeviceSynchronize());  // queued work may still read the old buffer
            pool_free(ptr, cap);
        }
        ptr = nullptr;
        size_t b = bytes;
        ptr = pool_alloc(b);
        cap = b;
    }
    return ptr;
}
void Workspace::release() {
    if (ptr) {
        cudaDeviceSynchronize();
        pool_free(ptr, cap);
    }
    ptr = nullptr;
    cap = 0;
}

static Workspace g_ws;
static std::mutex g_ws_mu;

void spectral_release_plans() {
    g_plans.clear();
    std::lock_guard<std::mutex> lk(g_ws_mu);
    g_ws.release();
}

long long half_len(const Dims& g) { return (long long)g.n0 * g.n1 * (g.n2 / 2 + 1); }

template <typename R>
struct CT;
template <>
struct CT<float> {
    using C = cufftComplex;
    static constexpr int R2C = CUFFT_R2C, C2R = CUFFT_C2R;
};
template <>
struct CT<double> {
    using C = cufftDoubleComplex;
    static constexpr int R2C = CUFFT_D2Z, C2R = CUFFT_Z2D;
};

template <typename R>
void fwd(PlanCache& pc, const Dims& g, int batch, const R* in, typename CT<R>::C* out, cudaStream_t st) {
    cufftHandle h = pc.get(g, CT<R>::R2C, batch);
    FRG_CUFFT(cufftSetStream(h, st));
    if (sizeof(R) == 8)
        FRG_CUFFT(cufftExecD2Z(h, (cufftDoubleReal*)in, (cufftDoubleComplex*)out));
    else
        FRG_CUFFT(cufftExecR2C(h, (cufftReal*)in, (cufftComplex*)out));
}

template <typename R>
void inv(PlanCache& pc, const Dims& g, int batch, typename CT<R>::C* in, R* out, cudaStream_t st) {
    cufftHandle h = pc.get(g, CT<R>::C2R, batch);
    FRG_CUFFT(cufftSetStream(h, st));
    if (sizeof(R) == 8)
        FRG_CUFFT(cufftExecZ2D(h, (cufftDoubleComplex*)in, (cufftDoubleReal*)out));
    else
        FRG_CUFFT(cufftExecC2R(h, (cufftComplex*)in, (cufftReal*)out));
}

template void fwd<float>(PlanCache&, const Dims&, int, const float*, cufftComplex*, cudaStream_t);
template void fwd<double>(PlanCache&, const Dims&, int, const double*, cufftDoubleComplex*, cudaStream_t);
template void inv<float>(PlanCache&, const Dims&, int, cufftComplex*, float*, cudaStream_t);
template void inv<double>(PlanCache&, const Dims&, int, cufftDoubleComplex*, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// symbols
// ---------------------------------------------------------------------------
__device__ __forceinline__ int dft_freq(int i, int n) { return i < (n + 1) / 2 ? i : i - n; }

struct Bin {
    double m[3];  // integer frequencies per axis (numpy fftfreq convention)
    bool nyq[3];  // |m| == n/2 (for n > 1)
};

// half-spectrum launch geometry: block (32, 8) over (i2, i1), grid z over i0
inline dim3 spec_grid(const Dims& g) { return dim3((g.n2 / 2 + 1 + BX - 1) / BX, (g.n1 + BY - 1) / BY, g.n0); }

__device__ __forceinline__ bool spec_vox(const Dims& g, int& i0, int& i1, int& i2, int& p) {
    const int nh = g.n2 / 2 + 1;
    i2 = blockIdx.x * BX + threadIdx.x;
    i1 = blockIdx.y * BY + threadIdx.y;
    i0 = blockIdx.z;
    if (i2 >= nh || i1 >= g.n1) return false;
    p = (i0 * g.n1 + i1) * nh + i2;
    return true;
}

__device__ __forceinline__ Bin bin_of(const Dims& g, int i0, int i1, int i2) {
    Bin b;
    int f0 = dft_freq(i0, g.n0), f1 = dft_freq(i1, g.n1);
    int f2 = (i2 == g.n2 / 2) ? -(g.n2 / 2) : i2;
    b.m[0] = f0;
    b.m[1] = f1;
    b.m[2] = f2;
    b.nyq[0] = g.n0 > 1 && (f0 == -(g.n0 / 2));
    b.nyq[1] = g.n1 > 1 && (f1 == -(g.n1 / 2));
    b.nyq[2] = g.n2 > 1 && (i2 == g.n2 / 2);
    return b;
}

__device__ __forceinline__ double ipow(double x, int o) {
    double r = x;
    for (int i = 1; i < o; ++i) r *= x;
    return r;
}

// diffops.py:167-173
__device__ __forceinline__ double reg_sym(double ksq, const RegSpec& r) {
    return r.seminorm ? ipow(ksq, r.order) : ipow(1.0 + ksq, r.order);
}

__device__ __forceinline__ double symbol_of(const Dims& g, const Bin& b, int kind, const RegSpec& r) {
    double ksq = b.m[0] * b.m[0] + b.m[1] * b.m[1] + b.m[2] * b.m[2];
    switch (kind) {
        case SK_REG: return r.alpha * reg_sym(ksq, r);
        case SK_REG_INV: {
            double s = reg_sym(ksq, r);
            if (s == 0.0) s = 1.0;
            return 1.0 / (r.alpha * s);
        }
        case SK_REG_INV_SQRT: {
            double s = reg_sym(ksq, r);
            if (s == 0.0) s = 1.0;
            return 1.0 / sqrt(r.alpha * s);
        }
        case SK_REG_KC: {
            double s = reg_sym(ksq, r);
            if (s == 0.0) s = 1.0;
            return r.alpha * s;
        }
        case SK_LAPLACIAN: return -ksq;
        case SK_BSPLINE_PREFILTER: {
            // periodic cubic B-spline interpolation condition per axis: the
            // samples are (c_{j-1} + 4 c_j + c_{j+1}) / 6 of the coefficients
            double s = 1.0;
            for (int a = 0; a < 3; ++a) {
                const int n = g.axis_len(a);
                if (n > 1) s *= (4.0 + 2.0 * cos(TWO_PI * b.m[a] / n)) / 6.0;
            }
            return 1.0 / s;
        }
        case SK_LOWPASS:
        case SK_HIGHPASS: {
            // diffops.py:283-289 — keep |k_i| < n_i / 4 on every axis
            bool low = fabs(b.m[0]) < g.n0 / 4.0 && fabs(b.m[1]) < g.n1 / 4.0 && fabs(b.m[2]) < g.n2 / 4.0;
            if (g.n0 == 1) low = fabs(b.m[1]) < g.n1 / 4.0 && fabs(b.m[2]) < g.n2 / 4.0;
            return (kind == SK_LOWPASS) == low ? 1.0 : 0.0;
        }
    }
    return 0.0;
}

// diffops.py:222-242, 245-280: factor M(k)/|k|^2 with Nyquist-zeroed k
__device__ __forceinline__ void proj_k(const Dims& g, const Bin& b, const RegSpec& r, double k[3], double& mfac) {
    for (int a = 0; a < 3; ++a) k[a] = b.nyq[a] ? 0.0 : b.m[a];
    double ksq = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
    if (ksq == 0.0 || r.incomp == 0) {
        mfac = 0.0;
        return;
    }
    double mult;
    if (r.incomp == 1) {
        mult = 1.0;
    } else {
        double inner = r.beta * (1.0 / ksq + 1.0);
        mult = 1.0 / (r.alpha / inner + 1.0);
    }
    mfac = mult / ksq;
}

template <typename C>
struct CR;
template <>
struct CR<cufftComplex> {
    using R = float;
};
template <>
struct CR<cufftDoubleComplex> {
    using R = double;
};

template <typename C>
__global__ void k_spec_scale(Dims g, long long nh, int ncomp, C* __restrict__ x, int kind, RegSpec r, double invN) {
    int i0, i1, i2, p;
    if (!spec_vox(g, i0, i1, i2, p)) return;
    Bin b = bin_of(g, i0, i1, i2);
    double s = symbol_of(g, b, kind, r) * invN;
    using R = typename CR<C>::R;
    // three components per round: their loads all issue before the stores
    // (in place, so a later load could not be hoisted above an earlier store)
    for (int c0 = 0; c0 < ncomp; c0 += 3) {
        C v[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            if (c0 + c < ncomp) v[c] = x[(long long)(c0 + c) * nh + p];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            if (c0 + c < ncomp) {
                v[c].x = (R)(v[c].x * s);
                v[c].y = (R)(v[c].y * s);
                x[(long long)(c0 + c) * nh + p] = v[c];
            }
    }
}

// out = alpha sym a + P(b), both normalised; written into a's spectrum.
// a may be null (P(b) only, written into b's spectrum converted to A).
// The per-bin arithmetic runs in the wider of the two spectra's precisions
// (fp32 spectra: fp32 math, no fp64 divisions on the fp32 path).
template <typename CA, typename CB>
__global__ void k_spec_combine(Dims g, long long nh, CA* __restrict__ a, const CB* __restrict__ bsp, RegSpec r,
                               double invN, bool have_a, bool project) {
    using RA = typename CR<CA>::R;
    using RB = typename CR<CB>::R;
    using M = typename std::conditional<(sizeof(RA) > sizeof(RB)), RA, RB>::type;
    int i0, i1, i2, p;
    if (!spec_vox(g, i0, i1, i2, p)) return;
    const Bin bn = bin_of(g, i0, i1, i2);
    M sa = M(0);
    if (have_a) {
        const M ksq = M(bn.m[0] * bn.m[0] + bn.m[1] * bn.m[1] + bn.m[2] * bn.m[2]);
        M s = r.seminorm ? ksq : M(1) + ksq;
        const M base = s;
        for (int o = 1; o < r.order; ++o) s *= base;
        sa = M(r.alpha) * s * M(invN);
    }
    M br[3], bi[3], k[3] = {M(0), M(0), M(0)}, mfac = M(0);
    for (int c = 0; c < g.d; ++c) {
        CB v = bsp[(long long)c * nh + p];
        br[c] = (M)v.x;
        bi[c] = (M)v.y;
    }
    if (project && r.incomp != 0) {
        for (int q = 0; q < 3; ++q) k[q] = bn.nyq[q] ? M(0) : M(bn.m[q]);
        const M ksq = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
        if (ksq != M(0)) {
            M mult = M(1);
            if (r.incomp == 2) {
                const M inner = M(r.beta) * (M(1) / ksq + M(1));
                mult = M(1) / (M(r.alpha) / inner + M(1));
            }
            mfac = mult / ksq;
        }
    }
    M dr = M(0), di = M(0);
    for (int c = 0; c < g.d; ++c) {
        const M kc = k[g.comp_axis(c)];
        dr += kc * br[c];
        di += kc * bi[c];
    }
    const M iN = M(invN);
    for (int c = 0; c < g.d; ++c) {
        const M kc = k[g.comp_axis(c)];
        M orr = (br[c] - kc * mfac * dr) * iN;
        M oi = (bi[c] - kc * mfac * di) * iN;
        CA o;
        if (have_a) {
            CA av = a[(long long)c * nh + p];
            orr += sa * (M)av.x;
            oi += sa * (M)av.y;
        }
        o.x = (RA)orr;
        o.y = (RA)oi;
        a[(long long)c * nh + p] = o;
    }
}

// spectral gradient of a scalar: out_c = -i m_axis(c) u  (Nyquist zeroed), diffops.py:56-73
template <typename C>
__global__ void k_spec_grad(Dims g, long long nh, const C* __restrict__ u, C* __restrict__ out, double invN) {
    int i0, i1, i2, p;
    if (!spec_vox(g, i0, i1, i2, p)) return;
    Bin b = bin_of(g, i0, i1, i2);
    C v = u[p];
    using R = typename CR<C>::R;
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        double m = b.nyq[a] ? 0.0 : b.m[a];
        // (-i m)(x + i y) = m y - i m x
        C o;
        o.x = (R)(m * v.y * invN);
        o.y = (R)(-m * v.x * invN);
        out[(long long)c * nh + p] = o;
    }
}

template <typename C>
__global__ void k_spec_div(Dims g, long long nh, const C* __restrict__ v, C* __restrict__ out, double invN) {
    int i0, i1, i2, p;
    if (!spec_vox(g, i0, i1, i2, p)) return;
    Bin b = bin_of(g, i0, i1, i2);
    double orr = 0.0, oi = 0.0;
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        double m = b.nyq[a] ? 0.0 : b.m[a];
        C x = v[(long long)c * nh + p];
        orr += m * x.y;
        oi += -m * x.x;
    }
    using R = typename CR<C>::R;
    C o;
    o.x = (R)(orr * invN);
    o.y = (R)(oi * invN);
    out[p] = o;
}

// Parseval: per-bin weight (1 on the i2 = 0 and i2 = n2/2 planes, else 2)
template <typename C>
__global__ void k_spec_energy(Dims g, long long nh, const C* __restrict__ v, RegSpec r, double* __restrict__ out) {
    int i0, i1, i2, p;
    if (!spec_vox(g, i0, i1, i2, p)) return;
    Bin b = bin_of(g, i0, i1, i2);
    double w = (i2 == 0 || i2 == g.n2 / 2) ? 1.0 : 2.0;
    double ksq = b.m[0] * b.m[0] + b.m[1] * b.m[1] + b.m[2] * b.m[2];
    double s = r.alpha * reg_sym(ksq, r);
    double acc = 0.0;
    for (int c = 0; c < g.d; ++c) {
        C x = v[(long long)c * nh + p];
        acc += (double)x.x * (double)x.x + (double)x.y * (double)x.y;
    }
    out[p] = w * s * acc;
}

// restriction: coarse spectrum from fine (diffops.py:304-326)
__device__ __forceinline__ int coarse_to_fine_full(int j, int c, int n) {
    // kept coarse bins: [0, c/2) and [c - c/2 + 1, c); the coarse Nyquist c/2 is dropped
    if (n == 1) return 0;
    if (j < c / 2) return j;
    if (j >= c - c / 2 + 1) return j + (n - c);
    return -1;
}

template <typename C>
__global__ void k_restrict_spec(Dims gf, Dims gc, const C* __restrict__ fine, C* __restrict__ coarse, double scale) {
    long long nhc = (long long)gc.n0 * gc.n1 * (gc.n2 / 2 + 1);
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nhc) return;
    int nh_c = gc.n2 / 2 + 1, nh_f = gf.n2 / 2 + 1;
    int j2 = (int)(p % nh_c);
    long long r = p / nh_c;
    int j1 = (int)(r % gc.n1);
    int j0 = (int)(r / gc.n1);
    int f0 = coarse_to_fine_full(j0, gc.n0, gf.n0);
    int f1 = coarse_to_fine_full(j1, gc.n1, gf.n1);
    int f2 = j2 < gc.n2 / 2 ? j2 : -1;
    C o;
    o.x = 0;
    o.y = 0;
    if (f0 >= 0 && f1 >= 0 && f2 >= 0) {
        C v = fine[((long long)f0 * gf.n1 + f1) * nh_f + f2];
        o.x = (typename CR<C>::R)(v.x * scale);
        o.y = (typename CR<C>::R)(v.y * scale);
    }
    coarse[p] = o;
}

__device__ __forceinline__ int fine_to_coarse_full(int f, int c, int n) {
    if (n == 1) return 0;
    if (f < c / 2) return f;
    if (f >= n - c / 2 + 1) return f - (n - c);
    return -1;
}

template <typename C>
__global__ void k_prolong_spec(Dims gf, Dims gc, const C* __restrict__ coarse, C* __restrict__ fine, double scale) {
    long long nhf = (long long)gf.n0 * gf.n1 * (gf.n2 / 2 + 1);
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nhf) return;
    int nh_c = gc.n2 / 2 + 1, nh_f = gf.n2 / 2 + 1;
    int f2 = (int)(p % nh_f);
    long long r = p / nh_f;
    int f1 = (int)(r % gf.n1);
    int f0 = (int)(r / gf.n1);
    int j0 = fine_to_coarse_full(f0, gc.n0, gf.n0);
    int j1 = fine_to_coarse_full(f1, gc.n1, gf.n1);
    int j2 = f2 < gc.n2 / 2 ? f2 : -1;
    C o;
    o.x = 0;
    o.y = 0;
    if (j0 >= 0 && j1 >= 0 && j2 >= 0) {
        C v = coarse[((long long)j0 * gc.n1 + j1) * nh_c + j2];
        o.x = (typename CR<C>::R)(v.x * scale);
        o.y = (typename CR<C>::R)(v.y * scale);
    }
    fine[p] = o;
}

// ---------------------------------------------------------------------------
// host entry points
// ---------------------------------------------------------------------------
constexpr int S_TPB = 256;

template <typename R>
static void spectral_apply_t(PlanCache& pc, void* ws, const Dims& g, int ncomp, const R* in, R* out, int kind,
                             const RegSpec& r, cudaStream_t st) {
    using C = typename CT<R>::C;
    long long nh = half_len(g);
    C* sp = (C*)ws;
    fwd<R>(pc, g, ncomp, in, sp, st);
    k_spec_scale<C><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, ncomp, sp, kind, r, 1.0 / (double)g.N);
    FRG_CHECK_LAUNCH();
    inv<R>(pc, g, ncomp, sp, out, st);
}

size_t spectral_ws_bytes(const Dims& g, int dtype, int ncomp) {
    return (size_t)half_len(g) * (dtype == F64 ? 16 : 8) * ncomp + (size_t)half_len(g) * 8;
}

void spectral_apply_ex(PlanCache& pc, void* ws, const Dims& g, int dtype, int ncomp, const void* in, void* out,
                       int kind, const RegSpec& r, cudaStream_t st) {
    if (dtype == F64)
        spectral_apply_t<double>(pc, ws, g, ncomp, (const double*)in, (double*)out, kind, r, st);
    else
        spectral_apply_t<float>(pc, ws, g, ncomp, (const float*)in, (float*)out, kind, r, st);
}

void spectral_apply(const Dims& g, int dtype, int ncomp, const void* in, void* out, int kind, const RegSpec& r,
                    cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    void* ws = g_ws.get(spectral_ws_bytes(g, dtype, ncomp));
    spectral_apply_ex(g_plans, ws, g, dtype, ncomp, in, out, kind, r, st);
}

void slab_combine_flat(const Dims& g, void* a, const void* b, const RegSpec& r, bool have_a, bool project, bool f64,
                       cudaStream_t st);

template <typename RA, typename RB>
static void combine_t(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, const RA* a, const RB* b, RA* out,
                      const RegSpec& r, bool project_on, cudaStream_t st) {
    using CA = typename CT<RA>::C;
    using CB = typename CT<RB>::C;
    long long nh = half_len(g);
    CA* sa = (CA*)ws_a;
    CB* sb = (CB*)ws_b;
    if (a) fwd<RA>(pc, g, g.d, a, sa, st);
    fwd<RB>(pc, g, g.d, b, sb, st);
    if constexpr (std::is_same<CA, CB>::value) {
        // flat grid-stride combine (no idle lanes on the n2/2+1 rows)
        if (g.n0 > 1 && g.d == 3) {
            slab_combine_flat(g, (void*)sa, (const void*)sb, r, a != nullptr, project_on, sizeof(RA) == 8, st);
            inv<RA>(pc, g, g.d, sa, out, st);
            return;
        }
    }
    k_spec_combine<CA, CB><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, sa, sb, r, 1.0 / (double)g.N, a != nullptr,
                                                                     project_on);
    FRG_CHECK_LAUNCH();
    inv<RA>(pc, g, g.d, sa, out, st);
}

void reg_plus_project_ex(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, int adtype, const void* a,
                         int bdtype, const void* b, void* out, const RegSpec& r, bool project_on, cudaStream_t st) {
    if (adtype == F64 && bdtype == F64)
        combine_t<double, double>(pc, ws_a, ws_b, g, (const double*)a, (const double*)b, (double*)out, r, project_on, st);
    else if (adtype == F32 && bdtype == F32)
        combine_t<float, float>(pc, ws_a, ws_b, g, (const float*)a, (const float*)b, (float*)out, r, project_on, st);
    else if (adtype == F64 && bdtype == F32)
        combine_t<double, float>(pc, ws_a, ws_b, g, (const double*)a, (const float*)b, (double*)out, r, project_on, st);
    else
        throw Error(E_ARG, "reg_plus_project: unsupported dtypes");
}

void reg_plus_project(const Dims& g, int adtype, const void* a, int bdtype, const void* b, void* out,
                      const RegSpec& r, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    size_t sa = (size_t)half_len(g) * (adtype == F64 ? 16 : 8) * g.d;
    size_t sb = (size_t)half_len(g) * (bdtype == F64 ? 16 : 8) * g.d;
    char* ws = (char*)g_ws.get(sa + sb);
    reg_plus_project_ex(g_plans, ws, ws + sa, g, adtype, a, bdtype, b, out, r, true, st);
}

void project(const Dims& g, int dtype, const void* b, void* out, const RegSpec& r, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    size_t sb = (size_t)half_len(g) * (dtype == F64 ? 16 : 8) * g.d;
    char* ws = (char*)g_ws.get(sb);
    // P(b) only: the combine kernel writes into the "a" spectrum -> use the same buffer
    if (dtype == F64) {
        using C = cufftDoubleComplex;
        long long nh = half_len(g);
        fwd<double>(g_plans, g, g.d, (const double*)b, (C*)ws, st);
        k_spec_combine<C, C><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, (C*)ws, (const C*)ws, r,
                                                                       1.0 / (double)g.N, false, true);
        FRG_CHECK_LAUNCH();
        inv<double>(g_plans, g, g.d, (C*)ws, (double*)out, st);
    } else {
        using C = cufftComplex;
        long long nh = half_len(g);
        fwd<float>(g_plans, g, g.d, (const float*)b, (C*)ws, st);
        k_spec_combine<C, C><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, (C*)ws, (const C*)ws, r,
                                                                       1.0 / (double)g.N, false, true);
        FRG_CHECK_LAUNCH();
        inv<float>(g_plans, g, g.d, (C*)ws, (float*)out, st);
    }
}

template <typename R>
static void spec_grad_t(const Dims& g, const R* u, R* out, cudaStream_t st) {
    using C = typename CT<R>::C;
    long long nh = half_len(g);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    C* ws = (C*)g_ws.get(sizeof(C) * nh * (g.d + 1));
    fwd<R>(g_plans, g, 1, u, ws, st);
    k_spec_grad<C><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, ws, ws + nh, 1.0 / (double)g.N);
    FRG_CHECK_LAUNCH();
    inv<R>(g_plans, g, g.d, ws + nh, out, st);
}

void spectral_gradient(const Dims& g, int dtype, const void* u, void* out, cudaStream_t st) {
    if (dtype == F64)
        spec_grad_t<double>(g, (const double*)u, (double*)out, st);
    else
        spec_grad_t<float>(g, (const float*)u, (float*)out, st);
}

template <typename R>
static void spec_div_t(const Dims& g, const R* v, R* out, cudaStream_t st) {
    using C = typename CT<R>::C;
    long long nh = half_len(g);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    C* ws = (C*)g_ws.get(sizeof(C) * nh * (g.d + 1));
    fwd<R>(g_plans, g, g.d, v, ws, st);
    k_spec_div<C><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, ws, ws + (long long)g.d * nh, 1.0 / (double)g.N);
    FRG_CHECK_LAUNCH();
    inv<R>(g_plans, g, 1, ws + (long long)g.d * nh, out, st);
}

void spectral_divergence(const Dims& g, int dtype, const void* v, void* out, cudaStream_t st) {
    if (dtype == F64)
        spec_div_t<double>(g, (const double*)v, (double*)out, st);
    else
        spec_div_t<float>(g, (const float*)v, (float*)out, st);
}

template <typename R>
static double reg_energy_t(PlanCache& pc, void* wsv, const Dims& g, const R* v, const RegSpec& r, cudaStream_t st) {
    using C = typename CT<R>::C;
    long long nh = half_len(g);
    C* ws = (C*)wsv;
    double* vals = (double*)(ws + (long long)g.d * nh);
    fwd<R>(pc, g, g.d, v, ws, st);
    k_spec_energy<C><<<spec_grid(g), vox_block(), 0, st>>>(g, nh, ws, r, vals);
    FRG_CHECK_LAUNCH();
    double mms[3];
    min_max_sum(F64, vals, nh, mms, st);
    double cellvol = (TWO_PI / g.n0) * (TWO_PI / g.n1) * (TWO_PI / g.n2);
    if (g.n0 == 1) cellvol = (TWO_PI / g.n1) * (TWO_PI / g.n2);
    // sum_x (aLv) v = (1/N) sum_k a sym |v^|^2
    return 0.5 * mms[2] / (double)g.N * cellvol;
}

double reg_energy_ex(PlanCache& pc, void* ws, const Dims& g, int dtype, const void* v, const RegSpec& r,
                     cudaStream_t st) {
    if (dtype == F64) return reg_energy_t<double>(pc, ws, g, (const double*)v, r, st);
    return reg_energy_t<float>(pc, ws, g, (const float*)v, r, st);
}

double reg_energy(const Dims& g, int dtype, const void* v, const RegSpec& r, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    void* ws = g_ws.get(spectral_ws_bytes(g, dtype, g.d));
    return reg_energy_ex(g_plans, ws, g, dtype, v, r, st);
}

Dims coarse_dims(const Dims& gf) {
    Dims gc = gf;
    gc.n0 = gf.n0 == 1 ? 1 : gf.n0 / 2;
    gc.n1 = gf.n1 / 2;
    gc.n2 = gf.n2 / 2;
    gc.N = (long long)gc.n0 * gc.n1 * gc.n2;
    return gc;
}

template <typename R>
static void restrict_t(PlanCache& pc, void* wsv, const Dims& gf, const R* in, R* out, cudaStream_t st) {
    using C = typename CT<R>::C;
    Dims gc = coarse_dims(gf);
    long long nhf = half_len(gf), nhc = half_len(gc);
    C* wf = (C*)wsv;
    C* wc = wf + nhf;
    fwd<R>(pc, gf, 1, in, wf, st);
    // (Nc/Nf) amplitude scale times the 1/Nc of the coarse inverse
    k_restrict_spec<C><<<blocks_for(nhc, S_TPB), S_TPB, 0, st>>>(gf, gc, wf, wc, 1.0 / (double)gf.N);
    FRG_CHECK_LAUNCH();
    inv<R>(pc, gc, 1, wc, out, st);
}

template <typename R>
static void prolong_t(PlanCache& pc, void* wsv, const Dims& gf, const R* in, R* out, cudaStream_t st) {
    using C = typename CT<R>::C;
    Dims gc = coarse_dims(gf);
    long long nhf = half_len(gf), nhc = half_len(gc);
    C* wf = (C*)wsv;
    C* wc = wf + nhf;
    fwd<R>(pc, gc, 1, in, wc, st);
    // (Nf/Nc) amplitude scale times the 1/Nf of the fine inverse
    k_prolong_spec<C><<<blocks_for(nhf, S_TPB), S_TPB, 0, st>>>(gf, gc, wc, wf, 1.0 / (double)gc.N);
    FRG_CHECK_LAUNCH();
    inv<R>(pc, gf, 1, wf, out, st);
}

size_t restrict_ws_bytes(const Dims& gf, int dtype) {
    Dims gc = coarse_dims(gf);
    return (size_t)(half_len(gf) + half_len(gc)) * (dtype == F64 ? 16 : 8);
}

void restrict_field_ex(PlanCache& pc, void* ws, const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st) {
    if (dtype == F64)
        restrict_t<double>(pc, ws, gf, (const double*)in, (double*)out, st);
    else
        restrict_t<float>(pc, ws, gf, (const float*)in, (float*)out, st);
}

void prolong_field_ex(PlanCache& pc, void* ws, const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st) {
    if (dtype == F64)
        prolong_t<double>(pc, ws, gf, (const double*)in, (double*)out, st);
    else
        prolong_t<float>(pc, ws, gf, (const float*)in, (float*)out, st);
}

void restrict_field(const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st) {
    FRG_REQUIRE((gf.n0 == 1 || gf.n0 % 4 == 0) && gf.n1 % 4 == 0 && gf.n2 % 4 == 0,
                "coarsening requires n_i divisible by 4");
    std::lock_guard<std::mutex> lk(g_ws_mu);
    void* ws = g_ws.get(restrict_ws_bytes(gf, dtype));
    restrict_field_ex(g_plans, ws, gf, dtype, in, out, st);
}

void prolong_field(const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    void* ws = g_ws.get(restrict_ws_bytes(gf, dtype));
    prolong_field_ex(g_plans, ws, gf, dtype, in, out, st);
}

}  // namespace frg

namespace frg {

// ===========================================================================
// Slab-decomposed spectral operators (multi-GPU, dist.py).
//
// Rank r owns planes [r n0/P, (r+1) n0/P) of the real field.  Forward:
//   (1) batched 2D R2C over axes (1, 2) of every owned plane  -> (n0/P, n1, nh)
//   (2) pack to (P, n0/P, n1/P, nh) and all-to-all (host, NCCL)  -> (n0, n1/P, nh)
//   (3) batched 1D C2C along axis 0 (stride n1/P * nh)
// The pointwise operators then act on the axis-1 split spectrum with global
// frequencies (i1 = r n1/P + local row); the inverse runs the steps backwards.
// ===========================================================================
namespace {
std::map<std::tuple<int, int, int, int>, cufftHandle> g_slab1d;
std::mutex g_slab1d_mu;
}  // namespace

template <typename R>
void slab_fft2_t(int n0_loc, int n1, int n2, int ncomp, int dir, const void* in, void* out, cudaStream_t st) {
    Dims p;  // one plane: rank-2 (n1, n2) plans from the shared cache, batched over planes x comps
    p.n0 = 1;
    p.n1 = n1;
    p.n2 = n2;
    p.N = (long long)n1 * n2;
    p.d = 3;
    if (dir > 0)
        fwd<R>(g_plans, p, n0_loc * ncomp, (const R*)in, (typename CT<R>::C*)out, st);
    else
        inv<R>(g_plans, p, n0_loc * ncomp, (typename CT<R>::C*)in, (R*)out, st);
}

void slab_fft2(int n0_loc, int n1, int n2, int dtype, int ncomp, int dir, const void* in, void* out, cudaStream_t st) {
    if (dtype == F64)
        slab_fft2_t<double>(n0_loc, n1, n2, ncomp, dir, in, out, st);
    else
        slab_fft2_t<float>(n0_loc, n1, n2, ncomp, dir, in, out, st);
}

void slab_fft1(int n0, int cols, int dtype, int ncomp, int dir, void* data, cudaStream_t st) {
    const int type = dtype == F64 ? CUFFT_Z2Z : CUFFT_C2C;
    cufftHandle h;
    {
        std::lock_guard<std::mutex> lk(g_slab1d_mu);
        auto key = std::make_tuple(n0, cols, type, 0);
        auto it = g_slab1d.find(key);
        if (it == g_slab1d.end()) {
            int n[1] = {n0};
            FRG_CUFFT(cufftPlanMany(&h, 1, n, n, cols, 1, n, cols, 1, (cufftType)type, cols));
            g_slab1d[key] = h;
        } else {
            h = it->second;
        }
    }
    FRG_CUFFT(cufftSetStream(h, st));
    const size_t es = dtype == F64 ? 16 : 8;
    for (int c = 0; c < ncomp; ++c) {
        char* x = (char*)data + (size_t)c * n0 * cols * es;
        if (dtype == F64)
            FRG_CUFFT(cufftExecZ2Z(h, (cufftDoubleComplex*)x, (cufftDoubleComplex*)x,
                                   dir > 0 ? CUFFT_FORWARD : CUFFT_INVERSE));
        else
            FRG_CUFFT(cufftExecC2C(h, (cufftComplex*)x, (cufftComplex*)x, dir > 0 ? CUFFT_FORWARD : CUFFT_INVERSE));
    }
}

// pack (dir > 0): (n0_loc, n1, nh) -> (P, n0_loc, n1/P, nh);  unpack (dir < 0): inverse.
// One thread per element, 8- or 16-byte complex elements, per component.
template <typename E>
__global__ void k_slab_transpose(int dir, int P, int n0_loc, int n1, int nh, int ncomp, const E* __restrict__ src,
                                 E* __restrict__ dst) {
    const long long per = (long long)n0_loc * n1 * nh;
    const long long total = per * ncomp;
    const int n1l = n1 / P;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / per;
        long long r = e - c * per;
        // natural index (i0, i1, i2) of the (n0_loc, n1, nh) layout
        const int i2 = (int)(r % nh);
        r /= nh;
        const int i1 = (int)(r % n1);
        const int i0 = (int)(r / n1);
        const int q = i1 / n1l, a = i1 - q * n1l;
        const long long packed = c * per + (((long long)q * n0_loc + i0) * n1l + a) * nh + i2;
        const long long natural = e;
        if (dir > 0)
            dst[packed] = src[natural];
        else
            dst[natural] = src[packed];
    }
}

void slab_transpose(int dir, int P, int n0_loc, int n1, int nh, int elem_bytes, int ncomp, const void* src, void* dst,
                    cudaStream_t st) {
    FRG_REQUIRE(P >= 1 && n1 % P == 0, "slab transpose: n1 must be divisible by the rank count");
    const long long total = (long long)n0_loc * n1 * nh * ncomp;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    if (elem_bytes == 16)
        k_slab_transpose<double2><<<blocks, 256, 0, st>>>(dir, P, n0_loc, n1, nh, ncomp, (const double2*)src,
                                                           (double2*)dst);
    else
        k_slab_transpose<float2><<<blocks, 256, 0, st>>>(dir, P, n0_loc, n1, nh, ncomp, (const float2*)src,
                                                          (float2*)dst);
    FRG_CHECK_LAUNCH();
}

// element (i0, a, i2) of the axis-1 split spectrum (n0, n1_loc, nh) -> global bin
__device__ __forceinline__ bool slab_spec_vox(const Dims& g, int i1_off, int n1_loc, long long e, int& i0, int& i1,
                                              int& i2) {
    const int nh = g.n2 / 2 + 1;
    i2 = (int)(e % nh);
    const long long r = e / nh;
    const int a = (int)(r % n1_loc);
    i0 = (int)(r / n1_loc);
    i1 = i1_off + a;
    return i0 < g.n0;
}

// x *= symbol(kind) / N for ncomp spectra (same symbols as k_spec_scale)
template <typename C>
__global__ void k_slab_spec_scale(Dims g, int i1_off, int n1_loc, int ncomp, C* __restrict__ x, int kind, RegSpec r,
                                  double invN) {
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
         e += (long long)gridDim.x * blockDim.x) {
        int i0, i1, i2;
        slab_spec_vox(g, i1_off, n1_loc, e, i0, i1, i2);
        const double s = symbol_of(g, bin_of(g, i0, i1, i2), kind, r) * invN;
        using R = typename CR<C>::R;
        for (int c = 0; c < ncomp; ++c) {
            C v = x[(long long)c * cnt + e];
            v.x = (R)(v.x * s);
            v.y = (R)(v.y * s);
            x[(long long)c * cnt + e] = v;
        }
    }
}

// out = alpha sym a + P(b), both normalised (k_spec_combine on the split
// spectrum); out may alias a or b (every input of a bin is read before its
// output is written); arithmetic in the output's precision (an f64 bin of a
// rounded to fp32 keeps its per-bin relative accuracy: the symbol multiplies
// the rounded value, it does not amplify global rounding)
template <typename CA, typename CB = CA, typename CO = CA>
__global__ void k_slab_combine(Dims g, int i1_off, int n1_loc, const CA* a, const CB* bsp, CO* out,
                               RegSpec r, double invN, bool have_a, bool project) {
    using M = typename CR<CO>::R;
    using RO = typename CR<CO>::R;
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
         e += (long long)gridDim.x * blockDim.x) {
        int i0, i1, i2;
        slab_spec_vox(g, i1_off, n1_loc, e, i0, i1, i2);
        const Bin bn = bin_of(g, i0, i1, i2);
        M sa = M(0);
        if (have_a) {
            const M ksq = M(bn.m[0] * bn.m[0] + bn.m[1] * bn.m[1] + bn.m[2] * bn.m[2]);
            M s = r.seminorm ? ksq : M(1) + ksq;
            const M base = s;
            for (int o = 1; o < r.order; ++o) s *= base;
            sa = M(r.alpha) * s * M(invN);
        }
        // every input of the bin is loaded before the first store (out may
        // alias a or b, so later loads could not be hoisted above a store)
        M br[3], bi[3], ar[3] = {M(0), M(0), M(0)}, ai[3] = {M(0), M(0), M(0)}, k[3] = {M(0), M(0), M(0)},
                                mfac = M(0);
        for (int c = 0; c < g.d; ++c) {
            const CB v = bsp[(long long)c * cnt + e];
            br[c] = M(v.x);
            bi[c] = M(v.y);
            if (have_a) {
                const CA av = a[(long long)c * cnt + e];
                ar[c] = M(av.x);
                ai[c] = M(av.y);
            }
        }
        if (project && r.incomp != 0) {
            for (int q = 0; q < 3; ++q) k[q] = bn.nyq[q] ? M(0) : M(bn.m[q]);
            const M ksq = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
            if (ksq != M(0)) {
                M mult = M(1);
                if (r.incomp == 2) {
                    const M inner = M(r.beta) * (M(1) / ksq + M(1));
                    mult = M(1) / (M(r.alpha) / inner + M(1));
                }
                mfac = mult / ksq;
            }
        }
        M dr = M(0), di = M(0);
        for (int c = 0; c < g.d; ++c) {
            const M kc = k[g.comp_axis(c)];
            dr += kc * br[c];
            di += kc * bi[c];
        }
        const M iN = M(invN);
        for (int c = 0; c < g.d; ++c) {
            const M kc = k[g.comp_axis(c)];
            M orr = (br[c] - kc * mfac * dr) * iN;
            M oi = (bi[c] - kc * mfac * di) * iN;
            if (have_a) {
                orr += sa * ar[c];
                oi += sa * ai[c];
            }
            CO o;
            o.x = RO(orr);
            o.y = RO(oi);
            out[(long long)c * cnt + e] = o;
        }
    }
}

static int slab_blocks(long long cnt) { return (int)std::min<long long>((cnt + 255) / 256, 148LL * 16); }

void slab_spec_scale(const Dims& g, int i1_off, int n1_loc, int dtype, int ncomp, void* x, int kind,
                     const RegSpec& r, cudaStream_t st) {
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    const double invN = 1.0 / ((double)g.n0 * g.n1 * g.n2);
    if (dtype == F64)
        k_slab_spec_scale<cufftDoubleComplex><<<slab_blocks(cnt), 256, 0, st>>>(g, i1_off, n1_loc, ncomp,
                                                                              (cufftDoubleComplex*)x, kind, r, invN);
    else
        k_slab_spec_scale<cufftComplex><<<slab_blocks(cnt), 256, 0, st>>>(g, i1_off, n1_loc, ncomp, (cufftComplex*)x,
                                                                        kind, r, invN);
    FRG_CHECK_LAUNCH();
}

void slab_spec_combine(const Dims& g, int i1_off, int n1_loc, int dtype, void* a, const void* b, const RegSpec& r,
                       bool project, cudaStream_t st) {
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    const double invN = 1.0 / ((double)g.n0 * g.n1 * g.n2);
    if (dtype == F64)
        k_slab_combine<cufftDoubleComplex><<<slab_blocks(cnt), 256, 0, st>>>(
            g, i1_off, n1_loc, (cufftDoubleComplex*)a, (const cufftDoubleComplex*)b, (cufftDoubleComplex*)a, r, invN,
            a != b, project);
    else
        k_slab_combine<cufftComplex><<<slab_blocks(cnt), 256, 0, st>>>(g, i1_off, n1_loc, (cufftComplex*)a,
                                                                     (const cufftComplex*)b, (cufftComplex*)a, r,
                                                                     invN, a != b, project);
    FRG_CHECK_LAUNCH();
}

void slab_spec_combine_mixed(const Dims& g, int i1_off, int n1_loc, const void* a, void* b, const RegSpec& r,
                             bool project, cudaStream_t st) {
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    const double invN = 1.0 / ((double)g.n0 * g.n1 * g.n2);
    k_slab_combine<cufftDoubleComplex, cufftComplex, cufftComplex><<<slab_blocks(cnt), 256, 0, st>>>(
        g, i1_off, n1_loc, (const cufftDoubleComplex*)a, (const cufftComplex*)b, (cufftComplex*)b, r, invN,
        a != nullptr, project);
    FRG_CHECK_LAUNCH();
}

// per-block partial sums of sum_k w_k |m'|^2 |x_k|^2 over the split spectrum
__global__ void k_slab_grad_energy(Dims g, int i1_off, int n1_loc, const cufftDoubleComplex* __restrict__ x,
                                   double* __restrict__ partial) {
    __shared__ double sw[8];
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    double acc = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
         e += (long long)gridDim.x * blockDim.x) {
        int i0, i1, i2;
        slab_spec_vox(g, i1_off, n1_loc, e, i0, i1, i2);
        const Bin bn = bin_of(g, i0, i1, i2);
        double kk = 0.0;
        for (int q = 0; q < 3; ++q) kk += bn.nyq[q] ? 0.0 : bn.m[q] * bn.m[q];
        const double w = (i2 == 0 || 2 * i2 == g.n2) ? 1.0 : 2.0;  // conjugate half of the spectrum
        const cufftDoubleComplex v = x[e];
        acc += w * kk * (v.x * v.x + v.y * v.y);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sw[q];
        partial[blockIdx.x] = t;
    }
}

double slab_grad_energy(const Dims& g, int i1_off, int n1_loc, const void* x_spec, cudaStream_t st) {
    const long long cnt = (long long)g.n0 * n1_loc * (g.n2 / 2 + 1);
    const int nb = slab_blocks(cnt);
    double* part = nullptr;
    FRG_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * nb, st));
    k_slab_grad_energy<<<nb, 256, 0, st>>>(g, i1_off, n1_loc, (const cufftDoubleComplex*)x_spec, part);
    FRG_CHECK_LAUNCH();
    std::vector<double> h(nb);
    FRG_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
    FRG_CUDA(cudaFreeAsync(part, st));
    FRG_CUDA(cudaStreamSynchronize(st));
    double t = 0.0;  // fixed order: deterministic
    for (double v : h) t += v;
    return t / ((double)g.n0 * g.n1 * g.n2);  // Parseval: sum_x |f|^2 = sum_k |F_k|^2 / N
}

void bspline_prefilter(const Dims& g, int dtype, const void* in, void* out, cudaStream_t st) {
    if (in != out && bspline_fir_applies(g, dtype) && !getenv("FRG_BSPLINE_SPECTRAL"))
        return bspline_prefilter_fir(g, dtype, in, out, st);
    RegSpec r{1.0, 1, 1, 0, 1e-4};
    spectral_apply(g, dtype, 1, in, out, SK_BSPLINE_PREFILTER, r, st);
}

// whole-grid combine through the flat split-spectrum kernel (i1 offset 0, all rows)
void slab_combine_flat(const Dims& g, void* a, const void* b, const RegSpec& r, bool have_a, bool project, bool f64,
                       cudaStream_t st) {
    const long long cnt = (long long)g.n0 * g.n1 * (g.n2 / 2 + 1);
    const double invN = 1.0 / ((double)g.n0 * g.n1 * g.n2);
    if (f64)
        k_slab_combine<cufftDoubleComplex><<<slab_blocks(cnt), 256, 0, st>>>(
            g, 0, g.n1, (cufftDoubleComplex*)a, (const cufftDoubleComplex*)b, (cufftDoubleComplex*)a, r, invN,
            have_a, project);
    else
        k_slab_combine<cufftComplex><<<slab_blocks(cnt), 256, 0, st>>>(g, 0, g.n1, (cufftComplex*)a,
                                                                     (const cufftComplex*)b, (cufftComplex*)a, r,
                                                                     invN, have_a, project);
    FRG_CHECK_LAUNCH();
}

// k_slab_combine<double2, float2, float2> over the whole 3D half spectrum, two
// consecutive bins per thread: b / out as float4, a as two double2, 32-bit bin
// index (same arithmetic, bin for bin)
__global__ void k_combine_mixed2(Dims g, int cnt, const double2* __restrict__ a, float4* bo, RegSpec r, float invN,
                                 bool project) {
    const int npair = cnt >> 1, nh = g.n2 / 2 + 1;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npair; q += gridDim.x * blockDim.x) {
        float4 bv[3];
        double2 av[3][2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            bv[c] = bo[(size_t)c * npair + q];
            av[c][0] = __ldg(a + (size_t)c * cnt + 2 * q);
            av[c][1] = __ldg(a + (size_t)c * cnt + 2 * q + 1);
        }
        float o[3][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = 2 * q + h;
            const int i2 = e % nh, rr = e / nh, i1 = rr % g.n1, i0 = rr / g.n1;
            const int f0 = dft_freq(i0, g.n0), f1 = dft_freq(i1, g.n1), f2 = (i2 == g.n2 / 2) ? -(g.n2 / 2) : i2;
            const float m0 = float(f0), m1 = float(f1), m2 = float(f2);
            const float ksq = m0 * m0 + m1 * m1 + m2 * m2;
            float s = r.seminorm ? ksq : 1.f + ksq;
            const float base = s;
            for (int oo = 1; oo < r.order; ++oo) s *= base;
            const float sa = float(r.alpha) * s * invN;
            float k[3] = {0.f, 0.f, 0.f}, mfac = 0.f;
            if (project && r.incomp != 0) {
                k[0] = (g.n0 > 1 && f0 == -(g.n0 / 2)) ? 0.f : m0;
                k[1] = (g.n1 > 1 && f1 == -(g.n1 / 2)) ? 0.f : m1;
                k[2] = (g.n2 > 1 && i2 == g.n2 / 2) ? 0.f : m2;
                const float kk = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
                if (kk != 0.f) {
                    float mult = 1.f;
                    if (r.incomp == 2) {
                        const float inner = float(r.beta) * (1.f / kk + 1.f);
                        mult = 1.f / (float(r.alpha) / inner + 1.f);
                    }
                    mfac = mult / kk;
                }
            }
            float br[3], bi[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                br[c] = h ? bv[c].z : bv[c].x;
                bi[c] = h ? bv[c].w : bv[c].y;
            }
            const float dr = k[0] * br[0] + k[1] * br[1] + k[2] * br[2];
            const float di = k[0] * bi[0] + k[1] * bi[1] + k[2] * bi[2];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                o[c][2 * h] = (br[c] - k[c] * mfac * dr) * invN + sa * float(av[c][h].x);
                o[c][2 * h + 1] = (bi[c] - k[c] * mfac * di) * invN + sa * float(av[c][h].y);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) bo[(size_t)c * npair + q] = make_float4(o[c][0], o[c][1], o[c][2], o[c][3]);
    }
}

// Mixed-precision alpha L a + P(b) (3D): a (f64) -> D2Z, b (fp32) -> R2C, the
// combine in f64 arithmetic written as an fp32 spectrum over b's, one C2R
// into out (fp32).  The forward transform of a must be f64: fp32 rounding of
// a smooth field (its own and the FFT's, ~1e-7 of |a| spread over every bin)
// is amplified by alpha |k|^2 at the high frequencies, 4x per grid doubling
// (measured 3.6e-4 rel-L2 on the 256^3 gradient); after the symbol is
// applied the inverse rounds relative to |out| only, so fp32 suffices there.
void mixed_forward_a(PlanCache& pc, void* ws_a, const Dims& g, const double* a, cudaStream_t st) {
    FRG_REQUIRE(g.d == 3, "reg_plus_project_mixed: 3D");
    fwd<double>(pc, g, g.d, a, (cufftDoubleComplex*)ws_a, st);
}

// second half: ws_a already holds the D2Z spectrum of a (mixed_forward_a,
// possibly issued on another stream the caller has joined)
void reg_plus_project_mixed_b(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, const float* b, float* out,
                              const RegSpec& r, bool project, cudaStream_t st) {
    auto* sa = (cufftDoubleComplex*)ws_a;
    auto* sb = (cufftComplex*)ws_b;
    fwd<float>(pc, g, g.d, b, sb, st);
    const long long cnt = (long long)g.n0 * g.n1 * (g.n2 / 2 + 1);
    const double invN = 1.0 / ((double)g.n0 * g.n1 * g.n2);
    if (cnt % 2 == 0 && cnt < (1LL << 31))
        k_combine_mixed2<<<slab_blocks(cnt / 2), 256, 0, st>>>(g, (int)cnt, (const double2*)sa, (float4*)sb, r,
                                                               (float)invN, project);
    else
        k_slab_combine<cufftDoubleComplex, cufftComplex, cufftComplex><<<slab_blocks(cnt), 256, 0, st>>>(
            g, 0, g.n1, sa, sb, sb, r, invN, true, project);
    FRG_CHECK_LAUNCH();
    inv<float>(pc, g, g.d, sb, out, st);
}

void reg_plus_project_mixed(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, const double* a, const float* b,
                            float* out, const RegSpec& r, bool project, cudaStream_t st) {
    mixed_forward_a(pc, ws_a, g, a, st);
    reg_plus_project_mixed_b(pc, ws_a, ws_b, g, b, out, r, project, st);
}

}  // namespace frg
