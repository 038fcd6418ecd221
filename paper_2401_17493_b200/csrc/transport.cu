// Semi-Lagrangian transport kernels (sm_100a).
//
// Departure points are stored once per velocity as DISPLACEMENTS in index
// units, disp = q(y) - j, instead of physical coordinates: the reference keeps
// y and recomputes q = n/2 - 1 - y/h per solve (transport.py:65-80,
// interp.py:22-34).  In index units the RK2 map of transport.py:37-45 reads
//   q~ = j + (h_t/h) v(x),   disp = (h_t/2h) (v(x) + v(q~)),
// exact for v = 0 and well conditioned in fp32 (|disp| is a few cells).
// Every gather then splits floor(disp) off exactly (common.cuh).
#include "ops.h"

namespace frg {

constexpr int TPB = 256;

// ---------------------------------------------------------------------------
// generic sample at f64 fractional indices (_kernels.sample_nd, :222-251)
// ---------------------------------------------------------------------------
template <typename V, typename O, int M>
__global__ void __launch_bounds__(TPB) k_sample_q(const V* __restrict__ vals, Dims g,
                                                  const double* __restrict__ q0,
                                                  const double* __restrict__ q1,
                                                  const double* __restrict__ q2, long long npts,
                                                  O* __restrict__ out) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    Stencil<double, M> s;
    make_stencil_q<double, M>(g, q0 ? q0[p] : 0.0, q1[p], q2[p], s);
    if (M == NEAREST)
        out[p] = (O)apply_stencil<V, double, M, V>(vals, s);
    else
        out[p] = (O)apply_stencil<double, double, M, V>(vals, s);
}

template <typename V, typename O>
static void sample_q_t(const V* vals, const Dims& g, const double* q0, const double* q1,
                       const double* q2, long long npts, int method, O* out, cudaStream_t st) {
    int nb = blocks_for(npts, TPB);
    if (npts == 0) return;
    switch (method) {
        case NEAREST: k_sample_q<V, O, NEAREST><<<nb, TPB, 0, st>>>(vals, g, q0, q1, q2, npts, out); break;
        case LINEAR: k_sample_q<V, O, LINEAR><<<nb, TPB, 0, st>>>(vals, g, q0, q1, q2, npts, out); break;
        case CUBIC: k_sample_q<V, O, CUBIC><<<nb, TPB, 0, st>>>(vals, g, q0, q1, q2, npts, out); break;
        default: throw Error(E_ARG, "unknown interpolation method");
    }
    FRG_CHECK_LAUNCH();
}

void sample_q(const void* vals, int dtype, const Dims& g, const double* q0, const double* q1,
              const double* q2, long long npts, int method, void* out, cudaStream_t st) {
    if (dtype == F64)
        sample_q_t((const double*)vals, g, q0, q1, q2, npts, method, (double*)out, st);
    else if (dtype == F32)
        sample_q_t((const float*)vals, g, q0, q1, q2, npts, method, (float*)out, st);
    else if (dtype == I32) {
        if (method == NEAREST)
            sample_q_t((const int*)vals, g, q0, q1, q2, npts, method, (int*)out, st);
        else  // non-float linear/cubic return f64 (_kernels.py:237)
            sample_q_t((const int*)vals, g, q0, q1, q2, npts, method, (double*)out, st);
    } else
        throw Error(E_ARG, "unsupported dtype");
}

// ---------------------------------------------------------------------------
// helpers: displacement components per grid axis (axis 0 is absent in 2D)
// ---------------------------------------------------------------------------
template <typename T>
struct DispPtrs {
    const T* a[3];  // per grid axis; nullptr -> zero displacement
};

template <typename T>
__host__ __device__ inline DispPtrs<T> disp_ptrs(const Dims& g, const T* disp) {
    DispPtrs<T> p;
    p.a[0] = p.a[1] = p.a[2] = nullptr;
    for (int c = 0; c < g.d; ++c) p.a[g.comp_axis(c)] = disp + (long long)c * g.N;
    return p;
}

template <typename T, int M>
__device__ __forceinline__ void stencil_at(const Dims& g, const DispPtrs<T>& dp, long long p,
                                           Stencil<T, M>& s) {
    int i, j, k;
    unflatten(g, p, i, j, k);
    T d0 = dp.a[0] ? dp.a[0][p] : T(0);
    T d1 = dp.a[1][p];
    T d2 = dp.a[2][p];
    make_stencil_disp<T, M>(g, i, j, k, d0, d1, d2, s);
}

// ---------------------------------------------------------------------------
// RK2 departure displacement (transport.py:37-45)
// ---------------------------------------------------------------------------
template <typename T, typename VI, int M>
__global__ void __launch_bounds__(TPB) k_departure(Dims g, const VI* __restrict__ v, double ht,
                                                   double h0, double h1, double h2, T* __restrict__ disp) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    int i, j, k;
    unflatten(g, p, i, j, k);
    const double hs[3] = {h0, h1, h2};
    T vx[3] = {T(0), T(0), T(0)};
    T dt[3] = {T(0), T(0), T(0)};
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        vx[c] = (T)v[(long long)c * g.N + p];
        dt[a] = (T)(ht / hs[a]) * vx[c];
    }
    Stencil<T, M> s;
    make_stencil_disp<T, M>(g, i, j, k, dt[0], dt[1], dt[2], s);
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        T va = apply_stencil<T, T, M, VI>(v + (long long)c * g.N, s);
        disp[(long long)c * g.N + p] = (T)(0.5 * ht / hs[a]) * (vx[c] + va);
    }
}

template <typename T, typename VI>
static void departure_t(const Dims& g, int method, double ht, const VI* v, T* disp, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    double h[3] = {TWO_PI / g.n0, TWO_PI / g.n1, TWO_PI / g.n2};
    switch (method) {
        case NEAREST: k_departure<T, VI, NEAREST><<<nb, TPB, 0, st>>>(g, v, ht, h[0], h[1], h[2], disp); break;
        case LINEAR: k_departure<T, VI, LINEAR><<<nb, TPB, 0, st>>>(g, v, ht, h[0], h[1], h[2], disp); break;
        case CUBIC: k_departure<T, VI, CUBIC><<<nb, TPB, 0, st>>>(g, v, ht, h[0], h[1], h[2], disp); break;
        default: throw Error(E_ARG, "unknown interpolation method");
    }
    FRG_CHECK_LAUNCH();
}

void departure(const Dims& g, int tdtype, int vdtype, int method, double h_t, const void* v, void* disp,
               cudaStream_t st) {
    if (tdtype == F64 && vdtype == F64)
        departure_t(g, method, h_t, (const double*)v, (double*)disp, st);
    else if (tdtype == F32 && vdtype == F32)
        departure_t(g, method, h_t, (const float*)v, (float*)disp, st);
    else if (tdtype == F32 && vdtype == F64)
        departure_t(g, method, h_t, (const double*)v, (float*)disp, st);
    else
        throw Error(E_ARG, "departure: unsupported dtype combination");
}

// y = x - h*disp   /   disp = (x - y)/h   (fields.py:105-114: x_j = (n/2-(j+1)) h)
template <typename T, bool TO_POINTS>
__global__ void k_disp_points(Dims g, const T* __restrict__ src, T* __restrict__ dst) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    int idx[3];
    unflatten(g, p, idx[0], idx[1], idx[2]);
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        int n = g.axis_len(a);
        T h = (T)(TWO_PI / n);
        T x = (T)((n / 2) - (idx[a] + 1.0)) * h;
        long long o = (long long)c * g.N + p;
        if (TO_POINTS)
            dst[o] = x - h * src[o];
        else
            dst[o] = (x - src[o]) / h;
    }
}

void disp_to_points(const Dims& g, int tdtype, const void* disp, void* y, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    if (tdtype == F64)
        k_disp_points<double, true><<<nb, TPB, 0, st>>>(g, (const double*)disp, (double*)y);
    else
        k_disp_points<float, true><<<nb, TPB, 0, st>>>(g, (const float*)disp, (float*)y);
    FRG_CHECK_LAUNCH();
}

void points_to_disp(const Dims& g, int tdtype, const void* y, void* disp, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    if (tdtype == F64)
        k_disp_points<double, false><<<nb, TPB, 0, st>>>(g, (const double*)y, (double*)disp);
    else
        k_disp_points<float, false><<<nb, TPB, 0, st>>>(g, (const float*)y, (float*)disp);
    FRG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// multi-field gather with one shared stencil
// ---------------------------------------------------------------------------
constexpr int MAXF = 9;
template <typename T>
struct FieldSet {
    const T* in[MAXF];
    T* out[MAXF];
    int nf;
};

template <typename T, int M>
__global__ void __launch_bounds__(TPB) k_gather(Dims g, DispPtrs<T> dp, FieldSet<T> fs) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    Stencil<T, M> s;
    stencil_at<T, M>(g, dp, p, s);
    for (int f = 0; f < fs.nf; ++f) fs.out[f][p] = apply_stencil<T, T, M, T>(fs.in[f], s);
}

template <typename T>
static void gather_t(const Dims& g, int method, const T* disp, int nf, const void* const* in,
                     void* const* out, cudaStream_t st) {
    DispPtrs<T> dp = disp_ptrs(g, disp);
    int nb = blocks_for(g.N, TPB);
    for (int f0 = 0; f0 < nf; f0 += MAXF) {
        FieldSet<T> fs;
        fs.nf = nf - f0 < MAXF ? nf - f0 : MAXF;
        for (int f = 0; f < fs.nf; ++f) {
            fs.in[f] = (const T*)in[f0 + f];
            fs.out[f] = (T*)out[f0 + f];
        }
        switch (method) {
            case NEAREST: k_gather<T, NEAREST><<<nb, TPB, 0, st>>>(g, dp, fs); break;
            case LINEAR: k_gather<T, LINEAR><<<nb, TPB, 0, st>>>(g, dp, fs); break;
            case CUBIC: k_gather<T, CUBIC><<<nb, TPB, 0, st>>>(g, dp, fs); break;
            default: throw Error(E_ARG, "unknown interpolation method");
        }
        FRG_CHECK_LAUNCH();
    }
}

void gather_fields(const Dims& g, int tdtype, int method, const void* disp, int nf,
                   const void* const* in, void* const* out, cudaStream_t st) {
    if (tdtype == F64)
        gather_t<double>(g, method, (const double*)disp, nf, in, out, st);
    else
        gather_t<float>(g, method, (const float*)disp, nf, in, out, st);
}

// transport.py:83-98 — homogeneous SL, one gather per step
void solve_state(const Dims& g, int tdtype, int method, int n_t, const void* disp, void* series,
                 cudaStream_t st) {
    size_t es = tdtype == F64 ? 8 : 4;
    for (int j = 0; j < n_t; ++j) {
        const void* in = (const char*)series + (size_t)j * g.N * es;
        void* out = (char*)series + (size_t)(j + 1) * g.N * es;
        gather_fields(g, tdtype, method, disp, 1, &in, &out, st);
    }
}

// ---------------------------------------------------------------------------
// adjoint / continuity equation (transport.py:105-135)
//   f0 = u(y) a, u_p = u(y) + h f0, f1 = u_p b, out = u(y) + h/2 (f0 + f1)
//   = u(y) * [1 + h/2 (a + b + h a b)],  a = div v(y_b), b = div v(x)
// The bracket is a per-velocity multiplier, built once per refresh.
// ---------------------------------------------------------------------------
template <typename T, int M>
__global__ void __launch_bounds__(TPB) k_adjoint_mult(Dims g, DispPtrs<T> dp, T ht,
                                                      const T* __restrict__ divv, T* __restrict__ cmul) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    Stencil<T, M> s;
    stencil_at<T, M>(g, dp, p, s);
    T a = apply_stencil<T, T, M, T>(divv, s);
    T b = divv[p];
    cmul[p] = T(1) + T(0.5) * ht * (a + b + ht * a * b);
}

template <typename T, int M>
__global__ void __launch_bounds__(TPB) k_adjoint_step(Dims g, DispPtrs<T> dp, const T* __restrict__ cmul,
                                                      const T* __restrict__ u, T* __restrict__ out) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    Stencil<T, M> s;
    stencil_at<T, M>(g, dp, p, s);
    out[p] = apply_stencil<T, T, M, T>(u, s) * cmul[p];
}

#define FRG_DISPATCH_METHOD(method, KERNEL, T, ...)                                      \
    switch (method) {                                                                    \
        case NEAREST: KERNEL<T, NEAREST><<<nb, TPB, 0, st>>>(__VA_ARGS__); break;        \
        case LINEAR: KERNEL<T, LINEAR><<<nb, TPB, 0, st>>>(__VA_ARGS__); break;          \
        case CUBIC: KERNEL<T, CUBIC><<<nb, TPB, 0, st>>>(__VA_ARGS__); break;            \
        default: throw Error(E_ARG, "unknown interpolation method");                     \
    }                                                                                    \
    FRG_CHECK_LAUNCH();

template <typename T>
static void adjoint_multiplier_t(const Dims& g, int method, double ht, const T* disp_b, const T* divv,
                                 T* cmul, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    DispPtrs<T> dp = disp_ptrs(g, disp_b);
    FRG_DISPATCH_METHOD(method, k_adjoint_mult, T, g, dp, (T)ht, divv, cmul);
}

void adjoint_multiplier(const Dims& g, int tdtype, int method, double h_t, const void* disp_b,
                        const void* divv, void* cmul, cudaStream_t st) {
    if (tdtype == F64)
        adjoint_multiplier_t(g, method, h_t, (const double*)disp_b, (const double*)divv, (double*)cmul, st);
    else
        adjoint_multiplier_t(g, method, h_t, (const float*)disp_b, (const float*)divv, (float*)cmul, st);
}

template <typename T>
static void adjoint_step_t(const Dims& g, int method, const T* disp_b, const T* cmul, const T* u, T* out,
                           cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    DispPtrs<T> dp = disp_ptrs(g, disp_b);
    FRG_DISPATCH_METHOD(method, k_adjoint_step, T, g, dp, cmul, u, out);
}

void adjoint_step(const Dims& g, int tdtype, int method, const void* disp_b, const void* cmul,
                  const void* u, void* out, cudaStream_t st) {
    if (tdtype == F64)
        adjoint_step_t(g, method, (const double*)disp_b, (const double*)cmul, (const double*)u, (double*)out, st);
    else
        adjoint_step_t(g, method, (const float*)disp_b, (const float*)cmul, (const float*)u, (float*)out, st);
}

void solve_adjoint(const Dims& g, int tdtype, int method, int n_t, const void* disp_b, const void* cmul,
                   void* series, cudaStream_t st) {
    size_t es = tdtype == F64 ? 8 : 4;
    for (int j = n_t; j > 0; --j) {
        const void* in = (const char*)series + (size_t)j * g.N * es;
        void* out = (char*)series + (size_t)(j - 1) * g.N * es;
        adjoint_step(g, tdtype, method, disp_b, cmul, in, out, st);
    }
}

// ---------------------------------------------------------------------------
// incremental state (transport.py:147-176)
//   m~_{j+1} = m~_j(y) + h/2 (f0 + f1),  f0 = -grad m_j(y) . v~(y),
//   f1 = -grad m_{j+1}(x) . v~(x);   m~_0 = 0.
// grad m_j(y) is gathered once per velocity (grads_y); v~(y) once per call.
// ---------------------------------------------------------------------------
template <typename T, typename CV, int M>
__global__ void __launch_bounds__(TPB) k_inc_first(Dims g, DispPtrs<T> dp, T ht, const CV* __restrict__ vt,
                                                   const T* __restrict__ gy0, const T* __restrict__ gx1,
                                                   T* __restrict__ vtT, T* __restrict__ vty, T* __restrict__ m1,
                                                   T* __restrict__ fin, T fsign) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    Stencil<T, M> s;
    stencil_at<T, M>(g, dp, p, s);
    T f0 = T(0), f1 = T(0);
    for (int c = 0; c < g.d; ++c) {
        long long o = (long long)c * g.N + p;
        T a = apply_stencil<T, T, M, CV>(vt + (long long)c * g.N, s);
        T b = (T)vt[o];
        vty[o] = a;
        vtT[o] = b;
        f0 -= gy0[o] * a;
        f1 -= gx1[o] * b;
    }
    T m = T(0.5) * ht * (f0 + f1);
    if (m1) m1[p] = m;
    if (fin) fin[p] = fsign * m;
}

template <typename T, int M>
__global__ void __launch_bounds__(TPB) k_inc_step(Dims g, DispPtrs<T> dp, T ht, const T* __restrict__ mj,
                                                  const T* __restrict__ vtT, const T* __restrict__ vty,
                                                  const T* __restrict__ gyj, const T* __restrict__ gx1,
                                                  T* __restrict__ mnext, T* __restrict__ fin, T fsign) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    Stencil<T, M> s;
    stencil_at<T, M>(g, dp, p, s);
    T my = apply_stencil<T, T, M, T>(mj, s);
    T f0 = T(0), f1 = T(0);
    for (int c = 0; c < g.d; ++c) {
        long long o = (long long)c * g.N + p;
        f0 -= gyj[o] * vty[o];
        f1 -= gx1[o] * vtT[o];
    }
    T m = my + T(0.5) * ht * (f0 + f1);
    if (mnext) mnext[p] = m;
    if (fin) fin[p] = fsign * m;
}

template <typename T, typename CV>
static void inc_state_t(const Dims& g, int method, int n_t, const T* disp, const T* grads, const T* grads_y,
                        const CV* vt, T* vtT, T* vty, T* series, T* fin, T fsign, bool keep, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    DispPtrs<T> dp = disp_ptrs(g, disp);
    T ht = (T)(1.0 / n_t);
    long long gs = (long long)g.d * g.N;  // gradient slice stride
    // slice buffers: keep == full series, else ping-pong in series[0..1]
    auto slice = [&](int j) -> T* { return keep ? series + (long long)j * g.N : series + (long long)(j & 1) * g.N; };
    if (keep) FRG_CUDA(cudaMemsetAsync(series, 0, sizeof(T) * g.N, st));
    {
        T* out = (n_t == 1 && !keep) ? nullptr : slice(1);
        T* f = (n_t == 1) ? fin : nullptr;
        switch (method) {
            case NEAREST:
                k_inc_first<T, CV, NEAREST><<<nb, TPB, 0, st>>>(g, dp, ht, vt, grads_y, grads + gs, vtT, vty, out, f, fsign);
                break;
            case LINEAR:
                k_inc_first<T, CV, LINEAR><<<nb, TPB, 0, st>>>(g, dp, ht, vt, grads_y, grads + gs, vtT, vty, out, f, fsign);
                break;
            case CUBIC:
                k_inc_first<T, CV, CUBIC><<<nb, TPB, 0, st>>>(g, dp, ht, vt, grads_y, grads + gs, vtT, vty, out, f, fsign);
                break;
            default: throw Error(E_ARG, "unknown interpolation method");
        }
        FRG_CHECK_LAUNCH();
    }
    for (int j = 1; j < n_t; ++j) {
        bool last = (j == n_t - 1);
        T* out = (last && !keep) ? nullptr : slice(j + 1);
        T* f = last ? fin : nullptr;
        FRG_DISPATCH_METHOD(method, k_inc_step, T, g, dp, ht, slice(j), vtT, vty, grads_y + (long long)j * gs,
                            grads + (long long)(j + 1) * gs, out, f, fsign);
    }
}

void inc_state(const Dims& g, int tdtype, int cdtype, int method, int n_t, const void* disp, const void* grads,
               const void* grads_y, const void* vt, void* vtT, void* vty, void* series, void* final_out,
               double final_sign, bool keep_series, cudaStream_t st) {
    if (tdtype == F64 && cdtype == F64)
        inc_state_t<double, double>(g, method, n_t, (const double*)disp, (const double*)grads,
                                    (const double*)grads_y, (const double*)vt, (double*)vtT, (double*)vty,
                                    (double*)series, (double*)final_out, final_sign, keep_series, st);
    else if (tdtype == F32 && cdtype == F32)
        inc_state_t<float, float>(g, method, n_t, (const float*)disp, (const float*)grads, (const float*)grads_y,
                                  (const float*)vt, (float*)vtT, (float*)vty, (float*)series, (float*)final_out,
                                  (float)final_sign, keep_series, st);
    else if (tdtype == F32 && cdtype == F64)
        inc_state_t<float, double>(g, method, n_t, (const float*)disp, (const float*)grads, (const float*)grads_y,
                                   (const double*)vt, (float*)vtT, (float*)vty, (float*)series, (float*)final_out,
                                   (float)final_sign, keep_series, st);
    else
        throw Error(E_ARG, "inc_state: unsupported dtype combination");
}

// ---------------------------------------------------------------------------
// trapezoid body force (kkt.py:225-231, fields.py:347-379)
// ---------------------------------------------------------------------------
template <typename T, typename O>
__global__ void __launch_bounds__(TPB) k_body_force(Dims g, int n_t, const T* __restrict__ lam,
                                                    const T* __restrict__ grads, O* __restrict__ out, bool acc) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    const T ht = T(1) / T(n_t);
    T b[3] = {T(0), T(0), T(0)};
    const long long gs = (long long)g.d * g.N;
    T l0 = lam[p], ln = lam[(long long)n_t * g.N + p];
    for (int c = 0; c < g.d; ++c)
        b[c] = T(0.5) * ht * (l0 * grads[(long long)c * g.N + p] + ln * grads[n_t * gs + (long long)c * g.N + p]);
    for (int j = 1; j < n_t; ++j) {
        T lj = lam[(long long)j * g.N + p];
        for (int c = 0; c < g.d; ++c) b[c] += ht * (lj * grads[j * gs + (long long)c * g.N + p]);
    }
    for (int c = 0; c < g.d; ++c) {
        long long o = (long long)c * g.N + p;
        if (acc)
            out[o] = out[o] + (O)b[c];
        else
            out[o] = (O)b[c];
    }
}

void body_force(const Dims& g, int tdtype, int odtype, int n_t, const void* lam, const void* grads, void* out,
                bool accumulate, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    if (tdtype == F64 && odtype == F64)
        k_body_force<double, double><<<nb, TPB, 0, st>>>(g, n_t, (const double*)lam, (const double*)grads,
                                                         (double*)out, accumulate);
    else if (tdtype == F32 && odtype == F32)
        k_body_force<float, float><<<nb, TPB, 0, st>>>(g, n_t, (const float*)lam, (const float*)grads,
                                                       (float*)out, accumulate);
    else if (tdtype == F32 && odtype == F64)
        k_body_force<float, double><<<nb, TPB, 0, st>>>(g, n_t, (const float*)lam, (const float*)grads,
                                                        (double*)out, accumulate);
    else
        throw Error(E_ARG, "body_force: unsupported dtype combination");
    FRG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// deformation tensor d_t F = (grad v) F, F(0) = I (transport.py:197-221)
// jac layout: (d, d, N) with J[i][k] = d v_i / d x_k (diffops.py:132-139)
// ---------------------------------------------------------------------------
template <typename T, int M>
__global__ void __launch_bounds__(TPB) k_deform_step(Dims g, DispPtrs<T> dp, T ht, const T* __restrict__ jac_y,
                                                     const T* __restrict__ jac, const T* __restrict__ Fin,
                                                     T* __restrict__ Fout, bool identity) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    const int d = g.d;
    T Fy[9], Jy[9], Jx[9], f0[9], Fp[9];
    Stencil<T, M> s;
    stencil_at<T, M>(g, dp, p, s);
    for (int e = 0; e < d * d; ++e) {
        Fy[e] = identity ? T((e / d) == (e % d)) : apply_stencil<T, T, M, T>(Fin + (long long)e * g.N, s);
        Jy[e] = jac_y[(long long)e * g.N + p];
        Jx[e] = jac[(long long)e * g.N + p];
    }
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            T acc = T(0);
            for (int k = 0; k < d; ++k) acc += Jy[i * d + k] * Fy[k * d + j];
            f0[i * d + j] = acc;
            Fp[i * d + j] = Fy[i * d + j] + ht * acc;
        }
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            T acc = T(0);
            for (int k = 0; k < d; ++k) acc += Jx[i * d + k] * Fp[k * d + j];
            Fout[(long long)(i * d + j) * g.N + p] = Fy[i * d + j] + T(0.5) * ht * (f0[i * d + j] + acc);
        }
}

template <typename T>
static void deformation_t(const Dims& g, int method, int n_t, const T* disp, const T* jac, T* F, T* work,
                          cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    DispPtrs<T> dp = disp_ptrs(g, disp);
    long long dd = (long long)g.d * g.d;
    T* jac_y = work;               // dd x N
    T* tmp = work + dd * g.N;      // dd x N
    const void* ins[9];
    void* outs[9];
    for (int e = 0; e < dd; ++e) {
        ins[e] = jac + e * g.N;
        outs[e] = jac_y + e * g.N;
    }
    gather_fields(g, sizeof(T) == 8 ? F64 : F32, method, disp, (int)dd, ins, outs, st);
    // ping-pong so that the final state lands in F
    T* bufs[2] = {(n_t % 2 == 1) ? F : tmp, (n_t % 2 == 1) ? tmp : F};
    const T* cur = nullptr;
    for (int s = 0; s < n_t; ++s) {
        T* out = bufs[s & 1];
        FRG_DISPATCH_METHOD(method, k_deform_step, T, g, dp, (T)(1.0 / n_t), jac_y, jac, cur, out, s == 0);
        cur = out;
    }
}

void deformation_tensor(const Dims& g, int tdtype, int method, int n_t, const void* disp, const void* jac,
                        void* F, void* work, cudaStream_t st) {
    if (tdtype == F64)
        deformation_t(g, method, n_t, (const double*)disp, (const double*)jac, (double*)F, (double*)work, st);
    else
        deformation_t(g, method, n_t, (const float*)disp, (const float*)jac, (float*)F, (float*)work, st);
}

// fields.py:302-312
template <typename T>
__global__ void k_det(Dims g, const T* __restrict__ a, T* __restrict__ det) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    const long long N = g.N;
    if (g.d == 2) {
        det[p] = a[p] * a[3 * N + p] - a[N + p] * a[2 * N + p];
    } else {
#define A(i, j) a[(long long)((i) * 3 + (j)) * N + p]
        det[p] = A(0, 0) * (A(1, 1) * A(2, 2) - A(1, 2) * A(2, 1)) -
                 A(0, 1) * (A(1, 0) * A(2, 2) - A(1, 2) * A(2, 0)) +
                 A(0, 2) * (A(1, 0) * A(2, 1) - A(1, 1) * A(2, 0));
#undef A
    }
}

void determinant(const Dims& g, int tdtype, const void* F, void* det, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    if (tdtype == F64)
        k_det<double><<<nb, TPB, 0, st>>>(g, (const double*)F, (double*)det);
    else
        k_det<float><<<nb, TPB, 0, st>>>(g, (const float*)F, (float*)det);
    FRG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// composed map (transport.py:224-247): D_{k+1} = D_k + disp(j + D_k)
// ---------------------------------------------------------------------------
template <typename T, int M>
__global__ void __launch_bounds__(TPB) k_compose_step(Dims g, DispPtrs<T> dstep, const T* __restrict__ Din,
                                                      T* __restrict__ Dout) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.N) return;
    DispPtrs<T> dcur = disp_ptrs(g, Din);
    Stencil<T, M> s;
    stencil_at<T, M>(g, dcur, p, s);
    for (int c = 0; c < g.d; ++c) {
        long long o = (long long)c * g.N + p;
        Dout[o] = Din[o] + apply_stencil<T, T, M, T>(dstep.a[g.comp_axis(c)], s);
    }
}

template <typename T>
static void compose_t(const Dims& g, int method, int n_t, const T* disp, T* out, T* work, cudaStream_t st) {
    int nb = blocks_for(g.N, TPB);
    DispPtrs<T> dp = disp_ptrs(g, disp);
    long long sz = (long long)g.d * g.N;
    // n_t - 1 compositions; ping-pong so that the result lands in `out`
    int steps = n_t - 1;
    T* bufs[2] = {(steps % 2 == 1) ? out : work, (steps % 2 == 1) ? work : out};
    if (steps == 0) {
        FRG_CUDA(cudaMemcpyAsync(out, disp, sizeof(T) * sz, cudaMemcpyDeviceToDevice, st));
        return;
    }
    const T* cur = disp;
    for (int s = 0; s < steps; ++s) {
        T* o = bufs[s & 1];
        FRG_DISPATCH_METHOD(method, k_compose_step, T, g, dp, cur, o);
        cur = o;
    }
}

void compose_disp(const Dims& g, int tdtype, int method, int n_t, const void* disp, void* out, void* work,
                  cudaStream_t st) {
    if (tdtype == F64)
        compose_t(g, method, n_t, (const double*)disp, (double*)out, (double*)work, st);
    else
        compose_t(g, method, n_t, (const float*)disp, (float*)out, (float*)work, st);
}

}  // namespace frg
