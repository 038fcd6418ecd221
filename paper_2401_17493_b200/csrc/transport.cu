// Semi-Lagrangian transport kernels (sm_100a).
//
// Departure points are stored once per velocity as DISPLACEMENTS in index
// units, disp = q(y) - j, instead of physical coordinates: the reference keeps
// y and recomputes q = n/2 - 1 - y/h per solve (transport.py:65-80,
// interp.py:22-34).  In index units the RK2 map of transport.py:37-45 reads
//   q~ = j + (h_t/h) v(x),   disp = (h_t/2h) (v(x) + v(q~)),
// exact for v = 0 and well conditioned in fp32 (|disp| is a few cells).
// Every SL time step is ONE launch of the shared-memory tiled gather engine
// (sl_tile.cuh) with the step's pointwise update fused into its epilogue.
#include "ops.h"
#include <cstdlib>
#include "sl_half.cuh"

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
    make_stencil_q<M>(g, q0 ? q0[p] : 0.0, q1[p], q2[p], s);
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
        case BSPLINE: k_sample_q<V, O, BSPLINE><<<nb, TPB, 0, st>>>(vals, g, q0, q1, q2, npts, out); break;
        default: throw Error(E_ARG, "unknown interpolation method");
    }
    FRG_CHECK_LAUNCH();
}

void sample_q(const void* vals, int dtype, const Dims& g, const double* q0, const double* q1,
              const double* q2, long long npts, int method, void* out, cudaStream_t st) {
    if (method == BSPLINE) {
        // B-spline: sample the prefiltered coefficients (float grids only)
        FRG_REQUIRE(dtype == F32 || dtype == F64, "bspline interpolation needs float values");
        void* c = bspline_scratch(0, (size_t)g.N * (dtype == F64 ? 8 : 4));
        bspline_prefilter(g, dtype, vals, c, st);
        vals = c;
    }
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
// RK2 departure displacement (transport.py:37-45)
// ---------------------------------------------------------------------------
template <typename T, typename VI, int D>
struct DepartureOp {
    using V = VI;
    static constexpr bool kLateDisp = true;  // displacement from the preceding launch (PDL, sl_fast.cuh)
    const VI* v[3];      // per component: gathered source (slab: with ghost planes)
    const VI* vl[3];     // per component: v at the output voxels
    T sc[3];             // per component: h_t / h_axis
    T* out[3];           // per component
    int axis_of[3];
    void set_field(int f, const VI* p) { v[f] = p; }
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const {
        T dd[3] = {T(0), T(0), T(0)};
#pragma unroll
        for (int c = 0; c < D; ++c) dd[axis_of[c]] = sc[c] * (T)vl[c][p];
        d0 = dd[0];
        d1 = dd[1];
        d2 = dd[2];
    }
    __host__ __device__ __forceinline__ const VI* field(int f) const { return v[f]; }
    __device__ __forceinline__ void done(int p, const T (&vals)[D]) const {
#pragma unroll
        for (int c = 0; c < D; ++c) out[c][p] = (T(0.5) * sc[c]) * ((T)vl[c][p] + vals[c]);
    }
};

template <typename T, typename VI, int D>
static void departure_d(const Dims& g, int method, double ht, const VI* v, const VI* vloc, T* disp,
                        cudaStream_t st) {
    DepartureOp<T, VI, D> op;
    const size_t Ns = (size_t)(g.n0 + 2 * g.h0) * g.n1 * g.n2;  // source component stride
    for (int c = 0; c < D; ++c) {
        int a = g.comp_axis(c);
        op.v[c] = v + (size_t)c * Ns;
        op.vl[c] = vloc + (size_t)c * g.N;
        op.out[c] = disp + (size_t)c * g.N;
        op.sc[c] = (T)(ht / (TWO_PI / g.axis_glob(a)));
        op.axis_of[c] = a;
    }
    launch_sl<T, D>(g, method, op, st);
}

template <typename T, typename VI>
static void departure_t(const Dims& g, int method, double ht, const VI* v, const VI* vloc, T* disp,
                        cudaStream_t st) {
    if (g.d == 3)
        departure_d<T, VI, 3>(g, method, ht, v, vloc, disp, st);
    else
        departure_d<T, VI, 2>(g, method, ht, v, vloc, disp, st);
}

void departure(const Dims& g, int tdtype, int vdtype, int method, double h_t, const void* v, void* disp,
               cudaStream_t st, const void* vloc) {
    if (!vloc) vloc = v;
    if (tdtype == F64 && vdtype == F64)
        departure_t(g, method, h_t, (const double*)v, (const double*)vloc, (double*)disp, st);
    else if (tdtype == F32 && vdtype == F32)
        departure_t(g, method, h_t, (const float*)v, (const float*)vloc, (float*)disp, st);
    else if (tdtype == F32 && vdtype == F64)
        departure_t(g, method, h_t, (const double*)v, (const double*)vloc, (float*)disp, st);
    else
        throw Error(E_ARG, "departure: unsupported dtype combination");
}

// y = x - h*disp   /   disp = (x - y)/h   (fields.py:105-114: x_j = (n/2-(j+1)) h)
template <typename T, bool TO_POINTS>
__global__ void k_disp_points(Dims g, const T* __restrict__ src, T* __restrict__ dst) {
    Vox v;
    if (!vox(g, v)) return;
    const int p = v.p;
    const int idx[3] = {v.i, v.j, v.k};
    for (int c = 0; c < g.d; ++c) {
        int a = g.comp_axis(c);
        int n = g.axis_len(a);
        T h = (T)(TWO_PI / n);
        T x = (T)((n / 2) - (idx[a] + 1.0)) * h;
        size_t o = (size_t)c * g.N + p;
        if (TO_POINTS)
            dst[o] = x - h * src[o];
        else
            dst[o] = (x - src[o]) / h;
    }
}

void disp_to_points(const Dims& g, int tdtype, const void* disp, void* y, cudaStream_t st) {
    if (tdtype == F64)
        k_disp_points<double, true><<<vox_grid(g), vox_block(), 0, st>>>(g, (const double*)disp, (double*)y);
    else
        k_disp_points<float, true><<<vox_grid(g), vox_block(), 0, st>>>(g, (const float*)disp, (float*)y);
    FRG_CHECK_LAUNCH();
}

void points_to_disp(const Dims& g, int tdtype, const void* y, void* disp, cudaStream_t st) {
    if (tdtype == F64)
        k_disp_points<double, false><<<vox_grid(g), vox_block(), 0, st>>>(g, (const double*)y, (double*)disp);
    else
        k_disp_points<float, false><<<vox_grid(g), vox_block(), 0, st>>>(g, (const float*)y, (float*)disp);
    FRG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// multi-field gather at one displacement map
// ---------------------------------------------------------------------------
template <typename T, int NF>
struct GatherOp {
    using V = T;
    DispSrc<T> ds;
    const T* in[NF];
    T* out[NF];
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const { ds.get(p, d0, d1, d2); }
    __host__ __device__ __forceinline__ const T* field(int f) const { return in[f]; }
    void set_field(int f, const T* p) { in[f] = p; }
    __device__ __forceinline__ void done(int p, const T (&vals)[NF]) const {
#pragma unroll
        for (int f = 0; f < NF; ++f) out[f][p] = vals[f];
    }
};

template <typename T, int NF>
static void gather_n(const Dims& g, int method, const T* disp, const void* const* in, void* const* out,
                     cudaStream_t st) {
    GatherOp<T, NF> op;
    op.ds = disp_src(g, disp);
    for (int f = 0; f < NF; ++f) {
        op.in[f] = (const T*)in[f];
        op.out[f] = (T*)out[f];
    }
    launch_sl<T, NF>(g, method, op, st);
}

template <typename T>
static void gather_t(const Dims& g, int method, const T* disp, int nf, const void* const* in, void* const* out,
                     cudaStream_t st) {
    int f = 0;
    // fp32 fields on a planned map: one launch per field.  The single-field
    // engine runs 4 CTAs/SM (the 3-field one 3, register-limited) and the
    // planned TMA needs no bounding-box phase, so re-reading the map per field
    // costs less than the lost residency (12-field grad m_j(y) gather at 256^3:
    // 2.16 -> 1.95 ms).  FRG_GATHER_GROUP=3 restores 3-field launches.
    static const int group = getenv("FRG_GATHER_GROUP") ? atoi(getenv("FRG_GATHER_GROUP")) : 1;
    if (sizeof(T) == 4 && group == 1 && disp_src(g, disp).plan) {
        for (; f < nf; ++f) gather_n<T, 1>(g, method, disp, in + f, out + f, st);
        return;
    }
    while (nf - f >= 3) {
        gather_n<T, 3>(g, method, disp, in + f, out + f, st);
        f += 3;
    }
    if (nf - f == 2) gather_n<T, 2>(g, method, disp, in + f, out + f, st);
    if (nf - f == 1) gather_n<T, 1>(g, method, disp, in + f, out + f, st);
}

void gather_fields(const Dims& g, int tdtype, int method, const void* disp, int nf, const void* const* in,
                   void* const* out, cudaStream_t st) {
    if (tdtype == F64)
        gather_t<double>(g, method, (const double*)disp, nf, in, out, st);
    else
        gather_t<float>(g, method, (const float*)disp, nf, in, out, st);
}

// transport.py:83-98 — homogeneous SL, one gather per step
void solve_state(const Dims& g, int tdtype, int method, int n_t, const void* disp, void* series, cudaStream_t st) {
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
template <typename T>
struct AdjMultOp {
    using V = T;
    DispSrc<T> ds;
    const T* divv;  // gathered source (slab: with ghost planes)
    const T* divl;  // div v at the output voxels
    T* cmul;
    T ht;
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const { ds.get(p, d0, d1, d2); }
    __host__ __device__ __forceinline__ const T* field(int) const { return divv; }
    void set_field(int, const T* p) { divv = p; }
    using Pre = T;
    __device__ __forceinline__ T pre(int p) const { return divl[p]; }
    __device__ __forceinline__ void done(int p, const T (&vals)[1], T b) const {
        T a = vals[0];
        cmul[p] = T(1) + T(0.5) * ht * (a + b + ht * a * b);
    }
};

template <typename T>
struct AdjStepOp {
    using V = T;
    DispSrc<T> ds;
    const T* u;
    const T* cmul;
    T* out;
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const { ds.get(p, d0, d1, d2); }
    __host__ __device__ __forceinline__ const T* field(int) const { return u; }
    void set_field(int, const T* p) { u = p; }
    using Pre = T;
    __device__ __forceinline__ T pre(int p) const { return cmul[p]; }
    __device__ __forceinline__ void done(int p, const T (&vals)[1], T c) const { out[p] = vals[0] * c; }
};

template <typename T>
static void adjoint_multiplier_t(const Dims& g, int method, double ht, const T* disp_b, const T* divv, T* cmul,
                                 cudaStream_t st, const T* divl) {
    AdjMultOp<T> op;
    op.ds = disp_src(g, disp_b);
    op.divv = divv;
    op.divl = divl ? divl : divv;
    op.cmul = cmul;
    op.ht = (T)ht;
    launch_sl<T, 1>(g, method, op, st);
}

void adjoint_multiplier(const Dims& g, int tdtype, int method, double h_t, const void* disp_b, const void* divv,
                        void* cmul, cudaStream_t st, const void* divl) {
    if (tdtype == F64)
        adjoint_multiplier_t(g, method, h_t, (const double*)disp_b, (const double*)divv, (double*)cmul, st,
                             (const double*)divl);
    else
        adjoint_multiplier_t(g, method, h_t, (const float*)disp_b, (const float*)divv, (float*)cmul, st,
                             (const float*)divl);
}

template <typename T>
static void adjoint_step_t(const Dims& g, int method, const T* disp_b, const T* cmul, const T* u, T* out,
                           cudaStream_t st) {
    AdjStepOp<T> op;
    op.ds = disp_src(g, disp_b);
    op.u = u;
    op.cmul = cmul;
    op.out = out;
    launch_sl<T, 1>(g, method, op, st);
}

void adjoint_step(const Dims& g, int tdtype, int method, const void* disp_b, const void* cmul, const void* u,
                  void* out, cudaStream_t st) {
    if (tdtype == F64)
        adjoint_step_t(g, method, (const double*)disp_b, (const double*)cmul, (const double*)u, (double*)out, st);
    else
        adjoint_step_t(g, method, (const float*)disp_b, (const float*)cmul, (const float*)u, (float*)out, st);
}

void solve_adjoint(const Dims& g, int tdtype, int method, int n_t, const void* disp_b, const void* cmul, void* series,
                   cudaStream_t st) {
    size_t es = tdtype == F64 ? 8 : 4;
    for (int j = n_t; j > 0; --j) {
        const void* in = (const char*)series + (size_t)j * g.N * es;
        void* out = (char*)series + (size_t)(j - 1) * g.N * es;
        adjoint_step(g, tdtype, method, disp_b, cmul, in, out, st);
    }
}

// ---------------------------------------------------------------------------
// trapezoid body force (kkt.py:225-231, fields.py:347-379)
// ---------------------------------------------------------------------------
template <typename T, typename O>
__global__ void __launch_bounds__(TPB) k_body_force(Dims g, int n_t, const T* __restrict__ lam,
                                                    const T* __restrict__ grads, O* __restrict__ out, bool acc) {
    Vox v;
    if (!vox(g, v)) return;
    const int p = v.p;
    const size_t N = g.N;
    const T ht = T(1) / T(n_t);
    T b[3] = {T(0), T(0), T(0)};
    const size_t gs = (size_t)g.d * N;
    T l0 = lam[p], ln = lam[(size_t)n_t * N + p];
    for (int c = 0; c < g.d; ++c)
        b[c] = T(0.5) * ht * (l0 * grads[c * N + p] + ln * grads[n_t * gs + c * N + p]);
    for (int j = 1; j < n_t; ++j) {
        T lj = lam[(size_t)j * N + p];
        for (int c = 0; c < g.d; ++c) b[c] += ht * (lj * grads[j * gs + c * N + p]);
    }
    for (int c = 0; c < g.d; ++c) {
        size_t o = c * N + p;
        if (acc)
            out[o] = out[o] + (O)b[c];
        else
            out[o] = (O)b[c];
    }
}

// fp32 streaming variant: 4 consecutive voxels per thread with 16-byte loads
// (5 lambda slices + 15 gradient fields in, 3 components out per voxel), same
// per-voxel expression order as k_body_force
__global__ void __launch_bounds__(TPB) k_body_force_f4(long long N4, int n_t, int d, const float4* __restrict__ lam,
                                                       long long ls4, const float4* __restrict__ grads,
                                                       float4* __restrict__ out, bool acc) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= N4) return;
    const float ht = 1.f / (float)n_t;
    const long long gs = (long long)d * N4;
    const float4 l0 = lam[q], ln = lam[(long long)n_t * ls4 + q];
    float4 b[3];
    for (int c = 0; c < d; ++c) {
        const float4 g0 = grads[c * N4 + q], gn = grads[n_t * gs + c * N4 + q];
        b[c].x = 0.5f * ht * (l0.x * g0.x + ln.x * gn.x);
        b[c].y = 0.5f * ht * (l0.y * g0.y + ln.y * gn.y);
        b[c].z = 0.5f * ht * (l0.z * g0.z + ln.z * gn.z);
        b[c].w = 0.5f * ht * (l0.w * g0.w + ln.w * gn.w);
    }
    for (int j = 1; j < n_t; ++j) {
        const float4 lj = lam[(long long)j * ls4 + q];
        for (int c = 0; c < d; ++c) {
            const float4 gj = grads[j * gs + c * N4 + q];
            b[c].x += ht * (lj.x * gj.x);
            b[c].y += ht * (lj.y * gj.y);
            b[c].z += ht * (lj.z * gj.z);
            b[c].w += ht * (lj.w * gj.w);
        }
    }
    for (int c = 0; c < d; ++c) {
        float4 o = b[c];
        if (acc) {
            const float4 x = out[c * N4 + q];
            o.x = x.x + o.x;
            o.y = x.y + o.y;
            o.z = x.z + o.z;
            o.w = x.w + o.w;
        }
        out[c * N4 + q] = o;
    }
}

void body_force(const Dims& g, int tdtype, int odtype, int n_t, const void* lam, const void* grads, void* out,
                bool accumulate, cudaStream_t st, long long lam_stride) {
    if (lam_stride <= 0) lam_stride = g.N;
    if (tdtype == F32 && odtype == F32 && g.N % 4 == 0 && lam_stride % 4 == 0 &&
        ((((uintptr_t)lam) | ((uintptr_t)grads) | ((uintptr_t)out)) & 15) == 0) {
        const long long N4 = g.N / 4;
        k_body_force_f4<<<blocks_for(N4, TPB), TPB, 0, st>>>(N4, n_t, g.d, (const float4*)lam, lam_stride / 4,
                                                             (const float4*)grads, (float4*)out, accumulate);
        FRG_CHECK_LAUNCH();
        return;
    }
    FRG_REQUIRE(lam_stride == g.N, "strided lambda series need the fp32 body force");
    if (tdtype == F64 && odtype == F64)
        k_body_force<double, double><<<vox_grid(g), vox_block(), 0, st>>>(g, n_t, (const double*)lam,
                                                                          (const double*)grads, (double*)out,
                                                                          accumulate);
    else if (tdtype == F32 && odtype == F32)
        k_body_force<float, float><<<vox_grid(g), vox_block(), 0, st>>>(g, n_t, (const float*)lam,
                                                                        (const float*)grads, (float*)out, accumulate);
    else if (tdtype == F32 && odtype == F64)
        k_body_force<float, double><<<vox_grid(g), vox_block(), 0, st>>>(g, n_t, (const float*)lam,
                                                                         (const float*)grads, (double*)out,
                                                                         accumulate);
    else
        throw Error(E_ARG, "body_force: unsupported dtype combination");
    FRG_CHECK_LAUNCH();
}

// fields.py:302-312
template <typename T>
__global__ void k_det(Dims g, const T* __restrict__ a, T* __restrict__ det) {
    Vox v;
    if (!vox(g, v)) return;
    const int p = v.p;
    const size_t N = g.N;
    if (g.d == 2) {
        det[p] = a[p] * a[3 * N + p] - a[N + p] * a[2 * N + p];
    } else {
#define A(i, j) a[(size_t)((i) * 3 + (j)) * N + p]
        det[p] = A(0, 0) * (A(1, 1) * A(2, 2) - A(1, 2) * A(2, 1)) - A(0, 1) * (A(1, 0) * A(2, 2) - A(1, 2) * A(2, 0)) +
                 A(0, 2) * (A(1, 0) * A(2, 1) - A(1, 1) * A(2, 0));
#undef A
    }
}

void determinant(const Dims& g, int tdtype, const void* F, void* det, cudaStream_t st) {
    if (tdtype == F64)
        k_det<double><<<vox_grid(g), vox_block(), 0, st>>>(g, (const double*)F, (double*)det);
    else
        k_det<float><<<vox_grid(g), vox_block(), 0, st>>>(g, (const float*)F, (float*)det);
    FRG_CHECK_LAUNCH();
}

}  // namespace frg
