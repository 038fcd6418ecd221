// Internal host-side launcher declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace frg {

// ---- gathers / transport (transport.cu) ------------------------------------
// generic sample at f64 fractional indices (sample_nd boundary)
void sample_q(const void* vals, int dtype, const Dims& g, const double* q0, const double* q1,
              const double* q2, long long npts, int method, void* out, cudaStream_t st);

// RK2 departure displacement (index units) from velocity v (vdtype), d comps
// (slab mode: v carries g.h0 ghost planes per component, vloc is v on the
// owned planes; vloc == nullptr: v itself)
void departure(const Dims& g, int tdtype, int vdtype, int method, double h_t, const void* v,
               void* disp, cudaStream_t st, const void* vloc = nullptr);
// physical departure points y = x - h*disp (tdtype) and the inverse map
void disp_to_points(const Dims& g, int tdtype, const void* disp, void* y, cudaStream_t st);
void points_to_disp(const Dims& g, int tdtype, const void* y, void* disp, cudaStream_t st);

// out_f = in_f(x + disp(x)) for nf fields (each N long, tdtype)
void gather_fields(const Dims& g, int tdtype, int method, const void* disp, int nf,
                   const void* const* in, void* const* out, cudaStream_t st);
// state: series[j+1] = series[j](y)
void solve_state(const Dims& g, int tdtype, int method, int n_t, const void* disp, void* series,
                 cudaStream_t st);
// adjoint multiplier c = 1 + h/2 (div(y_b) + div + h div(y_b) div)
void adjoint_multiplier(const Dims& g, int tdtype, int method, double h_t, const void* disp_b,
                        const void* divv, void* cmul, cudaStream_t st, const void* divl = nullptr);
// slab-mode incremental state pieces (fp32; sources with g.h0 ghost planes):
// first step (gathers v~, forms S_0..S_{n_t-1}; m1 = S_0) and one later step
void inc_first(const Dims& g, int method, int n_t, const float* disp, const float* grads, const float* grads_y,
               const float* vt_src, const float* vt_loc, float* m1, float* S, cudaStream_t st);
void inc_step(const Dims& g, int method, const float* disp, const float* m_src, const float* Sj, float* m_next,
              cudaStream_t st, float* fin = nullptr, float fsign = 0.f);
// one backward step: out = u(y_b) * c
void adjoint_step(const Dims& g, int tdtype, int method, const void* disp_b, const void* cmul,
                  const void* u, void* out, cudaStream_t st);
// adjoint series from a final condition (series[n_t] must hold it)
void solve_adjoint(const Dims& g, int tdtype, int method, int n_t, const void* disp_b,
                   const void* cmul, void* series, cudaStream_t st);
// incremental state. grads: (n_t+1) x d x N at x; grads_y: n_t x d x N gathered at y.
// vt: control dtype. Writes vtT (d x N, tdtype), the Heun sources S ((n_t-1) x N,
// tdtype) and the series slices
// (n_t+1) x N (slice 0 zeroed); if final_sign != 0 and final_out != nullptr the
// last slice is also written as final_sign * m~(1) into final_out.
void inc_state(const Dims& g, int tdtype, int cdtype, int method, int n_t, const void* disp,
               const void* grads, const void* grads_y, const void* vt, void* vtT, void* S,
               void* series, void* final_out, double final_sign, bool keep_series,
               cudaStream_t st);
// trapezoid body force b = sum_j w_j lam_j grad_j, written in odtype; if
// accumulate, out += b
void body_force(const Dims& g, int tdtype, int odtype, int n_t, const void* lam, const void* grads,
                void* out, bool accumulate, cudaStream_t st, long long lam_stride = 0);
// deformation tensor endpoint F(1) (d*d x N, tdtype) and jacobian at x
void deformation_tensor(const Dims& g, int tdtype, int method, int n_t, const void* disp,
                        const void* jac, void* F, void* work, cudaStream_t st);
void determinant(const Dims& g, int tdtype, const void* F, void* det, cudaStream_t st);
void deform_update(const Dims& g, int tdtype, double ht, bool first, const void* jac_y, const void* jac, void* F,
                   cudaStream_t st);
// composed departure displacement over n_t steps
void compose_disp(const Dims& g, int tdtype, int method, int n_t, const void* disp, void* out,
                  void* work, cudaStream_t st);

// ---- finite differences (fd8.cu) ---------------------------------------------
// gradient of nslices scalar fields (slice stride N) -> nslices x d x N
void fd8_gradient(const Dims& g, int tdtype, int nslices, const void* u, void* out, cudaStream_t st);
void fd8_divergence(const Dims& g, int tdtype, const void* v, void* out, cudaStream_t st);

// ---- reductions / pointwise (reduce.cu) --------------------------------------
// all return through a host pointer after a stream sync
double dot(int dtype, const void* a, const void* b, long long n, cudaStream_t st);
double abs_max(int dtype, const void* a, long long n, cudaStream_t st);
void min_max_sum(int dtype, const void* a, long long n, double out[3], cudaStream_t st);
bool all_finite(int dtype, const void* a, long long n, cudaStream_t st);
void convert(int sdtype, const void* src, int ddtype, void* dst, long long n, cudaStream_t st);
// y = a*x + b*y  (same dtype)
void axpby(int dtype, double a, const void* x, double b, void* y, long long n, cudaStream_t st);
// z = x + a*y
void xpay_to(int dtype, const void* x, double a, const void* y, void* z, long long n, cudaStream_t st);
// fused PCG update: x += k*s ; r -= k*hs ; returns <r, r> (unweighted)
double pcg_update(int dtype, double k, const void* s, const void* hs, void* x, void* r, long long n,
                  cudaStream_t st);
void fill(int dtype, void* a, double value, long long n, cudaStream_t st);
// out (odtype) += src (sdtype)
void add_into(int odtype, void* out, int sdtype, const void* src, long long n, cudaStream_t st);
void scale_diff(int dtype, const void* a, const void* b, double sa, void* out, long long n,
                cudaStream_t st);  // out = sa*(a - b)
// out = c1*a + c2*b + c3*c  (pointwise, same dtype; b/c may be null)
void lincomb3(int dtype, double c1, const void* a, double c2, const void* b, double c3, const void* c,
              void* out, long long n, cudaStream_t st);
// out = (sum_c g[c]*s[c]) * g   (rank-one h0 term, d comps); accumulate into out if acc
void rank_one(const Dims& g, int dtype, const void* gm, const void* s, void* out, bool acc,
              cudaStream_t st);

// ---- spectral (spectral.cu) ---------------------------------------------------
enum SpecKind {
    SK_REG = 0,          // alpha * sym
    SK_REG_INV = 1,      // 1/(alpha * sym), sym==0 -> 1
    SK_REG_INV_SQRT = 2, // 1/sqrt(alpha * sym), sym==0 -> 1
    SK_REG_KC = 3,       // alpha * sym, sym==0 -> 1 (h0 block)
    SK_LAPLACIAN = 4,    // -|k|^2
    SK_LOWPASS = 5,
    SK_HIGHPASS = 6,
    SK_BSPLINE_PREFILTER = 7,  // 1 / prod_a (4 + 2 cos(2 pi m_a / n_a)) / 6 (cubic B-spline coefficients)
};
struct RegSpec {
    double alpha;
    int order;
    int seminorm;
    int incomp;  // 0 none, 1 incompressible, 2 near-incompressible
    double beta;
};
// out = real(ifft(symbol * fft(in))) for ncomp fields (dtype); in/out may alias
void spectral_apply(const Dims& g, int dtype, int ncomp, const void* in, void* out, int kind,
                    const RegSpec& r, cudaStream_t st);
// out = alpha L a + P[b]  (a: adtype, b: bdtype, out: adtype); P = identity if incomp none.
// a may be null (then only P[b]).
void reg_plus_project(const Dims& g, int adtype, const void* a, int bdtype, const void* b, void* out,
                      const RegSpec& r, cudaStream_t st);
void project(const Dims& g, int dtype, const void* b, void* out, const RegSpec& r, cudaStream_t st);
void spectral_gradient(const Dims& g, int dtype, const void* u, void* out, cudaStream_t st);
void spectral_divergence(const Dims& g, int dtype, const void* v, void* out, cudaStream_t st);
// 0.5 * <alpha L v, v> (quadrature weighted) via Parseval on the half spectrum
double reg_energy(const Dims& g, int dtype, const void* v, const RegSpec& r, cudaStream_t st);
// spectral restriction (fine g -> coarse) and prolongation (coarse -> fine g), scalar fields
void restrict_field(const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st);
void prolong_field(const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st);
void spectral_release_plans();

// ---- slab-decomposed spectral pieces (spectral.cu; multi-GPU, dist.py) ------
// batched 2D R2C (dir > 0) / C2R (dir < 0, unnormalised) over axes (1, 2) of
// n0_loc planes x ncomp: real (ncomp, n0_loc, n1, n2) <-> complex (ncomp, n0_loc, n1, nh)
void slab_fft2(int n0_loc, int n1, int n2, int dtype, int ncomp, int dir, const void* in, void* out, cudaStream_t st);
// in-place batched 1D C2C along axis 0 of (ncomp, n0, cols) complex (cols = n1_loc * nh)
void slab_fft1(int n0, int cols, int dtype, int ncomp, int dir, void* data, cudaStream_t st);
// (n0_loc, n1, nh) <-> (P, n0_loc, n1/P, nh) per component (all-to-all staging)
void slab_transpose(int dir, int P, int n0_loc, int n1, int nh, int elem_bytes, int ncomp, const void* src, void* dst,
                    cudaStream_t st);
// on the axis-1 split spectrum (ncomp, n0, n1_loc, nh) of the GLOBAL grid g
void slab_spec_scale(const Dims& g, int i1_off, int n1_loc, int dtype, int ncomp, void* x, int kind,
                     const RegSpec& r, cudaStream_t st);
// a = alpha L a + P(b) (normalised); a == b: P(b) only
// mixed precision: a (f64 spectrum, or nullptr: P(b) only), b (f32 spectrum)
// in / out: b = alpha L a + P(b) in fp32 arithmetic per bin
void slab_spec_combine_mixed(const Dims& g, int i1_off, int n1_loc, const void* a, void* b, const RegSpec& r,
                             bool project, cudaStream_t st);
// sum over the split spectrum of |grad|^2 weights (Nyquist-zeroed integer
// wavenumbers) x |x_k|^2, half-spectrum bins doubled, / N (= sum_x |grad x|^2)
double slab_grad_energy(const Dims& g, int i1_off, int n1_loc, const void* x_spec, cudaStream_t st);
void slab_spec_combine(const Dims& g, int i1_off, int n1_loc, int dtype, void* a, const void* b, const RegSpec& r,
                       bool project, cudaStream_t st);

// peer windows of the slab path without ghost planes (tma.cu)
void peer_register(const float* local, int n0, int n1, int n2, int nranks, int rank, const float* const* peers);
void peer_unregister(const float* local);
void* ipc_alloc(size_t bytes, void* handle);
void* ipc_open(const void* handle);
void ipc_close(void* p);

// launch probe of the GN matvec's IncFirstOp kernel (transport_inc.cu)
void probe_arm(bool on);
void probe_read(double* total_ms, long long* count);

}  // namespace frg
