/*
 * libflowreg_b200 — C ABI of the B200-native GNK compute core.
 *
 * Drop-in boundary for the hot path of the reference `flowreg` package
 * (SURVEY.md §8b).  Every pointer argument is DEVICE memory owned by the
 * caller unless stated otherwise; every call is ordered on the CUDA stream
 * passed in (`stream`, a cudaStream_t; NULL = legacy default stream).
 * Functions that return a scalar to the host synchronise that stream.
 *
 * Return value: FRG_OK (0) or a negative status; frg_last_error() gives the
 * message of the most recent failure on the calling thread.
 *
 * Grid convention (fields.py:54-133): shape n[3] = {n0, n1, n2}, C-order,
 * last axis fastest.  2D grids pass n = {1, n0, n1}.  Vector fields hold d
 * components (d = 2 or 3) of N = n0*n1*n2 values each; component c belongs to
 * grid axis (3 - d) + c.  dtype codes: FRG_F32, FRG_F64, FRG_I32.
 */
#ifndef FLOWREG_B200_H
#define FLOWREG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRG_OK 0
#define FRG_E_ARG (-1)
#define FRG_E_NONFINITE (-2)
#define FRG_E_CUDA (-3)
#define FRG_E_CUFFT (-4)
#define FRG_E_STATE (-5)

#define FRG_F32 0
#define FRG_F64 1
#define FRG_I32 2

#define FRG_NEAREST 0
#define FRG_LINEAR 1
#define FRG_CUBIC 2
#define FRG_BSPLINE 3 /* cubic B-spline on spectrally prefiltered coefficients (no reference counterpart) */

#define FRG_FD8 0
#define FRG_SPECTRAL 1

#define FRG_SSD 0
#define FRG_NCC 1

#define FRG_INCOMP_NONE 0
#define FRG_INCOMP_HARD 1
#define FRG_INCOMP_NEAR 2

/* spectral symbols for frg_spectral_apply */
#define FRG_SYM_REG 0          /* alpha*L                           diffops.py:184 */
#define FRG_SYM_REG_INV 1      /* (alpha*L)^-1, zero symbol -> 1     diffops.py:190 */
#define FRG_SYM_REG_INV_SQRT 2 /* (alpha*L)^-1/2                     diffops.py:199 */
#define FRG_SYM_REG_KC 3       /* alpha*L with zero symbol -> 1      kkt.py:283-287 */
#define FRG_SYM_LAPLACIAN 4    /*                                    diffops.py:142 */
#define FRG_SYM_LOWPASS 5      /*                                    diffops.py:296 */
#define FRG_SYM_HIGHPASS 6     /*                                    diffops.py:300 */
#define FRG_SYM_BSPLINE_PREFILTER 7 /* 1 / prod_a (4 + 2 cos(2 pi m_a / n_a)) / 6 */

#define FRG_PRECOND_REG 0
#define FRG_PRECOND_H0 1
#define FRG_PRECOND_2LEVEL 2

typedef struct frg_reg {
    double alpha;      /* RegConfig.alpha                          kkt.py:60 */
    int32_t order;     /* RegOperatorSpec.order (1, 2, 3)          diffops.py:159 */
    int32_t seminorm;  /* RegOperatorSpec.seminorm                 diffops.py:160 */
    int32_t incomp;    /* IncompressibilityMode.mode               diffops.py:212 */
    double beta;       /* IncompressibilityMode.beta               diffops.py:213 */
} frg_reg;

typedef struct frg_config {
    int32_t n[3];            /* grid (n0 = 1 for 2D)                 fields.py:63 */
    int32_t d;               /* 2 or 3 */
    int32_t n_t;             /* time steps                           fields.py:64 */
    int32_t method;          /* FRG_NEAREST/LINEAR/CUBIC             kkt.py:145 */
    int32_t scheme;          /* FRG_FD8 / FRG_SPECTRAL               kkt.py:146 */
    int32_t distance;        /* FRG_SSD / FRG_NCC                    kkt.py:144 */
    int32_t transport_dtype; /* storage of transport fields (F32/F64) */
    int32_t control_dtype;   /* velocity / gradient / PCG vectors (F32/F64) */
    frg_reg reg;
} frg_config;

typedef struct frg_kkt frg_kkt;

const char* frg_last_error(void);
const char* frg_version(void);

/* ---- narrow boundary: _kernels.sample_nd (_kernels.py:222-251) ----------
 * values: dtype FRG_F32/F64/FRG_I32 on grid n; q[3]: f64 fractional indices
 * (q[0] ignored / may be NULL when n[0] == 1); out: npts values of the values
 * dtype (FRG_F64 for FRG_I32 with linear/cubic).  Unknown method -> FRG_E_ARG. */
int frg_sample(const void* values, int32_t dtype, const int32_t n[3], const double* q0, const double* q1,
               const double* q2, int64_t npts, int32_t method, void* out, void* stream);

/* ---- transport (transport.py) ------------------------------------------ */
/* departure displacement in index units, d x N (dtype), from v (vdtype)      transport.py:37-45 */
int frg_departure(const int32_t n[3], int32_t d, int32_t dtype, int32_t vdtype, int32_t method, double h_t,
                  const void* v, void* disp, void* stream);
/* physical departure points y = x - h*disp and back                         transport.py:37-45 */
int frg_disp_to_points(const int32_t n[3], int32_t d, int32_t dtype, const void* disp, void* y, void* stream);
int frg_points_to_disp(const int32_t n[3], int32_t d, int32_t dtype, const void* y, void* disp, void* stream);
/* nf scalar fields gathered at x + disp                                     interp.py:42-62 */
int frg_gather(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, const void* disp, int32_t nf,
               const void* const* in, void* const* out, void* stream);
/* SL tile plan of an fp32 displacement map (one int4 per 32x8x4 tile: the
 * stencil bounding box), built once per map and reused by every gather on it
 * (frg_gather_planned); the KKT context builds and binds its own plans. */
int64_t frg_tile_plan_count(const int32_t n[3]);
int frg_tile_plan(const int32_t n[3], int32_t d, int32_t method, const void* disp, void* plan, void* stream);
/* frg_gather for fp32 fields with a prebuilt plan of `disp` */
int frg_gather_planned(const int32_t n[3], int32_t d, int32_t method, const void* disp, const void* plan, int32_t nf,
                       const void* const* in, void* const* out, void* stream);

/* series[0] holds m0; fills series[1..n_t]                                   transport.py:83-98 */
int frg_solve_state(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t, const void* disp,
                    void* series, void* stream);
/* series[n_t] holds the final condition; fills series[0..n_t-1]             transport.py:105-135 */
int frg_solve_adjoint(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t,
                      const void* disp_b, const void* divv, void* series, void* stream);
/* incremental state; grads (n_t+1) x d x N at the mesh; vt in vdtype;
 * writes all slices (n_t+1) x N                                             transport.py:147-176 */
int frg_solve_inc_state(const int32_t n[3], int32_t d, int32_t dtype, int32_t vdtype, int32_t method,
                        int32_t n_t, const void* disp, const void* grads, const void* vt, void* series,
                        void* stream);
/* trapezoid body force sum_j w_j lam_j grad_j                                kkt.py:225-231 */
int frg_body_force(const int32_t n[3], int32_t d, int32_t dtype, int32_t n_t, const void* lam,
                   const void* grads, void* out, void* stream);
/* F(1) of d_t F = (grad v) F (d*d x N) from the departure disp and jac       transport.py:197-221 */
int frg_deformation_tensor(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t,
                           const void* disp, const void* jac, void* F, void* stream);
int frg_determinant(const int32_t n[3], int32_t d, int32_t dtype, const void* F, void* det, void* stream);
/* one Heun step of d_t F = (grad v) F at every voxel of a 3D grid (or slab):
 * first != 0: F = I + h/2 (J_y + J (I + h J_y)); else F holds F_j(y) on entry
 * and is updated in place (jac_y, jac, F: 9 x N)                transport.py:197-221 */
int frg_deform_update(const int32_t n[3], int32_t dtype, double h_t, int32_t first, const void* jac_y,
                      const void* jac, void* F, void* stream);
/* composed departure displacement over n_t steps                           transport.py:224-247 */
int frg_compose(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t, const void* disp,
                void* out, void* stream);

/* ---- differential operators (diffops.py) ---------------------------------- */
int frg_fd8_gradient(const int32_t n[3], int32_t d, int32_t dtype, int32_t nslices, const void* u, void* out,
                     void* stream);                                           /* diffops.py:98-106 */
int frg_fd8_divergence(const int32_t n[3], int32_t d, int32_t dtype, const void* v, void* out,
                       void* stream);                                         /* diffops.py:117-129 */
int frg_spectral_gradient(const int32_t n[3], int32_t d, int32_t dtype, const void* u, void* out,
                          void* stream);                                      /* diffops.py:67-73 */
int frg_spectral_divergence(const int32_t n[3], int32_t d, int32_t dtype, const void* v, void* out,
                            void* stream);                                    /* diffops.py:117-129 */
int frg_spectral_apply(const int32_t n[3], int32_t d, int32_t dtype, int32_t ncomp, const void* in, void* out,
                       int32_t symbol, const frg_reg* reg, void* stream);    /* diffops.py:176-205,283-301 */
int frg_project(const int32_t n[3], int32_t d, int32_t dtype, const void* b, void* out, const frg_reg* reg,
                void* stream);                                                /* diffops.py:245-280 */
int frg_restrict(const int32_t n[3], int32_t dtype, const void* in, void* out, void* stream); /* diffops.py:312 */
int frg_prolong(const int32_t n_fine[3], int32_t dtype, const void* in, void* out, void* stream); /* diffops.py:329 */

/* ---- reductions / vector updates (fields.py:320-344) ------------------------ */
int frg_dot(int32_t dtype, const void* a, const void* b, int64_t n, double* out, void* stream);
int frg_norm_inf(int32_t dtype, const void* a, int64_t n, double* out, void* stream);
int frg_min_max_sum(int32_t dtype, const void* a, int64_t n, double out[3], void* stream);
int frg_all_finite(int32_t dtype, const void* a, int64_t n, int32_t* out, void* stream);
int frg_axpby(int32_t dtype, double a, const void* x, double b, void* y, int64_t n, void* stream);
int frg_pcg_update(int32_t dtype, double k, const void* s, const void* hs, void* x, void* r, int64_t n,
                   double* rr, void* stream);                                 /* optimizer.py:129-133 */

/* ---- wide boundary: KktState (kkt.py:136-341) ------------------------------ */
int frg_kkt_create(const frg_config* cfg, void* stream, frg_kkt** out);
int frg_kkt_destroy(frg_kkt* k);
/* Destroyed contexts park their device buffers for the next context (capped
   at FRG_POOL_CAP_MB, default 1/4 of device memory); this frees them all. */
int frg_release_pool(void);
/* Measurement probe (bench.py): while armed, CUDA events on the launching
 * stream bracket every launch of the GN matvec's incremental-state first step
 * (the fused 3-field gather + Heun sources, its dominant kernel); read returns
 * the summed duration and the launch count and disarms nothing. */
int frg_probe_arm(int32_t on);
int frg_probe_read(double* total_ms, int64_t* count);
/* Peer windows of the slab path without ghost planes (dist.py peer mode; no
 * reference counterpart — the north star's off-rank departure-point exchange,
 * PAPER.md:545).  A window holds one rank's owned planes (n_loc) of a gathered
 * source field (fp32); frg_peer_alloc returns it with its 64-byte CUDA IPC
 * handle, the other ranks map it with frg_peer_open, and frg_peer_register
 * gives the library every rank's pointer (peers[rank] == local).  Slab SL
 * calls (frg_slab_*) with h0 == 0 whose sources are registered windows read
 * the stencil planes of other ranks straight from their windows (TMA / P2P
 * loads over NVLink): no ghost-plane exchange and no bound on |disp_0|. */
int frg_peer_alloc(int64_t bytes, void** ptr, void* handle);
int frg_peer_free(void* ptr);
int frg_peer_open(const void* handle, void** ptr);
int frg_peer_close(void* ptr);
int frg_peer_register(const void* local, const int32_t n_loc[3], int32_t nranks, int32_t rank,
                      const void* const* peers);
int frg_peer_unregister(const void* local);
int frg_kkt_set_stream(frg_kkt* k, void* stream);
/* images m0, m1 (N values, dtype) — copied into the context             kkt.py:139-162 */
/* Interpolation precision of the SL steps of the GN Hessian matvec: 32
 * (default; fp32 taps, 1e-5 parity) or 16 (north-star mixed-precision mode:
 * the gathered incremental fields are rounded to fp16 taps, weights /
 * accumulation / epilogues stay fp32; tolerance 1e-3 vs the f64 reference).
 * State, adjoint, gradient and objective stay fp32.  Needs fp32 transport. */
int frg_kkt_set_interp_precision(frg_kkt* k, int32_t bits);
int frg_kkt_set_images(frg_kkt* k, const void* m0, const void* m1, int32_t dtype);
/* all velocity-space vectors are control_dtype, d x N                      kkt.py:166-187 */
int frg_kkt_refresh(frg_kkt* k, const void* v);
int frg_kkt_objective(frg_kkt* k, double* J);                             /* kkt.py:198 */
int frg_kkt_objective_at(frg_kkt* k, const void* v_trial, double* J);    /* kkt.py:201-205 */
int frg_kkt_gradient(frg_kkt* k, void* g);                                /* kkt.py:233-235 */
int frg_kkt_hessian_matvec(frg_kkt* k, const void* vt, void* out);        /* kkt.py:237-260 */
/* kind FRG_PRECOND_*; outer_tol = eta; *fell_back set when an inner solve broke down
 *                                                                          kkt.py:308-341 */
int frg_kkt_apply_precond(frg_kkt* k, int32_t kind, double outer_tol, double inner_tol_factor,
                          int32_t inner_max_iterations, const void* r, void* z, int32_t* fell_back);
int frg_kkt_mismatch(frg_kkt* k, double* out);                           /* kkt.py:262-265 */
int frg_kkt_initial_mismatch(frg_kkt* k, double* out);
int frg_kkt_divergence_energy(frg_kkt* k, double* out);                  /* kkt.py:207-218 */
/* counters {matvecs, pde_solves, precond_fallbacks}; set overwrites them  */
int frg_kkt_counters(frg_kkt* k, int64_t out[3]);
int frg_kkt_set_counters(frg_kkt* k, const int64_t in[3]);
/* copy internal series to caller memory (transport dtype):
 * which 0 = state series (n_t+1)xN, 1 = adjoint series, 2 = departure disp dxN,
 * 3 = back departure disp dxN, 4 = div v N, 5 = state gradients (n_t+1)xdxN */
int frg_kkt_get(frg_kkt* k, int32_t which, void* dst);
/* determinant stats of F(1) for the current velocity {min, mean, max}   optimizer.py:169-171 */
int frg_kkt_detgrad(frg_kkt* k, double out[3]);

/* ---------------------------------------------------------------------------
 * Slab decomposition (multi-GPU; the reference has none — CLAIRE's MPI slab
 * decomposition is described in PAPER.md:500-545 and SURVEY.md §8e).  Rank r
 * owns n_loc[0] consecutive planes of a 3D grid with n0_glob planes along
 * axis 0.  Arrays named *_src carry h0 ghost planes before and after the
 * owned planes per component ((n_loc[0] + 2 h0) planes, filled by the caller's
 * halo exchange); all other arrays are (n_loc[0], n1, n2).  fp32 transport,
 * linear, cubic or B-spline.  For FRG_BSPLINE every *_src array holds the
 * B-spline COEFFICIENTS of its field (the prefilter is global: the caller runs
 * it with the slab FFT and frg_slab_spec_apply(FRG_SYM_BSPLINE_PREFILTER)
 * before the halo exchange); *_loc arrays keep the nodal values.  The host
 * (dist.py) exchanges ghost planes and runs the all-to-all transposes between
 * these calls.
 * ------------------------------------------------------------------------- */
int frg_slab_departure(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, double h_t,
                       const void* v_src, const void* v_loc, void* disp, void* stream);
int frg_slab_gather(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, const void* disp,
                    int32_t nf, const void* const* in_src, void* const* out, void* stream);
int frg_slab_adjoint_multiplier(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, double h_t,
                                const void* disp_b, const void* divv_src, const void* divv_loc, void* cmul,
                                void* stream);
int frg_slab_adjoint_step(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, const void* disp_b,
                          const void* cmul, const void* u_src, void* out, void* stream);
/* first incremental-state step: gathers v~ (vt_src), writes m~_1 and the Heun
 * sources S_1..S_{n_t-1} ((n_t-1) x N) from grad m_j (grads, (n_t+1) x 3 x N)
 * and grad m_j(y) (grads_y, n_t x 3 x N) */
int frg_slab_inc_first(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, int32_t n_t,
                       const void* disp, const void* grads, const void* grads_y, const void* vt_src,
                       const void* vt_loc, void* m1, void* S, void* stream);
/* fin (optional, owned planes): fin = fsign * m_next (SSD: lam~(1) = -m~(1)) */
int frg_slab_inc_step(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, const void* disp,
                      const void* m_src, const void* S_j, void* m_next, void* fin, double fsign, void* stream);
int frg_slab_fd8_gradient(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t nslices, const void* u_src,
                          void* out, void* stream);
int frg_slab_fd8_divergence(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, const void* v_src, void* out,
                            void* stream);
/* batched 2D R2C (dir = 1) / C2R (dir = -1, unnormalised) over axes (1, 2) of
 * the owned planes: real (ncomp, n0_loc, n1, n2) <-> complex (ncomp, n0_loc, n1, n2/2+1) */
int frg_slab_fft2(const int32_t n_loc[3], int32_t dtype, int32_t ncomp, int32_t dir, const void* in, void* out,
                  void* stream);
/* in-place 1D C2C along axis 0 of the axis-1 split spectrum (ncomp, n0_glob, n1_loc, n2/2+1) */
int frg_slab_fft1(int32_t n0_glob, int32_t n1_loc, int32_t n2, int32_t dtype, int32_t ncomp, int32_t dir, void* data,
                  void* stream);
/* dir = 1: (n0_loc, n1, nh) -> (nranks, n0_loc, n1/nranks, nh) per component; dir = -1: inverse */
int frg_slab_transpose(int32_t dir, int32_t nranks, const int32_t n_loc[3], int32_t dtype, int32_t ncomp,
                       const void* src, void* dst, void* stream);
/* symbol (FRG_SYM_*) / N on the split spectrum of rows [i1_off, i1_off + n1_loc) */
int frg_slab_spec_apply(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, int32_t dtype, int32_t ncomp,
                        void* x, int32_t kind, const frg_reg* reg, void* stream);
/* mixed precision (the single-GPU mixed path's arithmetic): a = f64 spectrum
 * of alpha L's argument (NULL: P(b) only), b = f32 spectrum, in / out:
 * b = alpha L a + P(b) (normalised) */
int frg_slab_spec_combine_mixed(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, const void* a, void* b,
                                const frg_reg* reg, int32_t project, void* stream);
/* sum_x |grad x|^2 (spectral gradient, Nyquist-zeroed) from this rank's share
 * of the f64 split spectrum of x: the local part, all-reduce to complete */
int frg_slab_grad_energy(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, const void* x_spec, double* out,
                         void* stream);
/* dst = (ddtype) src, f32 <-> f64 (vectorised) */
int frg_convert(int32_t sdtype, const void* src, int32_t ddtype, void* dst, int64_t n, void* stream);
/* a = alpha L a + P(b) (normalised); a == b: P(b) only */
int frg_slab_spec_combine(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, int32_t dtype, void* a,
                          const void* b, const frg_reg* reg, int32_t project, void* stream);

/* Bind a displacement map to its tile plan (frg_tile_plan) for the SL calls
 * this host thread makes until frg_clear_plans (two slots: forward / backward
 * map); used by the slab path, whose per-step calls carry only the map. */
int frg_bind_plan(int32_t slot, const void* disp, const void* plan, int32_t method);
int frg_clear_plans(void);
/* trapezoid body force with a lambda slice stride (elements; slab series
 * padded with ghost planes between slices) */
int frg_slab_body_force(const int32_t n_loc[3], int32_t n_t, const void* lam, int64_t lam_stride, const void* grads,
                        void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FLOWREG_B200_H */
