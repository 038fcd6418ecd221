// extern "C" boundary of libflowreg_b200 (include/flowreg_b200.h).
// Each entry point validates its arguments, converts exceptions into status
// codes and records the message for frg_last_error().
#include <string>
#include <vector>

#include "../../include/flowreg_b200.h"
#include "kkt.h"
#include "sl_fast.cuh"

using namespace frg;

static thread_local std::string g_last_error;

template <typename F>
static int guard(F&& f) {
    try {
        f();
        return FRG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FRG_E_STATE;
    }
}

static Dims dims_of(const int32_t n[3], int d) {
    FRG_REQUIRE(n != nullptr, "null grid");
    FRG_REQUIRE(n[0] >= 1 && n[1] >= 1 && n[2] >= 1, "grid sizes must be positive");
    FRG_REQUIRE(d == 2 || d == 3, "d must be 2 or 3");
    FRG_REQUIRE((d == 2) == (n[0] == 1), "2D grids are passed as n = {1, n0, n1}");
    return make_dims(n, d);
}

static void check_dtype(int dt) { FRG_REQUIRE(dt == FRG_F32 || dt == FRG_F64, "dtype must be FRG_F32 or FRG_F64"); }
static void check_method(int m) { FRG_REQUIRE(m >= 0 && m <= 3, "unknown interpolation method"); }

static RegSpec reg_of(const frg_reg* r) {
    FRG_REQUIRE(r != nullptr, "null frg_reg");
    FRG_REQUIRE(r->alpha > 0, "alpha must be positive");
    FRG_REQUIRE(r->order >= 1 && r->order <= 3, "order must be 1, 2 or 3");
    FRG_REQUIRE(r->incomp >= 0 && r->incomp <= 2, "unknown incompressibility mode");
    FRG_REQUIRE(r->incomp != 2 || r->beta > 0, "beta must be positive for the relaxed mode");
    RegSpec s;
    s.alpha = r->alpha;
    s.order = r->order;
    s.seminorm = r->seminorm;
    s.incomp = r->incomp;
    s.beta = r->beta;
    return s;
}

#define ST(s) ((cudaStream_t)(s))

extern "C" {

const char* frg_last_error(void) { return g_last_error.c_str(); }
const char* frg_version(void) { return "flowreg_b200 0.1.0 sm_100a"; }

int frg_sample(const void* values, int32_t dtype, const int32_t n[3], const double* q0, const double* q1,
               const double* q2, int64_t npts, int32_t method, void* out, void* stream) {
    return guard([&] {
        FRG_REQUIRE(dtype == FRG_F32 || dtype == FRG_F64 || dtype == FRG_I32, "unsupported dtype");
        check_method(method);
        FRG_REQUIRE(npts >= 0, "npts must be >= 0");
        Dims g = make_dims(n, n[0] == 1 ? 2 : 3);
        FRG_REQUIRE(npts == 0 || (q1 && q2 && (n[0] == 1 || q0)), "null query arrays");
        sample_q(values, dtype, g, n[0] == 1 ? nullptr : q0, q1, q2, npts, method, out, ST(stream));
    });
}

int frg_departure(const int32_t n[3], int32_t d, int32_t dtype, int32_t vdtype, int32_t method, double h_t,
                  const void* v, void* disp, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_dtype(vdtype);
        check_method(method);
        departure(dims_of(n, d), dtype, vdtype, method, h_t, v, disp, ST(stream));
    });
}

int frg_disp_to_points(const int32_t n[3], int32_t d, int32_t dtype, const void* disp, void* y, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        disp_to_points(dims_of(n, d), dtype, disp, y, ST(stream));
    });
}

int frg_points_to_disp(const int32_t n[3], int32_t d, int32_t dtype, const void* y, void* disp, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        points_to_disp(dims_of(n, d), dtype, y, disp, ST(stream));
    });
}

int frg_gather(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, const void* disp, int32_t nf,
               const void* const* in, void* const* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_method(method);
        FRG_REQUIRE(nf >= 0, "nf must be >= 0");
        gather_fields(dims_of(n, d), dtype, method, disp, nf, in, out, ST(stream));
    });
}

int64_t frg_tile_plan_count(const int32_t n[3]) {
    try {
        return (int64_t)tile_plan_count(dims_of(n, n[0] == 1 ? 2 : 3));
    } catch (...) {
        return -1;
    }
}

int frg_tile_plan(const int32_t n[3], int32_t d, int32_t method, const void* disp, void* plan, void* stream) {
    return guard([&] {
        FRG_REQUIRE(method == FRG_LINEAR || method == FRG_CUBIC || method == FRG_BSPLINE,
                    "tile plans are built for linear / cubic / bspline maps");
        build_tile_plan(dims_of(n, d), method, (const float*)disp, (int4*)plan, ST(stream));
    });
}

int frg_gather_planned(const int32_t n[3], int32_t d, int32_t method, const void* disp, const void* plan, int32_t nf,
                       const void* const* in, void* const* out, void* stream) {
    return guard([&] {
        check_method(method);
        FRG_REQUIRE(nf >= 0, "nf must be >= 0");
        PlanScope ps(0, disp, (const int4*)plan, method);
        gather_fields(dims_of(n, d), F32, method, disp, nf, in, out, ST(stream));
    });
}

int frg_solve_state(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t, const void* disp,
                    void* series, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_method(method);
        FRG_REQUIRE(n_t >= 1, "n_t must be >= 1");
        solve_state(dims_of(n, d), dtype, method, n_t, disp, series, ST(stream));
    });
}

int frg_solve_adjoint(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t, const void* disp_b,
                      const void* divv, void* series, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_method(method);
        FRG_REQUIRE(n_t >= 1, "n_t must be >= 1");
        Dims g = dims_of(n, d);
        void* cmul = nullptr;
        FRG_CUDA(cudaMallocAsync(&cmul, g.N * (dtype == FRG_F64 ? 8 : 4), ST(stream)));
        adjoint_multiplier(g, dtype, method, 1.0 / n_t, disp_b, divv, cmul, ST(stream));
        solve_adjoint(g, dtype, method, n_t, disp_b, cmul, series, ST(stream));
        FRG_CUDA(cudaFreeAsync(cmul, ST(stream)));
    });
}

int frg_solve_inc_state(const int32_t n[3], int32_t d, int32_t dtype, int32_t vdtype, int32_t method, int32_t n_t,
                        const void* disp, const void* grads, const void* vt, void* series, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_dtype(vdtype);
        check_method(method);
        FRG_REQUIRE(n_t >= 1, "n_t must be >= 1");
        Dims g = dims_of(n, d);
        size_t T = dtype == FRG_F64 ? 8 : 4;
        cudaStream_t st = ST(stream);
        char* work = nullptr;
        size_t per = (size_t)g.d * g.N * T;
        FRG_CUDA(cudaMallocAsync((void**)&work, per * (n_t + 1) + (size_t)(n_t > 1 ? n_t - 1 : 1) * g.N * T, st));
        void* grads_y = work;
        void* vtT = work + per * n_t;
        void* S = work + per * (n_t + 1);
        std::vector<const void*> in(g.d * n_t);
        std::vector<void*> out(g.d * n_t);
        for (long long e = 0; e < (long long)g.d * n_t; ++e) {
            in[e] = (const char*)grads + e * g.N * T;
            out[e] = work + e * g.N * T;
        }
        gather_fields(g, dtype, method, disp, g.d * n_t, in.data(), out.data(), st);
        inc_state(g, dtype, vdtype, method, n_t, disp, grads, grads_y, vt, vtT, S, series, nullptr, 0.0, true, st);
        FRG_CUDA(cudaFreeAsync(work, st));
    });
}

int frg_body_force(const int32_t n[3], int32_t d, int32_t dtype, int32_t n_t, const void* lam, const void* grads,
                   void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        FRG_REQUIRE(n_t >= 1, "time integral needs at least 2 slices");
        body_force(dims_of(n, d), dtype, dtype, n_t, lam, grads, out, false, ST(stream));
    });
}

int frg_deformation_tensor(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t,
                           const void* disp, const void* jac, void* F, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_method(method);
        Dims g = dims_of(n, d);
        size_t T = dtype == FRG_F64 ? 8 : 4;
        void* work = nullptr;
        FRG_CUDA(cudaMallocAsync(&work, 2 * (size_t)g.d * g.d * g.N * T, ST(stream)));
        deformation_tensor(g, dtype, method, n_t, disp, jac, F, work, ST(stream));
        FRG_CUDA(cudaFreeAsync(work, ST(stream)));
    });
}

int frg_deform_update(const int32_t n[3], int32_t dtype, double h_t, int32_t first, const void* jac_y,
                      const void* jac, void* F, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        deform_update(dims_of(n, 3), dtype, h_t, first != 0, jac_y, jac, F, ST(stream));
    });
}

int frg_determinant(const int32_t n[3], int32_t d, int32_t dtype, const void* F, void* det, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        determinant(dims_of(n, d), dtype, F, det, ST(stream));
    });
}

int frg_compose(const int32_t n[3], int32_t d, int32_t dtype, int32_t method, int32_t n_t, const void* disp,
                void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        check_method(method);
        Dims g = dims_of(n, d);
        void* work = nullptr;
        FRG_CUDA(cudaMallocAsync(&work, (size_t)g.d * g.N * (dtype == FRG_F64 ? 8 : 4), ST(stream)));
        compose_disp(g, dtype, method, n_t, disp, out, work, ST(stream));
        FRG_CUDA(cudaFreeAsync(work, ST(stream)));
    });
}

int frg_fd8_gradient(const int32_t n[3], int32_t d, int32_t dtype, int32_t nslices, const void* u, void* out,
                     void* stream) {
    return guard([&] {
        check_dtype(dtype);
        fd8_gradient(dims_of(n, d), dtype, nslices, u, out, ST(stream));
    });
}

int frg_fd8_divergence(const int32_t n[3], int32_t d, int32_t dtype, const void* v, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        fd8_divergence(dims_of(n, d), dtype, v, out, ST(stream));
    });
}

int frg_spectral_gradient(const int32_t n[3], int32_t d, int32_t dtype, const void* u, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        spectral_gradient(dims_of(n, d), dtype, u, out, ST(stream));
    });
}

int frg_spectral_divergence(const int32_t n[3], int32_t d, int32_t dtype, const void* v, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        spectral_divergence(dims_of(n, d), dtype, v, out, ST(stream));
    });
}

int frg_spectral_apply(const int32_t n[3], int32_t d, int32_t dtype, int32_t ncomp, const void* in, void* out,
                       int32_t symbol, const frg_reg* reg, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        FRG_REQUIRE(symbol >= 0 && symbol <= 7, "unknown spectral symbol");
        FRG_REQUIRE(ncomp >= 1, "ncomp must be >= 1");
        RegSpec r{1.0, 1, 1, 0, 1e-4};
        if (symbol <= FRG_SYM_REG_KC) r = reg_of(reg);
        spectral_apply(dims_of(n, d), dtype, ncomp, in, out, symbol, r, ST(stream));
    });
}

int frg_project(const int32_t n[3], int32_t d, int32_t dtype, const void* b, void* out, const frg_reg* reg,
                void* stream) {
    return guard([&] {
        check_dtype(dtype);
        project(dims_of(n, d), dtype, b, out, reg_of(reg), ST(stream));
    });
}

int frg_restrict(const int32_t n[3], int32_t dtype, const void* in, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        restrict_field(make_dims(n, n[0] == 1 ? 2 : 3), dtype, in, out, ST(stream));
    });
}

int frg_prolong(const int32_t n_fine[3], int32_t dtype, const void* in, void* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        prolong_field(make_dims(n_fine, n_fine[0] == 1 ? 2 : 3), dtype, in, out, ST(stream));
    });
}

int frg_dot(int32_t dtype, const void* a, const void* b, int64_t n, double* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        *out = dot(dtype, a, b, n, ST(stream));
    });
}

int frg_norm_inf(int32_t dtype, const void* a, int64_t n, double* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        *out = abs_max(dtype, a, n, ST(stream));
    });
}

int frg_min_max_sum(int32_t dtype, const void* a, int64_t n, double out[3], void* stream) {
    return guard([&] {
        check_dtype(dtype);
        min_max_sum(dtype, a, n, out, ST(stream));
    });
}

int frg_all_finite(int32_t dtype, const void* a, int64_t n, int32_t* out, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        *out = all_finite(dtype, a, n, ST(stream)) ? 1 : 0;
    });
}

int frg_axpby(int32_t dtype, double a, const void* x, double b, void* y, int64_t n, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        axpby(dtype, a, x, b, y, n, ST(stream));
    });
}

int frg_pcg_update(int32_t dtype, double k, const void* s, const void* hs, void* x, void* r, int64_t n, double* rr,
                   void* stream) {
    return guard([&] {
        check_dtype(dtype);
        *rr = pcg_update(dtype, k, s, hs, x, r, n, ST(stream));
    });
}

struct frg_kkt {
    KktCtx* ctx;
};

int frg_kkt_create(const frg_config* cfg, void* stream, frg_kkt** out) {
    return guard([&] {
        FRG_REQUIRE(cfg && out, "null argument");
        Dims g = dims_of(cfg->n, cfg->d);
        for (int c = 0; c < g.d; ++c) {
            int ni = g.axis_len(g.comp_axis(c));
            FRG_REQUIRE(ni >= 8 && ni % 2 == 0, "voxel counts must be even and >= 8");
        }
        auto* h = new frg_kkt;
        h->ctx = kkt_create(g, cfg->n_t, cfg->method, cfg->scheme, cfg->distance, cfg->transport_dtype,
                            cfg->control_dtype, reg_of(&cfg->reg), ST(stream));
        *out = h;
    });
}

int frg_peer_alloc(int64_t bytes, void** ptr, void* handle) {
    return guard([&] {
        FRG_REQUIRE(bytes > 0 && ptr && handle, "bad peer_alloc arguments");
        *ptr = ipc_alloc((size_t)bytes, handle);
    });
}
int frg_peer_free(void* ptr) {
    return guard([&] { FRG_CUDA(cudaFree(ptr)); });
}
int frg_peer_open(const void* handle, void** ptr) {
    return guard([&] {
        FRG_REQUIRE(handle && ptr, "bad peer_open arguments");
        *ptr = ipc_open(handle);
    });
}
int frg_peer_close(void* ptr) {
    return guard([&] { ipc_close(ptr); });
}
int frg_peer_register(const void* local, const int32_t n_loc[3], int32_t nranks, int32_t rank,
                      const void* const* peers) {
    return guard([&] {
        FRG_REQUIRE(local && n_loc && peers, "bad peer_register arguments");
        peer_register((const float*)local, n_loc[0], n_loc[1], n_loc[2], nranks, rank, (const float* const*)peers);
    });
}
int frg_peer_unregister(const void* local) {
    return guard([&] { peer_unregister((const float*)local); });
}

int frg_probe_arm(int32_t on) {
    return guard([&] { probe_arm(on != 0); });
}
int frg_probe_read(double* total_ms, int64_t* count) {
    return guard([&] {
        long long c = 0;
        probe_read(total_ms, &c);
        *count = c;
    });
}

int frg_release_pool(void) {
    return guard([&] { kkt_release_pool(); });
}

int frg_kkt_destroy(frg_kkt* k) {
    return guard([&] {
        if (!k) return;
        kkt_destroy(k->ctx);
        delete k;
    });
}

#define CTX(k)                                          \
    FRG_REQUIRE((k) != nullptr && (k)->ctx, "null kkt"); \
    KktCtx* c = (k)->ctx;

int frg_kkt_set_stream(frg_kkt* k, void* stream) {
    return guard([&] {
        CTX(k);
        kkt_set_stream(c, ST(stream));
    });
}

int frg_kkt_set_interp_precision(frg_kkt* k, int32_t bits) {
    return guard([&] {
        CTX(k);
        kkt_set_interp_bits(c, bits);
    });
}

int frg_kkt_set_images(frg_kkt* k, const void* m0, const void* m1, int32_t dtype) {
    return guard([&] {
        CTX(k);
        check_dtype(dtype);
        kkt_set_images(c, m0, m1, dtype);
    });
}

int frg_kkt_refresh(frg_kkt* k, const void* v) {
    return guard([&] {
        CTX(k);
        kkt_refresh(c, v);
    });
}

int frg_kkt_objective(frg_kkt* k, double* J) {
    return guard([&] {
        CTX(k);
        *J = kkt_objective(c);
    });
}

int frg_kkt_objective_at(frg_kkt* k, const void* v_trial, double* J) {
    return guard([&] {
        CTX(k);
        *J = kkt_objective_at(c, v_trial);
    });
}

int frg_kkt_gradient(frg_kkt* k, void* g) {
    return guard([&] {
        CTX(k);
        kkt_gradient(c, g);
    });
}

int frg_kkt_hessian_matvec(frg_kkt* k, const void* vt, void* out) {
    return guard([&] {
        CTX(k);
        kkt_hessian_matvec(c, vt, out);
    });
}

int frg_kkt_apply_precond(frg_kkt* k, int32_t kind, double outer_tol, double inner_tol_factor,
                          int32_t inner_max_iterations, const void* r, void* z, int32_t* fell_back) {
    return guard([&] {
        CTX(k);
        FRG_REQUIRE(kind >= 0 && kind <= 2, "unknown preconditioner");
        int fb = 0;
        kkt_apply_precond(c, kind, outer_tol, inner_tol_factor, inner_max_iterations, r, z, &fb);
        if (fell_back) *fell_back = fb;
    });
}

int frg_kkt_mismatch(frg_kkt* k, double* out) {
    return guard([&] {
        CTX(k);
        *out = kkt_mismatch(c);
    });
}

int frg_kkt_initial_mismatch(frg_kkt* k, double* out) {
    return guard([&] {
        CTX(k);
        *out = kkt_initial_mismatch(c);
    });
}

int frg_kkt_divergence_energy(frg_kkt* k, double* out) {
    return guard([&] {
        CTX(k);
        *out = kkt_divergence_energy(c);
    });
}

int frg_kkt_counters(frg_kkt* k, int64_t out[3]) {
    return guard([&] {
        CTX(k);
        long long o[3];
        kkt_counters(c, o);
        for (int i = 0; i < 3; ++i) out[i] = o[i];
    });
}

int frg_kkt_set_counters(frg_kkt* k, const int64_t in[3]) {
    return guard([&] {
        CTX(k);
        long long o[3] = {in[0], in[1], in[2]};
        kkt_set_counters(c, o);
    });
}

int frg_kkt_get(frg_kkt* k, int32_t which, void* dst) {
    return guard([&] {
        CTX(k);
        kkt_get(c, which, dst);
    });
}

int frg_kkt_detgrad(frg_kkt* k, double out[3]) {
    return guard([&] {
        CTX(k);
        kkt_detgrad(c, out);
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// slab decomposition (multi-GPU; dist.py drives these per rank, exchanges in
// between over torch.distributed / NCCL).  n_loc = {n0_loc, n1, n2} owned
// planes of a 3D grid with n0_glob planes; *_src arrays carry h0 ghost planes
// per component ((n0_loc + 2 h0) planes); fp32 transport.
// ---------------------------------------------------------------------------
static Dims slab_dims(const int32_t n_loc[3], int32_t n0_glob, int32_t h0) {
    FRG_REQUIRE(n_loc != nullptr && n_loc[0] >= 1 && n_loc[1] >= 1 && n_loc[2] >= 1, "bad slab grid");
    FRG_REQUIRE(n0_glob >= n_loc[0] && h0 >= 0, "bad slab decomposition");
    // h0 == 0: the sources are peer windows (frg_peer_register), planes off
    // the slab are read from the owning rank over NVLink
    Dims g = make_dims(n_loc, 3);
    g.h0 = h0;
    g.n0g = n0_glob;
    return g;
}
static void check_slab_method(int m) {
    FRG_REQUIRE(m == FRG_LINEAR || m == FRG_CUBIC || m == FRG_BSPLINE, "slab transport: linear, cubic or B-spline");
}

extern "C" {

int frg_slab_departure(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, double h_t,
                       const void* v_src, const void* v_loc, void* disp, void* stream) {
    return guard([&] {
        check_slab_method(method);
        departure(slab_dims(n_loc, n0_glob, h0), F32, F32, method, h_t, v_src, disp, ST(stream), v_loc);
    });
}

int frg_slab_gather(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, const void* disp,
                    int32_t nf, const void* const* in_src, void* const* out, void* stream) {
    return guard([&] {
        check_slab_method(method);
        FRG_REQUIRE(nf >= 1, "nf must be >= 1");
        gather_fields(slab_dims(n_loc, n0_glob, h0), F32, method, disp, nf, in_src, out, ST(stream));
    });
}

int frg_slab_adjoint_multiplier(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, double h_t,
                                const void* disp_b, const void* divv_src, const void* divv_loc, void* cmul,
                                void* stream) {
    return guard([&] {
        check_slab_method(method);
        adjoint_multiplier(slab_dims(n_loc, n0_glob, h0), F32, method, h_t, disp_b, divv_src, cmul, ST(stream),
                           divv_loc);
    });
}

int frg_slab_adjoint_step(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, const void* disp_b,
                          const void* cmul, const void* u_src, void* out, void* stream) {
    return guard([&] {
        check_slab_method(method);
        adjoint_step(slab_dims(n_loc, n0_glob, h0), F32, method, disp_b, cmul, u_src, out, ST(stream));
    });
}

int frg_slab_inc_first(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, int32_t n_t,
                       const void* disp, const void* grads, const void* grads_y, const void* vt_src,
                       const void* vt_loc, void* m1, void* S, void* stream) {
    return guard([&] {
        check_slab_method(method);
        FRG_REQUIRE(n_t >= 1, "n_t must be >= 1");
        inc_first(slab_dims(n_loc, n0_glob, h0), method, n_t, (const float*)disp, (const float*)grads,
                  (const float*)grads_y, (const float*)vt_src, (const float*)vt_loc, (float*)m1, (float*)S,
                  ST(stream));
    });
}

int frg_slab_inc_step(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t method, const void* disp,
                      const void* m_src, const void* S_j, void* m_next, void* fin, double fsign, void* stream) {
    return guard([&] {
        check_slab_method(method);
        inc_step(slab_dims(n_loc, n0_glob, h0), method, (const float*)disp, (const float*)m_src, (const float*)S_j,
                 (float*)m_next, ST(stream), (float*)fin, (float)fsign);
    });
}

int frg_slab_fd8_gradient(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, int32_t nslices, const void* u_src,
                          void* out, void* stream) {
    return guard([&] {
        FRG_REQUIRE(nslices >= 1, "nslices must be >= 1");
        fd8_gradient(slab_dims(n_loc, n0_glob, h0), F32, nslices, u_src, out, ST(stream));
    });
}

int frg_slab_fd8_divergence(const int32_t n_loc[3], int32_t n0_glob, int32_t h0, const void* v_src, void* out,
                            void* stream) {
    return guard([&] { fd8_divergence(slab_dims(n_loc, n0_glob, h0), F32, v_src, out, ST(stream)); });
}

int frg_slab_fft2(const int32_t n_loc[3], int32_t dtype, int32_t ncomp, int32_t dir, const void* in, void* out,
                  void* stream) {
    return guard([&] {
        check_dtype(dtype);
        FRG_REQUIRE(ncomp >= 1 && (dir == 1 || dir == -1), "bad slab fft2 arguments");
        slab_fft2(n_loc[0], n_loc[1], n_loc[2], dtype, ncomp, dir, in, out, ST(stream));
    });
}

int frg_slab_fft1(int32_t n0_glob, int32_t n1_loc, int32_t n2, int32_t dtype, int32_t ncomp, int32_t dir, void* data,
                  void* stream) {
    return guard([&] {
        check_dtype(dtype);
        FRG_REQUIRE(ncomp >= 1 && (dir == 1 || dir == -1), "bad slab fft1 arguments");
        slab_fft1(n0_glob, n1_loc * (n2 / 2 + 1), dtype, ncomp, dir, data, ST(stream));
    });
}

int frg_slab_transpose(int32_t dir, int32_t nranks, const int32_t n_loc[3], int32_t dtype, int32_t ncomp,
                       const void* src, void* dst, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        slab_transpose(dir, nranks, n_loc[0], n_loc[1], n_loc[2] / 2 + 1, dtype == FRG_F64 ? 16 : 8, ncomp, src, dst,
                       ST(stream));
    });
}

int frg_slab_spec_apply(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, int32_t dtype, int32_t ncomp,
                        void* x, int32_t kind, const frg_reg* reg, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        FRG_REQUIRE(kind >= 0 && kind <= 7, "unknown symbol kind");
        slab_spec_scale(dims_of(n_glob, 3), i1_off, n1_loc, dtype, ncomp, x, kind, reg_of(reg), ST(stream));
    });
}

int frg_slab_spec_combine_mixed(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, const void* a, void* b,
                                const frg_reg* reg, int32_t project, void* stream) {
    return guard([&] {
        FRG_REQUIRE(b != nullptr, "slab_spec_combine_mixed: b spectrum required");
        slab_spec_combine_mixed(dims_of(n_glob, 3), i1_off, n1_loc, a, b, reg_of(reg), project != 0, ST(stream));
    });
}

int frg_slab_grad_energy(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, const void* x_spec, double* out,
                         void* stream) {
    return guard([&] { *out = slab_grad_energy(dims_of(n_glob, 3), i1_off, n1_loc, x_spec, ST(stream)); });
}

int frg_convert(int32_t sdtype, const void* src, int32_t ddtype, void* dst, int64_t n, void* stream) {
    return guard([&] {
        check_dtype(sdtype);
        check_dtype(ddtype);
        convert(sdtype, src, ddtype, dst, n, ST(stream));
    });
}

int frg_slab_spec_combine(const int32_t n_glob[3], int32_t i1_off, int32_t n1_loc, int32_t dtype, void* a,
                          const void* b, const frg_reg* reg, int32_t project, void* stream) {
    return guard([&] {
        check_dtype(dtype);
        slab_spec_combine(dims_of(n_glob, 3), i1_off, n1_loc, dtype, a, b, reg_of(reg), project != 0, ST(stream));
    });
}

}  // extern "C"

extern "C" {

// thread-local binding of a displacement map to its tile plan for the SL calls
// this host thread makes afterwards (slab path: the C-ABI gathers receive the
// map pointer only)
int frg_bind_plan(int32_t slot, const void* disp, const void* plan, int32_t method) {
    return guard([&] {
        FRG_REQUIRE(slot == 0 || slot == 1, "plan slot must be 0 or 1");
        g_plan_bind[slot].disp = disp;
        g_plan_bind[slot].plan = (const int4*)plan;
        g_plan_bind[slot].method = method;
    });
}

int frg_clear_plans(void) {
    return guard([&] { g_plan_bind[0] = g_plan_bind[1] = PlanBinding(); });
}

int frg_slab_body_force(const int32_t n_loc[3], int32_t n_t, const void* lam, int64_t lam_stride, const void* grads,
                        void* out, void* stream) {
    return guard([&] {
        FRG_REQUIRE(n_t >= 1, "time integral needs at least 2 slices");
        body_force(make_dims(n_loc, 3), F32, F32, n_t, lam, grads, out, false, ST(stream), lam_stride);
    });
}

}  // extern "C"

