// KKT context interface (kkt.cu) used by the C ABI (abi.cu).
#pragma once

#include "ops.h"
#include "spectral.h"

namespace frg {

struct KktCtx;

KktCtx* kkt_create(const Dims& g, int n_t, int method, int scheme, int distance, int tdt, int cdt, const RegSpec& reg,
                   cudaStream_t st);
void kkt_destroy(KktCtx* k);
void kkt_set_stream(KktCtx* k, cudaStream_t st);
// 16: single-field SL steps with fp16 taps (mixed-precision interpolation); 32: fp32
void kkt_set_interp_bits(KktCtx* k, int bits);
void kkt_set_images(KktCtx* k, const void* m0, const void* m1, int dtype);
void kkt_refresh(KktCtx* k, const void* v);
double kkt_objective(KktCtx* k);
double kkt_objective_at(KktCtx* k, const void* v_trial);
void kkt_gradient(KktCtx* k, void* g_out);
void kkt_hessian_matvec(KktCtx* k, const void* vt, void* out);
void kkt_apply_precond(KktCtx* k, int kind, double outer_tol, double inner_tol_factor, int inner_max, const void* r,
                       void* z, int* fell_back);
double kkt_mismatch(KktCtx* k);
double kkt_initial_mismatch(KktCtx* k);
double kkt_divergence_energy(KktCtx* k);
void kkt_counters(KktCtx* k, long long out[3]);
void kkt_set_counters(KktCtx* k, const long long in[3]);
void kkt_get(KktCtx* k, int which, void* dst);
void kkt_detgrad(KktCtx* k, double out[3]);
// free every context buffer parked for reuse (all devices)
void kkt_release_pool();

}  // namespace frg
