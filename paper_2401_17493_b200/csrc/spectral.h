// cuFFT plan cache / workspace shared by spectral.cu and kkt.cu.
#pragma once

#include <cufft.h>

#include <map>
#include <mutex>
#include <tuple>

#include "ops.h"

namespace frg {

struct PlanCache {
    std::map<std::tuple<int, int, int, int, int>, cufftHandle> plans;
    std::mutex mu;
    cufftHandle get(const Dims& g, int type, int batch);
    void clear();
    ~PlanCache();
};

// process-wide device buffer pool (kkt.cu): callers guarantee no queued work
// still uses a buffer they hand back
void* pool_alloc(size_t& bytes);
void pool_free(void* p, size_t bytes);

struct Workspace {
    void* ptr = nullptr;
    size_t cap = 0;
    void* get(size_t bytes);
    void release();
    ~Workspace();
};

// process-wide plan cache (plans are keyed by shape/type/batch; the stream is set per call)
PlanCache& shared_plans();
long long half_len(const Dims& g);
Dims coarse_dims(const Dims& gf);
size_t spectral_ws_bytes(const Dims& g, int dtype, int ncomp);
size_t restrict_ws_bytes(const Dims& gf, int dtype);
void spectral_apply_ex(PlanCache& pc, void* ws, const Dims& g, int dtype, int ncomp, const void* in, void* out,
                       int kind, const RegSpec& r, cudaStream_t st);
// mixed precision alpha L a + P(b): a f64 (D2Z), b / out fp32 (spectral.cu)
void reg_plus_project_mixed(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, const double* a, const float* b,
                            float* out, const RegSpec& r, bool project, cudaStream_t st);
// the same in two halves: the D2Z of a (any stream), then b's part
void mixed_forward_a(PlanCache& pc, void* ws_a, const Dims& g, const double* a, cudaStream_t st);
void reg_plus_project_mixed_b(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, const float* b, float* out,
                              const RegSpec& r, bool project, cudaStream_t st);
// out = alpha L a + P[b] (project_on) or alpha L a + b; ws_a/ws_b hold d half spectra each
void reg_plus_project_ex(PlanCache& pc, void* ws_a, void* ws_b, const Dims& g, int adtype, const void* a,
                         int bdtype, const void* b, void* out, const RegSpec& r, bool project_on, cudaStream_t st);
double reg_energy_ex(PlanCache& pc, void* ws, const Dims& g, int dtype, const void* v, const RegSpec& r,
                     cudaStream_t st);
void restrict_field_ex(PlanCache& pc, void* ws, const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st);
void prolong_field_ex(PlanCache& pc, void* ws, const Dims& gf, int dtype, const void* in, void* out, cudaStream_t st);

// B-spline prefilter as separable FIR passes (bspline.cu): applies to whole
// grids whose axes are all 1 or >= 2K + 2 long (K = 16 fp32, 32 f64)
bool bspline_fir_applies(const Dims& g, int dtype);
void bspline_prefilter_fir(const Dims& g, int dtype, const void* in, void* out, cudaStream_t st);

}  // namespace frg
