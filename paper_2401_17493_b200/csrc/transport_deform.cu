// Deformation tensor (transport.py:197-221) and composed map (transport.py:224-247).
#include "ops.h"
#include "sl_half.cuh"

namespace frg {

// ---------------------------------------------------------------------------
// deformation tensor d_t F = (grad v) F, F(0) = I (transport.py:197-221)
// jac layout: (d, d, N) with J[i][k] = d v_i / d x_k (diffops.py:132-139)
// ---------------------------------------------------------------------------
template <typename T, int D>
__device__ __forceinline__ void deform_update(int p, size_t N, T ht, const T* Fy, const T* __restrict__ jac_y,
                                              const T* __restrict__ jac, T* __restrict__ Fout) {
    T f0[D * D], Fp[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < D; ++k) acc += jac_y[(i * D + k) * N + p] * Fy[k * D + j];
            f0[i * D + j] = acc;
            Fp[i * D + j] = Fy[i * D + j] + ht * acc;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < D; ++k) acc += jac[(i * D + k) * N + p] * Fp[k * D + j];
            Fout[(i * D + j) * N + p] = Fy[i * D + j] + T(0.5) * ht * (f0[i * D + j] + acc);
        }
}

// later steps: F holds F_j(y) (gathered in place), updated pointwise in place
template <typename T, int D>
__global__ void k_deform_step(Dims g, T ht, const T* __restrict__ jac_y, const T* __restrict__ jac, T* F) {
    Vox v;
    if (!vox(g, v)) return;
    T Fy[D * D];
#pragma unroll
    for (int e = 0; e < D * D; ++e) Fy[e] = F[e * g.N + v.p];
    deform_update<T, D>(v.p, g.N, ht, Fy, jac_y, jac, F);
}

// first step: F_y = I exactly (no gather)
template <typename T, int D>
__global__ void k_deform_first(Dims g, T ht, const T* __restrict__ jac_y, const T* __restrict__ jac,
                               T* __restrict__ Fout) {
    Vox v;
    if (!vox(g, v)) return;
    T I[D * D];
#pragma unroll
    for (int e = 0; e < D * D; ++e) I[e] = T((e / D) == (e % D));
    deform_update<T, D>(v.p, g.N, ht, I, jac_y, jac, Fout);
}

template <typename T, int D>
static void deformation_d(const Dims& g, int method, int n_t, const T* disp, const T* jac, T* F, T* work,
                          cudaStream_t st) {
    const size_t dd = D * D;
    T* jac_y = work;           // dd x N
    T* tmp = work + dd * g.N;  // dd x N
    const void* ins[9];
    void* outs[9];
    for (size_t e = 0; e < dd; ++e) {
        ins[e] = jac + e * g.N;
        outs[e] = jac_y + e * g.N;
    }
    gather_fields(g, tcode(T(0)), method, disp, (int)dd, ins, outs, st);
    // ping-pong so that the final state lands in F
    T* bufs[2] = {(n_t % 2 == 1) ? F : tmp, (n_t % 2 == 1) ? tmp : F};
    T ht = (T)(1.0 / n_t);
    k_deform_first<T, D><<<vox_grid(g), vox_block(), 0, st>>>(g, ht, jac_y, jac, bufs[0]);
    FRG_CHECK_LAUNCH();
    // F_{s+1} = F_s(y) + Heun update: multi-field gather (3 fields per launch)
    // into the output slot, then the 3x3 update in place
    for (int s = 1; s < n_t; ++s) {
        const T* Fin = bufs[(s - 1) & 1];
        T* Fout = bufs[s & 1];
        for (size_t e = 0; e < dd; ++e) {
            ins[e] = Fin + e * g.N;
            outs[e] = Fout + e * g.N;
        }
        gather_fields(g, tcode(T(0)), method, disp, (int)dd, ins, outs, st);
        k_deform_step<T, D><<<vox_grid(g), vox_block(), 0, st>>>(g, ht, jac_y, jac, Fout);
        FRG_CHECK_LAUNCH();
    }
}

// one pointwise Heun update of F (first: F_y = I, F written; else F holds
// F_j(y) and is updated in place) — the slab path's deformation step
void deform_update(const Dims& g, int tdtype, double ht, bool first, const void* jac_y, const void* jac, void* F,
                   cudaStream_t st) {
    FRG_REQUIRE(g.d == 3, "deform_update: 3D");
    if (tdtype == F64) {
        if (first)
            k_deform_first<double, 3><<<vox_grid(g), vox_block(), 0, st>>>(g, ht, (const double*)jac_y,
                                                                           (const double*)jac, (double*)F);
        else
            k_deform_step<double, 3><<<vox_grid(g), vox_block(), 0, st>>>(g, ht, (const double*)jac_y,
                                                                          (const double*)jac, (double*)F);
    } else {
        if (first)
            k_deform_first<float, 3><<<vox_grid(g), vox_block(), 0, st>>>(g, (float)ht, (const float*)jac_y,
                                                                          (const float*)jac, (float*)F);
        else
            k_deform_step<float, 3><<<vox_grid(g), vox_block(), 0, st>>>(g, (float)ht, (const float*)jac_y,
                                                                         (const float*)jac, (float*)F);
    }
    FRG_CHECK_LAUNCH();
}

void deformation_tensor(const Dims& g, int tdtype, int method, int n_t, const void* disp, const void* jac, void* F,
                        void* work, cudaStream_t st) {
    if (tdtype == F64) {
        if (g.d == 3)
            deformation_d<double, 3>(g, method, n_t, (const double*)disp, (const double*)jac, (double*)F,
                                     (double*)work, st);
        else
            deformation_d<double, 2>(g, method, n_t, (const double*)disp, (const double*)jac, (double*)F,
                                     (double*)work, st);
    } else {
        if (g.d == 3)
            deformation_d<float, 3>(g, method, n_t, (const float*)disp, (const float*)jac, (float*)F, (float*)work,
                                    st);
        else
            deformation_d<float, 2>(g, method, n_t, (const float*)disp, (const float*)jac, (float*)F, (float*)work,
                                    st);
    }
}

// ---------------------------------------------------------------------------
// composed map (transport.py:224-247): D_{k+1} = D_k + disp(j + D_k)
// ---------------------------------------------------------------------------
template <typename T, int D>
struct ComposeOp {
    using V = T;
    static constexpr bool kLateDisp = true;  // displacement from the preceding launch (PDL, sl_fast.cuh)
    DispSrc<T> cur;
    const T* step[D];
    const T* Din[D];
    T* Dout[D];
    __device__ __forceinline__ void disp(int p, T& d0, T& d1, T& d2) const { cur.get(p, d0, d1, d2); }
    __host__ __device__ __forceinline__ const T* field(int f) const { return step[f]; }
    void set_field(int f, const T* p) { step[f] = p; }
    __device__ __forceinline__ void done(int p, const T (&vals)[D]) const {
#pragma unroll
        for (int c = 0; c < D; ++c) Dout[c][p] = Din[c][p] + vals[c];
    }
};

template <typename T, int D>
static void compose_d(const Dims& g, int method, int n_t, const T* disp, T* out, T* work, cudaStream_t st) {
    const size_t sz = (size_t)D * g.N;
    int steps = n_t - 1;
    T* bufs[2] = {(steps % 2 == 1) ? out : work, (steps % 2 == 1) ? work : out};
    if (steps == 0) {
        FRG_CUDA(cudaMemcpyAsync(out, disp, sizeof(T) * sz, cudaMemcpyDeviceToDevice, st));
        return;
    }
    const T* cur = disp;
    for (int s = 0; s < steps; ++s) {
        T* o = bufs[s & 1];
        ComposeOp<T, D> op;
        op.cur = disp_src(g, cur);
        for (int c = 0; c < D; ++c) {
            op.step[c] = disp + c * g.N;
            op.Din[c] = cur + c * g.N;
            op.Dout[c] = o + c * g.N;
        }
        launch_sl<T, D>(g, method, op, st);
        cur = o;
    }
}

void compose_disp(const Dims& g, int tdtype, int method, int n_t, const void* disp, void* out, void* work,
                  cudaStream_t st) {
    if (tdtype == F64) {
        if (g.d == 3)
            compose_d<double, 3>(g, method, n_t, (const double*)disp, (double*)out, (double*)work, st);
        else
            compose_d<double, 2>(g, method, n_t, (const double*)disp, (double*)out, (double*)work, st);
    } else {
        if (g.d == 3)
            compose_d<float, 3>(g, method, n_t, (const float*)disp, (float*)out, (float*)work, st);
        else
            compose_d<float, 2>(g, method, n_t, (const float*)disp, (float*)out, (float*)work, st);
    }
}

}  // namespace frg
