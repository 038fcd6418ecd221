// fp16-tap SL gather engine: the north star's mixed-precision interpolation
// path (tolerance 1e-3 vs the f64 reference).
//
// The gathered field is rounded to fp16 (one conversion pass per gather,
// `to_half`), the TMA box holds fp16 (12 x 16 x 64 halves = 24 KB) and a copy
// shifted by one element (another 24 KB) is built from it in shared memory,
// so the four taps of every stencil row are TWO aligned 32-bit loads (half2
// pairs (c, c+1), (c+2, c+3) from the copy matching the parity of c) instead
// of four: 32 shared-memory loads per cubic point instead of 64, i.e. half of
// the shared-memory bytes that bound the fp32 engine (sl_fast.cuh).  Weights,
// accumulation, displacements and every epilogue stay fp32.  Single-field
// steps with a tile plan (the state / adjoint / incremental SL steps); other
// launches fall back to the fp32 engine.
#pragma once

#include <cuda_fp16.h>

#include "sl_fast.cuh"
#include "sl_pipe.cuh"

namespace frg {

// host: 2D map over an fp16 field viewed as ((n0 + 2 h0) n1) rows x n2, box 16 x 64 halves
void encode_field_map_half(CUtensorMap* map, const __half* ptr, const Dims& g);
// host: fp32 -> fp16 copy of one source field (n0 + 2 h0 planes) into per-thread scratch
const __half* half_copy(const Dims& g, const float* src, cudaStream_t st);
// interpolation precision of the SL steps launched by this host thread (16 or 32)
int& sl_interp_bits();

// scope: SL steps launched by this host thread use `bits`-bit taps
struct InterpScope {
    int old;
    explicit InterpScope(int bits) : old(sl_interp_bits()) { sl_interp_bits() = bits; }
    ~InterpScope() { sl_interp_bits() = old; }
};

// the shifted copy starts SLH_SKEW halves (16 words = half the banks) past
// the box: lanes alternate between the copies (neighbouring voxels' columns
// differ by one, so their parities alternate) and read the same word offset in
// each; without the skew the copy sits at TB_VOL / 2 = 0 mod 32 words and every
// such lane pair is a 2-way bank conflict (ncu: 2.45 shared wavefronts per
// voxel for 39 LDS)
constexpr int SLH_SKEW = 32;
struct SlhSmem {
    static constexpr size_t bytes = (2 * (size_t)TB_VOL + SLH_SKEW) * sizeof(__half) + 1024;
};

__device__ __forceinline__ float2 h2f(unsigned w) {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    return __half22float2(h);
}

__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<unsigned*>(&h); }

// f16 x f16 + f32 -> f32 (one FHFMA; the compiler folds the half selection
// into .H0 / .H1 operand selectors)
__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
    float r;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(r) : "h"(a), "h"(b), "f"(c));
    return r;
}

// one stencil row: taps t01 = (c, c+1), t23 = (c+2, c+3), weights likewise
__device__ __forceinline__ float row_fhfma(unsigned t01, unsigned t23, unsigned w01, unsigned w23) {
    float r = fhfma((unsigned short)(w01 & 0xffffu), (unsigned short)(t01 & 0xffffu), 0.f);
    r = fhfma((unsigned short)(w01 >> 16), (unsigned short)(t01 >> 16), r);
    r = fhfma((unsigned short)(w23 & 0xffffu), (unsigned short)(t23 & 0xffffu), r);
    return fhfma((unsigned short)(w23 >> 16), (unsigned short)(t23 >> 16), r);
}

// one stencil row: taps (c, c+1, c+2, c+3) as two half2 words -> w . taps
__device__ __forceinline__ float row_dot(const unsigned* __restrict__ rw, float2 w01, float2 w23) {
    float2 acc = __fmul2_rn(w01, h2f(rw[0]));
    acc = __ffma2_rn(w23, h2f(rw[1]), acc);
    return acc.x + acc.y;
}

// fp16 twin of patch_axis (sl_fast.cuh): only the out-of-range rows / columns
__device__ __forceinline__ void patch_axis_half(__half* __restrict__ box, const __half* __restrict__ src,
                                                const Dims& g, int lo0, int lo1, int lo2, int S0, int S1, int S2,
                                                int axis, int tid) {
    const int lo = axis == 1 ? lo1 : lo2;
    const int S = axis == 1 ? S1 : S2;
    const int n = axis == 1 ? g.n1 : g.n2;
    const int a_end = lo < 0 ? min(-lo, S) : 0;
    const int b_beg = lo + S > n ? max(n - lo, 0) : S;
    const int cnt = a_end + (S - b_beg);
    if (cnt == 0) return;
    const int E1 = S0;              // planes
    int E2 = axis == 2 ? S1 : S2;  // the other in-plane extent
    int r0 = 0;
    if (axis == 2) {  // rows outside [0, n1) were written by the axis-1 patch
        r0 = lo1 < 0 ? min(-lo1, S1) : 0;
        E2 = (lo1 + S1 > g.n1 ? max(g.n1 - lo1, 0) : S1) - r0;
        if (E2 <= 0) return;
    }
    const int total = cnt * E1 * E2;
    for (int e = tid; e < total; e += BX * BY) {
        const int r = e / E2;
        const int in2 = e - r * E2;
        const int q = r / E1;
        const int a = r - q * E1;
        const int x = q < a_end ? q : b_beg + (q - a_end);
        const int b = axis == 1 ? x : r0 + in2, c = axis == 1 ? in2 : x;
        const int gi = src_plane(g, lo0 + a), gj = wrap_near(lo1 + b, g.n1), gk = wrap_near(lo2 + c, g.n2);
        box[(a * TB_J + b) * TB_K + c] = src[((size_t)gi * g.n1 + gj) * g.n2 + gk];
    }
}

template <int M, class Op>
__global__ void __launch_bounds__(BX* BY, 4)
    k_slh(Dims g, Op op, const __grid_constant__ TmaMaps<1> maps, const __half* __restrict__ src16) {
    static_assert(M == LINEAR || M == CUBIC || M == BSPLINE, "k_slh: linear / cubic / B-spline");
    extern __shared__ __align__(16) unsigned char sdyn[];
    __half* b0 = reinterpret_cast<__half*>(sdyn + ((1024u - (smem_u32(sdyn) & 1023u)) & 1023u));
    __half* b1 = b0 + TB_VOL + SLH_SKEW;  // b1[x] = b0[x + 1]
    __shared__ __align__(8) uint64_t bar;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
    const int k = blockIdx.x * BX + tx;
    const int j = blockIdx.y * BY + ty;
    const int i_base = blockIdx.z * SL_TI;
    const bool in_kj = (k < g.n2) && (j < g.n1);
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();  // barrier initialised before anyone waits on it (nothing in flight yet)
    const int4 pe = __ldg(op.ds.plan + (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
    bool ok[SL_TI];
    float dsp[SL_TI][3];
#pragma unroll
    for (int u = 0; u < SL_TI; ++u) {
        const int i = i_base + u;
        ok[u] = in_kj && i < g.n0;
        dsp[u][0] = dsp[u][1] = dsp[u][2] = 0.f;
        if (ok[u]) op.disp((i * g.n1 + j) * g.n2 + k, dsp[u][0], dsp[u][1], dsp[u][2]);
    }
    using PreT = typename PreOf<Op>::type;
    PreT pre[SL_TI];
    if constexpr (HasPre<Op>::value) {
#pragma unroll
        for (int u = 0; u < SL_TI; ++u)
            if (ok[u]) pre[u] = op.pre(((i_base + u) * g.n1 + j) * g.n2 + k);
    }
    if (pe.w < 0) return;  // empty tile
    const int lo0 = pe.x, lo1 = pe.y, lo2 = pe.z & ~7;  // fp16 TMA box start: 16-byte aligned
    const int S0 = pe.w & 1023, S1 = (pe.w >> 10) & 1023, S2 = ((pe.w >> 20) & 1023) + (pe.z - lo2);
    const bool fits = S0 <= TB_I && S1 <= TB_J && S2 <= TB_K;
    if (tid == 0 && fits) {
        mbar_expect_tx(&bar, (unsigned)(S0 * TB_PLANE * sizeof(__half)));
        for (int a = 0; a < S0; ++a)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];\n" ::"r"(smem_u32(b0 + a * TB_PLANE)),
                "l"((unsigned long long)&maps.m[0]), "r"(lo2), "r"(src_plane(g, lo0 + a) * g.n1 + lo1),
                "r"(smem_u32(&bar))
                : "memory");
    }

    int base0[SL_TI], base1[SL_TI], base2[SL_TI];
    float fr0[SL_TI], fr1[SL_TI], fr2[SL_TI];
#pragma unroll
    for (int u = 0; u < SL_TI; ++u) {
        const float f0 = floorf(dsp[u][0]), f1 = floorf(dsp[u][1]), f2 = floorf(dsp[u][2]);
        base0[u] = i_base + u + (int)f0;
        base1[u] = j + (int)f1;
        base2[u] = k + (int)f2;
        fr0[u] = dsp[u][0] - f0;
        fr1[u] = dsp[u][1] - f1;
        fr2[u] = dsp[u][2] - f2;
    }
    float vals[SL_TI][1];
    if (fits) {
        mbar_wait_sleep(&bar, 0u);
        if (lo1 < 0 || lo1 + S1 > g.n1 || lo2 < 0 || lo2 + S2 > g.n2) {
            // rows / columns leaving the grid: copy from their periodic images
            patch_axis_half(b0, src16, g, lo0, lo1, lo2, S0, S1, S2, 1, tid);
            patch_axis_half(b0, src16, g, lo0, lo1, lo2, S0, S1, S2, 2, tid);
            __syncthreads();
        }
        // shifted copy: word w of b1 = (b0[2w + 1], b0[2w + 2])
        {
            const unsigned* w0 = reinterpret_cast<const unsigned*>(b0);
            unsigned* w1 = reinterpret_cast<unsigned*>(b1);
            const int words = S0 * TB_PLANE / 2;
            for (int w = tid; w < words; w += BX * BY) w1[w] = __byte_perm(w0[w], w0[w + 1], 0x5432);
        }
        __syncthreads();
        const unsigned* W0 = reinterpret_cast<const unsigned*>(b0);
        const unsigned* W1 = reinterpret_cast<const unsigned*>(b1);
        if (M == LINEAR) {
#pragma unroll
            for (int u = 0; u < SL_TI; ++u) {
                // taps (c, c + 1) of four rows from the parity-matched copy
                const int o = ok[u] ? ((base0[u] - lo0) * TB_J + (base1[u] - lo1)) * TB_K + (base2[u] - lo2) : 0;
                const unsigned* P = ((o & 1) ? W1 : W0) + (o >> 1);
                const float t0 = fr0[u], t1 = fr1[u], t2 = fr2[u];
                const float2 c00 = h2f(P[0]), c01 = h2f(P[TB_K / 2]), c10 = h2f(P[TB_PLANE / 2]),
                             c11 = h2f(P[(TB_PLANE + TB_K) / 2]);
                const float e00 = (1.f - t2) * c00.x + t2 * c00.y, e01 = (1.f - t2) * c01.x + t2 * c01.y;
                const float e10 = (1.f - t2) * c10.x + t2 * c10.y, e11 = (1.f - t2) * c11.x + t2 * c11.y;
                vals[u][0] = (1.f - t0) * ((1.f - t1) * e00 + t1 * e01) + t0 * ((1.f - t1) * e10 + t1 * e11);
            }
        } else {
            // two voxels per paired FMA, as the fp32 engine: each stencil row is
            // two half2 words per voxel, converted straight into the (A, B)
            // register pairs of FFMA2
#pragma unroll
            for (int u = 0; u < SL_TI; u += 2) {
                const int oA = ok[u] ? ((base0[u] - 1 - lo0) * TB_J + (base1[u] - 1 - lo1)) * TB_K +
                                           (base2[u] - 1 - lo2)
                                     : 0;
                const int oB = ok[u + 1] ? ((base0[u + 1] - 1 - lo0) * TB_J + (base1[u + 1] - 1 - lo1)) * TB_K +
                                               (base2[u + 1] - 1 - lo2)
                                         : 0;
                const unsigned* PA = ((oA & 1) ? W1 : W0) + (oA >> 1);
                const unsigned* PB = ((oB & 1) ? W1 : W0) + (oB >> 1);
                float2 w0[4], w1[4], w2[4];
                weights4f_x2<M>(make_float2(fr0[u], fr0[u + 1]), w0);
                weights4f_x2<M>(make_float2(fr1[u], fr1[u + 1]), w1);
                weights4f_x2<M>(make_float2(fr2[u], fr2[u + 1]), w2);
                // x-direction weights as fp16 pairs: each stencil row is 4
                // FHFMA (f16 x f16 + f32 accumulate, .H0/.H1 operand
                // selectors: no conversions), rows / planes combine in fp32
                const unsigned wA01 = h2u(__floats2half2_rn(w2[0].x, w2[1].x)),
                               wA23 = h2u(__floats2half2_rn(w2[2].x, w2[3].x));
                const unsigned wB01 = h2u(__floats2half2_rn(w2[0].y, w2[1].y)),
                               wB23 = h2u(__floats2half2_rn(w2[2].y, w2[3].y));
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    float2 plane = make_float2(0.f, 0.f);
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        const int ro = (a * TB_PLANE + bb * TB_K) / 2;
                        const float rA = row_fhfma(PA[ro], PA[ro + 1], wA01, wA23);
                        const float rB = row_fhfma(PB[ro], PB[ro + 1], wB01, wB23);
                        plane = __ffma2_rn(w1[bb], make_float2(rA, rB), plane);
                    }
                    acc = __ffma2_rn(w0[a], plane, acc);
                }
                vals[u][0] = acc.x;
                vals[u + 1][0] = acc.y;
            }
        }
    } else {
        // the box does not fit: fp32 gathers from global memory (rare)
        Dims gsrc = g;
        gsrc.n0 = g.n0 + 2 * g.h0;
        const float* src = op.field(0);
#pragma unroll
        for (int u = 0; u < SL_TI; ++u)
            vals[u][0] = ok[u] ? global_interp<float, M, float>(gsrc, src, base0[u] + g.h0, base1[u], base2[u], fr0[u],
                                                                fr1[u], fr2[u])
                               : 0.f;
    }
#pragma unroll
    for (int u = 0; u < SL_TI; ++u)
        if (ok[u]) {
            const int p = ((i_base + u) * g.n1 + j) * g.n2 + k;
            if constexpr (HasPre<Op>::value)
                op.done(p, vals[u], pre[u]);
            else
                op.done(p, vals[u]);
        }
}

// true when the fp16-tap engine ran this launch
template <int M, class Op>
bool launch_slh(const Dims& g, const Op& op, cudaStream_t st) {
    if constexpr (HasDs<Op>::value) {
        if (!op.ds.plan || plan_method(op.ds.plan) != M || !tma_grid_ok(g)) return false;
        const __half* h = half_copy(g, op.field(0), st);
        TmaMaps<1> maps;
        encode_field_map_half(&maps.m[0], h, g);
        static bool attr = false;
        if (!attr) {
            FRG_CUDA(cudaFuncSetAttribute(k_slh<M, Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)SlhSmem::bytes));
            attr = true;
        }
        k_slh<M, Op><<<sl_grid(g), vox_block(), SlhSmem::bytes, st>>>(g, op, maps, h);
        FRG_CHECK_LAUNCH();
        return true;
    }
    return false;
}

// B-spline prefilter (spectral.cu): out = coefficients of the periodic cubic
// B-spline interpolant of in (one field of g, dtype)
void bspline_prefilter(const Dims& g, int dtype, const void* in, void* out, cudaStream_t st);
// stream-ordered per-thread scratch for prefiltered copies (slot per field)
void* bspline_scratch(int slot, size_t bytes);

// Every SL launch: fp32 linear / cubic / B-spline gathers of fp32 fields take
// the TMA engine (single-field steps the fp16-tap engine when the host thread
// selected 16-bit interpolation and the map has a tile plan), everything else (f64 parity path, nearest, converting
// sources) the generic staged engine of sl_tile.cuh.  BSPLINE on a whole grid
// first replaces every gathered source by its prefiltered coefficients; on a
// slab (h0 > 0) the sources already are coefficients (the prefilter is a
// global FFT the host ran before the halo exchange, include/flowreg_b200.h).
template <typename T, int NF, class Op>
void launch_sl(const Dims& g, int method, const Op& op_in, cudaStream_t st) {
    Op op = op_in;
    if (method == BSPLINE && g.h0 == 0 && g.n0g == 0) {  // slab sources (ghosted or peer windows) are coefficients
        using V = typename Op::V;
        for (int f = 0; f < NF; ++f) {
            V* c = (V*)bspline_scratch(f, sizeof(V) * (size_t)g.N);
            bspline_prefilter(g, tcode(V(0)), op.field(f), c, st);
            op.set_field(f, c);
        }
    }
    if constexpr (std::is_same<T, float>::value && std::is_same<typename Op::V, float>::value) {
        if constexpr (NF == 1) {
            if (sl_interp_bits() == 16) {
                if (method == CUBIC && launch_slh<CUBIC, Op>(g, op, st)) return;
                if (method == BSPLINE && launch_slh<BSPLINE, Op>(g, op, st)) return;
                if (method == LINEAR && launch_slh<LINEAR, Op>(g, op, st)) return;
            }
        }
        if (method == CUBIC && launch_slp<CUBIC, NF, Op>(g, op, st)) return;
        if (method == BSPLINE && launch_slp<BSPLINE, NF, Op>(g, op, st)) return;
        if (method == LINEAR && launch_slp<LINEAR, NF, Op>(g, op, st)) return;
        if (method == CUBIC) return launch_slf<CUBIC, NF, Op>(g, op, st);
        if (method == BSPLINE) return launch_slf<BSPLINE, NF, Op>(g, op, st);
        if (method == LINEAR) return launch_slf<LINEAR, NF, Op>(g, op, st);
    }
    launch_sl_generic<T, NF, Op>(g, method, op, st);
}

}  // namespace frg
