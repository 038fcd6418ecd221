// Shared-memory crossbar microbenchmark: cycles per warp-instruction for LDS
// widths and lane-address patterns (does broadcast across lanes make a wide
// LDS cheaper than its byte count?).  nvcc -arch=sm_100a -O3 lds_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NW = 8192;  // words of smem
constexpr int IT = 4096;

template <int PAT>
__global__ void __launch_bounds__(512) k(float* out, int shift) {
    __shared__ __align__(16) float s[NW];
    for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = (float)i;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    const int base = ((w * 97) & 1023) & ~3;
#pragma unroll 1
    for (int it0 = 0; it0 < IT; it0 += 32)
#pragma unroll
    for (int it = 0; it < 32; ++it) {
        const int row = base + it * 72;  // compile-time offsets from one base; 72 = 64 + 8 words
        if (PAT == 0) {  // LDS.32, 32 distinct consecutive words
            float v;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(s + row + lane + shift)));
            acc.x += v;
        } else if (PAT == 1) {  // LDS.128, 32 distinct aligned blocks (128 words)
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row + 4 * lane)));
            acc.x += v.x;
        } else if (PAT == 2) {  // LDS.128, groups of 4 lanes on one block (8 blocks = 32 words)
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row + 4 * (lane >> 2))));
            acc.x += v.x;
        } else if (PAT == 3) {  // stencil-like: block floor((lane+shift)/4) (9 distinct blocks)
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row + 4 * ((lane + shift) >> 2))));
            acc.x += v.x;
        } else if (PAT == 4) {  // LDS.64, pairs of lanes on one 8-byte word (16 distinct = 32 words)
            float2 v;
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row + 2 * (lane >> 1))));
            acc.x += v.x;
        } else if (PAT == 5) {  // LDS.64, 32 distinct (64 words)
            float2 v;
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row + 2 * lane)));
            acc.x += v.x;
        } else if (PAT == 6) {  // LDS.128 all lanes one block (pure broadcast)
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row)));
            acc.x += v.x;
        } else if (PAT == 7) {  // LDS.128, 2 lanes per block (16 blocks = 64 words)
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(s + row + 4 * (lane >> 1))));
            acc.x += v.x;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int PAT>
void run(const char* name, int shift) {
    int blocks = 148 * 4, tpb = 512;
    float* out = nullptr;
    cudaError_t e = cudaMalloc(&out, sizeof(float) * blocks * tpb);
    if (e != cudaSuccess) { printf("malloc: %s\n", cudaGetErrorString(e)); fflush(stdout); return; }
    k<PAT><<<blocks, tpb>>>(out, shift);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); fflush(stdout); return; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<PAT><<<blocks, tpb>>>(out, shift);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double instr_per_sm = 5.0 * blocks / 148.0 * (tpb / 32) * IT;  // warp-instructions per SM
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-44s shift %d: %.3f cycles / warp-LDS per SM  (%.2f ms)\n", name, shift, cyc / instr_per_sm, ms / 5);
    cudaFree(out);
}

int main() {
    printf("start\n"); fflush(stdout);
    run<0>("LDS.32 distinct", 0);
    run<5>("LDS.64 distinct", 0);
    run<4>("LDS.64 2 lanes/word", 0);
    run<1>("LDS.128 distinct", 0);
    run<7>("LDS.128 2 lanes/block", 0);
    run<2>("LDS.128 4 lanes/block", 0);
    run<3>("LDS.128 stencil floor((lane+s)/4)", 0);
    run<3>("LDS.128 stencil floor((lane+s)/4)", 1);
    run<3>("LDS.128 stencil floor((lane+s)/4)", 3);
    run<6>("LDS.128 broadcast", 0);
    return 0;
}
