// Host-side TMA descriptors for the SL engine (sl_fast.cuh).  The driver entry
// point is resolved once through the runtime (no -lcuda link dependency).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <array>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "sl_half.cuh"

namespace frg {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    if (!fn) throw Error(E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

void encode_field_map(CUtensorMap* map, const float* ptr, const Dims& g, int box_k, int box_j) {
    FRG_REQUIRE(((uintptr_t)ptr & 15) == 0, "TMA field must be 16-byte aligned");
    const cuuint64_t dims[2] = {(cuuint64_t)g.n2, (cuuint64_t)(g.n0 + 2 * g.h0) * g.n1};
    const cuuint64_t strides[1] = {(cuuint64_t)g.n2 * 4};
    const cuuint32_t box[2] = {(cuuint32_t)box_k, (cuuint32_t)box_j};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

void encode_tile_stream_map(CUtensorMap* map, const float* ptr, int n1, int n2, long long planes) {
    FRG_REQUIRE(((uintptr_t)ptr & 15) == 0 && n2 % 4 == 0, "tile-stream TMA: 16-byte aligned rows");
    const cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)n2 * 4, (cuuint64_t)n1 * n2 * 4};
    const cuuint32_t box[3] = {BX, BY, SL_TI};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)ptr, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(E_CUDA, "cuTensorMapEncodeTiled (tile stream) failed (" + std::to_string((int)r) + ")");
}

void encode_field_map_half(CUtensorMap* map, const __half* ptr, const Dims& g) {
    FRG_REQUIRE(((uintptr_t)ptr & 15) == 0, "TMA field must be 16-byte aligned");
    FRG_REQUIRE(g.n2 % 8 == 0, "fp16 TMA rows must be multiples of 16 bytes");
    const cuuint64_t dims[2] = {(cuuint64_t)g.n2, (cuuint64_t)(g.n0 + 2 * g.h0) * g.n1};
    const cuuint64_t strides[1] = {(cuuint64_t)g.n2 * 2};
    const cuuint32_t box[2] = {TB_K, TB_J};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)ptr, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(E_CUDA, "cuTensorMapEncodeTiled (fp16) failed (" + std::to_string((int)r) + ")");
}

__global__ void k_to_half(const float4* __restrict__ s, __half2* __restrict__ d, long long n4) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n4) {
        const float4 x = s[i];
        d[2 * i] = __floats2half2_rn(x.x, x.y);
        d[2 * i + 1] = __floats2half2_rn(x.z, x.w);
    }
}

namespace {
struct HalfScratch {
    void* p = nullptr;
    size_t cap = 0;
};
thread_local HalfScratch g_half_scratch;
thread_local int g_interp_bits = 32;
}  // namespace

int& sl_interp_bits() { return g_interp_bits; }

const __half* half_copy(const Dims& g, const float* src, cudaStream_t st) {
    const long long n = (long long)(g.n0 + 2 * g.h0) * g.n1 * g.n2;
    FRG_REQUIRE(n % 4 == 0 && ((uintptr_t)src & 15) == 0, "fp16 copy needs 16-byte aligned fields");
    HalfScratch& s = g_half_scratch;
    const size_t bytes = (size_t)n * sizeof(__half);
    if (bytes > s.cap) {
        if (s.p) FRG_CUDA(cudaFree(s.p));
        s.p = nullptr;
        FRG_CUDA(cudaMalloc(&s.p, bytes));
        s.cap = bytes;
    }
    k_to_half<<<blocks_for(n / 4, 256), 256, 0, st>>>((const float4*)src, (__half2*)s.p, n / 4);
    FRG_CHECK_LAUNCH();
    return (const __half*)s.p;
}

void build_tile_plan(const Dims& g, int method, const float* disp, int4* plan, cudaStream_t st) {
    DispSrc<float> ds = disp_src(g, disp);
    ds.plan = nullptr;
    if (method == CUBIC || method == BSPLINE)  // same stencil geometry
        k_tile_plan<float, CUBIC><<<sl_grid(g), vox_block(), 0, st>>>(g, ds, plan);
    else if (method == LINEAR)
        k_tile_plan<float, LINEAR><<<sl_grid(g), vox_block(), 0, st>>>(g, ds, plan);
    else
        throw Error(E_ARG, "tile plans are built for linear / cubic maps");
    FRG_CHECK_LAUNCH();
}

namespace {
struct Scratch {
    void* p = nullptr;
    size_t cap = 0;
};
thread_local Scratch g_bs_scratch[16];
}  // namespace

void* bspline_scratch(int slot, size_t bytes) {
    FRG_REQUIRE(slot >= 0 && slot < 16, "too many B-spline sources in one launch");
    Scratch& s = g_bs_scratch[slot];
    if (bytes > s.cap) {
        if (s.p) FRG_CUDA(cudaFree(s.p));
        s.p = nullptr;
        FRG_CUDA(cudaMalloc(&s.p, bytes));
        s.cap = bytes;
    }
    return s.p;
}

// ---------------------------------------------------------------------------
// Peer windows (dist.py peer mode): device buffers exported to / imported from
// the other ranks with CUDA IPC, and per local window the tensor maps of every
// rank's copy (device-resident: k_slf reads them by address).
namespace {
struct PeerWin {
    int n0, n1, n2, nranks, rank;
    CUtensorMap* dev_maps;
    const float* peer[PEER_MAX];
};
std::mutex g_peer_mu;
std::unordered_map<const void*, PeerWin>& peer_wins() {
    static std::unordered_map<const void*, PeerWin> m;
    return m;
}
std::unordered_map<void*, void*>& ipc_opened() {  // mapped pointer -> IPC base
    static std::unordered_map<void*, void*> m;
    return m;
}
}  // namespace

void peer_register(const float* local, int n0, int n1, int n2, int nranks, int rank, const float* const* peers) {
    FRG_REQUIRE(nranks >= 1 && nranks <= PEER_MAX && rank >= 0 && rank < nranks, "peer windows: 1..8 ranks");
    FRG_REQUIRE(n1 >= TB_J && n2 >= TB_K && n2 % 4 == 0, "peer windows need n1 >= 16, n2 >= 64, n2 % 4 == 0");
    FRG_REQUIRE(peers[rank] == local, "peer windows: this rank's entry must be the local window");
    CUtensorMap h[PEER_MAX];
    Dims w = make_dims(std::array<int32_t, 3>{n0, n1, n2}.data(), 3);
    for (int r = 0; r < nranks; ++r) encode_field_map(&h[r], peers[r], w);
    PeerWin e;
    e.n0 = n0;
    e.n1 = n1;
    e.n2 = n2;
    e.nranks = nranks;
    e.rank = rank;
    for (int r = 0; r < PEER_MAX; ++r) e.peer[r] = r < nranks ? peers[r] : nullptr;
    FRG_CUDA(cudaMalloc(&e.dev_maps, sizeof(CUtensorMap) * nranks));
    FRG_CUDA(cudaMemcpy(e.dev_maps, h, sizeof(CUtensorMap) * nranks, cudaMemcpyHostToDevice));
    std::lock_guard<std::mutex> lk(g_peer_mu);
    auto it = peer_wins().find(local);
    if (it != peer_wins().end()) {
        cudaFree(it->second.dev_maps);
        peer_wins().erase(it);
    }
    peer_wins()[local] = e;
}

void peer_unregister(const float* local) {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    auto it = peer_wins().find(local);
    if (it == peer_wins().end()) return;
    cudaFree(it->second.dev_maps);
    peer_wins().erase(it);
}

bool peer_planes_of(const Dims& g, const float* const* fields, int nf, PeerPlanes& pp) {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    if (peer_wins().empty()) return false;
    FRG_REQUIRE(nf <= 3, "peer gathers take at most 3 fields");
    for (int f = 0; f < nf; ++f) {
        auto it = peer_wins().find(fields[f]);
        if (it == peer_wins().end()) {
            FRG_REQUIRE(f == 0, "peer gather: every source must be a registered window");
            return false;
        }
        const PeerWin& e = it->second;
        FRG_REQUIRE(e.n0 == g.n0 && e.n1 == g.n1 && e.n2 == g.n2 && e.nranks * g.n0 == g.n0g,
                    "peer window does not match the slab grid");
        pp.nranks = e.nranks;
        pp.rank = e.rank;
        pp.maps[f] = e.dev_maps;
        for (int r = 0; r < PEER_MAX; ++r) pp.base[f][r] = e.peer[r];
    }
    return true;
}

void* ipc_alloc(size_t bytes, void* handle) {
    void* p = nullptr;
    FRG_CUDA(cudaMalloc(&p, bytes));
    FRG_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), p));
    return p;
}

void* ipc_open(const void* handle) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    FRG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    std::lock_guard<std::mutex> lk(g_peer_mu);
    ipc_opened()[p] = p;
    return p;
}

void ipc_close(void* p) {
    {
        std::lock_guard<std::mutex> lk(g_peer_mu);
        ipc_opened().erase(p);
    }
    FRG_CUDA(cudaIpcCloseMemHandle(p));
}

}  // namespace frg
