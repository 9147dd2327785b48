// SPDX-License-Identifier: Apache-2.0
// Fused all-gather of a head-sharded decode over NVLink peer memory: CUDA IPC plumbing and
// the arrival kernel (K4). The data movement itself happens in K2's epilogue / K3, which store
// every finished O / LSE row into each rank's peer-mapped output (OutMap, etap_mla_kernels.cuh).
// No reference analog: etaplab is single-process.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/etap_mla.h"
#include "sm100_ptx.cuh"

namespace etap_b200 {
int host_fail(int code, const char* msg);  // etap_mla.cu
}

namespace {

struct PeerFlags {
    int world, rank;
    uint32_t* flags[ETAP_MLA_MAX_PEERS];  // flags[r] = rank r's arrival words (mapped here)
};

// K4: one warp. Lane r publishes `epoch` into rank r's word [rank] (release, system scope:
// orders this GPU's earlier K2 / K3 stores into every peer buffer, which happen-before this
// kernel through the stream), then lane r waits for rank r's word in the local array.
__global__ void __launch_bounds__(32) etap_peer_arrive_kernel(const __grid_constant__ PeerFlags pf,
                                                               uint32_t epoch) {
    const int lane = threadIdx.x;
    if (lane < pf.world) {
        __threadfence_system();
        uint32_t* dst = pf.flags[lane] + pf.rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
        const uint32_t* mine = pf.flags[pf.rank] + lane;
        const uint64_t t0 = etap_b200::ptx::global_timer_ns();
        uint32_t v = 0;
        for (uint32_t it = 0;; ++it) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
            if (static_cast<int32_t>(v - epoch) >= 0) break;  // >=: a fast peer may already be one epoch ahead
            if ((it & 1023u) == 1023u && etap_b200::ptx::global_timer_ns() - t0 > 4000000000ull)
                __trap();  // a peer never arrived (4 s): fail loudly instead of hanging
        }
    }
    __syncwarp();
}

}  // namespace

namespace etap_b200 {

int peer_signal_wait(const etap_mla_peer_gather* pg, uint32_t epoch, void* stream) {
    PeerFlags pf = {};
    pf.world = pg->world;
    pf.rank = pg->rank;
    for (int r = 0; r < pg->world; ++r) pf.flags[r] = pg->flags[r];
    // a plain launch (no programmatic serialisation): K4 starts after K2 and K3 completed
    etap_peer_arrive_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(pf, epoch);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}

}  // namespace etap_b200

extern "C" {

int etap_mla_ipc_alloc(size_t bytes, void** dev_ptr, void* handle) {
    if (!dev_ptr || !handle || bytes == 0) return etap_b200::host_fail(ETAP_ERR_SHAPE, "ipc_alloc: bad arguments");
    static_assert(sizeof(cudaIpcMemHandle_t) <= ETAP_MLA_IPC_HANDLE_BYTES, "IPC handle size");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return etap_b200::host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    }
    std::memset(handle, 0, ETAP_MLA_IPC_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof(h));
    *dev_ptr = p;
    return ETAP_OK;
}

int etap_mla_ipc_open(const void* handle, void** dev_ptr) {
    if (!handle || !dev_ptr) return etap_b200::host_fail(ETAP_ERR_SHAPE, "ipc_open: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return etap_b200::host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}

int etap_mla_ipc_close(void* dev_ptr) {
    const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return etap_b200::host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}

int etap_mla_ipc_free(void* dev_ptr) {
    const cudaError_t e = cudaFree(dev_ptr);
    if (e != cudaSuccess) return etap_b200::host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}

}  // extern "C"
