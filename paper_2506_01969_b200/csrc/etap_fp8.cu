// SPDX-License-Identifier: Apache-2.0
// FP8 (e4m3) latent-KV path: the kind::f8f6f4 UMMA self-test of the operand layouts in
// etap_fp8.cuh (one tile, operands staged by plain loads).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/etap_mla.h"
#include "etap_fp8.cuh"

namespace etap_b200 {
int host_fail(int code, const char* msg);  // etap_mla.cu
}


namespace {

using namespace etap_b200;

// One tile through both fp8 GEMMs with operands staged by plain loads in the layouts above.
// k8 [64][576], q8 [48][576] (three terms x 16 heads, K-major), p8 [64][48] (P^T rows) ->
// s_out [64][48], o_out [512][48].
__global__ void __launch_bounds__(256, 1) etap_fp8_selftest_kernel(const uint8_t* k8, const uint8_t* q8,
                                                                   const uint8_t* p8, float* s_out, float* o_out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* tile = smem;
    uint8_t* q = smem + fp8::TILE_BYTES + 1024;  // keep 1 KB alignment
    q = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(q) + 1023) & ~uintptr_t(1023));
    uint8_t* p = q + fp8::Q_BYTES;
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(p + fp8::P_BYTES);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 576; i += 256) {
        const int r = i / 576, col = i % 576;
        if (col < 512) tile[(col >> 7) * fp8::VCH_BYTES + fp8::sw128_off(r, col & 127)] = k8[i];
        else tile[fp8::ROPE_OFF + fp8::sw64_off(r, col - 512)] = k8[i];
    }
    for (int i = threadIdx.x; i < fp8::NQ * 576; i += 256) {
        const int n = i / 576, col = i % 576;
        if (col < 512) q[(col >> 7) * fp8::Q_VBLK + fp8::sw128_off(n, col & 127)] = q8[i];
        else q[fp8::VCH * fp8::Q_VBLK + fp8::sw64_off(n, col - 512)] = q8[i];
    }
    for (int i = threadIdx.x; i < 64 * fp8::NQ; i += 256) p[fp8::p_off(i / fp8::NQ, i % fp8::NQ)] = p8[i];
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar[0], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tslot, 512);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    constexpr uint32_t TCOL_O = 64;
    if (warp == 1) {
        fp8::issue_gemm1(tmem, ptx::smem_u32(tile), ptx::smem_u32(q));
        for (int c = 0; c < fp8::VCH; ++c)
            fp8::issue_gemm2(tmem + TCOL_O + c * fp8::NQ, ptx::smem_u32(tile + c * fp8::VCH_BYTES), ptx::smem_u32(p),
                             true);
        ptx::umma_commit_elect(&bar[0]);
    }
    if (warp >= 4) {
        ptx::mbar_wait(&bar[0], 0);
        ptx::tc_fence_after();
        const int wq = warp & 3;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
        // S^T (M = 64 layout: row m in lane m%16 + 32*(m/16)): lanes 0-15 of each quadrant
        for (int c0 = 0; c0 < fp8::NQ; c0 += 16) {
            uint32_t r[16];
            ptx::tmem_ld16(t_lane + c0, r);
            ptx::tmem_wait_ld();
            if (lane < 16)
                for (int j = 0; j < 16; ++j) s_out[(wq * 16 + lane) * fp8::NQ + c0 + j] = __uint_as_float(r[j]);
        }
        for (int c = 0; c < fp8::VCH; ++c)
            for (int c0 = 0; c0 < fp8::NQ; c0 += 16) {
                uint32_t r[16];
                ptx::tmem_ld16(t_lane + TCOL_O + c * fp8::NQ + c0, r);
                ptx::tmem_wait_ld();
                for (int j = 0; j < 16; ++j)
                    o_out[(c * 128 + wq * 32 + lane) * fp8::NQ + c0 + j] = __uint_as_float(r[j]);
            }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

}  // namespace

extern "C" int etap_mla_selftest_fp8(const void* k8, const void* q8, const void* p8, float* s_t, float* o_t,
                                     void* stream) {
    constexpr int SMEM = fp8::TILE_BYTES + fp8::Q_BYTES + fp8::P_BYTES + 4 * 1024;
    static const cudaError_t a = cudaFuncSetAttribute(etap_fp8_selftest_kernel,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (a != cudaSuccess) return etap_b200::host_fail(ETAP_ERR_CUDA, cudaGetErrorString(a));
    etap_fp8_selftest_kernel<<<1, 256, SMEM, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(k8), static_cast<const uint8_t*>(q8), static_cast<const uint8_t*>(p8), s_t, o_t);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return etap_b200::host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}
