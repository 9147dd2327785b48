// SPDX-License-Identifier: Apache-2.0
// FP8 (e4m3) latent-KV path of the ETAP MLA decode: operand layouts and their UMMA check.
//
// A page of the FP8 latent cache is [64 rows][576 B]. In shared memory one tile (page) is
//   4 V chunks of 128 columns: 64 rows x 128 B, SW128, K-major for GEMM1 / MN-major (V^T)
//     for GEMM2 (128 fp8 = one 128 B swizzle row, so a d-block of 128 is one chunk);
//   1 rope chunk of 64 columns: 64 rows x 64 B, SW64, K-major (GEMM1 only).
// GEMM1 (kind::f8f6f4, M = 64, N = 48, K = 32 per MMA) multiplies the page with three fp8
// terms of Q (q = q0 + q1/16 + q2/256, exact for bf16 q in the normal range); GEMM2
// (M = 128, N = 48) multiplies V^T with three fp8 terms of P (P = p0 + p1/16 + p2/256, about
// 12 significant bits). Both read the fp8 page straight from shared memory: no dequantising
// pass over the KV bytes.
#include <cuda.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/etap_mla.h"
#include "sm100_ptx.cuh"

namespace etap_b200 {
int host_fail(int code, const char* msg);  // etap_mla.cu
}

namespace etap_b200 {
namespace fp8 {

constexpr int ROWS = 64;                  // KV rows per tile
constexpr int VCH = 4;                    // V chunks of 128 fp8 columns
constexpr int VCH_BYTES = ROWS * 128;     // 8 KB
constexpr int ROPE_OFF = VCH * VCH_BYTES; // rope chunk: 64 rows x 64 B (SW64)
constexpr int TILE_BYTES = ROPE_OFF + ROWS * 64;  // 36 KB
constexpr int NT = 3;                     // fp8 terms of Q and of P
constexpr int HGF = 16;                   // heads per work unit
constexpr int NQ = NT * HGF;              // UMMA N of both GEMMs (48)
constexpr int Q_VBLK = NQ * 128;          // Q^T V block: 48 rows x 128 B
constexpr int Q_BYTES = VCH * Q_VBLK + NQ * 64;
constexpr int P_ROWGRP = (NQ / 16) * 128; // P^T (MN-major, no swizzle): bytes per 8-row group
constexpr int P_BYTES = ROWS / 8 * P_ROWGRP;

// instruction descriptor, kind::f8f6f4: E4M3 A and B, f32 D
__host__ __device__ constexpr uint32_t idesc_e4m3_f32(uint32_t m, uint32_t n, uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (a_mn << 15) | (b_mn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void umma_f8_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// byte offset of (row, byte b) in a swizzled K-major / MN-major block with 128 B rows (SW128)
// or 64 B rows (SW64): 16-byte units XOR-permuted within 1024 B / 512 B atoms
__host__ __device__ inline uint32_t sw128_off(uint32_t row, uint32_t b) {
    return row * 128 + ((((b >> 4) ^ (row & 7)) << 4) | (b & 15));
}
__host__ __device__ inline uint32_t sw64_off(uint32_t row, uint32_t b) {
    return row * 64 + ((((b >> 4) ^ ((row >> 1) & 3)) << 4) | (b & 15));
}
// P^T element (KV row r, column n = term * 16 + head), MN-major without swizzle
__host__ __device__ inline uint32_t p_off(uint32_t r, uint32_t n) {
    return (r >> 3) * P_ROWGRP + (n >> 4) * 128 + (r & 7) * 16 + (n & 15);
}

// GEMM1: S^T[64 x 48] = K[64 x 576] . Q3^T (18 MMAs of K = 32). Whole-warp call.
__device__ __forceinline__ void issue_gemm1(uint32_t s_tmem, uint32_t tile, uint32_t q) {
    constexpr uint32_t idesc = idesc_e4m3_f32(64, NQ, 0, 0);
#pragma unroll
    for (int c = 0; c < VCH; ++c) {
        const uint64_t a0 = ptx::smem_desc(tile + c * VCH_BYTES, 16, 1024, ptx::LAYOUT_SW128);
        const uint64_t b0 = ptx::smem_desc(q + c * Q_VBLK, 16, 1024, ptx::LAYOUT_SW128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // +32 B (32 fp8) along K inside the 128 B row
            umma_f8_elect(s_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, (c == 0 && kk == 0) ? 0u : 1u);
    }
    const uint64_t a0 = ptx::smem_desc(tile + ROPE_OFF, 16, 512, ptx::LAYOUT_SW64);
    const uint64_t b0 = ptx::smem_desc(q + VCH * Q_VBLK, 16, 512, ptx::LAYOUT_SW64);
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) umma_f8_elect(s_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, 1u);
}

// GEMM2 for d-block c (128 latent columns = V chunk c): O^T[128 x 48] (+)= V^T[128 x 64] . P3^T
__device__ __forceinline__ void issue_gemm2(uint32_t o_tmem, uint32_t vchunk, uint32_t p, bool zero_init) {
    constexpr uint32_t idesc = idesc_e4m3_f32(128, NQ, 1, 1);
    const uint64_t a0 = ptx::smem_desc(vchunk, VCH_BYTES, 1024, ptx::LAYOUT_SW128);
    const uint64_t b0 = ptx::smem_desc(p, P_ROWGRP, 128, ptx::LAYOUT_NONE);
#pragma unroll
    for (int kk = 0; kk < ROWS / 32; ++kk)  // 32 KV rows per MMA: 4 swizzle atoms of V^T, 4 row groups of P^T
        umma_f8_elect(o_tmem, a0 + kk * (4096 >> 4), b0 + kk * ((4 * P_ROWGRP) >> 4), idesc,
                      (zero_init && kk == 0) ? 0u : 1u);
}

}  // namespace fp8
}  // namespace etap_b200

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
