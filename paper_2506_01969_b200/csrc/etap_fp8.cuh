// SPDX-License-Identifier: Apache-2.0
// FP8 (e4m3) latent-KV path of the ETAP MLA decode: shared-memory operand layouts, UMMA
// kind::f8f6f4 issue helpers and the fp8 term splits of Q and P.
//
// A page of the FP8 latent cache is [64 rows][576 B]. In shared memory one tile (page) is
//   4 V chunks of 128 columns: 64 rows x 128 B, SW128, K-major for GEMM1 / MN-major (V^T)
//     for GEMM2 (128 fp8 = one 128 B swizzle row, so a d-block of 128 is one chunk);
//   1 rope chunk of 64 columns: 64 rows x 64 B, SW64, K-major (GEMM1 only).
// GEMM1 (kind::f8f6f4, M = 64, N = 48, K = 32 per MMA) multiplies the page with three fp8
// terms of Q (q = q0 + q1/16 + q2/256: exact for bf16 q in the normal range); GEMM2
// (M = 128, N = 48) multiplies V^T with three fp8 terms of P (P = p0 + p1/16 + p2/256, about
// 12 significant bits, the role the bf16 hi/lo split plays in the bf16 kernel). Both read
// the fp8 page straight from shared memory: there is no dequantising pass over the KV
// bytes, and the per-tensor KV scale folds into the softmax scale and 1/l.
#pragma once

#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <cstdint>

#include "sm100_ptx.cuh"

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

#ifndef ETAP_FP8_UMMA_X4
#define ETAP_FP8_UMMA_X4 0  // four-MMA issue blocks in GEMM1: 0.5% slower here (A/B), unlike the bf16 kernels
#endif
// four MMAs along K in one warp-uniform block (see ptx::umma_f16_x4_elect)
__device__ __forceinline__ void umma_f8_x4_elect(uint32_t d_tmem, uint64_t a0, uint64_t a_step, uint64_t b0,
                                                 uint64_t b_step, uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "add.s64 a1, %1, %2;\n\tadd.s64 a2, a1, %2;\n\tadd.s64 a3, a2, %2;\n\t"
        "add.s64 b1, %3, %4;\n\tadd.s64 b2, b1, %4;\n\tadd.s64 b3, b2, %4;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a1, b1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a2, b2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a3, b3, %5, 1;\n\t}" ::"r"(d_tmem),
        "l"(a0), "l"(a_step), "l"(b0), "l"(b_step), "r"(idesc), "r"(acc0)
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
#if ETAP_FP8_UMMA_X4
        umma_f8_x4_elect(s_tmem, a0, 2, b0, 2, idesc, c == 0 ? 0u : 1u);  // +32 B (32 fp8) along K per MMA
#else
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // +32 B (32 fp8) along K inside the 128 B row
            umma_f8_elect(s_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, (c == 0 && kk == 0) ? 0u : 1u);
#endif
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

// e4m3 (saturating RNE) of two floats -> two bytes (a low, b high), and back
__device__ __forceinline__ uint16_t to_e4m3x2(float a, float b) {
    return static_cast<uint16_t>(__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3));
}
__device__ __forceinline__ float2 from_e4m3x2(uint16_t v) {
    const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2(static_cast<__nv_fp8x2_storage_t>(v), __NV_E4M3);
    return __half22float2(*reinterpret_cast<const __half2*>(&h));
}

// x = t0 + t1/16 + t2/256 with e4m3 terms (two values at a time): returns the three byte
// pairs (low byte = a)
__device__ __forceinline__ void split3(float a, float b, uint16_t (&t)[NT]) {
    t[0] = to_e4m3x2(a, b);
    float2 f = from_e4m3x2(t[0]);
    const float ra = a - f.x, rb = b - f.y;
    t[1] = to_e4m3x2(ra * 16.f, rb * 16.f);
    f = from_e4m3x2(t[1]);
    t[2] = to_e4m3x2((ra - f.x * 0.0625f) * 256.f, (rb - f.y * 0.0625f) * 256.f);
}

// The three fp8 terms of 8 consecutive bf16 query values (one 16-byte vector): term t as 8
// bytes (x = t0 + t1/16 + t2/256, exact for bf16 values in the normal range).
__device__ __forceinline__ void quant_q_vec(const uint4 v, uint2 (&t)[NT]) {
    const uint32_t x[4] = {v.x, v.y, v.z, v.w};
    uint16_t tt[4][NT];
#pragma unroll
    for (int k = 0; k < 4; ++k) split3(__uint_as_float(x[k] << 16), __uint_as_float(x[k] & 0xffff0000u), tt[k]);
#pragma unroll
    for (int term = 0; term < NT; ++term)
        t[term] = make_uint2(static_cast<uint32_t>(tt[0][term]) | (static_cast<uint32_t>(tt[1][term]) << 16),
                             static_cast<uint32_t>(tt[2][term]) | (static_cast<uint32_t>(tt[3][term]) << 16));
}

// Byte offset of the 8-byte group (GEMM1 B-operand row n = term * 16 + head, vector cv of the
// 72 per query row) in the shared-memory Q buffer: V blocks of 48 rows x 128 B (SW128), then
// the rope block of 48 rows x 64 B (SW64).
__device__ __forceinline__ uint32_t q_smem_off(uint32_t n, int cv) {
    return cv < 64 ? (cv >> 4) * Q_VBLK + sw128_off(n, (cv & 15) * 8) : VCH * Q_VBLK + sw64_off(n, (cv - 64) * 8);
}

// One warp: the three terms of a work unit's 16 query rows into a global scratch slot,
// row-major [48][576] bytes (the layout the Q3 tensor maps read); nine loads in flight.
__device__ __forceinline__ void quant_q_global_warp(const void* __restrict__ q16, uint8_t* __restrict__ q3, int lane) {
    constexpr int VPR = 576 / 8, PER_LANE = HGF * VPR / 32;  // 36
#pragma unroll 1
    for (int i0 = 0; i0 < PER_LANE; i0 += 9) {
        uint4 v[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) v[i] = __ldg(static_cast<const uint4*>(q16) + lane + 32 * (i0 + i));
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            const int vi = lane + 32 * (i0 + i), h = vi / VPR, cv = vi - h * VPR;
            uint2 t[NT];
            quant_q_vec(v[i], t);
#pragma unroll
            for (int term = 0; term < NT; ++term)
                *reinterpret_cast<uint2*>(q3 + (term * HGF + h) * 576 + cv * 8) = t[term];
        }
    }
}

}  // namespace fp8
}  // namespace etap_b200