// SPDX-License-Identifier: Apache-2.0
// Device side of the B200 ETAP MLA decode path.
//
// Reference algorithm (what is computed): etaplab::run_etap / block_update_impl
//   /root/reference/proj/src/etap.cpp:15-79   per-KV-block update (S^T = scale K Q^T,
//                                              column max, P = exp(S^T - m), colsum, rescale,
//                                              O^T_half += V_half^T P)
//   /root/reference/proj/src/etap.cpp:102-148 driver: block loop, epilogue O = (O^T / l)^T,
//                                              L = m + log l
// How it is computed here (B200-native, not a translation):
//   * KV tile of 128 latent rows on the UMMA M axis, the 16 heads of a head group on N:
//     S^T[128 x 16] = K_tile[128 x 576] . Q^T  -> TMEM (fp32), 36 tcgen05.mma (K=16 each)
//   * column-wise online softmax by one warpgroup: thread = KV row = TMEM lane
//   * O^T[512 x 16] += V^T[512 x 128] . P^T[128 x 16] -> TMEM (4 M=128 blocks), with P split
//     into bf16 hi + lo parts (two MMAs) so the bf16 P rounding does not limit accuracy
//   * V^T is read from the SAME smem tile as K (MN-major descriptor over the TMA SW128 tile)
//   * paged latent-KV TMA loads into a 12-slot ring; one persistent CTA per SM
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

namespace etap_b200 {

constexpr int D_QK = 576;
constexpr int D_V = 512;
constexpr int PAGE = 64;        // rows per KV page
constexpr int TILE = 128;       // KV rows per UMMA tile (two pages)
constexpr int HG = 16;          // heads per head group (UMMA N)
constexpr int NCHUNK = 9;       // 576 / 64 column chunks (SW128 atoms are 64 bf16 wide)
constexpr int NVCHUNK = 8;      // 512 / 64 chunks that are also V
constexpr int NSLOT = 12;       // ring depth in chunk slots
constexpr int SLOT_BYTES = TILE * 128;          // 128 rows x 128 B = 16 KiB
constexpr int HALF_SLOT = PAGE * 128;           // one page of one chunk = 8 KiB
constexpr int Q_CHUNK_BYTES = HG * 128;         // 2 KiB
constexpr int Q_BYTES = NCHUNK * Q_CHUNK_BYTES; // 18 KiB
constexpr int P_BYTES = TILE * HG * 2;          // 4 KiB (one of hi / lo)

constexpr int OFF_RING = 0;
constexpr int OFF_Q = OFF_RING + NSLOT * SLOT_BYTES;  // 196608
constexpr int OFF_P = OFF_Q + Q_BYTES;                // 215040
constexpr int OFF_RED = OFF_P + 2 * P_BYTES;          // 223232
constexpr int RED_BYTES = 1024;                       // [2][4][16] max + [4][16] sum (floats)
constexpr int OFF_BAR = OFF_RED + RED_BYTES;          // 224256
constexpr int NBAR = 2 * NSLOT + 8;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
constexpr int SMEM_USED = OFF_TMEM + 16;
constexpr int SMEM_ALLOC = SMEM_USED + 1024;  // slack for manual 1024 B alignment

// barrier indices
constexpr int BAR_FULL = 0;
constexpr int BAR_EMPTY = NSLOT;
constexpr int BAR_Q_FULL = 2 * NSLOT + 0;
constexpr int BAR_Q_EMPTY = 2 * NSLOT + 1;
constexpr int BAR_S_FULL = 2 * NSLOT + 2;  // [2]
constexpr int BAR_S_FREE = 2 * NSLOT + 4;  // [2]
constexpr int BAR_P_FULL = 2 * NSLOT + 6;
constexpr int BAR_O_DONE = 2 * NSLOT + 7;

// TMEM columns (128 lanes x 32 bit each)
constexpr uint32_t TMEM_COLS = 128;
constexpr uint32_t TCOL_S = 0;    // S^T double buffer: cols [0,16) and [16,32)
constexpr uint32_t TCOL_O = 32;   // O^T d-block i at cols [32+16i, 48+16i)

constexpr int NUM_THREADS = 192;  // warp0 TMA, warp1 MMA, warps 2..5 softmax/epilogue
constexpr float LAZY_RESCALE_LOG2 = 8.0f;  // rescale O^T only when the max grows by > 2^8

constexpr int SCHED_INTS = 8;
constexpr int META_FIXED_COST = 2;  // per-split overhead in tile units for the scheduler

enum : unsigned { FLAG_NEGATE_RESCALE = 1u, FLAG_EAGER_RESCALE = 2u };

// P^T operand layouts (B of GEMM2). 0: MN-major, no swizzle (core matrices 8 rows x 8 heads);
// 1: K-major SW128 (P stored head-major).
template <int P_LAYOUT>
struct PLayout;

template <>
struct PLayout<0> {
    static constexpr uint32_t kMajorMN = 1;
    // rows 16kk..16kk+15; LBO = K-direction core stride, SBO = MN-direction core stride
    __device__ static uint64_t desc(uint32_t base, int kk) {
        return ptx::smem_desc(base + kk * 512, 256, 128, ptx::LAYOUT_NONE);
    }
    __device__ static void write_row(uint8_t* p, int r, const uint32_t (&pk)[8]) {
        uint8_t* dst = p + (r >> 3) * 256 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(dst + 128) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
};

template <>
struct PLayout<1> {
    static constexpr uint32_t kMajorMN = 0;
    __device__ static uint64_t desc(uint32_t base, int kk) {
        return ptx::smem_desc(base + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024,
                              ptx::LAYOUT_SW128);
    }
    __device__ static void write_row(uint8_t* p, int r, const uint32_t (&pk)[8]) {
        const int rr = r & 63;
        uint8_t* base = p + (r >> 6) * 2048 + (rr & 7) * 2;
#pragma unroll
        for (int h = 0; h < 16; ++h) {
            const uint32_t w = pk[h >> 1];
            const uint16_t v = (h & 1) ? static_cast<uint16_t>(w >> 16) : static_cast<uint16_t>(w);
            uint8_t* dst = base + (h >> 3) * 1024 + (h & 7) * 128 + ((((rr >> 3) ^ (h & 7))) << 4);
            *reinterpret_cast<uint16_t*>(dst) = v;
        }
    }
};

// Ring position -> latent column chunk. Every tile consumes 9 ring positions starting at
// 9*gt; V chunks (2i, 2i+1) must sit in adjacent slots so one MN-major descriptor covers
// 128 d-rows (LBO = one slot). 12 is even, so pairs starting at even positions never wrap:
// even tiles start on an even position ([V0..V7, rope]), odd tiles on an odd one
// ([rope, V0..V7]).
__device__ __forceinline__ int chunk_at(int pos, uint32_t gt) {
    if (gt & 1u) return pos == 0 ? 8 : pos - 1;
    return pos;
}
__device__ __forceinline__ int pos_of_chunk(int chunk, uint32_t gt) {
    if (gt & 1u) return chunk == 8 ? 0 : chunk + 1;
    return chunk;
}

// GEMM1 part for one latent column chunk: S^T[128x16] (+)= K[128 x 64] . Q^T[64 x 16]
__device__ __forceinline__ void issue_gemm1_chunk(uint32_t s_tmem, uint32_t slot_addr,
                                                  uint32_t q_chunk_addr, bool first_chunk) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 16, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const uint64_t a = ptx::smem_desc(slot_addr + kk * 32, 16, 1024, ptx::LAYOUT_SW128);
        const uint64_t b = ptx::smem_desc(q_chunk_addr + kk * 32, 16, 1024, ptx::LAYOUT_SW128);
        ptx::umma_f16(s_tmem, a, b, idesc, (first_chunk && kk == 0) ? 0u : 1u);
    }
}

// GEMM2 part for one d-block (128 latent columns = chunks 2i, 2i+1 in slots s, s+1):
// O^T[128 x 16] (+)= V^T[128 x rows] . P^T[rows x 16], P = hi + lo.
template <int P_LAYOUT>
__device__ __forceinline__ void issue_gemm2_block(uint32_t o_tmem, uint32_t slot_addr,
                                                  uint32_t p_hi, uint32_t p_lo, int n_k,
                                                  bool zero_init) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 16, 1, PLayout<P_LAYOUT>::kMajorMN);
    for (int kk = 0; kk < n_k; ++kk) {
        // MN-major SW128: LBO = stride between 64-wide MN atoms (next slot), SBO = 8-row group
        const uint64_t a = ptx::smem_desc(slot_addr + kk * 2048, SLOT_BYTES, 1024, ptx::LAYOUT_SW128);
        ptx::umma_f16(o_tmem, a, PLayout<P_LAYOUT>::desc(p_hi, kk), idesc,
                      (zero_init && kk == 0) ? 0u : 1u);
        ptx::umma_f16(o_tmem, a, PLayout<P_LAYOUT>::desc(p_lo, kk), idesc, 1u);
    }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_elem, float hi_elem) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
    return *reinterpret_cast<uint32_t*>(&v);
}

// P (fp32, 16 heads of one KV row) -> bf16 hi and lo parts, written as row r of P^T.
template <int P_LAYOUT>
__device__ __forceinline__ void write_p_hilo(uint8_t* p_hi, uint8_t* p_lo, int r,
                                             const float (&p)[16]) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(p[2 * i]);
        const __nv_bfloat16 h1 = __float2bfloat16_rn(p[2 * i + 1]);
        const float r0 = p[2 * i] - __bfloat162float(h0);
        const float r1 = p[2 * i + 1] - __bfloat162float(h1);
        __nv_bfloat162 hh;
        hh.x = h0;
        hh.y = h1;
        hi[i] = *reinterpret_cast<uint32_t*>(&hh);
        lo[i] = pack_bf16x2(r0, r1);
    }
    PLayout<P_LAYOUT>::write_row(p_hi, r, hi);
    PLayout<P_LAYOUT>::write_row(p_lo, r, lo);
}

// Butterfly transpose-reduction: 16 per-lane values (one per head) reduced over the 32 lanes
// of a warp with 16 shuffles; on return lane l holds the reduction for head (l >> 1).
template <bool kMax>
__device__ __forceinline__ float warp_reduce16(const float (&x)[16], int lane) {
    auto op = [](float a, float b) { return kMax ? fmaxf(a, b) : a + b; };
    float y[8];
    const bool b4 = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float keep = b4 ? x[i + 8] : x[i];
        const float send = b4 ? x[i] : x[i + 8];
        y[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
    float z[4];
    const bool b3 = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float keep = b3 ? y[i + 4] : y[i];
        const float send = b3 ? y[i] : y[i + 4];
        z[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
    float w[2];
    const bool b2 = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float keep = b2 ? z[i + 2] : z[i];
        const float send = b2 ? z[i] : z[i + 2];
        w[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
    const bool b1 = lane & 2;
    float v = op(b1 ? w[1] : w[0], __shfl_xor_sync(0xffffffffu, b1 ? w[0] : w[1], 2));
    v = op(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return v;
}

struct DecodeParams {
    const int32_t* block_table;
    const int32_t* seqlens;
    const int32_t* sched;
    const int32_t* split_off;
    float* out;
    float* lse;
    float* ws_o;
    float* ws_lse;
    int max_pages;
    int heads;
    int groups;  // heads / 16
    float scale_log2;
    unsigned flags;
};

}  // namespace etap_b200
