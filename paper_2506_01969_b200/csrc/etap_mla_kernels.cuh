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
//   * one 64-row latent-KV page per tile, KV rows on the UMMA M axis, the 16 heads of a head
//     group on N:  S^T[64 x 16] = K_page[64 x 576] . Q^T  -> TMEM (fp32), 36 tcgen05.mma
//   * column-wise online softmax (thread = KV row = TMEM lane) with a thresholded lazy
//     rescale decided by one barrier-reduction (bar.red.or) per tile
//   * O^T[512 x 32] += V^T[512 x 64] . [P_hi | P_lo]^T -> TMEM (4 M=128 d-blocks, N=32):
//     P is split into bf16 hi + lo so the bf16 rounding of P does not limit accuracy, and both
//     parts share one MMA (the A = V^T smem read dominates, N=32 costs the same as N=16)
//   * V^T is read from the SAME smem chunks as K (MN-major descriptor over the TMA SW128 tile)
//   * paged TMA loads into a 24-slot ring (2.6 pages in flight); one persistent CTA per SM
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

namespace etap_b200 {

constexpr int D_QK = 576;
constexpr int D_V = 512;
constexpr int PAGE = 64;        // rows per KV page
constexpr int TILE = 64;        // KV rows per tile (one page)
constexpr int HG = 16;          // heads per head group (UMMA N of GEMM1)
constexpr int NCHUNK = 9;       // 576 / 64 column chunks (SW128 atoms are 64 bf16 wide)
constexpr int NVCHUNK = 8;      // 512 / 64 chunks that are also V
constexpr int NSLOT = 24;       // ring depth in chunk slots
constexpr int SLOT_BYTES = TILE * 128;          // 64 rows x 128 B = 8 KiB
constexpr int Q_CHUNK_BYTES = HG * 128;         // 2 KiB
constexpr int Q_BYTES = NCHUNK * Q_CHUNK_BYTES; // 18 KiB
constexpr int PN = 32;                          // GEMM2 N: 16 heads hi | 16 heads lo
constexpr int P_BYTES = TILE * PN * 2;          // 4 KiB per P buffer

constexpr int OFF_RING = 0;
constexpr int OFF_Q = OFF_RING + NSLOT * SLOT_BYTES;  // 196608
constexpr int OFF_P = OFF_Q + Q_BYTES;                // 215040 (2 buffers)
constexpr int OFF_RED = OFF_P + 2 * P_BYTES;          // 223232
constexpr int RED_BYTES = 1024;                       // [2][4][16] max + [4][16] sum (floats)
constexpr int OFF_BAR = OFF_RED + RED_BYTES;          // 224256
constexpr int NTB = 4;          // tile-barrier ring depth (tiles in flight <= NSLOT/9 + 1)
constexpr int NBAR = 4 * NTB + 8;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
// in-kernel split schedule (fused K1): cost prefix, split offsets, tiles per virtual sequence
constexpr int MAX_FUSED_VB = 256;
constexpr int OFF_SCHED = OFF_TMEM + 16;
constexpr int SCHED_SMEM_INTS = 4 * MAX_FUSED_VB + 2 + 8 + 8;  // pref, soff, tiles, len, sched, wt
constexpr int SMEM_USED = OFF_SCHED + SCHED_SMEM_INTS * 4;
constexpr int SMEM_ALLOC = SMEM_USED + 1024;  // slack for manual 1024 B alignment

// barrier indices
constexpr int BAR_FULL_A = 0;           // [NTB] ring positions 0..5 of tile gt landed (gt % NTB)
constexpr int BAR_FULL_B = NTB;         // [NTB] ring positions 6..8 of tile gt landed
constexpr int BAR_G2_DONE = 2 * NTB;    // [NTB] GEMM2 of tile gt complete: its 9 ring slots
                                        //       and its P buffer are free (gt % NTB)
constexpr int BAR_G2_HALF = 3 * NTB;    // [NTB] GEMM2 d-blocks 0-1 of tile gt complete: the
                                        //       rope slot and V chunks 0-3 are free
constexpr int BAR_Q_FULL = 4 * NTB + 0;
constexpr int BAR_Q_EMPTY = 4 * NTB + 1;
constexpr int BAR_S_FULL = 4 * NTB + 2;  // [2]
constexpr int BAR_S_FREE = 4 * NTB + 4;  // [2]
constexpr int BAR_P_FULL = 4 * NTB + 6;  // [2]
constexpr int SPLIT_POS = 6;             // positions 0..5 reuse tile gt-3's slots, 6..8 gt-2's

// TMEM columns (128 lanes x 32 bit each)
constexpr uint32_t TMEM_COLS = 256;
constexpr uint32_t TCOL_S = 0;    // S^T double buffer: cols [0,16) and [16,32), M=64 lane layout
constexpr uint32_t TCOL_O = 32;   // O^T d-block i at cols [32+32i, 64+32i): 16 hi | 16 lo

// warp 0 TMA producer, warp 1 GEMM1 issuer (+TMEM alloc), warp 2 GEMM2 issuer, warp 3 idle,
// warps 4..7 softmax / epilogue (warp % 4 = TMEM lane quadrant)
constexpr int NUM_THREADS = 256;
constexpr int SOFTMAX_WARP0 = 4;
constexpr float LAZY_RESCALE_LOG2 = 8.0f;  // rescale O^T only when the max grows by > 2^8

constexpr int SCHED_INTS = 8;
constexpr int META_FIXED_COST = 3;  // per-split overhead in tile (page) units for the scheduler

enum : unsigned {
    FLAG_NEGATE_RESCALE = 1u,
    FLAG_EAGER_RESCALE = 2u,
    FLAG_SKIP_COMBINE = 4u,
    FLAG_EXTERNAL_SCHEDULE = 8u
};

// P^T operand (B of GEMM2): MN-major, no swizzle. Core matrices of 8 KV rows x 8 columns
// (16 B per row); columns 0-15 = P_hi heads 0-15, 16-31 = P_lo heads 0-15.
//   offset(r, n) = (r/8)*512 + (n/8)*128 + (r%8)*16 + (n%8)*2
// LBO = K-direction core stride (512), SBO = N-direction core stride (128).
__device__ __forceinline__ uint64_t p_desc(uint32_t base, int kk) {
    return ptx::smem_desc(base + kk * 1024, 512, 128, ptx::LAYOUT_NONE);
}

// M=64 accumulator layout (cta_group::1): row m lives in TMEM lane (m % 16) + 32 * (m / 16),
// i.e. lanes 0-15 of each 32-lane quadrant. Warp q of the softmax group owns rows
// 16q .. 16q+15; with the 16x32bx2 TMEM load, lane l handles row 16q + (l % 16) and heads
// 8*(l / 16) .. 8*(l / 16) + 7.
__device__ __forceinline__ int s_row_of(int quadrant, int lane) { return quadrant * 16 + (lane & 15); }

// Ring position -> latent column chunk. Every tile consumes 9 ring positions starting at
// 9*gt; V chunks (2i, 2i+1) must sit in adjacent slots so one MN-major descriptor covers
// 128 d-rows (LBO = one slot). NSLOT is even, so pairs starting at even positions never
// wrap: even tiles start on an even position ([V0..V7, rope]), odd tiles on an odd one
// ([rope, V0..V7]).
__device__ __forceinline__ int chunk_at(int pos, uint32_t gt) {
    if (gt & 1u) return pos == 0 ? 8 : pos - 1;
    return pos;
}
__device__ __forceinline__ int pos_of_chunk(int chunk, uint32_t gt) {
    if (gt & 1u) return chunk == 8 ? 0 : chunk + 1;
    return chunk;
}

// GEMM1 of one tile: S^T[64x16] = K[64 x 576] . Q^T[576 x 16], 9 chunks x 4 MMAs (K=16),
// ring positions [POS_BEGIN, POS_END). Whole-warp call (elect inside). pos0 = ring slot of
// the tile's first position.
template <int POS_BEGIN, int POS_END>
__device__ __forceinline__ void issue_gemm1_tile(uint32_t s_tmem, uint32_t ring_addr,
                                                 uint32_t q_addr, uint32_t pos0, uint32_t gt) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(64, 16, 0, 0);
    const uint64_t a_ring = ptx::smem_desc(ring_addr, 16, 1024, ptx::LAYOUT_SW128);
    const uint64_t b_q = ptx::smem_desc(q_addr, 16, 1024, ptx::LAYOUT_SW128);
#pragma unroll
    for (int pos = POS_BEGIN; pos < POS_END; ++pos) {
        uint32_t s = pos0 + pos;
        s = s >= NSLOT ? s - NSLOT : s;
        const int chunk = chunk_at(pos, gt);
        const uint64_t a0 = a_ring + static_cast<uint64_t>(s * (SLOT_BYTES >> 4));
        const uint64_t b0 = b_q + static_cast<uint64_t>(chunk * (Q_CHUNK_BYTES >> 4));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // +32 B along K inside the 128 B swizzle row
            ptx::umma_f16_elect(s_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc,
                                (pos == 0 && kk == 0) ? 0u : 1u);
    }
}

// GEMM2 part for one d-block (128 latent columns = chunks 2i, 2i+1 in slots s, s+1):
// O^T[128 x 32] (+)= V^T[128 x 64] . [P_hi | P_lo]^T[64 x 32]. Whole-warp call.
__device__ __forceinline__ void issue_gemm2_block(uint32_t o_tmem, uint32_t slot_addr,
                                                  uint32_t p_addr, bool zero_init) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, PN, 1, 1);
    // MN-major SW128: LBO = stride between 64-wide MN atoms (next slot), SBO = 8-row group
    const uint64_t a0 = ptx::smem_desc(slot_addr, SLOT_BYTES, 1024, ptx::LAYOUT_SW128);
    const uint64_t b0 = p_desc(p_addr, 0);
#pragma unroll
    for (int kk = 0; kk < TILE / 16; ++kk)
        ptx::umma_f16_elect(o_tmem, a0 + kk * (2048 >> 4), b0 + kk * (1024 >> 4), idesc,
                            (zero_init && kk == 0) ? 0u : 1u);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_elem, float hi_elem) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
    return *reinterpret_cast<uint32_t*>(&v);
}

// P (fp32, 8 heads [8*half, 8*half+8) of KV row r) -> bf16 hi and lo parts, written into row r
// of [P_hi | P_lo]^T: hi heads at columns 8*half.., lo heads at 16 + 8*half..
__device__ __forceinline__ void write_p_hilo8(uint8_t* p, int r, int half, const float (&pv)[8]) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(pv[2 * i]);
        const __nv_bfloat16 h1 = __float2bfloat16_rn(pv[2 * i + 1]);
        __nv_bfloat162 hh;
        hh.x = h0;
        hh.y = h1;
        hi[i] = *reinterpret_cast<uint32_t*>(&hh);
        lo[i] = pack_bf16x2(pv[2 * i] - __bfloat162float(h0), pv[2 * i + 1] - __bfloat162float(h1));
    }
    uint8_t* dst = p + (r >> 3) * 512 + (r & 7) * 16 + half * 128;
    *reinterpret_cast<uint4*>(dst) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(dst + 256) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// Butterfly transpose-reduction of 8 per-lane values (heads) over the 16 lanes of a half-warp
// (8 shuffles); on return lane l holds the reduction for head (l & 15) >> 1 of its half.
template <bool kMax>
__device__ __forceinline__ float halfwarp_reduce8(const float (&x)[8], int lane) {
    auto op = [](float a, float b) { return kMax ? fmaxf(a, b) : a + b; };
    float y[4];
    const bool b3 = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float keep = b3 ? x[i + 4] : x[i];
        const float send = b3 ? x[i] : x[i + 4];
        y[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
    float z[2];
    const bool b2 = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float keep = b2 ? y[i + 2] : y[i];
        const float send = b2 ? y[i] : y[i + 2];
        z[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
    const bool b1 = lane & 2;
    float v = op(b1 ? z[1] : z[0], __shfl_xor_sync(0xffffffffu, b1 ? z[0] : z[1], 2));
    v = op(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return v;
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
    int32_t* sched_out;      // in-kernel schedule published here (same buffers as K1 writes)
    int32_t* split_off_out;
    float* out;
    float* lse;
    float* ws_o;
    float* ws_lse;
    int max_pages;
    int batch;
    int heads;
    int groups;  // heads / 16
    int inkernel_sched;  // 1: compute the split schedule in the prologue (and publish it)
    float scale_log2;
    unsigned flags;
    unsigned long long* trace;  // debug: [cta][TRACE_TILES][8] globaltimer stamps, or null
    float* state;               // debug: per-tile softmax state [vb][state_tiles][4][16], or null
    int state_tiles;
};

constexpr int TRACE_TILES = 256;
#define ETAP_TRACE(prm, gt, slot)                                                              \
    do {                                                                                       \
        if ((prm).trace != nullptr && (gt) < TRACE_TILES)                                      \
            (prm).trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + (gt)) * 8 + (slot)] = \
                ptx::global_timer_ns();                                                        \
    } while (0)

}  // namespace etap_b200
