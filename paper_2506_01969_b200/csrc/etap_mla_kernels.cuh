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
constexpr int NCHUNK = 9;       // 576 / 64 column chunks (SW128 atoms are 64 bf16 wide)
constexpr int NVCHUNK = 8;      // 512 / 64 chunks that are also V
constexpr int SLOT_BYTES = TILE * 128;  // 64 rows x 128 B = 8 KiB per ring slot
constexpr int NTB = 4;          // tile-barrier ring depth (tiles in flight <= NSLOT/9 + 1)
constexpr int NBAR = 8 * NTB + 10;
// Longest line (batch * head groups, or batch with lanes) whose split schedule the decode
// kernel computes itself (the block-wide scan takes one line entry per thread of the >= 256-
// thread CTA); longer lines run K1 first.
constexpr int MAX_FUSED_VB = 256;
constexpr int sched_smem_ints(int max_vb) { return 3 * max_vb + 2 + 8 + 32; }  // pref, soff, len, sched, wt (<= 32 warps)

// warp 0 TMA producer, warp 1 GEMM1 issuer (+TMEM alloc), warp 2 GEMM2 issuer, warp 3 idle,
// warps 4..7 softmax / epilogue (warp % 4 = TMEM lane quadrant)
#ifndef ETAP_HG32_NSLOT
#define ETAP_HG32_NSLOT 22
#endif
constexpr int NUM_THREADS = 256;
constexpr int SOFTMAX_WARP0 = 4;
constexpr float LAZY_RESCALE_LOG2 = 8.0f;  // rescale O^T only when the max grows by > 2^8

constexpr int SCHED_INTS = 8;
#ifndef ETAP_META_FIXED_COST
#define ETAP_META_FIXED_COST 2
#endif
constexpr int META_FIXED_COST = ETAP_META_FIXED_COST;  // per-split overhead in tile units (scheduler)
// The FP8 path's tiles stream half the bytes in about half the time, while a split's fixed
// work (epilogue, the next split's first-tile latency) stays: about 2.4 us, 3-4 FP8 tiles
#ifndef ETAP_FP8_FIXED_COST
#define ETAP_FP8_FIXED_COST 4
#endif
constexpr int FP8_FIXED_COST = ETAP_FP8_FIXED_COST;

enum : unsigned {
    FLAG_NEGATE_RESCALE = 1u,
    FLAG_EAGER_RESCALE = 2u,
    FLAG_SKIP_COMBINE = 4u,
    FLAG_EXTERNAL_SCHEDULE = 8u
};

// barrier indices
constexpr int BAR_FULL_A = 0;           // [NTB] ring positions [0, SPLIT_POS) of tile gt landed
constexpr int BAR_FULL_B = NTB;         // [NTB] ring positions [SPLIT_POS, SPLIT_POS2) of tile gt landed
constexpr int BAR_G2_DONE = 2 * NTB;    // [NTB] GEMM2 of tile gt complete: its 9 ring slots
                                        //       and its P buffer are free (gt % NTB)
constexpr int BAR_G2_HALF = 3 * NTB;    // [NTB] GEMM2 d-blocks 0-1 of tile gt complete: the
                                        //       rope slot and V chunks 0-3 are free
constexpr int BAR_FULL_C = 4 * NTB + 8;  // [NTB] ring positions [SPLIT_POS2, 9) of tile gt landed
constexpr int BAR_G2_3Q = 5 * NTB + 8;   // [NTB] GEMM2 d-blocks 0-2 of tile gt complete (V0..V5 free)
constexpr int BAR_G2_Q1 = 6 * NTB + 8;   // [NTB] GEMM2 d-block 0 of tile gt complete (its first two positions free)
constexpr int BAR_G2_P1 = 7 * NTB + 8;   // [NTB] GEMM2 pass 1 (P_hi) of tile gt complete (two-pass GEMM2, !P_LO_BUF)
constexpr int BAR_P2_FULL = 8 * NTB + 8; // [2] P_lo written (two-pass GEMM2, !P_LO_BUF), count 128 * NWG
constexpr int BAR_Q_FULL = 4 * NTB + 0;
constexpr int BAR_Q_EMPTY = 4 * NTB + 1;
constexpr int BAR_S_FULL = 4 * NTB + 2;  // [2]
constexpr int BAR_S_FREE = 4 * NTB + 4;  // [2]
constexpr int BAR_P_FULL = 4 * NTB + 6;  // [2]

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

// Everything that depends on the head-group width HG (the UMMA N of GEMM1; GEMM2 uses
// N = 2*HG for the hi|lo parts of P, or two N = HG MMAs into one accumulator for HG = 64).
// HG = 16 fits a 24-slot ring (2.67 pages in flight), HG = 32 (twice the heads per KV byte,
// used for 32 / 96 heads) a 22-slot ring, HG = 64 (64 / 128 heads: half the GEMM1 issue
// cycles per head of HG = 32) a 16-slot ring beside its 72 KB of Q.
template <int HG_>
struct Cfg {
    static constexpr int HG = HG_;
    // softmax warpgroups: HG >= 32 splits its heads over two warpgroups, so a thread handles 8
    // (HG = 32) or 16 (HG = 64) heads
#ifndef ETAP_HG64_NWG
#define ETAP_HG64_NWG 4
#endif
    static constexpr int NWG = HG == 64 ? ETAP_HG64_NWG : (HG >= 32 ? 2 : 1);
    static constexpr int HW = HG / NWG;                  // heads per softmax warpgroup
    static constexpr int HH = HW / 2;                    // heads per softmax thread
    static constexpr int THREADS = 128 * (1 + NWG);      // warps 0-3 roles, then the warpgroups
    // ring depth in 8 KB chunk slots; HG = 32 affords 22 with a single P buffer (the softmax
    // writes P(gt) once GEMM2(gt-1) has read P(gt-1), which it has long done by then)
    static constexpr int NSLOT = HG == 16 ? 24 : (HG == 32 ? ETAP_HG32_NSLOT : 18);
    // HG = 64: O^T for 64 heads with separate hi / lo columns would take all 512 TMEM columns,
    // and 72 KB of Q leave room for only two whole tiles: P lives in the tile's own rope slot
    // (free once GEMM1 of the tile completed; the rope chunk feeds GEMM1 only) and GEMM2 runs
    // in two passes into one accumulator, O^T += V^T P_hi^T, then the softmax overwrites the
    // slot with P_lo and O^T += V^T P_lo^T. Tile gt then occupies ring half gt % 2 and the next
    // tile loads whole while GEMM2 of this one runs.
    static constexpr bool P_IN_ROPE = HG == 64;
    static constexpr bool SAME_D = P_IN_ROPE;
    static constexpr int P_BUFS = P_IN_ROPE ? 0 : ((HG == 16 || (HG == 32 && NSLOT <= 20)) ? 2 : 1);
    // P_LO_BUF (HG = 64, round 2): P_lo gets its own 8 KB buffer, so GEMM2 issues each d-block's
    // hi and lo MMAs back to back and commits per d-block; the next tile of the ring half then
    // lands in three groups in the order GEMM2 frees the slots (V0-V1 after d-block 0, V2-V5
    // after d-block 2, V6-V7 + rope after the whole GEMM2) instead of after the whole two-pass
    // GEMM2. The 8 KB come from a 64-entry fused-schedule line, a single-buffered max exchange,
    // the epilogue's sums and output rows aliased into buffers it does not use, and no 1 KB
    // alignment slack (the dynamic smem base is 1024-aligned; the kernel traps if it is not).
#ifndef ETAP_HG64_PLO
#define ETAP_HG64_PLO 1
#endif
    static constexpr bool P_LO_BUF = P_IN_ROPE && ETAP_HG64_PLO;
    static constexpr int RED_MAX_BUFS = P_LO_BUF ? 1 : 2;  // the per-tile vote separates consecutive uses
    // >= 20 slots: tile gt's ring positions [0, SPLIT_POS) reuse tile gt-3's last slots (free
    // after its GEMM2), positions p >= SPLIT_POS reuse tile gt-2's position p - SPLIT_POS. Of
    // those, gt-2's positions [0, 4) hold {V0..V3} or {rope, V0..V2}: free once GEMM2 d-blocks
    // 0-1 of gt-2 completed (G2_HALF), so tile gt's positions [SPLIT_POS, SPLIT_POS2) go out
    // then and only [SPLIT_POS2, 9) wait for the whole GEMM2 of gt-2 (an empty group for HG = 16).
    // 18 slots (P_IN_ROPE): tile gt reuses tile gt-2's slots, all free after GEMM2(gt-2); the
    // three landing groups only let GEMM1 start on the first chunks while the rest stream in.
    // Landing groups are ranges of "items" [0, SPLIT_POS), [SPLIT_POS, SPLIT_POS2), [SPLIT_POS2, 9):
    // ring positions (chunk = chunk_at(pos)), or with P_LO_BUF chunks (pos = pos_of_chunk(chunk)):
    // V0-V1 | V2-V5 | V6, V7, rope, the order GEMM2 of the tile two back frees their slots.
    static constexpr int SPLIT_POS = P_LO_BUF ? 2 : (P_IN_ROPE ? 3 : NSLOT - 18);
    static constexpr int SPLIT_POS2 = P_IN_ROPE ? 6 : (SPLIT_POS + 4 < NCHUNK ? SPLIT_POS + 4 : NCHUNK);
    static constexpr bool THIRD_GROUP = SPLIT_POS2 < NCHUNK;
    // the third group reuses gt-2's positions [4, 9 - SPLIT_POS): V chunks up to V(8 - SPLIT_POS),
    // free after GEMM2 d-blocks 0-2 (G2_3Q) when that is at most V5
    static constexpr bool G3_AFTER_3Q = SPLIT_POS >= 3;
    static constexpr int Q_CHUNK_BYTES = HG * 128;
    static constexpr int Q_BYTES = NCHUNK * Q_CHUNK_BYTES;
    static constexpr int PN = P_IN_ROPE ? HG : 2 * HG;   // P^T columns: HG heads hi | HG heads lo (or one part)
    static constexpr int GN = SAME_D ? HG : PN;          // GEMM2 MMA N
    static constexpr int P_ROWGRP = PN * 16;             // bytes per 8-row group of P^T
    static constexpr int P_BYTES = TILE * PN * 2;
    static constexpr int OFF_RING = 0;
    static constexpr int OFF_Q = OFF_RING + NSLOT * SLOT_BYTES;
    static constexpr int OFF_P = OFF_Q + Q_BYTES;        // P_BUFS buffers, or the P_lo buffer
    static constexpr int P_TOTAL = P_LO_BUF ? P_BYTES : P_BUFS * P_BYTES;
    // red_max[RED_MAX_BUFS][4][HG], then (without P_LO_BUF) red_sum[4][HG], m[HG], alpha[HG],
    // row[HG]; with P_LO_BUF the epilogue's red_sum aliases red_max, 1/l aliases alpha and the
    // output rows sit in the warpgroup's own column stripe of the (then idle) P_lo buffer
    static constexpr int OFF_RED = OFF_P + P_TOTAL;
    static constexpr int RED_FLOATS = RED_MAX_BUFS * 4 * HG + (P_LO_BUF ? 0 : 4 * HG) + HG + HG + (P_LO_BUF ? 0 : HG);
    static constexpr int OFF_BAR = align_up(OFF_RED + RED_FLOATS * 4, 16);
    static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr int OFF_SCHED = OFF_TMEM + 16;
    static constexpr int MAX_VB = P_LO_BUF ? 64 : MAX_FUSED_VB;  // fused-schedule line limit (longer lines: K1)
    static constexpr int SMEM_USED = OFF_SCHED + sched_smem_ints(MAX_VB) * 4;
    static constexpr int SMEM_ALLOC = SMEM_USED + (P_LO_BUF ? 0 : 1024);  // slack for manual 1024 B alignment
    // TMEM columns (128 lanes x 32 bit): S^T double buffer [0, 2HG) (M=64 lane layout), then
    // four O^T d-blocks of GN columns (HG hi | HG lo, or HG summed for SAME_D)
    static constexpr uint32_t TCOL_S = 0;
    static constexpr uint32_t TCOL_O = 2 * HG;
    static constexpr uint32_t OBLK = GN;
    static constexpr int OSEG = SAME_D ? 1 : 2;          // accumulator segments per d-block (hi, lo)
    static constexpr uint32_t TMEM_COLS = (TCOL_O + 4 * OBLK) <= 256 ? 256 : 512;
    static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
    static_assert(NSLOT % 2 == 0 && NSLOT >= 18 && NSLOT <= 27, "ring must hold two tiles, even slots");
    static_assert(!P_IN_ROPE || (NSLOT == 18 && P_BYTES == SLOT_BYTES), "P part fills exactly the rope slot");
    static_assert(!P_LO_BUF || (OFF_P % 1024 == 0 && P_BYTES == 8 * 1024 && HW * 16 == 256),
                  "P_lo buffer: 8 row groups of 1024 B, a warpgroup's heads are one 256 B stripe per row group");
    static_assert(TCOL_O + 4 * OBLK <= 512, "TMEM budget");
    static_assert(HW % 16 == 0, "a warpgroup handles whole 16-column TMEM loads");
};

// P^T operand (B of GEMM2): MN-major, no swizzle. Core matrices of 8 KV rows x 8 columns
// (16 B per row); columns [0, HG) = P_hi, [HG, 2HG) = P_lo.
//   offset(r, n) = (r/8)*P_ROWGRP + (n/8)*128 + (r%8)*16 + (n%8)*2
// LBO = K-direction core stride (P_ROWGRP), SBO = N-direction core stride (128).
template <class C>
__device__ __forceinline__ uint64_t p_desc(uint32_t base) {
    return ptx::smem_desc(base, C::P_ROWGRP, 128, ptx::LAYOUT_NONE);
}

// M=64 accumulator layout (cta_group::1): row m lives in TMEM lane (m % 16) + 32 * (m / 16),
// i.e. lanes 0-15 of each 32-lane quadrant. Warp q of the softmax group owns rows
// 16q .. 16q+15; with the 16x32bx2 TMEM load, lane l handles row 16q + (l % 16) and heads
// HH*(l / 16) .. HH*(l / 16) + HH-1.
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

// Landing-group item i of tile gt: its ring position and its latent column chunk (Cfg::SPLIT_POS)
template <class C>
__device__ __forceinline__ int item_pos(int i, uint32_t gt) { return C::P_LO_BUF ? pos_of_chunk(i, gt) : i; }
template <class C>
__device__ __forceinline__ int item_chunk(int i, uint32_t gt) { return C::P_LO_BUF ? i : chunk_at(i, gt); }

#ifndef ETAP_UMMA_X4
#define ETAP_UMMA_X4 1  // four K-steps per issue block (ptx::umma_f16_x4_elect); 0: one MMA per block (A/B)
#endif
// GEMM1 of one tile: S^T[64 x HG] = K[64 x 576] . Q^T[576 x HG], 9 chunks x 4 MMAs (K=16),
// landing-group items [POS_BEGIN, POS_END). Whole-warp call (elect inside). pos0 = ring slot of
// the tile's first position. The tile's first MMA (item 0) zero-initialises S^T.
template <class C, int POS_BEGIN, int POS_END>
__device__ __forceinline__ void issue_gemm1_tile(uint32_t s_tmem, uint32_t ring_addr,
                                                 uint32_t q_addr, uint32_t pos0, uint32_t gt) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(64, C::HG, 0, 0);
    const uint64_t a_ring = ptx::smem_desc(ring_addr, 16, 1024, ptx::LAYOUT_SW128);
    const uint64_t b_q = ptx::smem_desc(q_addr, 16, 1024, ptx::LAYOUT_SW128);
#pragma unroll
    for (int pos = POS_BEGIN; pos < POS_END; ++pos) {
        uint32_t s = pos0 + item_pos<C>(pos, gt);
        s = s >= C::NSLOT ? s - C::NSLOT : s;
        const int chunk = item_chunk<C>(pos, gt);
        const uint64_t a0 = a_ring + static_cast<uint64_t>(s * (SLOT_BYTES >> 4));
        const uint64_t b0 = b_q + static_cast<uint64_t>(chunk * (C::Q_CHUNK_BYTES >> 4));
#if ETAP_UMMA_X4
        ptx::umma_f16_x4_elect(s_tmem, a0, 2, b0, 2, idesc, pos == 0 ? 0u : 1u);  // +32 B along K per MMA
#else
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // +32 B along K inside the 128 B swizzle row
            ptx::umma_f16_elect(s_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc,
                                (pos == 0 && kk == 0) ? 0u : 1u);
#endif
    }
}

// GEMM2 part for one d-block (128 latent columns = chunks 2i, 2i+1 in slots s, s+1):
// O^T[128 x 2HG] (+)= V^T[128 x 64] . [P_hi | P_lo]^T[64 x 2HG], or for SAME_D
// O^T[128 x HG] (+)= V^T . P_hi^T + V^T . P_lo^T (two N = HG MMAs, one accumulator). Whole-warp call.
template <class C>
__device__ __forceinline__ void issue_gemm2_block(uint32_t o_tmem, uint32_t slot_addr,
                                                  uint32_t p_addr, bool zero_init) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, C::GN, 1, 1);
    // MN-major SW128: LBO = stride between 64-wide MN atoms (next slot), SBO = 8-row group
    const uint64_t a0 = ptx::smem_desc(slot_addr, SLOT_BYTES, 1024, ptx::LAYOUT_SW128);
    const uint64_t b0 = p_desc<C>(p_addr);
#if ETAP_UMMA_X4
    static_assert(TILE / 16 == 4, "four MMAs per d-block");
    ptx::umma_f16_x4_elect(o_tmem, a0, 2048 >> 4, b0, (2 * C::P_ROWGRP) >> 4, idesc, zero_init ? 0u : 1u);
#else
#pragma unroll
    for (int kk = 0; kk < TILE / 16; ++kk)  // 16 KV rows = 2 row groups per MMA
        ptx::umma_f16_elect(o_tmem, a0 + kk * (2048 >> 4), b0 + kk * ((2 * C::P_ROWGRP) >> 4),
                            idesc, (zero_init && kk == 0) ? 0u : 1u);
#endif
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_elem, float hi_elem) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
    return *reinterpret_cast<uint32_t*>(&v);
}

// P (fp32, HH heads [HH*half, HH*half+HH) of KV row r) -> bf16 hi and lo parts, written into
// row r of [P_hi | P_lo]^T: hi heads at columns HH*half.., lo heads at HG + HH*half..
template <class C>
__device__ __forceinline__ void write_p_hilo(uint8_t* p, int r, int half, const float (&pv)[C::HH], int hoff = 0) {
    uint32_t hi[C::HH / 2], lo[C::HH / 2];
#pragma unroll
    for (int i = 0; i < C::HH / 2; ++i) {
        // one packed RNE conversion per pair (F2FP) instead of two scalar F2F; widening a bf16
        // back to fp32 is a 16-bit shift
        hi[i] = pack_bf16x2(pv[2 * i], pv[2 * i + 1]);
        const float h0 = __uint_as_float(hi[i] << 16), h1 = __uint_as_float(hi[i] & 0xffff0000u);
        lo[i] = pack_bf16x2(pv[2 * i] - h0, pv[2 * i + 1] - h1);
    }
    uint8_t* row = p + (r >> 3) * C::P_ROWGRP + (r & 7) * 16;
#pragma unroll
    for (int c = 0; c < C::HH / 8; ++c) {  // 8 heads = one 16 B core-matrix row
        const int n_hi = hoff + half * C::HH + 8 * c, n_lo = C::HG + n_hi;
        *reinterpret_cast<uint4*>(row + (n_hi >> 3) * 128) =
            make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(row + (n_lo >> 3) * 128) =
            make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
    }
}

// One part (hi or lo, HH heads of KV row r as bf16 pairs) into row r of a P^T tile of PN = HG
// columns (two-pass GEMM2, C::P_IN_ROPE).
template <class C>
__device__ __forceinline__ void write_p_part(uint8_t* p, int r, int half, const uint32_t (&v)[C::HH / 2], int hoff) {
    uint8_t* row = p + (r >> 3) * C::P_ROWGRP + (r & 7) * 16;
#pragma unroll
    for (int c = 0; c < C::HH / 8; ++c) {  // 8 heads = one 16 B core-matrix row
        const int n = hoff + half * C::HH + 8 * c;
        *reinterpret_cast<uint4*>(row + (n >> 3) * 128) = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
}

// Butterfly transpose-reduction of N per-lane values (heads) over the 16 lanes of a half-warp.
// N = 8: 8 shuffles, lane l then holds head (l & 15) >> 1; N = 16: 15 shuffles, head l & 15.
template <bool kMax, int N>
__device__ __forceinline__ float halfwarp_reduce(const float (&x)[N], int lane) {
    static_assert(N == 8 || N == 16, "8 or 16 values per lane");
    auto op = [](float a, float b) { return kMax ? fmaxf(a, b) : a + b; };
    float y[N / 2];
    const bool b3 = lane & 8;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        const float keep = b3 ? x[i + N / 2] : x[i];
        const float send = b3 ? x[i] : x[i + N / 2];
        y[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
    float z[N / 4];
    const bool b2 = lane & 4;
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
        const float keep = b2 ? y[i + N / 4] : y[i];
        const float send = b2 ? y[i] : y[i + N / 4];
        z[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
    float w[N / 8 > 0 ? N / 8 : 1];
    const bool b1 = lane & 2;
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
        const float keep = b1 ? z[i + N / 8] : z[i];
        const float send = b1 ? z[i] : z[i + N / 8];
        w[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 2));
    }
    if constexpr (N == 8) {
        return op(w[0], __shfl_xor_sync(0xffffffffu, w[0], 1));
    } else {
        const bool b0 = lane & 1;
        return op(b0 ? w[1] : w[0], __shfl_xor_sync(0xffffffffu, b0 ? w[0] : w[1], 1));
    }
}

// head (within the half's HH heads) that halfwarp_reduce leaves in this lane
template <int N>
__device__ __forceinline__ int halfwarp_reduce_head(int lane) {
    return N == 8 ? ((lane & 15) >> 1) : (lane & 15);
}

// Split-KV work line. Virtual sequences are numbered head-group-major, vb = g * batch + b.
// With several head groups the SMs are dealt into `lanes` = groups equal lanes of p_line CTAs;
// every lane partitions the same line of `line_n` = batch sequences identically, so CTA
// (lane, k') and CTA (lane', k') stream the same KV pages at the same time and all but one
// of the head groups' reads of a page hit L2. One lane (lanes = 1, line of batch * groups
// virtual sequences) when there is one group, fewer CTAs than groups, or lanes are disabled.
struct LineShape {
    int lanes, line_n, p_line;
};

__host__ __device__ inline LineShape line_shape(int batch, int groups, int parts, bool lanes_on) {
    LineShape s;
    s.lanes = (lanes_on && groups > 1 && parts >= groups) ? groups : 1;
    s.line_n = s.lanes > 1 ? batch : batch * groups;
    s.p_line = parts / s.lanes;
    return s;
}

// Where final O / LSE rows go. Query row f (tokens folded into heads) of sequence b lands at
// output row (b * q_tokens + f / heads_per_token) * out_heads + out_head0 + f % heads_per_token
// of every one of the n_out copies: one local buffer, or (peer gather, fused all-gather of a
// head-sharded decode) every rank's full-head buffer through peer-mapped NVLink memory.
constexpr int MAX_OUT_COPIES = 8;
struct OutMap {
    int q_tokens, heads_per_token, out_heads, out_head0, n_out;
    float* out[MAX_OUT_COPIES];
    float* lse[MAX_OUT_COPIES];

    __device__ __forceinline__ size_t row(int b, int f) const {
        const int tok = f / heads_per_token;
        return (static_cast<size_t>(b) * q_tokens + tok) * out_heads + out_head0 + (f - tok * heads_per_token);
    }
};

struct DecodeParams {
    const int32_t* block_table;
    const int32_t* seqlens;
    const int32_t* sched;
    const int32_t* split_off;
    int32_t* sched_out;      // in-kernel schedule published here (same buffers as K1 writes)
    int32_t* split_off_out;
    OutMap om;               // final outputs (sequences finished by one split)
    float* ws_o;
    float* ws_lse;
    const void* kv_pool;     // raw pool / Q (L2 prefetch hints before the grid dependency)
    const void* q;
    int64_t num_pages;
    int max_pages;
    int batch;
    int heads;            // query rows per sequence (all tokens folded)
    int groups;  // heads / HG
    int q_tokens;         // query tokens per sequence (MTP: > 1); heads = q_tokens * heads_per_token
    int heads_per_token;
    int causal;           // q_tokens > 1: token j sees KV rows [0, seqlen - q_tokens + j]
    int inkernel_sched;  // 1: compute the split schedule in the prologue (and publish it)
    int early_meta;      // 1: read seqlens / block_table before the grid dependency (decode_prologue)
    int fixed_cost;      // per-split overhead in tile units of the split schedule
    int lanes_on;        // head-group lanes enabled (line_shape)
    int pair;            // 1: CTA-pair kernel, a schedule part is a pair of CTAs (part = blockIdx.x >> 1)
    int defer_dep;       // 1 (ETAP_FLAG_INDEPENDENT_INPUTS): the grid dependency is waited for only before
                         // the first global write (schedule publish, epilogue), not before the loads
    float scale_log2;
    unsigned flags;
    unsigned long long* trace;  // debug: [cta][TRACE_TILES][TRACE_SLOTS] stamps (ETAP_TRACE), or null
    unsigned long long* span;   // [cta][2] %globaltimer at grid-dependency resolution / exit, or null
    float* state;               // debug: per-tile softmax state [vb][state_tiles][4][16], or null
    int state_tiles;
};

// Split-schedule part of this CTA, number of parts, and whether this CTA publishes the part's
// schedule row (the CTA-pair kernel schedules pairs: both CTAs compute the same range).
__device__ __forceinline__ int sched_part(const DecodeParams& prm) { return static_cast<int>(blockIdx.x) >> prm.pair; }
__device__ __forceinline__ int sched_parts(const DecodeParams& prm) { return static_cast<int>(gridDim.x) >> prm.pair; }
__device__ __forceinline__ bool sched_publisher(const DecodeParams& prm) { return (blockIdx.x & prm.pair) == 0; }

// Debug stamps and the softmax-state dump are compiled into the DBG instantiations of the
// decode kernels only (selected at launch when a debug buffer is registered): in the product
// instantiation kDebug is false and every stamp vanishes, so the hot loops keep their schedule
// (the runtime-checked stamps cost ~1% of the step, 10% on the MTP FP8 path). Helpers outside
// the kernels see this namespace-scope value and keep the runtime check.
constexpr bool kDebug = true;
constexpr int TRACE_TILES = 256;
constexpr int TRACE_SLOTS = 16;
// Debug stamps: [cta][TRACE_TILES][TRACE_SLOTS]. Tile rows hold %clock64 (SM cycles, fine
// grained); the last row holds %globaltimer ns (entry / schedule done / exit, comparable
// across SMs) plus %clock64 at entry and exit (slots 5, 6) to convert cycles to ns.
#define ETAP_TRACE(prm, gt, slot)                                                                   \
    do {                                                                                            \
        if (kDebug && (prm).trace != nullptr && (gt) < TRACE_TILES - 1)                             \
            (prm).trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + (gt)) * TRACE_SLOTS + (slot)] = \
                clock64();                                                                          \
    } while (0)
#define ETAP_TRACE_G(prm, slot)                                                                     \
    do {                                                                                            \
        if (kDebug && (prm).trace != nullptr)                                                       \
            (prm).trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + TRACE_TILES - 1) * TRACE_SLOTS + \
                        (slot)] = ptx::global_timer_ns();                                           \
    } while (0)
// Prologue clock64 stamps in the second-to-last trace row (debug instantiation; that row is a
// tile row only for CTAs with more than 254 tiles): slots 0-7, see decode_prologue
#define ETAP_TRACE_PRO(prm, slot)                                                                   \
    do {                                                                                            \
        if (kDebug && (prm).trace != nullptr)                                                       \
            (prm).trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + TRACE_TILES - 2) * TRACE_SLOTS + \
                        (slot)] = clock64();                                                        \
    } while (0)
// SM id of the CTA in global slot 3 (debug instantiation): per-SM gaps between launches
#define ETAP_TRACE_SMID(prm)                                                                        \
    do {                                                                                            \
        if (kDebug && (prm).trace != nullptr) {                                                     \
            uint32_t smid_;                                                                         \
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                                      \
            (prm).trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + TRACE_TILES - 1) * TRACE_SLOTS + 3] = smid_; \
        }                                                                                           \
    } while (0)
#define ETAP_TRACE_CLK(prm, slot)                                                                   \
    do {                                                                                            \
        if (kDebug && (prm).trace != nullptr)                                                       \
            (prm).trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + TRACE_TILES - 1) * TRACE_SLOTS + \
                        (slot)] = clock64();                                                        \
    } while (0)

}  // namespace etap_b200
