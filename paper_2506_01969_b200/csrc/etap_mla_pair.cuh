// SPDX-License-Identifier: Apache-2.0
// K2-pair: the decode for 128 heads per work unit on a CTA pair (tcgen05 cta_group::2).
// Included by etap_mla.cu inside its anonymous namespace (shares the split schedule, the
// prologue and the output map of the single-CTA kernels).
//
// Reference algorithm: etaplab::run_etap / block_update_impl (/root/reference/proj/src/etap.cpp
// :15-79 per-block update, :102-148 driver, epilogue L = m + log l at :144), with the heads of the
// decode folded into the query rows as the reference's cmd_bench does (cli.cpp:214).
//
// Why a pair (DESIGN.md §3 "CTA pair"): at 128 heads per GPU the single-CTA kernels are bound by
// tensor-pipe instruction cost, not HBM. A 1-SM UMMA of M64 N64 takes 32.7 cycles for 64x64x16,
// a pair UMMA of M128 N64 takes 25.8 cycles for twice that work, and a pair M128 N256 with A in
// tensor memory runs at the math rate (66 cycles; scripts/probe_pair*.cu). TMEM also caps one SM
// at O for ~96 heads; a pair holds O for 64 heads per SM over all 512 latent columns.
//
// The work unit is (sequence, 128 heads); CTA r of the pair owns heads [64r, 64r + 64).
//   GEMM1  S[128 heads x 64 rows] = Q . K^T   pair SS UMMA M=128 N=64: A = this CTA's 64 Q rows
//          (smem, 72 KB per split), B = K^T split by N: CTA r supplies KV rows [32r, 32r+32) of
//          the page (9 chunks of 32 x 64, 36 KB). D lands in the 2x2 layout: lane h holds head h
//          x rows 0-31, lane 64+h head h x rows 32-63 (32 TMEM columns per page).
//   softmax  thread = (head, 16 rows): online max with the thresholded lazy rescale, P = 2^(x-m)
//          split into bf16 hi + lo (the bf16 rounding of P would cost the 2e-5 RMSE bar).
//   GEMM2  O[128 heads x 512] += P . V   pair TS UMMA M=128 N=256, A = P from tensor memory
//          (duplicated in lanes 0-63 / 64-127 as the 2-SM A layout requires), B = V split by N:
//          CTA r supplies latent chunks {2r, 2r+1} (N block 0) and {2r+4, 2r+5} (block 1) of all
//          64 rows (32 KB). O of this CTA's 64 heads (all 512 columns) stays in its TMEM, so the
//          rescale and the epilogue never cross SMs.
// Shared memory per CTA: Q 72 KB + two pages x (36 + 32) KB + the P exchange buffer 16 KB.
#pragma once

namespace pairk {
constexpr int HPC = 64;                        // heads per CTA
constexpr int UNIT = 2 * HPC;                  // heads per pair work unit
constexpr int G1_BYTES = 32 * 128;             // GEMM1 B half-chunk: 32 KV rows x 64 columns
constexpr int V_BYTES = PAGE * 128;            // V chunk: 64 KV rows x 64 columns
constexpr int STAGE_G1 = NCHUNK * G1_BYTES;    // 36 KB
constexpr int STAGE = STAGE_G1 + 4 * V_BYTES;  // 68 KB per page
constexpr int Q_CHUNK = HPC * 128;
constexpr int Q_BYTES = NCHUNK * Q_CHUNK;      // 72 KB
constexpr int OFF_STAGE = 0;                   // two pages
constexpr int OFF_Q = 2 * STAGE;
constexpr int OFF_X = OFF_Q + Q_BYTES;         // P exchange [2 wg][128 lanes][16 u32]
constexpr int X_BYTES = 2 * 128 * 64;
constexpr int OFF_RED = OFF_X + X_BYTES;       // [4][64] floats: per-(row quarter) head max / sum
constexpr int OFF_MREF = OFF_RED + 4 * HPC * 4;  // [2][64] running max handed between warpgroups
constexpr int OFF_BAR = OFF_MREF + 2 * HPC * 4;
constexpr int NB = 22;
constexpr int OFF_TMEM = OFF_BAR + NB * 8;
constexpr int OFF_SCHED = OFF_TMEM + 16;
constexpr int MAX_VB = 64;                     // fused-schedule line limit (longer lines: K1)
constexpr int SMEM = OFF_SCHED + sched_smem_ints(MAX_VB) * 4;
constexpr int THREADS = 384;                   // warps 0-3 roles, 4-11 two softmax warpgroups
constexpr int SM_WARP0 = 4;
// TMEM columns (512 allocated per CTA): O [0, 256): N block n at 128n (lane h: head h, d 256n +
// c; lane 64+h: head h, d 256n + 128 + c); S [256, 320) two pages; P [320, 512) three pages of
// 64 columns, k-step j of a page at [16j, 16j + 8) (hi) and [16j + 8, 16j + 16) (lo), bf16 pairs
// along the KV rows. Three P buffers: the softmax writes P of page gp while GEMM2 of gp-1 and
// gp-2 may still be queued on the tensor pipe.
constexpr uint32_t TC_O = 0, TC_S = 256, TC_P = 320, TMEM_COLS = 512;
constexpr int NPB = 3;   // P buffers (tensor memory)
constexpr int P_TILE = HPC * 128;  // P in shared memory: one [64 heads][64 rows] bf16 tile (hi, then lo)
constexpr int NG2 = 4;   // GEMM2-done barriers (waits reach back three pages: a ring of four keeps
                         // every waited phase the newest or the one before on its barrier)
// barriers (same offsets in both CTAs); "L" = only the leader's copy is used
enum : int {
    B_FULL_G1 = 0,   // [2] L: both CTAs' GEMM1 halves of the page landed (tx from both)
    B_FULL_Q = 2,    // L: both CTAs' Q of the split landed
    B_V_LAND = 3,    // [2] local: this CTA's V chunks of the page landed
    B_V_READY = 5,   // [2] L: both CTAs' V chunks landed and tail rows zeroed (2 arrivals)
    B_S_FULL = 7,    // [2] both: GEMM1 of the page complete (S ready, GEMM1 halves free)
    B_Q_EMPTY = 9,   // both: GEMM1 of the split's last page complete (Q buffer free)
    B_G2_DONE = 10,  // [NG2] both: GEMM2 of the page complete (V chunks, P columns free; O final)
    B_S_FREE = 14,   // [2] L: both CTAs' softmax read S of the page (16 warp arrivals)
    B_P_FULL = 16,   // [2] L: both CTAs' P of the page in TMEM, O rescaled (16 warp arrivals)
    B_MREF = 18,     // [2] local (PINGPONG): warpgroup w published the running max of its page
};
static_assert(SMEM <= 232448, "shared memory budget");
// timing experiments only (wrong results): fewer GEMM1 chunks / GEMM2 MMAs, no P stores
#ifndef ETAP_PAIR_G1_CHUNKS
#define ETAP_PAIR_G1_CHUNKS 9
#endif
#ifndef ETAP_PAIR_G2_KSTEPS
#define ETAP_PAIR_G2_KSTEPS 4
#endif
#ifndef ETAP_PAIR_P_STORE
#define ETAP_PAIR_P_STORE 1
#endif
// GEMM2's A operand: 0 = P in tensor memory (TS UMMA, duplicated lanes: an exchange between the
// two row halves of each head through shared memory), 1 = P in shared memory (SS UMMA, K-major
// SW128 [64 heads][64 rows] hi and lo tiles in the exchange buffer's 16 KB, single-buffered)
#ifndef ETAP_PAIR_P_SMEM
#define ETAP_PAIR_P_SMEM 1
#endif
// 1: the two softmax warpgroups take alternate pages (each thread all 32 columns of its lane),
// the running max is handed from one to the other per page, and P goes to tensor memory (TS
// GEMM2), so the ~0.9k-cycle tcgen05.st and the duplicate-lane exchange get two page periods.
// Measured slower than the SS default on the same box (400.4 vs 377.7 us at 128 heads,
// profiles/r02e/trace_pair6.txt): thread-side TMEM stores beside a busy pipe cost more than the
// 66 vs 76.8 cycles per GEMM2 UMMA save. Kept for A/B runs.
#ifndef ETAP_PAIR_PINGPONG
#define ETAP_PAIR_PINGPONG 0
#endif
constexpr bool PINGPONG = ETAP_PAIR_PINGPONG != 0;
constexpr bool P_IN_SMEM = !PINGPONG && ETAP_PAIR_P_SMEM != 0;
// Arrivals on the leader's barriers: 0 = every CTA arrives through the cluster window with
// release.cluster, 1 = the leader's own warps arrive locally (release.cta), 2 = as 1 and the
// partner arrives relaxed.cluster. A cluster-scope release costs ~1k cycles per arrival on B200
// (trace_pair.py: 5.5k -> 3.4k cycles per page), and the orderings these arrivals publish do not
// need it: P is in tensor memory and complete (tcgen05.wait::st) before the arrival is issued,
// and an S_FREE arrival follows tcgen05.wait::ld. The V-ready arrival after zeroing smem rows
// (generic-proxy stores read by the partner's half of the MMA) keeps release.cluster.
#ifndef ETAP_PAIR_ARRIVE
#define ETAP_PAIR_ARRIVE 2
#endif
static_assert(OFF_Q % 1024 == 0 && STAGE % 1024 == 0 && STAGE_G1 % 1024 == 0, "SW128 alignment");
static_assert(B_P_FULL + 2 <= NB && B_G2_DONE + NG2 <= B_S_FREE, "barrier count");
static_assert(TC_P + NPB * 64 <= TMEM_COLS, "TMEM budget");
// V chunk i (0..3) of CTA r: N block i/2, 64-column atom i%2
__host__ __device__ constexpr int v_chunk(int r, int i) { return 2 * r + (i & 1) + 4 * (i >> 1); }
}  // namespace pairk

// one arrival of a softmax warp on the leader's barrier
__device__ __forceinline__ void pair_arrive(uint64_t* bar, bool leader) {
    if (ETAP_PAIR_ARRIVE >= 1 && leader) {
        ptx::mbar_arrive(bar);
    } else if (ETAP_PAIR_ARRIVE == 2) {
        asm volatile(
            "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, 0;\n\t"
            "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(ptx::smem_u32(bar))
            : "memory");
    } else {
        ptx::mbar_arrive_cluster(bar, 0);
    }
}

template <bool DBG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pairk::THREADS, 1)
    etap_mla_decode_pair_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_kv32,
                                const __grid_constant__ CUtensorMap tm_q, const DecodeParams prm) {
    using namespace pairk;
    constexpr bool kDebug = DBG;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    if (smem != smem_raw) asm volatile("trap;");  // no slack allocated: the base must be 1024-aligned
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    if (threadIdx.x == 0) {
        ETAP_TRACE_G(prm, 0);
        ETAP_TRACE_CLK(prm, 5);
    }

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_kv);
        ptx::prefetch_tmap(&tm_kv32);
        ptx::prefetch_tmap(&tm_q);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&bars[B_FULL_G1 + i], 1);
            ptx::mbar_init(&bars[B_V_LAND + i], 1);
            ptx::mbar_init(&bars[B_V_READY + i], 2);
            ptx::mbar_init(&bars[B_S_FULL + i], 1);
            ptx::mbar_init(&bars[B_S_FREE + i], PINGPONG ? 8 : 16);
            ptx::mbar_init(&bars[B_P_FULL + i], PINGPONG ? 8 : 16);
            ptx::mbar_init(&bars[B_MREF + i], 4);
        }
        for (int i = 0; i < NG2; ++i) ptx::mbar_init(&bars[B_G2_DONE + i], 1);
        ptx::mbar_init(&bars[B_FULL_Q], 1);
        ptx::mbar_init(&bars[B_Q_EMPTY], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_pair(tmem_slot, TMEM_COLS);
    ptx::tc_fence_before();
    ptx::cluster_sync_all();  // barriers of both CTAs initialised before any remote arrival / tx
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const Prologue pro = decode_prologue<kDebug, MAX_VB>(prm, smem + OFF_SCHED, UNIT, PAGE * D_QK * 2, true, warp, lane);
    const int32_t* sch = pro.sch;
    const int32_t* soff = pro.soff;
    const int idx_off = pro.idx_off;
    const bool fused = prm.inkernel_sched != 0;
    const int* s_len = pro.s_len;
    const int vb_begin = sch[0], vb_end = sch[2];
    const int B = prm.batch;
    auto seqlen_of = [&](int i) { return fused ? s_len[i] : max(0, prm.seqlens[(sch[5] + i) % B]); };
    const uint32_t stage_addr = ptx::smem_u32(smem + OFF_STAGE);

    if (warp == 0) {
        // ===================================================== TMA producer: GEMM1 halves + Q (both CTAs)
        // (every KV byte is read by both CTAs of the pair within a page: evict-normal)
        const uint64_t pol_kv = ptx::policy_evict_normal();
        const uint64_t pol_q = ptx::policy_evict_last();
        uint32_t bar_g1[2], bar_q;
        bar_g1[0] = ptx::mapa_u32(&bars[B_FULL_G1], 0);
        bar_g1[1] = ptx::mapa_u32(&bars[B_FULL_G1 + 1], 0);
        bar_q = ptx::mapa_u32(&bars[B_FULL_Q], 0);
        uint32_t gp = 0, nsplit = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            const int32_t* bt = prm.block_table + static_cast<size_t>(sd.b) * prm.max_pages;
            int base = sd.t0;
            int pg;
            if (nsplit == 0 && sd.b == pro.hint_b && sd.t0 == pro.hint_t0) pg = pro.hint_pg;
            else pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
            bool q_pending = true;
            for (int t = sd.t0; t < sd.t1; ++t) {
                if (t - base >= 32) {
                    base = t;
                    pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
                }
                const int page = __shfl_sync(0xffffffffu, pg, t - base);
                const uint32_t buf = gp & 1;
                uint8_t* stage = smem + OFF_STAGE + buf * STAGE;
                if (gp == 0 && pro.late_wait) dep_wait_producer<kDebug>(prm);
                // GEMM1 halves of page gp-2 are free once its GEMM1 completed
                if (gp >= 2) ptx::mbar_wait(&bars[B_S_FULL + buf], ((gp - 2) >> 1) & 1);
                if (lane == 0) {
                    ETAP_TRACE(prm, gp, 0);
                    if (leader) ptx::mbar_arrive_expect_tx(&bars[B_FULL_G1 + buf], 2 * STAGE_G1);
#pragma unroll 1
                    for (int c = 0; c < NCHUNK; ++c)
                        ptx::tma_load_2d_pair(stage + c * G1_BYTES, &tm_kv32, bar_g1[buf], c * 64,
                                              page * PAGE + 32 * static_cast<int>(rank), pol_kv);
                }
                __syncwarp();
                if (q_pending) {
                    q_pending = false;
                    if (nsplit > 0) ptx::mbar_wait(&bars[B_Q_EMPTY], (nsplit - 1) & 1);
                    if (lane == 0) {
                        if (leader) ptx::mbar_arrive_expect_tx(&bars[B_FULL_Q], 2 * Q_BYTES);
                        const int qrow = sd.b * prm.heads + sd.g * UNIT + HPC * static_cast<int>(rank);
#pragma unroll 1
                        for (int c = 0; c < NCHUNK; ++c)
                            ptx::tma_load_2d_pair(smem + OFF_Q + c * Q_CHUNK, &tm_q, bar_q, c * 64, qrow, pol_q);
                    }
                    __syncwarp();
                    ++nsplit;
                }
                ++gp;
            }
        }
        if (gp == 0 && pro.late_wait) dep_wait_producer<kDebug>(prm);
    } else if (warp == 1) {
        // ===================================================== GEMM1 issuer (leader)
        uint32_t nsplit = 0;
        if (leader) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 64, 0, 0);
            const uint64_t q_desc = ptx::smem_desc(ptx::smem_u32(smem + OFF_Q), 16, 1024, ptx::LAYOUT_SW128);
            uint32_t gp = 0;
            for (int vb = vb_begin; vb <= vb_end; ++vb) {
                SplitDesc sd;
                if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
                ptx::mbar_wait(&bars[B_FULL_Q], nsplit & 1);
                for (int t = sd.t0; t < sd.t1; ++t) {
                    const uint32_t buf = gp & 1;
                    if (gp >= 2) ptx::mbar_wait(&bars[B_S_FREE + buf], ((gp - 2) >> 1) & 1);
                    ptx::mbar_wait(&bars[B_FULL_G1 + buf], (gp >> 1) & 1);
                    __syncwarp();
                    ptx::tc_fence_after();
                    if (lane == 0) ETAP_TRACE(prm, gp, 3);
                    const uint64_t k_desc =
                        ptx::smem_desc(stage_addr + buf * STAGE, 16, 1024, ptx::LAYOUT_SW128);
                    const uint32_t s_tmem = tmem_base + TC_S + 32 * buf;
#pragma unroll
                    for (int c = 0; c < ETAP_PAIR_G1_CHUNKS; ++c)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            ptx::umma_pair_ss(s_tmem, q_desc + c * (Q_CHUNK >> 4) + 2 * kk,
                                              k_desc + c * (G1_BYTES >> 4) + 2 * kk, idesc, (c | kk) ? 1u : 0u);
                    ptx::umma_commit_pair(&bars[B_S_FULL + buf]);
                    if (lane == 0) ETAP_TRACE(prm, gp, 4);
                    if (t == sd.t1 - 1) ptx::umma_commit_pair(&bars[B_Q_EMPTY]);
                    ++gp;
                }
                ++nsplit;
            }
        } else {
            for (int vb = vb_begin; vb <= vb_end; ++vb) {
                SplitDesc sd;
                if (split_at(sch, seqlen_of(vb), B, vb, sd)) ++nsplit;
            }
        }
        // the last Q_EMPTY commit lands in both CTAs: wait for it before either CTA may exit
        if (nsplit > 0) ptx::mbar_wait(&bars[B_Q_EMPTY], (nsplit - 1) & 1);
    } else if (warp == 2) {
        // ===================================================== GEMM2 issuer (leader)
        if (leader) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 256, 0, 1);
            uint32_t gp = 0;
            for (int vb = vb_begin; vb <= vb_end; ++vb) {
                SplitDesc sd;
                if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
                for (int t = sd.t0; t < sd.t1; ++t) {
                    const uint32_t buf = gp & 1;
                    ptx::mbar_wait(&bars[B_P_FULL + buf], (gp >> 1) & 1);
                    if (lane == 0) ETAP_TRACE(prm, gp, 9);
                    // (acquire.cluster after zeroed tail rows: the release.cluster arrivals)
                    if (sd.seqlen - t * PAGE < PAGE) ptx::mbar_wait_cluster(&bars[B_V_READY + buf], (gp >> 1) & 1);
                    else ptx::mbar_wait(&bars[B_V_READY + buf], (gp >> 1) & 1);
                    __syncwarp();
                    ptx::tc_fence_after();
                    if (lane == 0) ETAP_TRACE(prm, gp, 10);
                    const uint32_t v0 = stage_addr + buf * STAGE + STAGE_G1;
                    const uint32_t p0 = tmem_base + TC_P + 64 * (gp % NPB);
                    const uint64_t p_desc = ptx::smem_desc(ptx::smem_u32(smem + OFF_X), 16, 1024, ptx::LAYOUT_SW128);
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        // MN-major SW128 B: LBO = the next 64-column atom (chunk), SBO = 8-row group
                        const uint64_t v_desc = ptx::smem_desc(v0 + 2 * n * V_BYTES, V_BYTES, 1024, ptx::LAYOUT_SW128);
#pragma unroll
                        for (int j = 0; j < ETAP_PAIR_G2_KSTEPS; ++j)
#pragma unroll
                            for (int part = 0; part < 2; ++part) {
                                const uint32_t acc = (t == sd.t0 && j == 0 && part == 0) ? 0u : 1u;
                                if (P_IN_SMEM)  // K-major SW128 A: +32 B per 16 rows of K
                                    ptx::umma_pair_ss(tmem_base + TC_O + 128 * n,
                                                      p_desc + part * (P_TILE >> 4) + 2 * j, v_desc + j * (2048 >> 4),
                                                      idesc, acc);
                                else
                                    ptx::umma_pair_ts(tmem_base + TC_O + 128 * n, p0 + 16 * j + 8 * part,
                                                      v_desc + j * (2048 >> 4), idesc, acc);
                            }
                    }
                    ptx::umma_commit_pair(&bars[B_G2_DONE + (gp % NG2)]);
                    if (lane == 0) ETAP_TRACE(prm, gp, 11);
                    ++gp;
                }
            }
        }
    } else if (warp == 3) {
        // ===================================================== TMA producer: V chunks (both CTAs)
        // rows of a split's last page past seqlen were loaded from HBM and may hold non-finite
        // garbage; their P is 0 but 0 * NaN = NaN in the MMA, so they are zeroed before GEMM2
        const uint64_t pol_kv = ptx::policy_evict_normal();
        uint32_t gp = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            const int32_t* bt = prm.block_table + static_cast<size_t>(sd.b) * prm.max_pages;
            int base = sd.t0;
            int pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
            for (int t = sd.t0; t < sd.t1; ++t) {
                if (t - base >= 32) {
                    base = t;
                    pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
                }
                const int page = __shfl_sync(0xffffffffu, pg, t - base);
                const uint32_t buf = gp & 1;
                // V chunks of page gp-2 are free once its GEMM2 completed
                if (gp >= 2) ptx::mbar_wait(&bars[B_G2_DONE + (gp - 2) % NG2], ((gp - 2) / NG2) & 1);
                if (lane == 0) {
                    ETAP_TRACE(prm, gp, 1);
                    ptx::mbar_arrive_expect_tx(&bars[B_V_LAND + buf], 4 * V_BYTES);
#pragma unroll 1
                    for (int i = 0; i < 4; ++i)
                        ptx::tma_load_2d(smem + OFF_STAGE + buf * STAGE + STAGE_G1 + i * V_BYTES, &tm_kv,
                                         &bars[B_V_LAND + buf], v_chunk(static_cast<int>(rank), i) * 64, page * PAGE,
                                         pol_kv);
                }
                __syncwarp();
                ptx::mbar_wait(&bars[B_V_LAND + buf], (gp >> 1) & 1);
                if (lane == 0) ETAP_TRACE(prm, gp, 2);
                const int r0 = sd.seqlen - t * PAGE;
                if (r0 < PAGE) {
                    uint8_t* v = smem + OFF_STAGE + buf * STAGE + STAGE_G1;
                    for (int i = lane; i < (PAGE - r0) * 4 * 8; i += 32) {
                        const int row = r0 + i / 32, ch = (i / 8) & 3, q16 = i & 7;
                        *reinterpret_cast<uint4*>(v + ch * V_BYTES + row * 128 + q16 * 16) = make_uint4(0, 0, 0, 0);
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                }
                if (lane == 0) {
                    if (r0 < PAGE) ptx::mbar_arrive_cluster(&bars[B_V_READY + buf], 0);
                    else pair_arrive(&bars[B_V_READY + buf], leader);
                }
                ++gp;
            }
        }
    } else if constexpr (PINGPONG) {
        // ===================================================== softmax + epilogue, ping-pong (both CTAs)
        // warpgroup wg takes the pages gp with gp % 2 == wg; thread = TMEM lane L of its quadrant
        // (head h = L % 64, row half r = L / 64) x all 32 columns: KV rows 32r + [0, 32) = GEMM2
        // k-steps 2r, 2r + 1. The running max of a page goes to the other warpgroup through
        // s_mref[wg] and the B_MREF[wg] barrier; l is kept per thread relative to the max it last
        // used and rescaled when the handed-over max moved.
        const int wg = (warp - SM_WARP0) >> 2;
        const int q = warp & 3;
        const int L = 32 * q + lane;
        const int h = L & (HPC - 1), r = L >> 6;
        const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
        const uint32_t wg_bar = 3 + wg;
        float* red = reinterpret_cast<float*>(smem + OFF_RED);    // [2 wg][2 r][64]
        float* s_mref = reinterpret_cast<float*>(smem + OFF_MREF);  // [2 wg][64]
        uint4* xb = reinterpret_cast<uint4*>(smem + OFF_X) + wg * 128 * 4;  // this warpgroup: [128][4] uint4
        const bool negate = prm.flags & FLAG_NEGATE_RESCALE;
        const bool eager = negate || (prm.flags & FLAG_EAGER_RESCALE);
        const float thresh = eager ? 0.f : LAZY_RESCALE_LOG2;
        const bool mtp = prm.q_tokens > 1;
        const bool tracer = threadIdx.x == SM_WARP0 * 32;
        uint32_t gp = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            const int head = sd.g * UNIT + HPC * static_cast<int>(rank) + h;  // query row of the sequence
            const int tok = head / prm.heads_per_token;
            const int row_lim = sd.seqlen - (prm.causal ? prm.q_tokens - 1 - tok : 0);
            float m_seen = -INFINITY, l_part = 0.f;  // l_part relative to m_seen
            for (int t = sd.t0; t < sd.t1; ++t, ++gp) {
                if ((gp & 1) != static_cast<uint32_t>(wg)) continue;
                const uint32_t buf = gp & 1;
                const bool first = t == sd.t0;
                wg_wait(&bars[B_S_FULL + buf], (gp >> 1) & 1, wg_bar, q);
                ptx::tc_fence_after();
                if (tracer) ETAP_TRACE(prm, gp, 5);
                uint32_t sr[32];
                ptx::tmem_ld32(t_lane + TC_S + 32 * buf, sr);
                ptx::tmem_wait_ld();
                if (tracer) ETAP_TRACE(prm, gp, 13);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) pair_arrive(&bars[B_S_FREE + buf], leader);
                if (tracer) ETAP_TRACE(prm, gp, 12);
                const int row0 = t * PAGE + 32 * r;
                float x[32];
                if (row0 + 32 <= row_lim) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(sr[i]) * prm.scale_log2;
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) x[i] = row0 + i < row_lim ? __uint_as_float(sr[i]) * prm.scale_log2 : -INFINITY;
                }
                float lm = x[0];
#pragma unroll
                for (int i = 1; i < 32; ++i) lm = fmaxf(lm, x[i]);
                red[(2 * wg + r) * HPC + h] = lm;
                ptx::named_bar_sync(wg_bar, 128);
                const float pagemax = fmaxf(red[2 * wg * HPC + h], red[(2 * wg + 1) * HPC + h]);
                // the running max after page gp-1 (the other warpgroup); also orders that
                // warpgroup's read of s_mref[wg] (page gp-2) before this page's write
                if (gp >= 1) ptx::mbar_wait(&bars[B_MREF + ((gp - 1) & 1)], ((gp - 1) >> 1) & 1);
                const float m_prev = first ? -INFINITY : s_mref[((gp - 1) & 1) * HPC + h];
                float m_cur = m_prev, alpha = first ? 0.f : 1.f;
                bool upd = false;
                if (first) {
                    m_cur = pagemax;
                } else if (pagemax > m_prev + thresh) {
                    m_cur = pagemax;
                    alpha = ptx::exp2_ftz(m_prev - m_cur);
                    upd = true;
                }
                if (r == 0) s_mref[wg * HPC + h] = m_cur;
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bars[B_MREF + wg]);
                if (tracer) ETAP_TRACE(prm, gp, 6);
                // a column may have no visible row yet (multi-token causal mask): m = -inf
                const float mu = (mtp && m_cur == -INFINITY) ? 0.f : m_cur;
                if (m_seen != m_cur) {
                    l_part = l_part == 0.f ? 0.f : l_part * ptx::exp2_ftz(m_seen - m_cur);
                    m_seen = m_cur;
                }
                float ps = 0.f;
                uint32_t pk[32];  // k-step 2r: [0, 8) hi, [8, 16) lo; k-step 2r + 1: [16, 24) hi, [24, 32) lo
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float p0 = ptx::exp2_ftz(x[16 * k + 2 * i] - mu), p1 = ptx::exp2_ftz(x[16 * k + 2 * i + 1] - mu);
                        ps += p0 + p1;
                        const uint32_t hi = pack_bf16x2(p0, p1);
                        pk[16 * k + i] = hi;
                        pk[16 * k + 8 + i] = pack_bf16x2(p0 - __uint_as_float(hi << 16), p1 - __uint_as_float(hi & 0xffff0000u));
                    }
                l_part += ps;
                // P columns of this buffer: GEMM2 of page gp-NPB must have read them
                if (gp >= NPB) wg_wait(&bars[B_G2_DONE + (gp - NPB) % NG2], ((gp - NPB) / NG2) & 1, wg_bar, q);
                if (tracer) ETAP_TRACE(prm, gp, 7);
                const bool resc = __any_sync(0xffffffffu, upd) || (negate && !first);
                if (resc) {
                    // O must contain GEMM2 of page gp-1 before it is rescaled (this lane's 256 columns)
                    ptx::mbar_wait(&bars[B_G2_DONE + (gp - 1) % NG2], ((gp - 1) / NG2) & 1);
                    ptx::tc_fence_after();
                    const float a = negate ? -alpha : alpha;
#pragma unroll 1
                    for (int c = 0; c < 8; ++c) {
                        uint32_t o[32];
                        const uint32_t ta = t_lane + TC_O + 32 * c;
                        ptx::tmem_ld32(ta, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
                        ptx::tmem_st32(ta, o);
                    }
                }
                // own 32 columns [32r, 32r + 32) of the P buffer, and (two rounds through this
                // warpgroup's 8 KB of the exchange buffer) the duplicate lane L ^ 64's
                const uint32_t pcol = t_lane + TC_P + 64 * (gp % NPB);
                uint32_t th[32];
#pragma unroll
                for (int round = 0; round < 2; ++round) {
                    uint4* mine = xb + L * 4;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int b0 = (i >> 1) * 16 + round * 8 + (i & 1) * 4;  // k-step i/2, hi (round 0) / lo (1)
                        mine[i] = make_uint4(pk[b0], pk[b0 + 1], pk[b0 + 2], pk[b0 + 3]);
                    }
                    ptx::named_bar_sync(wg_bar, 128);
                    const uint4* theirs = xb + (L ^ 64) * 4;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 v = theirs[i];
                        const int b0 = (i >> 1) * 16 + round * 8 + (i & 1) * 4;
                        th[b0] = v.x; th[b0 + 1] = v.y; th[b0 + 2] = v.z; th[b0 + 3] = v.w;
                    }
                    if (round == 0) ptx::named_bar_sync(wg_bar, 128);  // partner read before the lo round
                }
                if (tracer) ETAP_TRACE(prm, gp, 14);
                ptx::tmem_st32(pcol + 32 * r, pk);
                ptx::tmem_st32(pcol + 32 * (r ^ 1), th);
                ptx::tmem_wait_st();
                if (tracer) ETAP_TRACE(prm, gp, 15);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) pair_arrive(&bars[B_P_FULL + buf], leader);
                if (tracer) ETAP_TRACE(prm, gp, 8);
            }

            // ---- epilogue: the split's final max, l over the four (warpgroup, row half) parts,
            // O = O / l, L = m + log l (etap.cpp:140-144)
            const uint32_t last = gp - 1;
            float m_fin;
            if ((last & 1) == static_cast<uint32_t>(wg)) {
                m_fin = m_seen;
            } else {
                ptx::mbar_wait(&bars[B_MREF + (last & 1)], (last >> 1) & 1);
                m_fin = s_mref[(last & 1) * HPC + h];
            }
            const float l_fin = l_part == 0.f ? 0.f : l_part * ptx::exp2_ftz(m_seen - m_fin);
            ptx::named_bar_sync(2, 256);  // both warpgroups are past their last page's use of red
            red[(2 * wg + r) * HPC + h] = l_fin;
            ptx::named_bar_sync(2, 256);
            const float l = red[h] + red[HPC + h] + red[2 * HPC + h] + red[3 * HPC + h];
            const float inv = l > 0.f ? 1.f / l : 0.f;  // l = 0: the row saw no KV row (O = 0, L = -inf)
            wg_wait(&bars[B_G2_DONE + last % NG2], (last / NG2) & 1, wg_bar, q);
            ptx::tc_fence_after();
            const int ns = soff[vb + 1] - soff[vb];
            const bool direct = ns == 1;
            const int idx = (vb == sch[0]) ? sch[4] : soff[vb] + idx_off;
            const size_t orow = direct ? prm.om.row(sd.b, head) : 0;
            float* part_o = prm.ws_o + (static_cast<size_t>(idx) * UNIT + HPC * rank + h) * D_V;
            const int d0 = 256 * wg + 128 * r;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t o[32];
                ptx::tmem_ld32(t_lane + TC_O + 128 * wg + 32 * c, o);
                ptx::tmem_wait_ld();
                float4 v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    v[i] = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                                       __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
                if (direct) {
#pragma unroll 1
                    for (int k = 0; k < prm.om.n_out; ++k) {
                        float4* dst = reinterpret_cast<float4*>(prm.om.out[k] + orow * D_V + d0 + 32 * c);
#pragma unroll
                        for (int i = 0; i < 8; ++i) dst[i] = v[i];
                    }
                } else {
                    float4* dst = reinterpret_cast<float4*>(part_o + d0 + 32 * c);
#pragma unroll
                    for (int i = 0; i < 8; ++i) dst[i] = v[i];
                }
            }
            if (wg == 0 && r == 0) {
                const float Lse = (m_fin + log2f(l)) * 0.69314718055994530942f;
                if (direct) {
                    for (int k = 0; k < prm.om.n_out; ++k) prm.om.lse[k][orow] = Lse;
                } else {
                    prm.ws_lse[static_cast<size_t>(idx) * UNIT + HPC * rank + h] = Lse;
                }
            }
            ptx::tc_fence_before();
            // both warpgroups have read O before either releases the next split's first GEMM2
            ptx::named_bar_sync(2, 256);
        }
    } else {
        // ===================================================== softmax + epilogue (both CTAs)
        // thread = TMEM lane L of its quadrant (head h = L % 64, row half r = L / 64) x the 16
        // columns of its warpgroup: KV rows 32r + 16wg + [0, 16) = GEMM2 k-step 2r + wg
        const int wg = (warp - SM_WARP0) >> 2;
        const int q = warp & 3;
        const int L = 32 * q + lane;
        const int h = L & (HPC - 1), r = L >> 6;
        const int kstep = 2 * r + wg;
        const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
        const uint32_t wg_bar = 3 + wg;
        float* red = reinterpret_cast<float*>(smem + OFF_RED);  // [4][64]
        uint4* xb = reinterpret_cast<uint4*>(smem + OFF_X);      // [2][128][4] uint4
        const bool negate = prm.flags & FLAG_NEGATE_RESCALE;
        const bool eager = negate || (prm.flags & FLAG_EAGER_RESCALE);
        const float thresh = eager ? 0.f : LAZY_RESCALE_LOG2;
        const bool mtp = prm.q_tokens > 1;
        const int quarter = 2 * wg + r;
        const bool tracer = threadIdx.x == SM_WARP0 * 32;
        uint32_t gp = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            const int head = sd.g * UNIT + HPC * static_cast<int>(rank) + h;  // query row of the sequence
            const int tok = head / prm.heads_per_token;
            const int row_lim = sd.seqlen - (prm.causal ? prm.q_tokens - 1 - tok : 0);
            float m_own = -INFINITY, m_thr = -INFINITY, mu = mtp ? 0.f : -INFINITY, l_part = 0.f;
            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gp & 1;
                const bool first = t == sd.t0;
                wg_wait(&bars[B_S_FULL + buf], (gp >> 1) & 1, wg_bar, q);
                ptx::tc_fence_after();
                if (tracer) ETAP_TRACE(prm, gp, 5);
                uint32_t sr[16];
                ptx::tmem_ld16(t_lane + TC_S + 32 * buf + 16 * wg, sr);
                ptx::tmem_wait_ld();
                if (tracer) ETAP_TRACE(prm, gp, 13);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) pair_arrive(&bars[B_S_FREE + buf], leader);
                if (tracer) ETAP_TRACE(prm, gp, 12);
                const int row0 = t * PAGE + 32 * r + 16 * wg;
                float x[16];
                if (row0 + 16 <= row_lim) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) x[i] = __uint_as_float(sr[i]) * prm.scale_log2;
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) x[i] = row0 + i < row_lim ? __uint_as_float(sr[i]) * prm.scale_log2 : -INFINITY;
                }
                bool exceed = false;
#pragma unroll
                for (int i = 0; i < 16; ++i) exceed |= x[i] > m_thr;
                // one barrier decides, CTA-uniformly, whether any running max must move
                const bool any = ptx::bar_red_or(1, 256, exceed || (negate && !first));
                float alpha = first ? 0.f : 1.f;
                bool upd = false;
                if (any) {
                    float lm = x[0];
#pragma unroll
                    for (int i = 1; i < 16; ++i) lm = fmaxf(lm, x[i]);
                    red[quarter * HPC + h] = lm;
                    ptx::named_bar_sync(2, 256);
                    const float mt = fmaxf(fmaxf(red[h], red[HPC + h]), fmaxf(red[2 * HPC + h], red[3 * HPC + h]));
                    if (first) {
                        m_own = mt;
                    } else {
                        const float mn = fmaxf(m_own, mt);
                        if (mn > m_own + thresh) {
                            alpha = ptx::exp2_ftz(m_own - mn);
                            m_own = mn;
                            upd = true;
                        }
                    }
                    m_thr = m_own + thresh;
                    mu = (mtp && m_own == -INFINITY) ? 0.f : m_own;
                }
                float ps = 0.f;
                uint32_t pk[16];  // [0, 8) hi pairs, [8, 16) lo pairs (rows 2i, 2i+1)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float p0 = ptx::exp2_ftz(x[2 * i] - mu), p1 = ptx::exp2_ftz(x[2 * i + 1] - mu);
                    ps += p0 + p1;
                    pk[i] = pack_bf16x2(p0, p1);
                    pk[8 + i] = pack_bf16x2(p0 - __uint_as_float(pk[i] << 16), p1 - __uint_as_float(pk[i] & 0xffff0000u));
                }
                l_part = fmaf(l_part, alpha, ps);  // first page: alpha = 0
                // this thread's k-step goes to its own lane and, via shared memory, to the
                // duplicate lane L ^ 64 of the 2-SM A layout (warp q ^ 2 of the same warpgroup)
                if (tracer) ETAP_TRACE(prm, gp, 6);
                if constexpr (P_IN_SMEM) {
                    // GEMM2 of page gp-1 must have read the single P tile (and O must hold it
                    // before a rescale): one wait covers both
                    if (gp >= 1) wg_wait(&bars[B_G2_DONE + (gp - 1) % NG2], ((gp - 1) / NG2) & 1, wg_bar, q);
                    if (tracer) ETAP_TRACE(prm, gp, 7);
                    const bool resc = __any_sync(0xffffffffu, upd) || (negate && !first);
                    if (resc) {
                        ptx::tc_fence_after();
                        const float a = negate ? -alpha : alpha;
#pragma unroll 1
                        for (int c = 0; c < 4; ++c) {
                            uint32_t o[32];
                            const uint32_t ta = t_lane + TC_O + 128 * wg + 32 * c;
                            ptx::tmem_ld32(ta, o);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
                            ptx::tmem_st32(ta, o);
                        }
                        ptx::tmem_wait_st();
                    }
                    // row h of the K-major SW128 tiles: rows 32r + 16wg + [0, 16) are 32 B = two
                    // 16 B chunks at chunk index 4r + 2wg (+1), XOR-swizzled with h % 8
                    uint8_t* prow = smem + OFF_X + (h >> 3) * 1024 + (h & 7) * 128;
                    const int c0 = 4 * r + 2 * wg;
#pragma unroll
                    for (int part = 0; part < 2; ++part) {
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const int i0 = part * 8 + 4 * k;
                            *reinterpret_cast<uint4*>(prow + part * P_TILE + (((c0 + k) ^ (h & 7)) << 4)) =
                                make_uint4(pk[i0], pk[i0 + 1], pk[i0 + 2], pk[i0 + 3]);
                        }
                    }
                    ptx::fence_proxy_async_smem();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (tracer) ETAP_TRACE(prm, gp, 15);
                    if (lane == 0) pair_arrive(&bars[B_P_FULL + buf], leader);
                    if (tracer) ETAP_TRACE(prm, gp, 8);
                    ++gp;
                    continue;
                }
                uint4* mine = xb + (wg * 128 + L) * 4;
#pragma unroll
                for (int i = 0; i < 4; ++i) mine[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
                // P columns of this buffer: GEMM2 of page gp-NPB must have read them
                if (gp >= NPB) wg_wait(&bars[B_G2_DONE + (gp - NPB) % NG2], ((gp - NPB) / NG2) & 1, wg_bar, q);
                if (tracer) ETAP_TRACE(prm, gp, 7);
                const bool resc = __any_sync(0xffffffffu, upd) || (negate && !first);
                if (resc) {
                    // O must contain GEMM2 of page gp-1 before it is rescaled
                    ptx::mbar_wait(&bars[B_G2_DONE + (gp - 1) % NG2], ((gp - 1) / NG2) & 1);
                    ptx::tc_fence_after();
                    const float a = negate ? -alpha : alpha;
#pragma unroll 1
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        const uint32_t ta = t_lane + TC_O + 128 * wg + 32 * c;
                        ptx::tmem_ld32(ta, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
                        ptx::tmem_st32(ta, o);
                    }
                }
                ptx::named_bar_sync(wg_bar, 128);  // exchange buffer written by the partner lane
                if (tracer) ETAP_TRACE(prm, gp, 14);
                const uint4* theirs = xb + (wg * 128 + (L ^ 64)) * 4;
                uint32_t ph[8], pl[8], oh[8], ol[8];
                {
                    const uint4 a0 = theirs[0], a1 = theirs[1], a2 = theirs[2], a3 = theirs[3];
                    oh[0] = a0.x; oh[1] = a0.y; oh[2] = a0.z; oh[3] = a0.w;
                    oh[4] = a1.x; oh[5] = a1.y; oh[6] = a1.z; oh[7] = a1.w;
                    ol[0] = a2.x; ol[1] = a2.y; ol[2] = a2.z; ol[3] = a2.w;
                    ol[4] = a3.x; ol[5] = a3.y; ol[6] = a3.z; ol[7] = a3.w;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) { ph[i] = pk[i]; pl[i] = pk[8 + i]; }
                const uint32_t pcol = t_lane + TC_P + 64 * (gp % NPB);
                if (ETAP_PAIR_P_STORE) {
                    uint32_t mine16[16], theirs16[16];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        mine16[i] = ph[i]; mine16[8 + i] = pl[i];
                        theirs16[i] = oh[i]; theirs16[8 + i] = ol[i];
                    }
                    ptx::tmem_st16(pcol + 16 * kstep, mine16);
                    ptx::tmem_st16(pcol + 16 * (kstep ^ 2), theirs16);
                    ptx::tmem_wait_st();
                }
                if (tracer) ETAP_TRACE(prm, gp, 15);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) pair_arrive(&bars[B_P_FULL + buf], leader);
                if (tracer) ETAP_TRACE(prm, gp, 8);
                ++gp;
            }

            // ---- epilogue: l over the four row quarters, O = O / l, L = m + log l (etap.cpp:140-144)
            ptx::named_bar_sync(2, 256);  // every thread is past its last read of red
            red[quarter * HPC + h] = l_part;
            ptx::named_bar_sync(2, 256);
            const float l = red[h] + red[HPC + h] + red[2 * HPC + h] + red[3 * HPC + h];
            const float inv = l > 0.f ? 1.f / l : 0.f;  // l = 0: the row saw no KV row (O = 0, L = -inf)
            const uint32_t last = gp - 1;
            wg_wait(&bars[B_G2_DONE + last % NG2], (last / NG2) & 1, wg_bar, q);
            ptx::tc_fence_after();
            const int ns = soff[vb + 1] - soff[vb];
            const bool direct = ns == 1;
            const int idx = (vb == sch[0]) ? sch[4] : soff[vb] + idx_off;
            const size_t orow = direct ? prm.om.row(sd.b, head) : 0;
            float* part_o = prm.ws_o + (static_cast<size_t>(idx) * UNIT + HPC * rank + h) * D_V;
            const int d0 = 256 * wg + 128 * r;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t o[32];
                ptx::tmem_ld32(t_lane + TC_O + 128 * wg + 32 * c, o);
                ptx::tmem_wait_ld();
                float4 v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    v[i] = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                                       __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
                if (direct) {
#pragma unroll 1
                    for (int k = 0; k < prm.om.n_out; ++k) {
                        float4* dst = reinterpret_cast<float4*>(prm.om.out[k] + orow * D_V + d0 + 32 * c);
#pragma unroll
                        for (int i = 0; i < 8; ++i) dst[i] = v[i];
                    }
                } else {
                    float4* dst = reinterpret_cast<float4*>(part_o + d0 + 32 * c);
#pragma unroll
                    for (int i = 0; i < 8; ++i) dst[i] = v[i];
                }
            }
            if (quarter == 0) {
                const float Lse = (m_own + log2f(l)) * 0.69314718055994530942f;
                if (direct) {
                    for (int k = 0; k < prm.om.n_out; ++k) prm.om.lse[k][orow] = Lse;
                } else {
                    prm.ws_lse[static_cast<size_t>(idx) * UNIT + HPC * rank + h] = Lse;
                }
            }
            ptx::tc_fence_before();
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync_all();  // the partner's remote arrivals and commits have landed
    if (threadIdx.x == 0) {
        span_stamp(prm, 1);
        ETAP_TRACE_G(prm, 2);
        ETAP_TRACE_CLK(prm, 6);
    }
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem_base, TMEM_COLS);
    }
}
