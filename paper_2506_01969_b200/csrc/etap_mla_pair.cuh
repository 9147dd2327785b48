// SPDX-License-Identifier: Apache-2.0
// K2-pair: the decode for 128 heads per work unit on a CTA pair (tcgen05 cta_group::2).
// Included by etap_mla.cu inside its anonymous namespace (shares the split schedule, the
// prologue and the output map of the single-CTA kernels).
//
// Reference algorithm: etaplab::run_etap / block_update_impl (/root/reference/proj/src/etap.cpp
// :15-79 per-block update, :102-148 driver, epilogue L = m + log l at :144), with the heads of the
// decode folded into the query rows as the reference's cmd_bench does (cli.cpp:214).
//
// Why a pair (DESIGN.md §3 "K2-pair"): at 128 heads per GPU the single-CTA kernels are bound by
// tensor-pipe instruction cost, not HBM. A 1-SM UMMA of M64 N64 takes 32.7 cycles for 64x64x16,
// a pair UMMA of M128 N64 takes 25.8 cycles for twice that work (scripts/probe_pair*.cu). TMEM
// also caps one SM at O for ~96 heads; a pair holds O for 64 heads per SM over all 512 latent
// columns.
//
// The work unit is (sequence, 128 heads); CTA r of the pair owns heads [64r, 64r + 64).
//   GEMM1  S[128 heads x 64 rows] = Q . K^T   pair SS UMMA M=128 N=64: A = this CTA's 64 Q rows
//          (smem, 72 KB per split), B = K^T split by N: CTA r supplies KV rows [32r, 32r+32) of
//          the page (9 chunks of 32 x 64, 36 KB). D lands in the 2x2 layout: lane h holds head h
//          x rows 0-31, lane 64+h head h x rows 32-63 (32 TMEM columns per page).
//   softmax  thread = (head, 16 rows): online max with the thresholded lazy rescale, P = 2^(x-m)
//          split into bf16 hi + lo (the bf16 rounding of P alone would cost the 2e-5 RMSE bar),
//          written to shared memory.
//   GEMM2  O[128 heads x 512] += P . V   pair SS UMMA M=128 N=256: A = P (K-major SW128
//          [64 heads][64 rows] hi and lo tiles), B = V split by N: CTA r supplies latent chunks
//          {2r, 2r+1} (N block 0) and {2r+4, 2r+5} (block 1) of all 64 rows (32 KB). O of this
//          CTA's 64 heads (all 512 columns) stays in its TMEM, so the rescale and the epilogue
//          never cross SMs.
// Shared memory per CTA: Q 72 KB + two pages x (36 + 32) KB + P 16 KB.
// Measured alternatives (DESIGN.md §3 "K2-pair", profiles/r02e): P in tensor memory (TS UMMA,
// 66 vs 76.8 cycles, but a duplicate-lane exchange and slow thread-side tcgen05.st: 395 vs 371 us),
// the same with two softmax warpgroups alternating pages (400 vs 378 us), and GEMM1 over two-page
// tiles (N = 128, 32.9 cycles per two pages' UMMA, but its 72 KB of halves then fit only single-
// buffered and their load latency sets the period: 422 vs 371 us).
#pragma once

#ifndef ETAP_PAIR_BOX3D
#define ETAP_PAIR_BOX3D 1  // 3-D page boxes: 1 TMA per GEMM1 half-page (was 9), 2 per V half (was 4); A/B: 0
#endif
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
constexpr int P_TILE = HPC * 128;              // one [64 heads][64 rows] bf16 tile (8 KB)
constexpr int OFF_P = OFF_Q + Q_BYTES;         // P hi tile, P lo tile
constexpr int OFF_RED = OFF_P + 2 * P_TILE;    // [4][64] floats: per-(row quarter) head max / sum
constexpr int OFF_BAR = OFF_RED + 4 * HPC * 4;
constexpr int NB = 18;
constexpr int OFF_TMEM = OFF_BAR + NB * 8;
constexpr int OFF_SCHED = OFF_TMEM + 16;
constexpr int MAX_VB = 64;                     // fused-schedule line limit (longer lines: K1)
constexpr int SMEM = OFF_SCHED + sched_smem_ints(MAX_VB) * 4;
constexpr int THREADS = 384;                   // warps 0-3 roles, 4-11 two softmax warpgroups
constexpr int SM_WARP0 = 4;
// TMEM columns (512 allocated per CTA): O [0, 256): N block n at 128n (lane h: head h, d 256n +
// c; lane 64+h: head h, d 256n + 128 + c); S [256, 320): two pages of 32 columns.
constexpr uint32_t TC_O = 0, TC_S = 256, TMEM_COLS = 512;
constexpr int NG2 = 4;   // GEMM2-done barriers (a ring of four keeps every waited phase the newest
                         // or the one before on its barrier)
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
    B_P_FULL = 16,   // [2] L: both CTAs' P of the page in shared memory, O rescaled (16 warp arrivals)
};
static_assert(SMEM <= 232448, "shared memory budget");
// Arrivals on the leader's barriers: 0 = every CTA arrives through the cluster window with
// release.cluster, 1 = the leader's own warps arrive locally (release.cta), 2 = as 1 and the
// partner arrives relaxed.cluster. A cluster-scope release costs ~1k cycles per arrival on B200
// (trace_pair.py: 5.5k -> 3.4k cycles per page), and the orderings these arrivals publish do not
// need it: an S_FREE arrival follows tcgen05.wait::ld, a P_FULL arrival the proxy fence of the
// P stores. The V-ready arrival after zeroing smem rows (generic-proxy stores read by the
// partner's half of the MMA) keeps release.cluster.
#ifndef ETAP_PAIR_ARRIVE
#define ETAP_PAIR_ARRIVE 2
#endif
static_assert(OFF_Q % 1024 == 0 && OFF_P % 1024 == 0 && STAGE % 1024 == 0 && STAGE_G1 % 1024 == 0,
              "SW128 alignment");
static_assert(B_P_FULL + 2 <= NB && B_G2_DONE + NG2 <= B_S_FREE, "barrier count");
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
            ptx::mbar_init(&bars[B_S_FREE + i], 16);
            ptx::mbar_init(&bars[B_P_FULL + i], 16);
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

    // (the leader's warp 3 streams V: the schedule publish, which waits for the grid
    // dependency, comes after its last page instead of before its first)
    const Prologue pro = decode_prologue<kDebug, MAX_VB>(prm, smem + OFF_SCHED, UNIT, PAGE * D_QK * 2, true, warp, lane,
                                                         true);
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
#if ETAP_PAIR_BOX3D
                    // this CTA's 32 rows of the page, all nine chunks, as [chunk][row][128 B]
                    ptx::tma_load_3d_pair(stage, &tm_kv32, bar_g1[buf], 0, page * PAGE + 32 * static_cast<int>(rank), 0,
                                          pol_kv);
#else
#pragma unroll 1
                    for (int c = 0; c < NCHUNK; ++c)
                        ptx::tma_load_2d_pair(stage + c * G1_BYTES, &tm_kv32, bar_g1[buf], c * 64,
                                              page * PAGE + 32 * static_cast<int>(rank), pol_kv);
#endif
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
                    for (int c = 0; c < NCHUNK; ++c)
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
                    const uint64_t p_desc = ptx::smem_desc(ptx::smem_u32(smem + OFF_P), 16, 1024, ptx::LAYOUT_SW128);
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        // MN-major SW128 B: LBO = the next 64-column atom (chunk), SBO = 8-row group
                        const uint64_t v_desc = ptx::smem_desc(v0 + 2 * n * V_BYTES, V_BYTES, 1024, ptx::LAYOUT_SW128);
#pragma unroll
                        for (int j = 0; j < 4; ++j)
#pragma unroll
                            for (int part = 0; part < 2; ++part)  // K-major SW128 A: +32 B per 16 rows of K
                                ptx::umma_pair_ss(tmem_base + TC_O + 128 * n, p_desc + part * (P_TILE >> 4) + 2 * j,
                                                  v_desc + j * (2048 >> 4), idesc,
                                                  (t == sd.t0 && j == 0 && part == 0) ? 0u : 1u);
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
#if ETAP_PAIR_BOX3D
                    // V chunks {2r, 2r+1} and {2r+4, 2r+5}: two boxes of two consecutive chunks
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        ptx::tma_load_3d(smem + OFF_STAGE + buf * STAGE + STAGE_G1 + 2 * h * V_BYTES, &tm_kv,
                                         &bars[B_V_LAND + buf], 0, page * PAGE, v_chunk(static_cast<int>(rank), 2 * h),
                                         pol_kv);
#else
#pragma unroll 1
                    for (int i = 0; i < 4; ++i)
                        ptx::tma_load_2d(smem + OFF_STAGE + buf * STAGE + STAGE_G1 + i * V_BYTES, &tm_kv,
                                         &bars[B_V_LAND + buf], v_chunk(static_cast<int>(rank), i) * 64, page * PAGE,
                                         pol_kv);
#endif
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
        publish_after_prologue(prm, pro, lane);
    } else {
        // ===================================================== softmax + epilogue (both CTAs)
        // thread = TMEM lane L of its quadrant (head h = L % 64, row half r = L / 64) x the 16
        // columns of its warpgroup: KV rows 32r + 16wg + [0, 16) = GEMM2 k-step 2r + wg
        const int wg = (warp - SM_WARP0) >> 2;
        const int q = warp & 3;
        const int L = 32 * q + lane;
        const int h = L & (HPC - 1), r = L >> 6;
        const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
        const uint32_t wg_bar = 3 + wg;
        float* red = reinterpret_cast<float*>(smem + OFF_RED);  // [4][64]
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
                if (tracer) ETAP_TRACE(prm, gp, 6);
                // GEMM2 of page gp-1 must have read the single P tile (and O must hold it before
                // a rescale): one wait covers both
                if (gp >= 1) wg_wait(&bars[B_G2_DONE + (gp - 1) % NG2], ((gp - 1) / NG2) & 1, wg_bar, q);
                if (tracer) ETAP_TRACE(prm, gp, 7);
                if (__any_sync(0xffffffffu, upd) || (negate && !first)) {
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
                // row h of the K-major SW128 tiles: rows 32r + 16wg + [0, 16) are 32 B = two 16 B
                // chunks at chunk index 4r + 2wg (+1), XOR-swizzled with h % 8
                uint8_t* prow = smem + OFF_P + (h >> 3) * 1024 + (h & 7) * 128;
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
                if (lane == 0) pair_arrive(&bars[B_P_FULL + buf], leader);
                if (tracer) ETAP_TRACE(prm, gp, 8);
                ++gp;
            }

            // ---- epilogue: l over the four row quarters, O = O / l, L = m + log l (etap.cpp:140-144)
            dep_wait_before_write(prm);
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
