// SPDX-License-Identifier: Apache-2.0
// B200 (sm_100a) ETAP MLA decode: kernels K1 (split-KV scheduler), K2 (transposed tcgen05
// pipeline), K3 (log-sum-exp combine), a UMMA layout self-test, and the C-ABI declared in
// include/etap_mla.h.
//
// Reference path replaced: etaplab::run_etap (/root/reference/proj/src/etap.cpp:102-148)
// with its per-block body block_update_impl (etap.cpp:15-79). See DESIGN.md for the data
// layout in HBM, the smem ring, the TMEM map and the roofline.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/etap_mla.h"
#include "etap_mla_kernels.cuh"
#include "etap_fp8.cuh"

using namespace etap_b200;

#ifndef ETAP_MLA_VERSION
#define ETAP_MLA_VERSION "etap_mla sm_100a r1"
#endif

// =============================================================================================
// K1: split-KV scheduler. One CTA of 1024 threads.
//
// Virtual sequences vb = g * batch + b (head group major). Each owns tiles(vb) =
// ceil(seqlen_b / 64) KV tiles and a cost of tiles + META_FIXED_COST (0 if empty). The CTAs
// are dealt into line_shape().lanes lanes of p_line CTAs; the cost line of one lane's
// line_n virtual sequences [0, total) is cut into p_line equal intervals and line CTA k takes
// [k*T, (k+1)*T) mapped back to (line position, tile). Every lane uses the same cut, so with
// several head groups the lanes stream the same pages in lock step (L2 sharing). Partials of
// one vb are numbered contiguously in CTA order: split_off[vb] .. split_off[vb+1].
// sched[cta] = {pos_begin, tile_begin, pos_end, tile_end (exclusive), first_partial_idx,
//               vb offset of the lane (vb = offset + pos), partial offset of the lane, 0}
// =============================================================================================
namespace {

constexpr int META_THREADS = 1024;
constexpr int META_MAX_VB = 2048;

__device__ int block_excl_scan(int v, int* warp_tot, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < (int)(blockDim.x >> 5)) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    const int before = (warp > 0 ? warp_tot[warp - 1] : 0) + x - v;
    if (total) *total = warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

// exclusive prefix over n values held in a[0..n); writes prefix to out[0..n], out[n] = total
__device__ void block_scan_array(const int* a, int* out, int n, int* warp_tot) {
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(n, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += a[i];
    int total;
    int run = block_excl_scan(s, warp_tot, &total);
    for (int i = lo; i < hi; ++i) {
        out[i] = run;
        run += a[i];
    }
    if (threadIdx.x == 0) out[n] = total;
    __syncthreads();
}

__global__ void __launch_bounds__(META_THREADS, 1)
    etap_mla_metadata_kernel(const int32_t* __restrict__ seqlens, int batch, int groups,
                             int num_parts, int lanes_on, int32_t* __restrict__ sched,
                             int32_t* __restrict__ split_off, int fixed_cost) {
    // seqlens may come from the kernel before this one, and the previous step's combine may
    // still read split_off: nothing is read or written before the grid dependency resolved
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    __shared__ int s_tiles[META_MAX_VB];
    __shared__ int s_pref[META_MAX_VB + 1];
    __shared__ int s_ns[META_MAX_VB];
    __shared__ int s_first[META_MAX_VB];
    __shared__ int s_soff[META_MAX_VB + 1];
    __shared__ int warp_tot[32];
    const LineShape ls = line_shape(batch, groups, num_parts, lanes_on != 0);
    const int n = ls.line_n;

    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int len = max(0, seqlens[i % batch]);
        s_tiles[i] = (len + TILE - 1) / TILE;
        s_ns[i] = s_tiles[i] > 0 ? s_tiles[i] + fixed_cost : 0;  // cost, reused below
        s_first[i] = 0x7fffffff;
    }
    __syncthreads();
    block_scan_array(s_ns, s_pref, n, warp_tot);
    const int total = s_pref[n];
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_ns[i] = 0;
    __syncthreads();

    const int T = max(1, (total + ls.p_line - 1) / ls.p_line);
    // map a cost coordinate x in [0, total) to (line index, tile)
    auto map = [&](int x, int& vb, int& t) {
        int lo = 0, hi = n - 1;  // largest index with s_pref <= x and nonzero cost
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= x) lo = mid; else hi = mid - 1;
        }
        // skip zero-cost sequences that share the same prefix value
        while (lo + 1 < n && s_pref[lo + 1] <= x) ++lo;
        vb = lo;
        t = min(max(0, x - s_pref[lo] - fixed_cost), s_tiles[lo]);
    };

    // line CTA kl's range [kl*T, (kl+1)*T) in (line index, tile) coordinates
    auto range = [&](int kl, int& b0, int& tb, int& b1, int& te) {
        const int x0 = kl * T, x1 = min(total, (kl + 1) * T);
        b0 = 0; tb = 0; b1 = -1; te = 0;
        if (x0 < total) {
            map(x0, b0, tb);
            if (x1 >= total) { b1 = n - 1; te = s_tiles[n - 1]; }
            else map(x1, b1, te);
        }
    };
    for (int kk = threadIdx.x; kk < ls.p_line; kk += blockDim.x) {
        int b0, tb, b1, te;
        range(kk, b0, tb, b1, te);
        {
            for (int vb = b0; vb <= b1; ++vb) {
                const int t0 = vb == b0 ? tb : 0;
                const int t1 = vb == b1 ? te : s_tiles[vb];
                if (t0 < t1) {
                    atomicAdd(&s_ns[vb], 1);
                    atomicMin(&s_first[vb], kk);
                }
            }
        }
    }
    __syncthreads();
    block_scan_array(s_ns, s_soff, n, warp_tot);  // split offsets along the line
    const int ns_line = s_soff[n];
    // split_off over all batch * groups virtual sequences: lane-major copies of the line's
    for (int v = threadIdx.x; v <= batch * groups; v += blockDim.x) {
        const int lane = v / n, i = v - lane * n;
        split_off[v] = lane * ns_line + s_soff[i];
    }
    for (int kk = threadIdx.x; kk < num_parts; kk += blockDim.x) {
        const int lane = kk / ls.p_line, kl = kk - lane * ls.p_line;
        int b0 = 0, tb = 0, b1 = -1, te = 0;  // CTAs past the last lane idle
        if (lane < ls.lanes) range(kl, b0, tb, b1, te);
        int first_idx = 0;
        if (b1 >= b0 && b0 < n) first_idx = lane * ns_line + s_soff[b0] + (kl - min(s_first[b0], kl));
        int32_t* s = sched + kk * SCHED_INTS;
        s[0] = b0; s[1] = tb; s[2] = b1; s[3] = te; s[4] = first_idx;
        s[5] = min(lane, ls.lanes - 1) * n; s[6] = min(lane, ls.lanes - 1) * ns_line; s[7] = 0;
    }
}

// =============================================================================================
// K2: the transposed pipeline. One persistent CTA per SM, 192 threads:
//   warp 0      TMA producer (paged latent-KV chunks into the ring, Q per split)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  softmax (thread = KV row = TMEM lane) and epilogue (thread = d row of O^T)
// =============================================================================================
__device__ __forceinline__ bool tracer_exit(int warp, int lane) { return warp == SOFTMAX_WARP0 && lane == 0; }

struct SplitDesc {
    int vb, b, g, seqlen, t0, t1;
};

// exclusive prefix over the 256 threads of the CTA (one value per thread)
__device__ __forceinline__ int cta_excl_scan256(int v, int* s_wt, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wt[warp] = x;
    __syncthreads();
    int pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
        const int t = s_wt[w];
        pre += (w < warp) ? t : 0;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return pre + x - v;
}

// The split schedule of etap_mla_metadata_kernel (K1) computed by every CTA for itself:
// cost prefix along the line -> closed-form split counts per line entry (line CTA k covers i
// iff (k+1)T > P[i]+F and kT < P[i+1]) -> split offsets -> this CTA's range. Identical output
// to K1 (GPU test); CTA 0 publishes split_off for the combine kernel, every CTA its sched row.
__device__ void schedule_own_range(const DecodeParams& prm, const LineShape& ls, const int* s_pref,
                                   const int* s_soff, const int* s_len, int* s_sched, int total, int T,
                                   bool publish) {
    const int n = ls.line_n;
    const int part = sched_part(prm);
    const int lane = part / ls.p_line, k = part - lane * ls.p_line;
    auto map = [&](int x, int& vb, int& t) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= x) lo = mid; else hi = mid - 1;
        }
        while (lo + 1 < n && s_pref[lo + 1] <= x) ++lo;
        vb = lo;
        t = min(max(0, x - s_pref[lo] - prm.fixed_cost), (s_len[lo] + TILE - 1) / TILE);
    };
    const int x0 = k * T, x1 = min(total, (k + 1) * T);
    int b0 = 0, tb = 0, b1 = -1, te = 0, first = 0;
    if (lane < ls.lanes && x0 < total) {
        map(x0, b0, tb);
        if (x1 >= total) { b1 = n - 1; te = (s_len[n - 1] + TILE - 1) / TILE; }
        else map(x1, b1, te);
        if (b1 >= b0) first = lane * s_soff[n] + s_soff[b0] + (k - (s_pref[b0] + prm.fixed_cost) / T);
    }
    s_sched[0] = b0; s_sched[1] = tb; s_sched[2] = b1; s_sched[3] = te; s_sched[4] = first;
    s_sched[5] = min(lane, ls.lanes - 1) * n;         // virtual-sequence offset of the lane
    s_sched[6] = min(lane, ls.lanes - 1) * s_soff[n];  // partial-index offset of the lane
    s_sched[7] = 0;
    if (!publish) return;
    int32_t* g = prm.sched_out + sched_part(prm) * SCHED_INTS;
    for (int i = 0; i < SCHED_INTS; ++i) g[i] = s_sched[i];
}

// split_off over all batch * groups virtual sequences (lane-major copies of the line's)
__device__ __forceinline__ void publish_split_off(const DecodeParams& prm, const LineShape& ls,
                                                  const int* s_soff, int tid, int nthreads) {
    const int n = ls.line_n, nv = prm.batch * prm.groups;
    for (int v = tid; v <= nv; v += nthreads) {
        const int lane = v / n, i = v - lane * n;
        prm.split_off_out[v] = lane * s_soff[n] + s_soff[i];
    }
}

// Warp-level variant for lines of up to 32 entries, run by warp 0 only: everything stays in
// registers (lane i = line entry i), the two range lookups are ballots instead of binary
// searches, so the producer can issue its first loads a few hundred cycles earlier.
// Same output as schedule_own_range / K1 (GPU test).
__device__ void inkernel_schedule_warp(const DecodeParams& prm, const LineShape& ls, int* s_soff,
                                       int* s_len, int* s_sched, bool publish) {
    const int n = ls.line_n;
    const int lane = threadIdx.x & 31;
    const bool live = lane < n;
    const int len = live ? max(0, prm.seqlens[lane % prm.batch]) : 0;
    const int tiles = (len + TILE - 1) / TILE;
    const int cost = tiles > 0 ? tiles + prm.fixed_cost : 0;
    int incl = cost;  // inclusive prefix = P[lane + 1]
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0) { ETAP_TRACE_G(prm, 8); ETAP_TRACE_CLK(prm, 13); }
    const int pref = incl - cost;
    const int T = max(1, (total + ls.p_line - 1) / ls.p_line);
    const int ns = (live && tiles > 0) ? ((incl + T - 1) / T - 1) - (pref + prm.fixed_cost) / T + 1 : 0;
    int so = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, so, o);
        if (lane >= o) so += y;
    }
    const int soff = so - ns;
    const int ns_line = __shfl_sync(0xffffffffu, so, 31);
    // this CTA's cost interval [x0, x1) -> (entry, tile) at both ends: the largest live entry
    // whose prefix is <= x (zero-cost entries sharing the prefix resolve to the last one)
    const int part = sched_part(prm);
    const int cl = part / ls.p_line, k = part - cl * ls.p_line;
    const int x0 = k * T, x1 = min(total, (k + 1) * T);
    const int b0 = 31 - __clz(__ballot_sync(0xffffffffu, live && pref <= x0) | 1u);
    const int b1m = 31 - __clz(__ballot_sync(0xffffffffu, live && pref <= x1) | 1u);
    const int p0 = __shfl_sync(0xffffffffu, pref, b0), t0n = __shfl_sync(0xffffffffu, tiles, b0);
    const int so0 = __shfl_sync(0xffffffffu, soff, b0);
    const int p1 = __shfl_sync(0xffffffffu, pref, b1m), t1n = __shfl_sync(0xffffffffu, tiles, b1m);
    const int tiles_last = __shfl_sync(0xffffffffu, tiles, max(0, n - 1));
    if (lane == 0) {
        int sb0 = 0, stb = 0, sb1 = -1, ste = 0, first = 0;
        if (cl < ls.lanes && x0 < total) {
            sb0 = b0;
            stb = min(max(0, x0 - p0 - prm.fixed_cost), t0n);
            if (x1 >= total) { sb1 = n - 1; ste = tiles_last; }
            else { sb1 = b1m; ste = min(max(0, x1 - p1 - prm.fixed_cost), t1n); }
            if (sb1 >= sb0) first = cl * ns_line + so0 + (k - (p0 + prm.fixed_cost) / T);
        }
        const int lc = min(cl, ls.lanes - 1);
        s_sched[0] = sb0; s_sched[1] = stb; s_sched[2] = sb1; s_sched[3] = ste; s_sched[4] = first;
        s_sched[5] = lc * n;         // virtual-sequence offset of the lane
        s_sched[6] = lc * ns_line;   // partial-index offset of the lane
        s_sched[7] = 0;
    }
    if (live) {
        s_len[lane] = len;
        s_soff[lane] = soff;
    }
    if (lane == 31) s_soff[n] = so;
    __syncwarp();
    // published for the combine kernel and external readers (not read back by this CTA)
    if (!publish) return;
    if (lane < SCHED_INTS) prm.sched_out[sched_part(prm) * SCHED_INTS + lane] = s_sched[lane];
    if (sched_part(prm) == 0) publish_split_off(prm, ls, s_soff, lane, 32);
}

// The schedule computed before the grid dependency (DecodeParams::early_meta) is published
// only after it: the previous step's combine may still read split_off until then.
__device__ __forceinline__ void publish_schedule(const DecodeParams& prm, const LineShape& ls, const int* s_soff,
                                                 const int* s_sched, int tid, int nthreads) {
    if (tid < SCHED_INTS) prm.sched_out[sched_part(prm) * SCHED_INTS + tid] = s_sched[tid];
    if (sched_part(prm) == 0) publish_split_off(prm, ls, s_soff, tid, nthreads);
}

__device__ void inkernel_schedule(const DecodeParams& prm, const LineShape& ls, int* s_pref, int* s_soff,
                                  int* s_len, int* s_sched, int* s_wt, bool publish) {
    const int n = ls.line_n;
    const int tid = threadIdx.x;
    int tiles = 0, cost = 0;
    if (tid < n) {
        const int len = max(0, prm.seqlens[tid % prm.batch]);
        tiles = (len + TILE - 1) / TILE;
        cost = tiles > 0 ? tiles + prm.fixed_cost : 0;
        s_len[tid] = len;
    }
    int total;
    const int pref = cta_excl_scan256(cost, s_wt, total);
    if (tid < n) s_pref[tid] = pref;
    if (tid == 0) s_pref[n] = total;
    __syncthreads();
    const int T = max(1, (total + ls.p_line - 1) / ls.p_line);
    int ns = 0;
    if (tid < n && tiles > 0) {
        const int kf = (pref + prm.fixed_cost) / T;
        const int kl = (s_pref[tid + 1] + T - 1) / T - 1;
        ns = kl - kf + 1;
    }
    int nsplits;
    const int so = cta_excl_scan256(ns, s_wt, nsplits);
    if (tid < n) s_soff[tid] = so;
    if (tid == 0) s_soff[n] = nsplits;
    __syncthreads();
    if (tid == 0) schedule_own_range(prm, ls, s_pref, s_soff, s_len, s_sched, total, T, publish);
    if (publish && sched_part(prm) == 0) publish_split_off(prm, ls, s_soff, tid, blockDim.x);
    __syncthreads();
}

// L2 prefetch depth before the grid dependency, in bytes of KV: 2 bf16 pages = 4 FP8 pages
// (measured best for each kernel; deeper prefetch competes with the previous step's tail)
#ifndef ETAP_HG64_PF_AHEAD
#define ETAP_HG64_PF_AHEAD 0  // L2 prefetch of the next tile's page: measured slower (pf1 290.0 vs 281.9 us at 64 heads)
#endif
#ifndef ETAP_TMA_ELECT
#define ETAP_TMA_ELECT 1  // the producer issues a landing group's boxes warp-uniformly (A/B: 0)
#endif
#ifndef ETAP_HINT_PAGES
#define ETAP_HINT_PAGES 1  // the producer takes its first page ids from the prologue's hint (A/B: 0)
#endif
#ifndef ETAP_HINT_BYTES
#define ETAP_HINT_BYTES (2 * 64 * 576 * 2)
#endif
// Before the grid dependency (while the previous kernel finishes): warm L2 with the first pages
// this CTA will most likely stream, guessed from its own range of the previous decode call (the
// fused schedule republishes it every call; a decode step moves it only when a sequence crosses
// a page), and return that guess (b, first tile). Hints only: every byte used is loaded after
// the grid dependency, and a wrong or stale guess merely wastes a prefetch. Whole warp.
__device__ __forceinline__ void prev_range_hint(const DecodeParams& prm, int hg, uint32_t page_bytes, bool q_rows,
                                                int lane, int& hint_b, int& hint_t0, int* s_hint = nullptr) {
#ifndef ETAP_NO_PREFETCH_HINT
    if (!prm.inkernel_sched) return;
    // one dependent load (the previous range), then the page ids on parallel lanes: the
    // schedule's __syncthreads waits for this warp, so no serial chain of block_table reads
    const int32_t* prev = prm.sched_out + sched_part(prm) * SCHED_INTS;
    int p0 = 0, tb = -1, p1 = -1, off = -1;
    if (lane == 0) { p0 = prev[0]; tb = prev[1]; p1 = prev[2]; off = prev[5]; }
    p0 = __shfl_sync(0xffffffffu, p0, 0);
    tb = __shfl_sync(0xffffffffu, tb, 0);
    p1 = __shfl_sync(0xffffffffu, p1, 0);
    off = __shfl_sync(0xffffffffu, off, 0);
    const int vb = off + p0, nvb = prm.batch * prm.groups;
    if (s_hint != nullptr && lane == 0) s_hint[0] = -1;
    if (p1 >= p0 && p0 >= 0 && vb >= 0 && vb < nvb && tb >= 0 && tb < prm.max_pages) {
        const int g = vb / prm.batch, b = vb - g * prm.batch;
        hint_b = b;
        hint_t0 = tb;
        const int32_t* bt = prm.block_table + static_cast<size_t>(b) * prm.max_pages;
        const int page = (s_hint != nullptr || lane < static_cast<int>(ETAP_HINT_BYTES / page_bytes)) &&
                                 tb + lane < prm.max_pages
                             ? bt[tb + lane]
                             : 0;
        if (lane < static_cast<int>(ETAP_HINT_BYTES / page_bytes) && page >= 0 && page < prm.num_pages)
            ptx::bulk_prefetch_l2(static_cast<const uint8_t*>(prm.kv_pool) + static_cast<size_t>(page) * page_bytes,
                                  page_bytes);
        if (s_hint != nullptr) {
            // the 32 page ids from (b, tb) for the producer: its first TMA needs no block_table
            // read of its own when this call's range starts where the previous one did
            s_hint[2 + lane] = page;
            if (lane == 0) { s_hint[0] = b; s_hint[1] = tb; }
        }
        if (q_rows && lane == 0)
            ptx::bulk_prefetch_l2(static_cast<const uint8_t*>(prm.q) +
                                      (static_cast<size_t>(b) * prm.heads + g * hg) * D_QK * 2,
                                  hg * D_QK * 2);
    }
#endif
}

// Split i of the CTA's range along the line: virtual sequence vb = lane_off + i (head-group
// major: b = vb % batch, g = vb / batch) and the tile interval this CTA owns of it.
__device__ __forceinline__ bool split_at(const int32_t* sch, int seqlen, int batch, int i,
                                         SplitDesc& d) {
    d.vb = sch[5] + i;
    d.g = d.vb / batch;
    d.b = d.vb - d.g * batch;
    d.seqlen = seqlen;
    const int n_tiles = (d.seqlen + TILE - 1) / TILE;
    d.t0 = (i == sch[0]) ? sch[1] : 0;
    d.t1 = (i == sch[2]) ? min(sch[3], n_tiles) : n_tiles;
    return d.t0 < d.t1;
}

// Split schedule and the producer's first page ids, around the grid dependency (all threads).
// With early_meta (opt-in, ETAP_FLAG_EARLY_METADATA) seqlens and block_table are read BEFORE
// griddepcontrol.wait: the caller guarantees that the kernel immediately before the decode in
// the stream does not write them (this library's decode / combine kernels do not; host copies
// are ordered anyway). By default both are read after the wait. The dependency then gates only
// the KV / Q loads and every global write: the schedule is published after it (the previous
// step's combine may still read split_off), and the producer's first TMA goes out right after
// it with its page ids already in registers. Without early_meta the previous call's range
// serves as an L2 prefetch guess and the schedule is computed after the dependency.
struct Prologue {
    const int32_t* sch;
    const int32_t* soff;
    const int* s_len;
    int idx_off;
    int hint_b, hint_t0, hint_pg;  // (b, first tile) of the producer's first split, its first 32 page ids
    bool late_wait;                // warp 0 has not waited for the grid dependency yet
};

// The producer's grid-dependency wait when decode_prologue deferred it (whole warp 0).
// Kernel span (bench roofline timing without breaking programmatic launch): when prm.span is
// set, thread 0 of every CTA records %globaltimer when its grid dependency resolved (the first
// moment it may touch KV) and at exit: span[cta][0..1]. Two stores per CTA outside every loop.
__device__ __forceinline__ void span_stamp(const DecodeParams& prm, int slot) {
    if (prm.span != nullptr) prm.span[blockIdx.x * 2 + slot] = ptx::global_timer_ns();
}

template <bool kDebug>
__device__ __forceinline__ void dep_wait_producer(const DecodeParams& prm) {
    if (!prm.defer_dep) {
        ptx::grid_dep_wait();
        ptx::grid_dep_launch();
    }
    // (deferred dependency: the first moment the kernel touches KV is its first TMA)
    if (threadIdx.x == 0) { span_stamp(prm, 0); ETAP_TRACE_G(prm, 7); ETAP_TRACE_CLK(prm, 12); }
}

// Before a warp's first global write under a deferred grid dependency (ETAP_FLAG_INDEPENDENT_
// INPUTS): the kernel before this one (the previous step's combine) may still read the split
// partials / split_off this kernel is about to write. Immediate once the dependency resolved.
__device__ __forceinline__ void dep_wait_before_write(const DecodeParams& prm) {
    if (prm.defer_dep) ptx::grid_dep_wait();
}

// defer_publish: under the early schedule the kernel publishes this CTA's schedule itself, later,
// with publish_after_prologue (warp 3 waits for the grid dependency first; a kernel whose
// prologue holds warp 3 in a named barrier with others must not let that wait stall them)
template <bool kDebug, int MAXVB>
__device__ __forceinline__ Prologue decode_prologue(const DecodeParams& prm, uint8_t* sched_smem, int hg,
                                                    uint32_t page_bytes, bool q_rows, int warp, int lane,
                                                    bool defer_publish = false) {
    int* s_pref = reinterpret_cast<int*>(sched_smem);
    int* s_soff = s_pref + MAXVB + 1;
    int* s_len = s_soff + MAXVB + 1;
    int* s_sched = s_len + MAXVB;
    const bool fused = prm.inkernel_sched != 0;
    const bool early = fused && prm.early_meta != 0;
    Prologue r{};
    r.s_len = s_len;
    r.hint_b = -1;
    LineShape ls{};
    if (fused) ls = line_shape(prm.batch, prm.groups, sched_parts(prm), prm.lanes_on != 0);
    auto schedule = [&](bool publish) {
        if (ls.line_n <= 32) {
            if (warp == 0) inkernel_schedule_warp(prm, ls, s_soff, s_len, s_sched, publish);
            __syncthreads();
        } else {
            inkernel_schedule(prm, ls, s_pref, s_soff, s_len, s_sched, s_sched + 8, publish);
        }
    };
    if (early) {
        // warp 2 (idle until the first tile) warms L2 with the previous call's first pages while
        // warp 0 computes this call's schedule (matters when nothing overlaps the prologue,
        // e.g. the first node of a CUDA graph replay)
        // (line <= 32 entries: the warp schedule leaves s_pref unused, and warp 2 leaves there the
        // page ids it read, s_hint = {b, t0, 32 ids})
#ifdef ETAP_NO_PREFETCH_HINT
        int* s_hint = nullptr;
#else
        int* s_hint = (ls.line_n <= 32 && ETAP_HINT_PAGES) ? s_pref : nullptr;
#endif
        if (warp == 2) {
            int gb = -1, gt0 = 0;
            prev_range_hint(prm, hg, page_bytes, q_rows, lane, gb, gt0, s_hint);
            if (lane == 0) ETAP_TRACE_PRO(prm, 0);
        }
        schedule(false);
        if (warp == 0 && lane == 0) ETAP_TRACE_PRO(prm, 1);
        if (warp == 0) {
            for (int vb = s_sched[0]; vb <= s_sched[2]; ++vb) {
                SplitDesc sd;
                if (!split_at(s_sched, s_len[vb], prm.batch, vb, sd)) continue;
                r.hint_b = sd.b;
                r.hint_t0 = sd.t0;
                if (s_hint != nullptr && s_hint[0] == sd.b && s_hint[1] == sd.t0) {
                    // the previous call's range starts here too: warp 2 read these page ids from
                    // this call's block_table and prefetched the first pages and Q already
                    r.hint_pg = (sd.t0 + lane < sd.t1) ? s_hint[2 + lane] : 0;
                    break;
                }
                r.hint_pg = (sd.t0 + lane < sd.t1) ? __ldg(prm.block_table + static_cast<size_t>(sd.b) * prm.max_pages +
                                                           sd.t0 + lane) : 0;
#ifndef ETAP_NO_PREFETCH_HINT
                // L2 warm-up only: the bytes used are loaded by TMA after the dependency
                if (lane < static_cast<int>(ETAP_HINT_BYTES / page_bytes) && sd.t0 + lane < sd.t1 && r.hint_pg >= 0 &&
                    r.hint_pg < prm.num_pages)
                    ptx::bulk_prefetch_l2(static_cast<const uint8_t*>(prm.kv_pool) +
                                              static_cast<size_t>(r.hint_pg) * page_bytes, page_bytes);
                if (q_rows && lane == 0)
                    ptx::bulk_prefetch_l2(static_cast<const uint8_t*>(prm.q) +
                                              (static_cast<size_t>(sd.b) * prm.heads + sd.g * hg) * D_QK * 2,
                                          hg * D_QK * 2);
#endif
                break;
            }
            if (kDebug && prm.trace != nullptr) {  // page ids in registers (waits for their load)
                const int pg0 = __shfl_sync(0xffffffffu, r.hint_pg, 0);
                if (lane == 0 && pg0 != (-2147483647 - 1)) ETAP_TRACE_PRO(prm, 2);
            }
        }
    } else if (warp == 0) {
        prev_range_hint(prm, hg, page_bytes, q_rows, lane, r.hint_b, r.hint_t0);
    }
    // With early_meta the producer warp (warp 0) has nothing left to do before its first TMA:
    // it waits for the dependency itself, right before issuing it (dep_wait_producer), with
    // the issue path already fetched and its page ids in registers.
    r.late_wait = early;
    if (early && prm.defer_dep) {
        // ETAP_FLAG_INDEPENDENT_INPUTS: the caller guarantees that the kernel before this one
        // writes none of the inputs, so the loads need not wait for it; every global write does
        // (dep_wait_before_write). The combine may be scheduled right away.
        ptx::grid_dep_launch();
    } else if (!(early && warp == 0)) {
        ptx::grid_dep_wait();     // KV / Q and the outputs of earlier kernels in the stream
        ptx::grid_dep_launch();   // let the combine kernel get scheduled
    }
    if (!early) {
        // the first page ids for the guessed range go out together with the seqlens loads of
        // the schedule (used only if the schedule confirms the guess)
        if (warp == 0 && r.hint_b >= 0 && r.hint_t0 + lane < prm.max_pages)
            r.hint_pg = prm.block_table[static_cast<size_t>(r.hint_b) * prm.max_pages + r.hint_t0 + lane];
    }
    if (threadIdx.x == 0 && !early) { span_stamp(prm, 0); ETAP_TRACE_G(prm, 7); ETAP_TRACE_CLK(prm, 12); }
    if (fused) {
        if (early) {
            if (warp == 3 && sched_publisher(prm) && !defer_publish) {
                dep_wait_before_write(prm);  // the previous step's combine may still read split_off
                publish_schedule(prm, ls, s_soff, s_sched, lane, 32);
            }
        } else {
            schedule(sched_publisher(prm));
        }
        r.sch = s_sched;
        r.soff = s_soff;  // line-local split offsets
        r.idx_off = s_sched[6];
    } else {
        r.sch = prm.sched + sched_part(prm) * SCHED_INTS;
        r.soff = prm.split_off + r.sch[5];  // indexed by line position like the fused copy
        r.idx_off = 0;
    }
    if (threadIdx.x == 0) { ETAP_TRACE_G(prm, 1); ETAP_TRACE_CLK(prm, 14); }
    return r;
}

// The early schedule's publish that decode_prologue(defer_publish = true) left out (warp 3).
__device__ __forceinline__ void publish_after_prologue(const DecodeParams& prm, const Prologue& pro, int lane) {
    if (prm.inkernel_sched != 0 && prm.early_meta != 0 && sched_publisher(prm)) {
        dep_wait_before_write(prm);  // the previous step's combine may still read split_off
        const LineShape ls = line_shape(prm.batch, prm.groups, sched_parts(prm), prm.lanes_on != 0);
        publish_schedule(prm, ls, pro.soff, pro.sch, lane, 32);
    }
}

// A softmax warpgroup's wait on an mbarrier: one warp polls it, the other three block on the
// warpgroup's named barrier (no issue slots while blocked), so four warps instead of sixteen
// re-issue the try_wait loop next to the softmax arithmetic. The named barrier is the thread
// synchronisation after which every warp's tcgen05.fence::after_thread_sync orders its TMEM /
// smem reads behind the observed phase.
#ifndef ETAP_WG_POLL
#define ETAP_WG_POLL 1
#endif
__device__ __forceinline__ void wg_wait(uint64_t* bar, uint32_t parity, uint32_t wg_bar, int wq) {
#if ETAP_WG_POLL
    if (wq == 0) ptx::mbar_wait(bar, parity);
    ptx::named_bar_sync(wg_bar, 128);
#else
    ptx::mbar_wait(bar, parity);
#endif
}

template <int HG_, bool DBG>
__global__ void __launch_bounds__(Cfg<HG_>::THREADS, 1)
    etap_mla_decode_kernel(const __grid_constant__ CUtensorMap tm_kv,
                           const __grid_constant__ CUtensorMap tm_q, const DecodeParams prm) {
    using C = Cfg<HG_>;
    constexpr bool kDebug = DBG;  // debug stamps / state dump (see etap_mla_kernels.cuh)
    constexpr int HG = C::HG, HH = C::HH;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    // no alignment slack allocated (P_LO_BUF): the dynamic smem base must already be 1024-aligned
    if constexpr (C::SMEM_ALLOC == C::SMEM_USED) {
        if (smem != smem_raw) asm volatile("trap;");
    }
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ETAP_TRACE_G(prm, 0);
        ETAP_TRACE_CLK(prm, 5);
        ETAP_TRACE_SMID(prm);
    }

    // ---- prologue (overlaps the previous kernel under programmatic dependent launch)
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_kv);
        ptx::prefetch_tmap(&tm_q);
        for (int i = 0; i < NTB; ++i) {
            ptx::mbar_init(&bars[BAR_FULL_A + i], 1);
            ptx::mbar_init(&bars[BAR_FULL_B + i], 1);
            ptx::mbar_init(&bars[BAR_FULL_C + i], 1);
            ptx::mbar_init(&bars[BAR_G2_DONE + i], 1);
            ptx::mbar_init(&bars[BAR_G2_HALF + i], 1);
            ptx::mbar_init(&bars[BAR_G2_3Q + i], 1);
            ptx::mbar_init(&bars[BAR_G2_Q1 + i], 1);
            ptx::mbar_init(&bars[BAR_G2_P1 + i], 1);
        }
        ptx::mbar_init(&bars[BAR_Q_FULL], 1);
        ptx::mbar_init(&bars[BAR_Q_EMPTY], 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&bars[BAR_S_FULL + i], 1);
            ptx::mbar_init(&bars[BAR_S_FREE + i], 128 * C::NWG);
            ptx::mbar_init(&bars[BAR_P_FULL + i], 128 * C::NWG);
            ptx::mbar_init(&bars[BAR_P2_FULL + i], 128 * C::NWG);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
    // (no ring zero-fill: every row a GEMM reads was written by a full-page TMA box of the
    // same tile; garbage rows past seqlen are zeroed by the softmax warps before GEMM2)
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // split schedule + the producer's first page ids, around the grid dependency
    const Prologue pro = decode_prologue<kDebug, C::MAX_VB>(prm, smem + C::OFF_SCHED, HG, PAGE * D_QK * 2, true, warp, lane);
    const int32_t* sch = pro.sch;
    const int32_t* soff = pro.soff;  // split offsets per virtual sequence
    const int idx_off = pro.idx_off; // partial-index offset of this CTA's lane (fused schedule)
    const int hint_b = pro.hint_b, hint_t0 = pro.hint_t0, hint_pg = pro.hint_pg;
    const bool fused = prm.inkernel_sched != 0;
    const int* s_len = pro.s_len;

    const int vb_begin = sch[0], vb_end = sch[2];  // line positions (vb = sch[5] + position)
    const int B = prm.batch;
    const uint32_t ring_addr = ptx::smem_u32(smem + C::OFF_RING);
    const uint32_t q_addr = ptx::smem_u32(smem + C::OFF_Q);
    const uint32_t p_addr = ptx::smem_u32(smem + C::OFF_P);
    auto seqlen_of = [&](int i) { return fused ? s_len[i] : max(0, prm.seqlens[(sch[5] + i) % B]); };

    if (warp == 0) {
        // ===================================================== TMA producer (whole warp)
        // Tile gt occupies ring positions [9gt, 9gt+9); positions [0, SPLIT_POS) reuse slots
        // of tile gt-3, the rest slots of tile gt-2: two waits on "GEMM2 done" per tile.
        // KV pages are streamed once per head group: with head-group lanes the other groups'
        // CTAs read the same page shortly after, so it stays evict-normal in L2
        const bool kv_shared = line_shape(B, prm.groups, gridDim.x, prm.lanes_on != 0).lanes > 1;
        const uint64_t pol_kv = kv_shared ? ptx::policy_evict_normal() : ptx::policy_evict_first();
        const uint64_t pol_q = ptx::policy_evict_last();
        uint32_t gt = 0, nsplit = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            // page ids of the split's first 32 tiles (one per lane) go out before anything else:
            // the first KV boxes wait on them, Q (usually L2-resident) is issued after those
            const int32_t* bt = prm.block_table + static_cast<size_t>(sd.b) * prm.max_pages;
            int base = sd.t0;
            int pg;
            if (nsplit == 0 && sd.b == hint_b && sd.t0 == hint_t0) pg = hint_pg;  // loaded already
            else pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
            bool q_pending = true;
            for (int t = sd.t0; t < sd.t1; ++t) {
                if (t - base >= 32) {  // page ids of the next 32 tiles, one per lane
                    base = t;
                    const int tt = base + lane;
                    pg = (tt < sd.t1) ? __ldg(bt + tt) : 0;
                }
                const int page = __shfl_sync(0xffffffffu, pg, t - base);
                const uint32_t tb = gt % NTB;
                const uint32_t pos0 = (gt * NCHUNK) % C::NSLOT;
                if (gt == 0 && pro.late_wait) dep_wait_producer<kDebug>(prm);
                // group A reuses slots of tile gt - A_LAG (all GEMM2 work of that tile done)
                constexpr uint32_t A_LAG = C::P_IN_ROPE ? 2 : 3;
                // two-tile ring (P_IN_ROPE): the page PF_AHEAD tiles ahead in this split is pulled
                // into L2 now, so its TMA load (issued only once GEMM2 two tiles back released
                // the slots) is an L2 hit instead of an HBM round trip on the tile chain
                int page_ahead = -1;
                if constexpr (C::P_IN_ROPE && ETAP_HG64_PF_AHEAD > 0) {
                    const int ta = t + ETAP_HG64_PF_AHEAD;
                    const int v = __shfl_sync(0xffffffffu, pg, min(ta - base, 31));
                    page_ahead = (ta < sd.t1 && ta - base < 32) ? v : -1;
                }
                if constexpr (C::P_LO_BUF) {  // V0-V1 of gt-2: free after its GEMM2 d-block 0
                    if (gt >= 2) ptx::mbar_wait(&bars[BAR_G2_Q1 + (gt - 2) % NTB], ((gt - 2) / NTB) & 1);
                } else if (gt >= A_LAG) {
                    ptx::mbar_wait(&bars[BAR_G2_DONE + (gt - A_LAG) % NTB], ((gt - A_LAG) / NTB) & 1);
                }
#if ETAP_TMA_ELECT
                // (the group's boxes are issued warp-uniformly: one elect inside each TMA)
                if (lane == 0) {
                    if (gt == 0) { ETAP_TRACE_G(prm, 9); ETAP_TRACE_CLK(prm, 15); }
                    ETAP_TRACE(prm, gt, 0);
                    ptx::mbar_arrive_expect_tx(&bars[BAR_FULL_A + tb], C::SPLIT_POS * SLOT_BYTES);
                }
                __syncwarp();
#pragma unroll
                for (int pos = 0; pos < C::SPLIT_POS; ++pos) {
                    uint32_t s = pos0 + item_pos<C>(pos, gt);
                    s = s >= C::NSLOT ? s - C::NSLOT : s;
                    ptx::tma_load_2d_elect(smem + C::OFF_RING + s * SLOT_BYTES, &tm_kv, &bars[BAR_FULL_A + tb],
                                           item_chunk<C>(pos, gt) * 64, page * PAGE, pol_kv);
                }
                if (lane == 0) {
#else
                if (lane == 0) {
                    if (gt == 0) { ETAP_TRACE_G(prm, 9); ETAP_TRACE_CLK(prm, 15); }
                    ETAP_TRACE(prm, gt, 0);
                    ptx::mbar_arrive_expect_tx(&bars[BAR_FULL_A + tb], C::SPLIT_POS * SLOT_BYTES);
#pragma unroll 1
                    for (int pos = 0; pos < C::SPLIT_POS; ++pos) {
                        const uint32_t s = (pos0 + item_pos<C>(pos, gt)) % C::NSLOT;
                        ptx::tma_load_2d(smem + C::OFF_RING + s * SLOT_BYTES, &tm_kv, &bars[BAR_FULL_A + tb],
                                         item_chunk<C>(pos, gt) * 64, page * PAGE, pol_kv);
                    }
#endif
                    if (page_ahead >= 0 && page_ahead < prm.num_pages)
                        ptx::bulk_prefetch_l2(static_cast<const uint8_t*>(prm.kv_pool) +
                                                  static_cast<size_t>(page_ahead) * PAGE * D_QK * 2,
                                              PAGE * D_QK * 2);
                }
                __syncwarp();
                if (q_pending) {
                    // Q of this split: its buffer is free once GEMM1 of the previous split's last
                    // tile completed
                    q_pending = false;
                    if (nsplit > 0) ptx::mbar_wait(&bars[BAR_Q_EMPTY], (nsplit - 1) & 1);
                    if (lane == 0) {
                        ptx::mbar_arrive_expect_tx(&bars[BAR_Q_FULL], C::Q_BYTES);
                        const int qrow = sd.b * prm.heads + sd.g * HG;
#pragma unroll 1
                        for (int c = 0; c < NCHUNK; ++c)
                            ptx::tma_load_2d(smem + C::OFF_Q + c * C::Q_CHUNK_BYTES, &tm_q, &bars[BAR_Q_FULL],
                                             c * 64, qrow, pol_q);
                    }
                    __syncwarp();
                    ++nsplit;
                }
                // positions [SPLIT_POS, SPLIT_POS2) reuse tile gt-2's first four positions: free
                // once GEMM2 d-blocks 0-1 of gt-2 completed (16-slot ring: tile gt-1's first two
                // positions, free once GEMM2 d-block 0 of gt-1 completed)
                // (P_LO_BUF: V2-V5 of gt-2, free after its GEMM2 d-blocks 0-2)
                if (!C::P_IN_ROPE && gt >= 2) ptx::mbar_wait(&bars[BAR_G2_HALF + (gt - 2) % NTB], ((gt - 2) / NTB) & 1);
                if (C::P_LO_BUF && gt >= 2) ptx::mbar_wait(&bars[BAR_G2_3Q + (gt - 2) % NTB], ((gt - 2) / NTB) & 1);
#if ETAP_TMA_ELECT
                if (lane == 0)
                    ptx::mbar_arrive_expect_tx(&bars[BAR_FULL_B + tb], (C::SPLIT_POS2 - C::SPLIT_POS) * SLOT_BYTES);
                __syncwarp();
#pragma unroll
                for (int pos = C::SPLIT_POS; pos < C::SPLIT_POS2; ++pos) {
                    uint32_t s = pos0 + item_pos<C>(pos, gt);
                    s = s >= C::NSLOT ? s - C::NSLOT : s;
                    ptx::tma_load_2d_elect(smem + C::OFF_RING + s * SLOT_BYTES, &tm_kv, &bars[BAR_FULL_B + tb],
                                           item_chunk<C>(pos, gt) * 64, page * PAGE, pol_kv);
                }
                if (lane == 0 && !C::THIRD_GROUP) ETAP_TRACE(prm, gt, 1);
#else
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(&bars[BAR_FULL_B + tb], (C::SPLIT_POS2 - C::SPLIT_POS) * SLOT_BYTES);
#pragma unroll 1
                    for (int pos = C::SPLIT_POS; pos < C::SPLIT_POS2; ++pos) {
                        const uint32_t s = (pos0 + item_pos<C>(pos, gt)) % C::NSLOT;
                        ptx::tma_load_2d(smem + C::OFF_RING + s * SLOT_BYTES, &tm_kv, &bars[BAR_FULL_B + tb],
                                         item_chunk<C>(pos, gt) * 64, page * PAGE, pol_kv);
                    }
                    if (!C::THIRD_GROUP) ETAP_TRACE(prm, gt, 1);
                }
#endif
                if constexpr (C::THIRD_GROUP) {
                    // the rest reuse gt-2's positions [4, 9 - SPLIT_POS): free after GEMM2 d-blocks
                    // 0-2 of gt-2 (22-slot ring) or the whole GEMM2
                    __syncwarp();
                    // (P_LO_BUF: V6, V7 and the rope slot, whose P_hi GEMM2 reads in every d-block,
                    // free after the whole GEMM2 of gt-2)
                    if (!C::P_IN_ROPE && gt >= 2)
                        ptx::mbar_wait(&bars[(C::G3_AFTER_3Q ? BAR_G2_3Q : BAR_G2_DONE) + (gt - 2) % NTB],
                                       ((gt - 2) / NTB) & 1);
                    if (C::P_LO_BUF && gt >= 2)
                        ptx::mbar_wait(&bars[BAR_G2_DONE + (gt - 2) % NTB], ((gt - 2) / NTB) & 1);
#if ETAP_TMA_ELECT
                    if (lane == 0)
                        ptx::mbar_arrive_expect_tx(&bars[BAR_FULL_C + tb], (NCHUNK - C::SPLIT_POS2) * SLOT_BYTES);
                    __syncwarp();
#pragma unroll
                    for (int pos = C::SPLIT_POS2; pos < NCHUNK; ++pos) {
                        uint32_t s = pos0 + item_pos<C>(pos, gt);
                        s = s >= C::NSLOT ? s - C::NSLOT : s;
                        ptx::tma_load_2d_elect(smem + C::OFF_RING + s * SLOT_BYTES, &tm_kv, &bars[BAR_FULL_C + tb],
                                               item_chunk<C>(pos, gt) * 64, page * PAGE, pol_kv);
                    }
                    if (lane == 0) ETAP_TRACE(prm, gt, 1);
#else
                    if (lane == 0) {
                        ptx::mbar_arrive_expect_tx(&bars[BAR_FULL_C + tb], (NCHUNK - C::SPLIT_POS2) * SLOT_BYTES);
#pragma unroll 1
                        for (int pos = C::SPLIT_POS2; pos < NCHUNK; ++pos) {
                            const uint32_t s = (pos0 + item_pos<C>(pos, gt)) % C::NSLOT;
                            ptx::tma_load_2d(smem + C::OFF_RING + s * SLOT_BYTES, &tm_kv, &bars[BAR_FULL_C + tb],
                                             item_chunk<C>(pos, gt) * 64, page * PAGE, pol_kv);
                        }
                        ETAP_TRACE(prm, gt, 1);
                    }
#endif
                }
                __syncwarp();
                ++gt;
            }
        }
        if (gt == 0 && pro.late_wait) dep_wait_producer<kDebug>(prm);  // no tiles in this CTA's range
    } else if (warp == 1) {
        // ===================================================== GEMM1 issuer (whole warp, elect)
        uint32_t gt = 0, nsplit = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            ptx::mbar_wait(&bars[BAR_Q_FULL], nsplit & 1);
            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gt & 1;
                const uint32_t s_tmem = tmem_base + C::TCOL_S + HG * buf;
                if (gt >= 2) ptx::mbar_wait(&bars[BAR_S_FREE + buf], ((gt >> 1) - 1) & 1);
                const uint32_t pos0 = (gt * NCHUNK) % C::NSLOT;
                ptx::mbar_wait(&bars[BAR_FULL_A + gt % NTB], (gt / NTB) & 1);
                __syncwarp();
                ptx::tc_fence_after();
                issue_gemm1_tile<C, 0, C::SPLIT_POS>(s_tmem, ring_addr, q_addr, pos0, gt);
                ptx::mbar_wait(&bars[BAR_FULL_B + gt % NTB], (gt / NTB) & 1);
                __syncwarp();
                ptx::tc_fence_after();
                if (!C::THIRD_GROUP) ETAP_TRACE(prm, gt, 2);
                issue_gemm1_tile<C, C::SPLIT_POS, C::SPLIT_POS2>(s_tmem, ring_addr, q_addr, pos0, gt);
                if constexpr (C::THIRD_GROUP) {
                    ptx::mbar_wait(&bars[BAR_FULL_C + gt % NTB], (gt / NTB) & 1);
                    __syncwarp();
                    ptx::tc_fence_after();
                    ETAP_TRACE(prm, gt, 2);
                    issue_gemm1_tile<C, C::SPLIT_POS2, NCHUNK>(s_tmem, ring_addr, q_addr, pos0, gt);
                }
                ptx::umma_commit_elect(&bars[BAR_S_FULL + buf]);
                ETAP_TRACE(prm, gt, 3);
                if (t == sd.t1 - 1) ptx::umma_commit_elect(&bars[BAR_Q_EMPTY]);
                ++gt;
            }
            ++nsplit;
        }
    } else if (warp == 2) {
        // ===================================================== GEMM2 issuer (whole warp, elect)
        uint32_t gt = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gt & 1;
                ptx::mbar_wait(&bars[BAR_P_FULL + buf], (gt >> 1) & 1);
                __syncwarp();
                ptx::tc_fence_after();
                ETAP_TRACE(prm, gt, 6);
                const uint32_t pos0 = (gt * NCHUNK) % C::NSLOT;
                if constexpr (C::P_LO_BUF) {
                    // per d-block: O^T += V^T P_hi^T (P_hi in the tile's rope slot) then
                    // O^T += V^T P_lo^T (the P_lo buffer), one accumulator; a commit after d-block 0
                    // and after d-block 2 releases V0-V1 / V2-V5 to the next tile of this ring half
                    const uint32_t pa = ring_addr + ((pos0 + pos_of_chunk(8, gt)) % C::NSLOT) * SLOT_BYTES;
#pragma unroll
                    for (int blk = 0; blk < 4; ++blk) {
                        uint32_t sa = pos0 + pos_of_chunk(2 * blk, gt);
                        sa = sa >= C::NSLOT ? sa - C::NSLOT : sa;
                        const uint32_t ot = tmem_base + C::TCOL_O + C::OBLK * blk;
                        issue_gemm2_block<C>(ot, ring_addr + sa * SLOT_BYTES, pa, t == sd.t0);
                        issue_gemm2_block<C>(ot, ring_addr + sa * SLOT_BYTES, p_addr, false);
                        if (blk == 0) ptx::umma_commit_elect(&bars[BAR_G2_Q1 + gt % NTB]);
                        if (blk == 2) ptx::umma_commit_elect(&bars[BAR_G2_3Q + gt % NTB]);
                    }
                } else if constexpr (C::P_IN_ROPE) {
                    // pass 1: O^T += V^T P_hi^T (P in the tile's rope slot), then the softmax
                    // replaces P_hi by P_lo in the same slot; pass 2: O^T += V^T P_lo^T
                    const uint32_t pa = ring_addr + ((pos0 + pos_of_chunk(8, gt)) % C::NSLOT) * SLOT_BYTES;
#pragma unroll
                    for (int pass = 0; pass < 2; ++pass) {
                        if (pass == 1) {
                            ptx::mbar_wait(&bars[BAR_P2_FULL + buf], (gt >> 1) & 1);
                            __syncwarp();
                            ptx::tc_fence_after();
                        }
#pragma unroll
                        for (int blk = 0; blk < 4; ++blk) {
                            uint32_t sa = pos0 + pos_of_chunk(2 * blk, gt);
                            sa = sa >= C::NSLOT ? sa - C::NSLOT : sa;
                            issue_gemm2_block<C>(tmem_base + C::TCOL_O + C::OBLK * blk, ring_addr + sa * SLOT_BYTES, pa,
                                                 pass == 0 && t == sd.t0);
                        }
                        if (pass == 0) ptx::umma_commit_elect(&bars[BAR_G2_P1 + gt % NTB]);
                    }
                } else {
#pragma unroll
                    for (int blk = 0; blk < 4; ++blk) {
                        uint32_t sa = pos0 + pos_of_chunk(2 * blk, gt);
                        sa = sa >= C::NSLOT ? sa - C::NSLOT : sa;
                        issue_gemm2_block<C>(tmem_base + C::TCOL_O + C::OBLK * blk, ring_addr + sa * SLOT_BYTES,
                                             p_addr + (buf % C::P_BUFS) * C::P_BYTES, t == sd.t0);
                        if (blk == 1) ptx::umma_commit_elect(&bars[BAR_G2_HALF + gt % NTB]);
                        if (C::G3_AFTER_3Q && C::THIRD_GROUP && blk == 2) ptx::umma_commit_elect(&bars[BAR_G2_3Q + gt % NTB]);
                    }
                }
                ptx::umma_commit_elect(&bars[BAR_G2_DONE + gt % NTB]);
                ETAP_TRACE(prm, gt, 7);
                ++gt;
            }
        }
    } else if (warp >= SOFTMAX_WARP0) {
        // ===================================================== softmax + epilogue (NWG x 128 threads)
        // warpgroup wg owns heads [hoff, hoff + HW); thread = (KV row, head half): lane l of
        // warp q owns row 16q + l%16, heads hoff + HH*(l/16)..; warpgroups synchronise only
        // among themselves (named barriers 1+2wg, 2+2wg)
        constexpr int HW = C::HW;
        const int wg = (warp - SOFTMAX_WARP0) >> 2;
        const int hoff = wg * HW;
        const uint32_t bar_a = 1 + 2 * wg, bar_b = 2 + 2 * wg;
        const int wq = warp & 3;               // TMEM lane quadrant accessible by this warp
        const int half = lane >> 4;
        const int row = s_row_of(wq, lane);    // KV row in the tile
        const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(wq * 32) << 16);
        float* red_max = reinterpret_cast<float*>(smem + C::OFF_RED);  // [RED_MAX_BUFS][4][HG]
        // [4][HG] column sums (epilogue; BlockHook dump): aliases red_max with P_LO_BUF (every use
        // lies between a vote and the next max exchange of the warpgroup's own heads)
        float* red_sum = C::P_LO_BUF ? red_max : red_max + 8 * HG;
        float* s_m = red_max + C::RED_MAX_BUFS * 4 * HG + (C::P_LO_BUF ? 0 : 4 * HG);  // [HG] running max (log2)
        float* s_alpha = s_m + HG;             // [HG] rescale factors of the current tile
        // [HG] output row of each head (epilogue): with P_LO_BUF in the warpgroup's own 256 B
        // column stripe of row group 0 of the P_lo buffer (idle from the split's last GEMM2 until
        // this warpgroup writes the next P_lo)
        int* s_row = C::P_LO_BUF ? reinterpret_cast<int*>(smem + C::OFF_P + wg * 256) - hoff
                                 : reinterpret_cast<int*>(s_alpha + HG);
        const bool negate = prm.flags & FLAG_NEGATE_RESCALE;
        const bool eager = negate || (prm.flags & FLAG_EAGER_RESCALE);
        const float thresh = eager ? 0.f : LAZY_RESCALE_LOG2;
        const bool tracer = (threadIdx.x == SOFTMAX_WARP0 * 32);
        const bool head_owner = wq == 0 && (lane & 15) == 0;  // writes s_m / s_alpha of its half
        const bool lane_head = wq == 0 && lane < HW;           // owner of head hoff + lane
        const bool mtp = prm.q_tokens > 1;
        const int rhead = halfwarp_reduce_head<HH>(lane);   // head (of the half) a reduction leaves here
        const bool rwriter = HH == 16 || (lane & 1) == 0;
        uint32_t gt = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            float m_own[HH];    // running max of this thread's heads (log2 units)
            // derived from m_own, refreshed only when it moves (the lazy-rescale branch), so the
            // per-tile path spends one compare and one subtraction per element on them:
            float m_thr[HH];    // m_own + thresh: the vote threshold
            float mu[HH];       // exp2 offset: m_own, or 0 while a causal column has seen no row
            float l_part[HH];   // partial column sums of this thread's rows, own heads
            float dbg_l = 0.f;  // debug state dump: running column sum of head `lane`
            int row_lim[HH];    // causal multi-token decode: rows visible to each column
            int row_all = sd.seqlen;  // rows below this are visible to every column of the thread
#pragma unroll
            for (int j = 0; j < HH; ++j) {
                m_own[j] = -INFINITY;
                m_thr[j] = -INFINITY;
                mu[j] = mtp ? 0.f : -INFINITY;
                l_part[j] = 0.f;
                const int tok = (sd.g * HG + hoff + half * HH + j) / prm.heads_per_token;
                row_lim[j] = sd.seqlen - (prm.causal ? prm.q_tokens - 1 - tok : 0);
                row_all = min(row_all, row_lim[j]);
                // a split whose first tile shows no row to any column skips the max exchange
                // (bar.red.or is false), so s_m must already read -inf for the epilogue
                // (the previous split's epilogue released s_m with its final barrier)
                if (head_owner) s_m[hoff + half * HH + j] = -INFINITY;
            }

            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gt & 1;
                wg_wait(&bars[BAR_S_FULL + buf], (gt >> 1) & 1, bar_a, wq);
                ptx::tc_fence_after();
                if (tracer) ETAP_TRACE(prm, gt, 4);
                uint32_t sr[HH];
                ptx::tmem_ld16x2<HH>(t_lane + C::TCOL_S + HG * buf + hoff, sr);
                ptx::tmem_wait_ld();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&bars[BAR_S_FREE + buf]);
                if (tracer) ETAP_TRACE(prm, gt, 12);  // (tile rows: slots 10-15 are the epilogue's on a split's last tile)

                const int grow = t * TILE + row;
                float x[HH];
                if (grow < row_all) {  // every row of a split but its last tile's tail
#pragma unroll
                    for (int j = 0; j < HH; ++j) x[j] = __uint_as_float(sr[j]) * prm.scale_log2;
                } else {
#pragma unroll
                    for (int j = 0; j < HH; ++j)
                        x[j] = grow < row_lim[j] ? __uint_as_float(sr[j]) * prm.scale_log2 : -INFINITY;
                }
                bool exceed = false;
#pragma unroll
                for (int j = 0; j < HH; ++j) exceed |= x[j] > m_thr[j];
                const bool first = (t == sd.t0);
                const bool debug = kDebug && prm.state != nullptr && t < prm.state_tiles;
                const float dbg_m_old = (debug && lane_head && !first) ? s_m[hoff + lane] : -INFINITY;
                // one barrier decides, CTA-uniformly, whether any running max must move
                const bool any = ptx::bar_red_or(bar_a, 128, exceed || (negate && !first));
                if (tracer) ETAP_TRACE(prm, gt, 13);
                bool need_rescale = false;
                float alpha_own[HH];
#pragma unroll
                for (int j = 0; j < HH; ++j) alpha_own[j] = first ? 0.f : 1.f;
                if (any) {
                    const float wm = halfwarp_reduce<true, HH>(x, lane);
                    float* rm = red_max + (C::RED_MAX_BUFS == 2 ? (gt & 1) : 0) * 4 * HG;
                    if (rwriter) rm[wq * HG + hoff + half * HH + rhead] = wm;
                    ptx::named_bar_sync(bar_b, 128);
                    bool upd = false;
#pragma unroll
                    for (int j = 0; j < HH; ++j) {
                        const int h = hoff + half * HH + j;
                        const float mt = fmaxf(fmaxf(rm[h], rm[HG + h]), fmaxf(rm[2 * HG + h], rm[3 * HG + h]));
                        if (first) {
                            m_own[j] = mt;
                        } else {
                            const float mn = fmaxf(m_own[j], mt);
                            if (mn > m_own[j] + thresh) {
                                alpha_own[j] = ptx::exp2_ftz(m_own[j] - mn);
                                m_own[j] = mn;
                                upd = true;
                            }
                        }
                    }
                    // CTA-uniform decision (also orders all reads of s_m before the writes below)
                    need_rescale = ptx::bar_red_or(bar_b, 128, upd) || (negate && !first);
                    if (head_owner) {
#pragma unroll
                        for (int j = 0; j < HH; ++j) {
                            s_m[hoff + half * HH + j] = m_own[j];
                            s_alpha[hoff + half * HH + j] = alpha_own[j];
                        }
                    }
#pragma unroll
                    for (int j = 0; j < HH; ++j) {
                        m_thr[j] = m_own[j] + thresh;
                        // a column may have no visible row yet (multi-token causal mask): m = -inf
                        mu[j] = (mtp && m_own[j] == -INFINITY) ? 0.f : m_own[j];
                    }
                }
                float pv[HH];
#pragma unroll
                for (int j = 0; j < HH; ++j) {
                    pv[j] = ptx::exp2_ftz(x[j] - mu[j]);
                    l_part[j] = fmaf(l_part[j], alpha_own[j], pv[j]);  // first tile: alpha = 0, l = 0
                }
                if (debug) {
                    // BlockHook replay: column sums of this tile's P, running l, m, rescale in
                    // natural-log units, as BlockStepInfo carries them (tiled_standard.hpp:32-40)
                    const float cs = halfwarp_reduce<false, HH>(pv, lane);
                    if (rwriter) red_sum[wq * HG + hoff + half * HH + rhead] = cs;
                    ptx::named_bar_sync(bar_b, 128);
                    if (lane_head) {
                        const int h = hoff + lane;
                        const float colsum = red_sum[h] + red_sum[HG + h] + red_sum[2 * HG + h] + red_sum[3 * HG + h];
                        const float mn = s_m[h];
                        const float al = first ? 0.f : (any ? s_alpha[h] : 1.f);
                        dbg_l = first ? colsum : fmaf(dbg_l, al, colsum);
                        float* st = prm.state + (static_cast<size_t>(sd.vb) * prm.state_tiles + t) * 4 * HG;
                        st[h] = dbg_m_old * 0.69314718055994530942f;
                        st[HG + h] = mn * 0.69314718055994530942f;
                        st[2 * HG + h] = al;
                        st[3 * HG + h] = dbg_l;
                    }
                    ptx::named_bar_sync(bar_b, 128);
                }
                if (tracer) ETAP_TRACE(prm, gt, 8);
                // head group 64: P_hi goes to the tile's own rope slot (free since GEMM1 of this tile
                // completed) before the wait for the P_lo buffer below
                uint32_t p_lo[HH / 2];  // two-pass GEMM2: written after pass 1
                uint8_t* p_rope = nullptr;
                if constexpr (C::P_IN_ROPE) {
                    uint32_t p_hi[HH / 2];
#pragma unroll
                    for (int i = 0; i < HH / 2; ++i) {
                        p_hi[i] = pack_bf16x2(pv[2 * i], pv[2 * i + 1]);
                        p_lo[i] = pack_bf16x2(pv[2 * i] - __uint_as_float(p_hi[i] << 16),
                                              pv[2 * i + 1] - __uint_as_float(p_hi[i] & 0xffff0000u));
                    }
                    const uint32_t pos0 = (gt * NCHUNK) % C::NSLOT;
                    p_rope = smem + C::OFF_RING + ((pos0 + pos_of_chunk(8, gt)) % C::NSLOT) * SLOT_BYTES;
                    write_p_part<C>(p_rope, row, half, p_hi, hoff);
                }
                // the P buffer is reused every P_BUFS tiles: GEMM2(gt - P_BUFS) must have read it
                if (C::P_BUFS > 0 && gt >= C::P_BUFS)
                    wg_wait(&bars[BAR_G2_DONE + (gt - C::P_BUFS) % NTB], ((gt - C::P_BUFS) / NTB) & 1, bar_a, wq);
                if (C::P_LO_BUF && gt >= 1)  // the P_lo buffer: GEMM2(gt - 1) must have read it
                    wg_wait(&bars[BAR_G2_DONE + (gt - 1) % NTB], ((gt - 1) / NTB) & 1, bar_a, wq);
                if (tracer) ETAP_TRACE(prm, gt, 9);
                if (need_rescale) {
                    // O^T must contain GEMM2(gt-1) before it is rescaled; s_alpha written above
                    ptx::named_bar_sync(bar_b, 128);
                    ptx::mbar_wait(&bars[BAR_G2_DONE + (gt - 1) % NTB], ((gt - 1) / NTB) & 1);
                    ptx::tc_fence_after();
                    // this warpgroup's heads: the hi columns [hoff, hoff+HW) and lo [HG+hoff, ...)
#pragma unroll 1
                    for (int blk = 0; blk < 4; ++blk) {
#pragma unroll
                        for (int seg = 0; seg < C::OSEG * (HW / 16); ++seg) {  // SAME_D: one accumulator
                            uint32_t o[16];
                            const int sub = seg % (HW / 16);
                            const uint32_t ta =
                                t_lane + C::TCOL_O + C::OBLK * blk + (seg / (HW / 16)) * HG + hoff + 16 * sub;
                            ptx::tmem_ld16(ta, o);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                const float a = s_alpha[hoff + 16 * sub + c];
                                o[c] = __float_as_uint(__uint_as_float(o[c]) * (negate ? -a : a));
                            }
                            ptx::tmem_st16(ta, o);
                        }
                    }
                    ptx::tmem_wait_st();
                }
                if constexpr (C::P_IN_ROPE) {
                    if constexpr (C::P_LO_BUF) write_p_part<C>(smem + C::OFF_P, row, half, p_lo, hoff);
                } else {
                    write_p_hilo<C>(smem + C::OFF_P + (buf % C::P_BUFS) * C::P_BYTES, row, half, pv, hoff);
                }
                // rows of the last page past seqlen were loaded from HBM and may hold
                // non-finite garbage; zero them in the V chunks (0 * NaN = NaN in the MMA)
                if (grow >= sd.seqlen) {
                    const uint32_t pos0 = (gt * NCHUNK) % C::NSLOT;
                    constexpr int ZC = 8 / (2 * C::NWG);  // V chunks zeroed per thread
#pragma unroll 1
                    for (int c = (wg * 2 + half) * ZC; c < (wg * 2 + half + 1) * ZC; ++c) {
                        const uint32_t s = (pos0 + pos_of_chunk(c, gt)) % C::NSLOT;
                        uint4* dst = reinterpret_cast<uint4*>(smem + C::OFF_RING + s * SLOT_BYTES + row * 128);
#pragma unroll
                        for (int j = 0; j < 8; ++j) dst[j] = make_uint4(0, 0, 0, 0);
                    }
                }
                ptx::fence_proxy_async_smem();
                ptx::tc_fence_before();
                if (tracer) ETAP_TRACE(prm, gt, 5);
                ptx::mbar_arrive(&bars[BAR_P_FULL + buf]);
                if constexpr (C::P_IN_ROPE && !C::P_LO_BUF) {
                    // P_lo replaces P_hi once GEMM2 pass 1 of this tile has read it
                    wg_wait(&bars[BAR_G2_P1 + gt % NTB], (gt / NTB) & 1, bar_a, wq);
                    ptx::tc_fence_after();
                    write_p_part<C>(p_rope, row, half, p_lo, hoff);
                    ptx::fence_proxy_async_smem();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bars[BAR_P2_FULL + buf]);
                }
                ++gt;
            }

            // ---- epilogue: wait for the last GEMM2, reduce l, O = (O^T_hi + O^T_lo) / l
            // (the single transpose of etap.cpp:140 is the TMEM lane -> d mapping),
            // L = m + log l (etap.cpp:144)
            const uint32_t last = gt - 1;
            dep_wait_before_write(prm);
            ptx::mbar_wait(&bars[BAR_G2_DONE + last % NTB], (last / NTB) & 1);
            ptx::tc_fence_after();
            if (tracer) ETAP_TRACE_G(prm, 10);
            // two d-blocks per TMEM load wait: this warpgroup's 16 hi + 16 lo columns each
            constexpr int BPW = 2;
            uint32_t o[BPW][C::OSEG * HW];  // SAME_D: the HW summed columns only
            const float wsum = halfwarp_reduce<false, HH>(l_part, lane);
            if (rwriter) red_sum[wq * HG + hoff + half * HH + rhead] = wsum;
            const int ns = soff[vb + 1] - soff[vb];
            const bool direct = ns == 1;  // one split: final O / L rows, else a split partial
            if (direct && lane_head) s_row[hoff + lane] = static_cast<int>(prm.om.row(sd.b, sd.g * HG + hoff + lane));
            if (tracer) ETAP_TRACE(prm, last, 10);
            ptx::named_bar_sync(bar_b, 128);
            if (tracer) ETAP_TRACE(prm, last, 11);
            // one owner thread per head finishes l, 1/l and L in parallel (a serial per-head loop
            // in every thread costs ~1.6k cycles); 1/l is broadcast through red_max, which no
            // one reads between tiles
            float L_own = 0.f;
            float* s_inv = C::P_LO_BUF ? s_alpha : red_max;  // (P_LO_BUF: red_max holds red_sum)
            if (lane_head) {
                const int h = hoff + lane;
                const float l = red_sum[h] + red_sum[HG + h] + red_sum[2 * HG + h] + red_sum[3 * HG + h];
                s_inv[h] = l > 0.f ? 1.f / l : 0.f;  // l = 0: column saw no row (O = 0, L = -inf)
                L_own = (s_m[h] + log2f(l)) * 0.69314718055994530942f;
            }
            ptx::named_bar_sync(bar_b, 128);
            float inv_l[HW];
#pragma unroll
            for (int h = 0; h < HW; h += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(s_inv + hoff + h);
                inv_l[h] = v4.x; inv_l[h + 1] = v4.y; inv_l[h + 2] = v4.z; inv_l[h + 3] = v4.w;
            }
            const int idx = (vb == sch[0]) ? sch[4] : soff[vb] + idx_off;  // partial index (ns > 1)
            float* part_o = prm.ws_o + static_cast<size_t>(idx) * HG * D_V;
            const int drow = wq * 32 + lane;  // M=128 layout: d row = TMEM lane
#pragma unroll 1
            for (int blk0 = 0; blk0 < 4; blk0 += BPW) {
#pragma unroll
                for (int bb = 0; bb < BPW; ++bb)
#pragma unroll
                    for (int seg = 0; seg < C::OSEG; ++seg)
#pragma unroll
                        for (int sub = 0; sub < HW / 16; ++sub)
                            ptx::tmem_ld16(t_lane + C::TCOL_O + C::OBLK * (blk0 + bb) + seg * HG + hoff + 16 * sub,
                                           *reinterpret_cast<uint32_t(*)[16]>(&o[bb][HW * seg + 16 * sub]));
                ptx::tmem_wait_ld();
                if (tracer && blk0 == 0) ETAP_TRACE(prm, last, 14);
#pragma unroll
                for (int bb = 0; bb < BPW; ++bb) {
                    const int d = (blk0 + bb) * 128 + drow;
                    float v[HW];
#pragma unroll
                    for (int h = 0; h < HW; ++h)
                        v[h] = (C::OSEG == 2 ? __uint_as_float(o[bb][h]) + __uint_as_float(o[bb][(C::OSEG - 1) * HW + h])
                                             : __uint_as_float(o[bb][h])) * inv_l[h];
                    if (direct) {
                        // every output copy (peer gather: each rank's buffer over NVLink)
#pragma unroll 1
                        for (int r = 0; r < prm.om.n_out; ++r) {
                            float* dst = prm.om.out[r] + d;
#pragma unroll
                            for (int h = 0; h < HW; ++h) dst[static_cast<size_t>(s_row[hoff + h]) * D_V] = v[h];
                        }
                    } else {
#pragma unroll
                        for (int h = 0; h < HW; ++h) part_o[(hoff + h) * D_V + d] = v[h];
                    }
                }
                if (tracer && blk0 == 0) ETAP_TRACE(prm, last, 15);
            }
            if (tracer) ETAP_TRACE(prm, last, 12);
            if (lane_head) {
                const float L = L_own;
                if (direct) {
                    for (int r = 0; r < prm.om.n_out; ++r) prm.om.lse[r][s_row[hoff + lane]] = L;
                } else {
                    prm.ws_lse[static_cast<size_t>(idx) * HG + hoff + lane] = L;
                }
            }
            ptx::tc_fence_before();
            // red_sum / s_m are rewritten by the next split only after this barrier
            ptx::named_bar_sync(bar_b, 128);
            if (tracer) ETAP_TRACE(prm, last, 13);
        }
    }

    if (tracer_exit(warp, lane)) ETAP_TRACE_G(prm, 11);
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        span_stamp(prm, 1);
        ETAP_TRACE_G(prm, 2);
        ETAP_TRACE_CLK(prm, 6);
        if (prm.trace != nullptr) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            prm.trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + TRACE_TILES - 1) * TRACE_SLOTS + 3] = smid;
        }
    }
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
    }
}

#include "etap_mla_pair.cuh"

// =============================================================================================
// K2-FP8: the transposed pipeline on an FP8 (e4m3) latent cache (etap_fp8.cuh for the operand
// layouts). Same roles, schedule, softmax and split partials as the bf16 kernel (HG = 16), but
//   * a tile is one 36 KB fp8 page in a ring of 5 page slots (5 pages in flight: the bytes per
//     page halve, the latency to hide does not), loaded by 4 SW128 boxes + 1 SW64 box;
//   * GEMM1 is 18 kind::f8f6f4 MMAs (K = 32) against three fp8 terms of Q (N = 48), GEMM2 is
//     8 MMAs per tile of V^T against three fp8 terms of P (N = 48), both straight from the
//     fp8 page: no dequantising pass; the KV scale folds into the softmax scale and 1/l.
// =============================================================================================
#ifndef ETAP_FP8_PAGE3D
#define ETAP_FP8_PAGE3D 1  // FP8 page = one 3-D box (V chunks) + the rope box; 0: five 2-D boxes (A/B)
#endif
// One FP8 page (64 rows x 576 B) into a ring slot: V chunks 0-3 as [chunk][row][128 B] SW128,
// the rope chunk as [row][64 B] SW64, all completing one mbarrier (lane 0 of the producer).
__device__ __forceinline__ void fp8_page_load(uint8_t* slot, const CUtensorMap* kv128, const CUtensorMap* kv64,
                                              uint64_t* full, int page, uint64_t pol) {
#if ETAP_FP8_PAGE3D
    ptx::tma_load_3d(slot, kv128, full, 0, page * PAGE, 0, pol);
#else
#pragma unroll 1
    for (int c = 0; c < fp8::VCH; ++c)
        ptx::tma_load_2d(slot + c * fp8::VCH_BYTES, kv128, full, c * 128, page * PAGE, pol);
#endif
    ptx::tma_load_2d(slot + fp8::ROPE_OFF, kv64, full, 512, page * PAGE, pol);
}

namespace kfp8 {
constexpr int NPS = 5;                               // page slots in the ring
constexpr int NTB8 = 8;                              // tile-barrier ring depth (>= NPS + 1)
constexpr int OFF_RING = 0;
constexpr int OFF_Q = NPS * fp8::TILE_BYTES;         // 180 KB
constexpr int OFF_P = OFF_Q + fp8::Q_BYTES;          // 2 buffers
constexpr int OFF_RED = OFF_P + 2 * fp8::P_BYTES;
constexpr int HG8 = fp8::HGF, HH8 = HG8 / 2;
constexpr int RED_FLOATS = 8 * HG8 + 4 * HG8 + 3 * HG8;
constexpr int BAR_FULL = 0;                          // [NTB8] page of tile gt landed
constexpr int BAR_G2D = NTB8;                        // [NTB8] GEMM2 of tile gt complete
constexpr int BAR_QF = 2 * NTB8, BAR_QE = 2 * NTB8 + 1;
constexpr int BAR_SF = 2 * NTB8 + 2, BAR_SR = 2 * NTB8 + 4, BAR_PF = 2 * NTB8 + 6;  // [2] each
constexpr int NSCR = 3;                              // per-CTA scratch slots: Q terms of later splits
constexpr int BAR_SCF = 2 * NTB8 + 8;                // [NSCR] slot written
constexpr int BAR_SCE = BAR_SCF + NSCR;              // [NSCR] slot read (its Q landed in smem)
constexpr int NBAR8 = BAR_SCE + NSCR;
constexpr int QPRO_THREADS = NUM_THREADS - 64;       // warps 2..7 quantise Q in the prologue
constexpr int QPRO_VEC = fp8::HGF * (D_QK / 8) / QPRO_THREADS;  // 16-byte vectors per thread per split
static_assert(fp8::HGF * (D_QK / 8) % QPRO_THREADS == 0, "prologue Q split");
constexpr int OFF_BAR = align_up(OFF_RED + RED_FLOATS * 4, 16);
constexpr int OFF_TMEM = OFF_BAR + NBAR8 * 8;
constexpr int OFF_SCHED = OFF_TMEM + 16;
constexpr int SMEM_USED = OFF_SCHED + sched_smem_ints(MAX_FUSED_VB) * 4;
constexpr int SMEM_ALLOC = SMEM_USED + 1024;
constexpr uint32_t TCOL_S = 0;                       // S^T: 2 buffers x 48 columns
constexpr uint32_t TCOL_O = 2 * fp8::NQ;             // O^T: 4 d-blocks x 48 columns
constexpr uint32_t TMEM_COLS = 512;
static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
static_assert(OFF_Q % 1024 == 0 && OFF_P % 1024 == 0, "alignment");
}  // namespace kfp8

// At most 176 registers (256 threads: 45056 of the SM's 65536): one 80-register combine CTA
// (256 threads) fits beside the decode CTA, so the next step's decode CTA takes each SM the
// moment this step's leaves it instead of waiting behind combine CTAs that hold the SM until
// the whole decode grid is done (DESIGN §3 "step overlap"; 0: the compiler's 241, A/B)
#ifndef ETAP_FP8_MAXNREG
#define ETAP_FP8_MAXNREG 176
#endif
#if ETAP_FP8_MAXNREG > 0
#define ETAP_FP8_BOUNDS __maxnreg__(ETAP_FP8_MAXNREG)
#else
#define ETAP_FP8_BOUNDS __launch_bounds__(NUM_THREADS, 1)
#endif
template <bool DBG>
__global__ void ETAP_FP8_BOUNDS
    etap_mla_decode_fp8_kernel(const __grid_constant__ CUtensorMap tm_kv128, const __grid_constant__ CUtensorMap tm_kv64,
                               const __grid_constant__ CUtensorMap tm_q128, const __grid_constant__ CUtensorMap tm_q64,
                               const DecodeParams prm, float kv_scale, uint8_t* __restrict__ q3s) {
    using namespace kfp8;
    constexpr bool kDebug = DBG;
    constexpr int HG = HG8, HH = HH8, NQ = fp8::NQ;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ETAP_TRACE_G(prm, 0);
        ETAP_TRACE_CLK(prm, 5);
        ETAP_TRACE_SMID(prm);
    }
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_kv128);
        ptx::prefetch_tmap(&tm_kv64);
        ptx::prefetch_tmap(&tm_q128);
        ptx::prefetch_tmap(&tm_q64);
        for (int i = 0; i < NTB8; ++i) {
            ptx::mbar_init(&bars[BAR_FULL + i], 1);
            ptx::mbar_init(&bars[BAR_G2D + i], 1);
        }
        ptx::mbar_init(&bars[BAR_QF], 1);
        ptx::mbar_init(&bars[BAR_QE], 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&bars[BAR_SF + i], 1);
            ptx::mbar_init(&bars[BAR_SR + i], 128);
            ptx::mbar_init(&bars[BAR_PF + i], 128);
        }
        for (int i = 0; i < NSCR; ++i) {
            ptx::mbar_init(&bars[BAR_SCF + i], 1);
            ptx::mbar_init(&bars[BAR_SCE + i], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // (the schedule publish waits for the grid dependency: warp 3 does it after the Q prologue,
    // whose named barrier it shares with warps 2 and 4-7, so the first split's Q terms do not
    // wait for the previous step's combine under a deferred dependency)
    const Prologue pro = decode_prologue<kDebug, MAX_FUSED_VB>(prm, smem + OFF_SCHED, HG, PAGE * D_QK, false, warp, lane,
                                                               true);
    const int32_t* sch = pro.sch;
    const int32_t* soff = pro.soff;
    const int idx_off = pro.idx_off;
    const int hint_b = pro.hint_b, hint_t0 = pro.hint_t0, hint_pg = pro.hint_pg;
    const bool fused = prm.inkernel_sched != 0;
    const int* s_len = pro.s_len;
    const int vb_begin = sch[0], vb_end = sch[2];
    const int B = prm.batch;
    const uint32_t ring_addr = ptx::smem_u32(smem + OFF_RING);
    const uint32_t q_addr = ptx::smem_u32(smem + OFF_Q);
    const uint32_t p_addr = ptx::smem_u32(smem + OFF_P);
    auto seqlen_of = [&](int i) { return fused ? s_len[i] : max(0, prm.seqlens[(sch[5] + i) % B]); };
    auto q_rows = [&](const SplitDesc& sd) {
        return static_cast<const uint4*>(prm.q) + (static_cast<size_t>(sd.b) * prm.heads + sd.g * HG) * (D_QK / 8);
    };
    auto scratch = [&](uint32_t slot_q) { return q3s + (static_cast<size_t>(blockIdx.x) * NSCR + slot_q) * NQ * D_QK; };

    if (warp >= 2) {
        // ---- Q terms of the CTA's first 1 + NSCR splits, while the first pages load: warps 2..7
        // quantise the first split's Q straight into the shared-memory operand and the next
        // NSCR splits' into this CTA's scratch slots, from which the producer loads them like
        // any operand (there is no separate quantisation kernel in front of the decode)
        const int pt = threadIdx.x - 64;
        int nq = 0;
        uint4 v[1 + NSCR][QPRO_VEC];
        {
            int vb = vb_begin;
#pragma unroll
            for (int j = 0; j < 1 + NSCR; ++j) {  // the next split with tiles, loads in flight
                SplitDesc sd;
                bool found = false;
                for (; vb <= vb_end && !found; ++vb) found = split_at(sch, seqlen_of(vb), B, vb, sd);
                if (found) {
                    nq = j + 1;
                    const uint4* src = q_rows(sd);
#pragma unroll
                    for (int i = 0; i < QPRO_VEC; ++i) v[j][i] = __ldg(src + pt + QPRO_THREADS * i);
                }
            }
        }
        // the first split's terms go to shared memory at once; the scratch slots are global
        // writes, after the grid dependency under ETAP_FLAG_INDEPENDENT_INPUTS (the previous
        // call's CTAs may still read them until then)
#pragma unroll
        for (int j = 0; j < 1 + NSCR; ++j) {
            if (j >= nq) break;
            if (j == 1) {
                ptx::fence_proxy_async_smem();
                ptx::named_bar_sync(5, QPRO_THREADS);
                if (pt == 0) ptx::mbar_arrive(&bars[BAR_QF]);
                dep_wait_before_write(prm);
            }
#pragma unroll
            for (int i = 0; i < QPRO_VEC; ++i) {
                const int vi = pt + QPRO_THREADS * i, h = vi / (D_QK / 8), cv = vi - h * (D_QK / 8);
                uint2 t[fp8::NT];
                fp8::quant_q_vec(v[j][i], t);
#pragma unroll
                for (int term = 0; term < fp8::NT; ++term) {
                    if (j == 0)
                        *reinterpret_cast<uint2*>(smem + OFF_Q + fp8::q_smem_off(term * HG + h, cv)) = t[term];
                    else
                        *reinterpret_cast<uint2*>(scratch(j - 1) + (term * HG + h) * D_QK + cv * 8) = t[term];
                }
            }
        }
        if (nq == 1) ptx::fence_proxy_async_smem();
        else ptx::fence_proxy_async_global();
        ptx::named_bar_sync(5, QPRO_THREADS);
        if (pt == 0) {
            if (nq == 1) ptx::mbar_arrive(&bars[BAR_QF]);
            for (int j = 1; j < nq; ++j) ptx::mbar_arrive(&bars[BAR_SCF + j - 1]);
        }
    }

    if (warp == 0) {
        // ===================================================== TMA producer
        if (lane == 0) ETAP_TRACE_PRO(prm, 3);
        const bool kv_shared = line_shape(B, prm.groups, gridDim.x, prm.lanes_on != 0).lanes > 1;
        const uint64_t pol_kv = kv_shared ? ptx::policy_evict_normal() : ptx::policy_evict_first();
        const uint64_t pol_q = ptx::policy_evict_first();
        if (lane == 0) ETAP_TRACE_PRO(prm, 4);
        uint32_t gt = 0, nsplit = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            const int32_t* bt = prm.block_table + static_cast<size_t>(sd.b) * prm.max_pages;
            int base = sd.t0;
            int pg;
            if (nsplit == 0 && sd.b == hint_b && sd.t0 == hint_t0) pg = hint_pg;  // loaded already
            else pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
            if (nsplit == 0 && lane == 0) ETAP_TRACE_PRO(prm, 5);
            bool q_pending = nsplit > 0;  // the first split's Q terms come from the prologue
            for (int t = sd.t0; t < sd.t1; ++t) {
                if (t - base >= 32) {
                    base = t;
                    pg = (base + lane < sd.t1) ? __ldg(bt + base + lane) : 0;
                }
                const int page = __shfl_sync(0xffffffffu, pg, t - base);
                if (gt == 0 && pro.late_wait) dep_wait_producer<kDebug>(prm);
                if (gt >= NPS) ptx::mbar_wait(&bars[BAR_G2D + (gt - NPS) % NTB8], ((gt - NPS) / NTB8) & 1);
                if (lane == 0) {
                    if (gt == 0) { ETAP_TRACE_G(prm, 9); ETAP_TRACE_CLK(prm, 15); }
                    ETAP_TRACE(prm, gt, 0);
                    uint8_t* slot = smem + OFF_RING + (gt % NPS) * fp8::TILE_BYTES;
                    uint64_t* full = &bars[BAR_FULL + gt % NTB8];
                    ptx::mbar_arrive_expect_tx(full, fp8::TILE_BYTES);
                    fp8_page_load(slot, &tm_kv128, &tm_kv64, full, page, pol_kv);
                    ETAP_TRACE(prm, gt, 1);
                }
                __syncwarp();
                if (q_pending) {
                    // a later split's Q terms from the scratch slot the prologue (or warp 3) filled,
                    // once GEMM1 of the previous split's last tile released the buffer
                    q_pending = false;
                    const uint32_t slot_q = (nsplit - 1) % NSCR;
                    ptx::mbar_wait(&bars[BAR_QE], (nsplit - 1) & 1);
                    ptx::mbar_wait(&bars[BAR_SCF + slot_q], ((nsplit - 1) / NSCR) & 1);
                    if (lane == 0) {
                        ptx::mbar_arrive_expect_tx(&bars[BAR_QF], fp8::Q_BYTES);
                        const int qrow = (blockIdx.x * NSCR + slot_q) * NQ;
#pragma unroll 1
                        for (int c = 0; c < fp8::VCH; ++c)
                            ptx::tma_load_2d(smem + OFF_Q + c * fp8::Q_VBLK, &tm_q128, &bars[BAR_QF], c * 128, qrow,
                                             pol_q);
                        ptx::tma_load_2d(smem + OFF_Q + fp8::VCH * fp8::Q_VBLK, &tm_q64, &bars[BAR_QF], 512, qrow, pol_q);
                    }
                    __syncwarp();
                }
                ++gt;
            }
            ++nsplit;
        }
        if (gt == 0 && pro.late_wait) dep_wait_producer<kDebug>(prm);  // no tiles in this CTA's range
    } else if (warp == 1) {
        // ===================================================== GEMM1 issuer
        uint32_t gt = 0, nsplit = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            ptx::mbar_wait(&bars[BAR_QF], nsplit & 1);
            if (nsplit == 0 && lane == 0) ETAP_TRACE_PRO(prm, 6);  // first split's Q terms in shared memory
            if (nsplit > 0 && lane == 0) ptx::mbar_arrive(&bars[BAR_SCE + (nsplit - 1) % NSCR]);  // slot read
            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gt & 1;
                if (gt >= 2) ptx::mbar_wait(&bars[BAR_SR + buf], ((gt >> 1) - 1) & 1);
                ptx::mbar_wait(&bars[BAR_FULL + gt % NTB8], (gt / NTB8) & 1);
                __syncwarp();
                ptx::tc_fence_after();
                ETAP_TRACE(prm, gt, 2);
                fp8::issue_gemm1(tmem_base + TCOL_S + NQ * buf, ring_addr + (gt % NPS) * fp8::TILE_BYTES, q_addr);
                ptx::umma_commit_elect(&bars[BAR_SF + buf]);
                ETAP_TRACE(prm, gt, 3);
                if (t == sd.t1 - 1) ptx::umma_commit_elect(&bars[BAR_QE]);
                ++gt;
            }
            ++nsplit;
        }
    } else if (warp == 2) {
        // ===================================================== GEMM2 issuer
        uint32_t gt = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gt & 1;
                ptx::mbar_wait(&bars[BAR_PF + buf], (gt >> 1) & 1);
                __syncwarp();
                ptx::tc_fence_after();
                ETAP_TRACE(prm, gt, 6);
                const uint32_t slot = ring_addr + (gt % NPS) * fp8::TILE_BYTES;
#pragma unroll
                for (int c = 0; c < fp8::VCH; ++c)
                    fp8::issue_gemm2(tmem_base + TCOL_O + c * NQ, slot + c * fp8::VCH_BYTES, p_addr + buf * fp8::P_BYTES,
                                     t == sd.t0);
                ptx::umma_commit_elect(&bars[BAR_G2D + gt % NTB8]);
                ETAP_TRACE(prm, gt, 7);
                ++gt;
            }
        }
    } else if (warp == 3) {
        publish_after_prologue(prm, pro, lane);
        // ===================================================== Q terms of splits past 1 + NSCR
        // (many short sequences per CTA): into scratch slot (j-1) % NSCR once GEMM1 saw the Q
        // that slot held land in shared memory
        uint32_t j = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            if (j > NSCR) {
                const uint32_t slot_q = (j - 1) % NSCR, u = (j - 1) / NSCR;
                ptx::mbar_wait(&bars[BAR_SCE + slot_q], (u - 1) & 1);
                dep_wait_before_write(prm);
                fp8::quant_q_global_warp(q_rows(sd), scratch(slot_q), lane);
                ptx::fence_proxy_async_global();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bars[BAR_SCF + slot_q]);
            }
            ++j;
        }
    } else if (warp >= SOFTMAX_WARP0) {
        // ===================================================== softmax + epilogue (128 threads)
        const int wq = warp & 3;
        const int half = lane >> 4;
        const int row = s_row_of(wq, lane);
        const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(wq * 32) << 16);
        float* red_max = reinterpret_cast<float*>(smem + OFF_RED);  // [2][4][HG]
        float* red_sum = red_max + 8 * HG;
        float* s_m = red_sum + 4 * HG;
        float* s_alpha = s_m + HG;
        int* s_row = reinterpret_cast<int*>(s_alpha + HG);
        const float thresh = (prm.flags & FLAG_EAGER_RESCALE) ? 0.f : LAZY_RESCALE_LOG2;
        const bool head_owner = wq == 0 && (lane & 15) == 0;
        const bool lane_head = wq == 0 && lane < HG;
        const bool mtp = prm.q_tokens > 1;
        const int rhead = halfwarp_reduce_head<HH>(lane);
        const bool rwriter = (lane & 1) == 0;
        const bool tracer = threadIdx.x == SOFTMAX_WARP0 * 32;
        uint32_t gt = 0;
        for (int vb = vb_begin; vb <= vb_end; ++vb) {
            SplitDesc sd;
            if (!split_at(sch, seqlen_of(vb), B, vb, sd)) continue;
            float m_own[HH], l_part[HH];
            float m_thr[HH], mu[HH];  // m_own + thresh, exp2 offset (refreshed when m_own moves)
            int row_lim[HH];
            int row_all = sd.seqlen;  // rows below this are visible to every column of the thread
#pragma unroll
            for (int j = 0; j < HH; ++j) {
                m_own[j] = -INFINITY;
                m_thr[j] = -INFINITY;
                mu[j] = mtp ? 0.f : -INFINITY;
                l_part[j] = 0.f;
                const int tok = (sd.g * HG + half * HH + j) / prm.heads_per_token;
                row_lim[j] = sd.seqlen - (prm.causal ? prm.q_tokens - 1 - tok : 0);
                row_all = min(row_all, row_lim[j]);
                if (head_owner) s_m[half * HH + j] = -INFINITY;
            }
            for (int t = sd.t0; t < sd.t1; ++t) {
                const uint32_t buf = gt & 1;
                ptx::mbar_wait(&bars[BAR_SF + buf], (gt >> 1) & 1);
                ptx::tc_fence_after();
                if (tracer) ETAP_TRACE(prm, gt, 4);
                uint32_t s0[HH], s1[HH], s2[HH];
                ptx::tmem_ld16x2<HH>(t_lane + TCOL_S + NQ * buf, s0);
                ptx::tmem_ld16x2<HH>(t_lane + TCOL_S + NQ * buf + 16, s1);
                ptx::tmem_ld16x2<HH>(t_lane + TCOL_S + NQ * buf + 32, s2);
                ptx::tmem_wait_ld();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&bars[BAR_SR + buf]);

                const int grow = t * TILE + row;
                float x[HH];
#pragma unroll
                for (int j = 0; j < HH; ++j)  // S = S_q0 + S_q1 / 16 + S_q2 / 256 (the three fp8 terms of Q)
                    x[j] = (__uint_as_float(s0[j]) +
                            (__uint_as_float(s1[j]) * 0.0625f + __uint_as_float(s2[j]) * 0.00390625f)) * prm.scale_log2;
                if (grow >= row_all) {  // a split's last tile: rows past the (per-token) context
#pragma unroll
                    for (int j = 0; j < HH; ++j) x[j] = grow < row_lim[j] ? x[j] : -INFINITY;
                }
                bool exceed = false;
#pragma unroll
                for (int j = 0; j < HH; ++j) exceed |= x[j] > m_thr[j];
                const bool first = (t == sd.t0);
                const bool any = ptx::bar_red_or(1, 128, exceed);
                bool need_rescale = false;
                float alpha_own[HH];
#pragma unroll
                for (int j = 0; j < HH; ++j) alpha_own[j] = first ? 0.f : 1.f;
                if (any) {
                    const float wm = halfwarp_reduce<true, HH>(x, lane);
                    float* rm = red_max + (gt & 1) * 4 * HG;
                    if (rwriter) rm[wq * HG + half * HH + rhead] = wm;
                    ptx::named_bar_sync(2, 128);
                    bool upd = false;
#pragma unroll
                    for (int j = 0; j < HH; ++j) {
                        const int h = half * HH + j;
                        const float mt = fmaxf(fmaxf(rm[h], rm[HG + h]), fmaxf(rm[2 * HG + h], rm[3 * HG + h]));
                        if (first) {
                            m_own[j] = mt;
                        } else {
                            const float mn = fmaxf(m_own[j], mt);
                            if (mn > m_own[j] + thresh) {
                                alpha_own[j] = ptx::exp2_ftz(m_own[j] - mn);
                                m_own[j] = mn;
                                upd = true;
                            }
                        }
                    }
                    need_rescale = ptx::bar_red_or(2, 128, upd);
                    if (head_owner) {
#pragma unroll
                        for (int j = 0; j < HH; ++j) {
                            s_m[half * HH + j] = m_own[j];
                            s_alpha[half * HH + j] = alpha_own[j];
                        }
                    }
#pragma unroll
                    for (int j = 0; j < HH; ++j) {
                        m_thr[j] = m_own[j] + thresh;
                        mu[j] = (mtp && m_own[j] == -INFINITY) ? 0.f : m_own[j];
                    }
                }
                float pv[HH];
#pragma unroll
                for (int j = 0; j < HH; ++j) {
                    pv[j] = ptx::exp2_ftz(x[j] - mu[j]);
                    l_part[j] = fmaf(l_part[j], alpha_own[j], pv[j]);  // first tile: alpha = 0, l = 0
                }
                // the P buffer is reused every other tile: GEMM2(gt-2) must have read it
                if (tracer) ETAP_TRACE(prm, gt, 8);
                if (gt >= 2) ptx::mbar_wait(&bars[BAR_G2D + (gt - 2) % NTB8], ((gt - 2) / NTB8) & 1);
                if (tracer) ETAP_TRACE(prm, gt, 9);
                if (need_rescale) {
                    ptx::named_bar_sync(2, 128);
                    ptx::mbar_wait(&bars[BAR_G2D + (gt - 1) % NTB8], ((gt - 1) / NTB8) & 1);
                    ptx::tc_fence_after();
#pragma unroll 1
                    for (int c = 0; c < fp8::VCH; ++c) {
#pragma unroll
                        for (int term = 0; term < fp8::NT; ++term) {
                            uint32_t o[16];
                            const uint32_t ta = t_lane + TCOL_O + c * NQ + term * 16;
                            ptx::tmem_ld16(ta, o);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int h = 0; h < 16; ++h) o[h] = __float_as_uint(__uint_as_float(o[h]) * s_alpha[h]);
                            ptx::tmem_st16(ta, o);
                        }
                    }
                    ptx::tmem_wait_st();
                }
                // P -> three e4m3 terms, this row's 8 heads per term: one 8-byte store each
                {
                    uint16_t tt[4][fp8::NT];
#pragma unroll
                    for (int i = 0; i < 4; ++i) fp8::split3(pv[2 * i], pv[2 * i + 1], tt[i]);
                    uint8_t* pb = smem + OFF_P + buf * fp8::P_BYTES;
#pragma unroll
                    for (int term = 0; term < fp8::NT; ++term) {
                        const uint32_t lo = static_cast<uint32_t>(tt[0][term]) | (static_cast<uint32_t>(tt[1][term]) << 16);
                        const uint32_t hi = static_cast<uint32_t>(tt[2][term]) | (static_cast<uint32_t>(tt[3][term]) << 16);
                        *reinterpret_cast<uint2*>(pb + fp8::p_off(row, term * 16 + half * HH)) = make_uint2(lo, hi);
                    }
                }
                // rows past seqlen may hold non-finite bytes: zero them in the V chunks
                if (grow >= sd.seqlen) {
                    uint8_t* slot = smem + OFF_RING + (gt % NPS) * fp8::TILE_BYTES;
#pragma unroll 1
                    for (int c = half * 2; c < half * 2 + 2; ++c) {
                        uint4* dst = reinterpret_cast<uint4*>(slot + c * fp8::VCH_BYTES + row * 128);
#pragma unroll
                        for (int j = 0; j < 8; ++j) dst[j] = make_uint4(0, 0, 0, 0);
                    }
                }
                ptx::fence_proxy_async_smem();
                ptx::tc_fence_before();
                if (tracer) ETAP_TRACE(prm, gt, 5);
                ptx::mbar_arrive(&bars[BAR_PF + buf]);
                ++gt;
            }

            // ---- epilogue: O = kv_scale * (O_0 + O_1/16 + O_2/256) / l, L = m + log l
            const uint32_t last = gt - 1;
            dep_wait_before_write(prm);
            ptx::mbar_wait(&bars[BAR_G2D + last % NTB8], (last / NTB8) & 1);
            ptx::tc_fence_after();
            if (tracer) { ETAP_TRACE_G(prm, 10); ETAP_TRACE(prm, last, 10); }
            const float wsum = halfwarp_reduce<false, HH>(l_part, lane);
            if (rwriter) red_sum[wq * HG + half * HH + rhead] = wsum;
            const int ns = soff[vb + 1] - soff[vb];
            const bool direct = ns == 1;
            if (direct && lane_head) s_row[lane] = static_cast<int>(prm.om.row(sd.b, sd.g * HG + lane));
            ptx::named_bar_sync(2, 128);
            float L_own = 0.f;
            float* s_inv = red_max;
            if (lane_head) {
                const float l = red_sum[lane] + red_sum[HG + lane] + red_sum[2 * HG + lane] + red_sum[3 * HG + lane];
                s_inv[lane] = l > 0.f ? kv_scale / l : 0.f;
                L_own = (s_m[lane] + log2f(l)) * 0.69314718055994530942f;
            }
            ptx::named_bar_sync(2, 128);
            float inv_l[HG];
#pragma unroll
            for (int h = 0; h < HG; h += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(s_inv + h);
                inv_l[h] = v4.x; inv_l[h + 1] = v4.y; inv_l[h + 2] = v4.z; inv_l[h + 3] = v4.w;
            }
            const int idx = (vb == sch[0]) ? sch[4] : soff[vb] + idx_off;
            float* part_o = prm.ws_o + static_cast<size_t>(idx) * HG * D_V;
            const int drow = wq * 32 + lane;
#pragma unroll 1
            for (int c = 0; c < fp8::VCH; ++c) {
                uint32_t o[fp8::NT][16];
#pragma unroll
                for (int term = 0; term < fp8::NT; ++term) ptx::tmem_ld16(t_lane + TCOL_O + c * NQ + term * 16, o[term]);
                ptx::tmem_wait_ld();
                const int d = c * 128 + drow;
                float v[HG];
#pragma unroll
                for (int h = 0; h < HG; ++h)
                    v[h] = (__uint_as_float(o[0][h]) + (__uint_as_float(o[1][h]) * 0.0625f +
                                                       __uint_as_float(o[2][h]) * 0.00390625f)) * inv_l[h];
                if (direct) {
#pragma unroll 1
                    for (int r = 0; r < prm.om.n_out; ++r) {
                        float* dst = prm.om.out[r] + d;
#pragma unroll
                        for (int h = 0; h < HG; ++h) dst[static_cast<size_t>(s_row[h]) * D_V] = v[h];
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < HG; ++h) part_o[h * D_V + d] = v[h];
                }
            }
            if (lane_head) {
                if (direct) {
                    for (int r = 0; r < prm.om.n_out; ++r) prm.om.lse[r][s_row[lane]] = L_own;
                } else {
                    prm.ws_lse[static_cast<size_t>(idx) * HG + lane] = L_own;
                }
            }
            ptx::tc_fence_before();
            ptx::named_bar_sync(2, 128);
            if (tracer) ETAP_TRACE(prm, last, 11);
        }
    }

    if (tracer_exit(warp, lane)) ETAP_TRACE_G(prm, 11);
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        span_stamp(prm, 1);
        ETAP_TRACE_G(prm, 2);
        ETAP_TRACE_CLK(prm, 6);
    }
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// =============================================================================================
// KV append (caller side of the path: the serving loop writes each step's new latent rows
// into the paged cache before the decode reads them). One CTA of 72 threads per new row,
// one 16 B vector each (576 bf16 = 1152 B). HBM-bound scatter of B * q_tokens rows.
// =============================================================================================
__global__ void __launch_bounds__(72)
    etap_mla_append_kv_kernel(const uint4* __restrict__ rows, uint4* __restrict__ pool, int64_t num_pages,
                              const int32_t* __restrict__ block_table, int max_pages,
                              const int32_t* __restrict__ seqlens, int q_tokens) {
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    const int r = blockIdx.x;                 // b * q_tokens + j
    const int b = r / q_tokens, j = r - b * q_tokens;
    const int pos = __ldg(seqlens + b) - q_tokens + j;
    if (pos < 0 || pos / PAGE >= max_pages) return;
    const int page = __ldg(block_table + static_cast<size_t>(b) * max_pages + pos / PAGE);
    if (page < 0 || page >= num_pages) return;
    const size_t dst_row = static_cast<size_t>(page) * PAGE + pos % PAGE;
    pool[dst_row * (D_QK * 2 / 16) + threadIdx.x] = rows[static_cast<size_t>(r) * (D_QK * 2 / 16) + threadIdx.x];
}

// Serving-step ingest (etap_mla_host_decode_step with page-locked host buffers): one kernel
// reads this step's Q, new latent rows and seqlens straight from mapped host memory over PCIe,
// writes Q and seqlens to their device buffers and appends the rows into the paged pool —
// instead of three host->device copies and the append kernel. Blocks [0, nq) copy one Q row
// (1152 B) each, blocks [nq, nq + B*T) append one latent row. It never triggers its dependents
// early: the decode launched after it reads seqlens before its own grid dependency.
__global__ void __launch_bounds__(72)
    etap_mla_ingest_kernel(const uint4* __restrict__ q_src, uint4* __restrict__ q_dst, int nq,
                           const uint4* __restrict__ rows, uint4* __restrict__ pool, int64_t num_pages,
                           const int32_t* __restrict__ block_table, int max_pages,
                           const int32_t* __restrict__ seqlens_src, int32_t* __restrict__ seqlens_dst,
                           int batch, int q_tokens) {
    constexpr int V = D_QK * 2 / 16;  // 16-byte vectors per row
    const int r = blockIdx.x;
    if (r < nq) {
        q_dst[static_cast<size_t>(r) * V + threadIdx.x] = q_src[static_cast<size_t>(r) * V + threadIdx.x];
        if (r == 0)
            for (int i = threadIdx.x; i < batch; i += blockDim.x) seqlens_dst[i] = seqlens_src[i];
        return;
    }
    const int rr = r - nq;  // b * q_tokens + j
    const int b = rr / q_tokens, j = rr - b * q_tokens;
    const int pos = seqlens_src[b] - q_tokens + j;
    if (pos < 0 || pos / PAGE >= max_pages) return;
    const int page = block_table[static_cast<size_t>(b) * max_pages + pos / PAGE];
    if (page < 0 || page >= num_pages) return;
    const size_t dst_row = static_cast<size_t>(page) * PAGE + pos % PAGE;
    pool[dst_row * V + threadIdx.x] = rows[static_cast<size_t>(rr) * V + threadIdx.x];
}

// =============================================================================================
// K3: log-sum-exp combine of split partials (no reference analog: split-KV is a SPEC
// non-goal; the math is pinned by L = m + log l, etap.cpp:144, and partition
// invariance, acceptance.cpp:209-229). Grid: one CTA of 128 threads per (vb, head).
// =============================================================================================
// Heads per CTA (template HPB, 128 threads each) and partial float4 loads in flight per thread
// (template COMBINE_BATCH, any value gives the same bits):
//   * 16-head units (the headline): HPB 2, batch 8 -> 128 CTAs of 72 registers, so one combine
//     CTA fits on an SM beside the decode CTA (43k registers, 224 KB): every combine CTA is
//     resident before the decode ends, and the next step's decode CTAs can launch beside the
//     running combine (with ETAP_FLAG_INDEPENDENT_INPUTS they then stream at once); two round
//     trips for the ~10 splits of a sequence instead of one;
//   * 32 / 64-head units: HPB 1, batch 16 (one round trip for up to 16 splits per sequence);
//   * the CTA-pair kernel's 128-head units: the dense combine, HPB 1, batch 4 (2048 rows at
//     B = 16 with ~6 splits each: 64 registers, 8 CTAs per SM; batch 8 at 72 registers measured
//     0.4% slower, batch 16 at 114 registers 1.2%).
constexpr int COMBINE_GROUP = 16;  // splits merged per rescale of the running sums
// K3 lets the next kernel launch before its own grid dependency (1) or after it (0). Early: the
// next step's decode CTAs take SMs as this step's decode CTAs exit (during its tail), and with
// ETAP_FLAG_INDEPENDENT_INPUTS they stream right away; without that flag they wait for this
// combine in their prologue as before. Either way every global write of the next decode is
// ordered after this combine (its grid dependency covers this grid's completion).
#ifndef ETAP_K3_EARLY_TRIGGER
#define ETAP_K3_EARLY_TRIGGER 1
#endif
template <int COMBINE_BATCH, int HPB>
__device__ __forceinline__ void combine_body(const float* __restrict__ ws_o, const float* __restrict__ ws_lse,
                                             const int32_t* __restrict__ split_off, int hg, int batch,
                                             const OutMap& om, unsigned long long* trace,
                                             const int32_t* __restrict__ seqlens, int parts, int lanes_on,
                                             int fixed_cost) {
    if (trace && threadIdx.x == 0) trace[blockIdx.x * 4 + 0] = ptx::global_timer_ns();
    const int units = hg / HPB;                   // CTAs per virtual sequence
    const int vb = blockIdx.x / units;
    const int h = (blockIdx.x - vb * units) * HPB + threadIdx.x / 128;
    const int t = threadIdx.x % 128;              // float4 of the 512-wide O row
    const int g = vb / batch, b = vb - g * batch;  // head-group-major virtual sequences
    int s0, ns;
    if (seqlens != nullptr) {
        // The decode used the in-kernel schedule on a line of <= 32 entries: this sequence's
        // split offset / count follow in closed form from seqlens (the same formula as
        // inkernel_schedule_warp), computed before the grid dependency resolves so the
        // partial loads go out right after it. seqlens are final here: the decode kernel
        // triggered this launch only after its own grid_dep_wait.
        __shared__ int s_info[2];
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            const LineShape ls = line_shape(batch, gridDim.x / units / batch, parts, lanes_on != 0);
            const int n = ls.line_n;
            const int lv = vb / n, pos = vb - lv * n;
            const int len = lane < n ? max(0, __ldg(seqlens + lane % batch)) : 0;
            const int tiles = (len + TILE - 1) / TILE;
            const int cost = tiles > 0 ? tiles + fixed_cost : 0;
            int incl = cost;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int pref = incl - cost;
            const int T = max(1, (total + ls.p_line - 1) / ls.p_line);
            const int nsi = (lane < n && tiles > 0) ? ((incl + T - 1) / T - 1) - (pref + fixed_cost) / T + 1 : 0;
            int so = nsi;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, so, o);
                if (lane >= o) so += y;
            }
            const int ns_line = __shfl_sync(0xffffffffu, so, 31);
            if (lane == pos) {
                s_info[0] = lv * ns_line + so - nsi;
                s_info[1] = nsi;
            }
        }
        __syncthreads();
        s0 = s_info[0];
        ns = s_info[1];
        if (ETAP_K3_EARLY_TRIGGER) ptx::grid_dep_launch();
        ptx::grid_dep_wait();
        if (!ETAP_K3_EARLY_TRIGGER) ptx::grid_dep_launch();  // the next decode step's prologue may overlap this combine
    } else {
        if (ETAP_K3_EARLY_TRIGGER) ptx::grid_dep_launch();
        ptx::grid_dep_wait();
        if (!ETAP_K3_EARLY_TRIGGER) ptx::grid_dep_launch();
        s0 = __ldg(split_off + vb);
        ns = __ldg(split_off + vb + 1) - s0;
    }
    if (trace && threadIdx.x == 0) trace[blockIdx.x * 4 + 1] = ptx::global_timer_ns();
    if (ns == 1) {
        if (trace && threadIdx.x == 0) trace[blockIdx.x * 4 + 2] = ptx::global_timer_ns();
        return;
    }
    const size_t orow = om.row(b, g * hg + h);
    if (ns <= 0) {  // empty context: O = 0, L = -inf
        for (int r = 0; r < om.n_out; ++r) {
            reinterpret_cast<float4*>(om.out[r] + orow * D_V)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t == 0) om.lse[r][orow] = -INFINITY;
        }
        return;
    }
    // Splits merge in groups of COMBINE_GROUP (the group's LSEs first: its max rescales the running
    // sums once), each group's partial float4s loaded COMBINE_BATCH at a time (registers): the
    // arithmetic, and so every output bit, is the same for every COMBINE_BATCH.
    const float* l_base = ws_lse + static_cast<size_t>(s0) * hg + h;
    const float4* p4 = reinterpret_cast<const float4*>(ws_o + (static_cast<size_t>(s0) * hg + h) * D_V) + t;
    const size_t stride4 = static_cast<size_t>(hg) * D_V / 4;
    float mx = -INFINITY, sum = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < ns; s += COMBINE_GROUP) {
        const int n = min(COMBINE_GROUP, ns - s);
        float l[COMBINE_GROUP];
        float4 v[COMBINE_BATCH];
#pragma unroll
        for (int j = 0; j < COMBINE_GROUP; ++j)
            if (j < n) l[j] = __ldg(l_base + static_cast<size_t>(s + j) * hg);
#pragma unroll
        for (int j = 0; j < COMBINE_BATCH; ++j)  // the first loads go out with the LSEs
            if (j < n) v[j] = __ldg(p4 + (s + j) * stride4);
        // online merge of this group (same algebra as L = m + log l, etap.cpp:144)
        float bm = mx;
#pragma unroll
        for (int j = 0; j < COMBINE_GROUP; ++j)
            if (j < n) bm = fmaxf(bm, l[j]);
        const float bs = bm == -INFINITY ? 0.f : bm;  // all partials empty so far (causal MTP)
        const float corr = __expf(mx - bs);  // 0 on the first group (mx = -inf)
        sum *= corr;
        acc.x *= corr; acc.y *= corr; acc.z *= corr; acc.w *= corr;
#pragma unroll
        for (int j0 = 0; j0 < COMBINE_GROUP; j0 += COMBINE_BATCH) {
            if (j0 > 0) {
#pragma unroll
                for (int j = 0; j < COMBINE_BATCH; ++j)
                    if (j0 + j < n) v[j] = __ldg(p4 + (s + j0 + j) * stride4);
            }
#pragma unroll
            for (int j = 0; j < COMBINE_BATCH; ++j) {
                if (j0 + j < n) {
                    const float w = __expf(l[j0 + j] - bs);
                    sum += w;
                    acc.x = fmaf(w, v[j].x, acc.x);
                    acc.y = fmaf(w, v[j].y, acc.y);
                    acc.z = fmaf(w, v[j].z, acc.z);
                    acc.w = fmaf(w, v[j].w, acc.w);
                }
            }
        }
        mx = bm;
    }
    const float inv = sum > 0.f ? 1.f / sum : 0.f;
    acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
    for (int r = 0; r < om.n_out; ++r) {  // every output copy (peer gather: each rank's buffer)
        if (t == 0) om.lse[r][orow] = mx + logf(sum);
        reinterpret_cast<float4*>(om.out[r] + orow * D_V)[t] = acc;
    }
    if (trace && threadIdx.x == 0) trace[blockIdx.x * 4 + 2] = ptx::global_timer_ns();
}

template <int COMBINE_BATCH>
__global__ void __launch_bounds__(128)
    etap_mla_combine_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_lse,
                            const int32_t* __restrict__ split_off, int hg, int batch,
                            const __grid_constant__ OutMap om, unsigned long long* trace,
                            const int32_t* __restrict__ seqlens, int parts, int lanes_on, int fixed_cost) {
    combine_body<COMBINE_BATCH, 1>(ws_o, ws_lse, split_off, hg, batch, om, trace, seqlens, parts, lanes_on, fixed_cost);
}
// at most 64 registers (8 CTAs of 128 threads per SM): the CTAs of one combine pack onto few SMs
__global__ void __launch_bounds__(128, 8)
    etap_mla_combine_dense_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_lse,
                                  const int32_t* __restrict__ split_off, int hg, int batch,
                                  const __grid_constant__ OutMap om, unsigned long long* trace,
                                  const int32_t* __restrict__ seqlens, int parts, int lanes_on, int fixed_cost) {
    combine_body<4, 1>(ws_o, ws_lse, split_off, hg, batch, om, trace, seqlens, parts, lanes_on, fixed_cost);
}
// two heads per CTA, at most 80 registers: one CTA beside a 16-head decode CTA (43k registers)
#ifdef ETAP_COMBINE2_MAXNREG
#define ETAP_COMBINE2_BOUNDS __maxnreg__(ETAP_COMBINE2_MAXNREG)
#else
#define ETAP_COMBINE2_BOUNDS __launch_bounds__(256, 3)
#endif
__global__ void ETAP_COMBINE2_BOUNDS
    etap_mla_combine2_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_lse,
                             const int32_t* __restrict__ split_off, int hg, int batch,
                             const __grid_constant__ OutMap om, unsigned long long* trace,
                             const int32_t* __restrict__ seqlens, int parts, int lanes_on, int fixed_cost) {
    combine_body<8, 2>(ws_o, ws_lse, split_off, hg, batch, om, trace, seqlens, parts, lanes_on, fixed_cost);
}

// =============================================================================================
// UMMA layout self-test: one CTA runs GEMM1 and GEMM2 of a single tile through exactly the
// descriptors / smem layouts of the decode kernel and dumps the TMEM accumulators.
// =============================================================================================
__global__ void __launch_bounds__(NUM_THREADS, 1)
    etap_mla_selftest_kernel(const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_q, const float* p_in,
                             float* s_out, float* o_out) {
    using C = Cfg<16>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars[0], 1);
        ptx::mbar_init(&bars[1], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t ring_addr = ptx::smem_u32(smem + C::OFF_RING);
    const uint32_t q_addr = ptx::smem_u32(smem + C::OFF_Q);
    const uint32_t p_addr = ptx::smem_u32(smem + C::OFF_P);

    if (threadIdx.x == 0) {
        const uint64_t pol = ptx::policy_evict_first();
        ptx::mbar_arrive_expect_tx(&bars[0], NCHUNK * SLOT_BYTES + C::Q_BYTES);
        for (int c = 0; c < NCHUNK; ++c) {  // chunk c in slot c
            ptx::tma_load_2d(smem + C::OFF_RING + c * SLOT_BYTES, &tm_k, &bars[0], c * 64, 0, pol);
            ptx::tma_load_2d(smem + C::OFF_Q + c * C::Q_CHUNK_BYTES, &tm_q, &bars[0], c * 64, 0, pol);
        }
    }
    // P = hi + lo of the input, written by the softmax warps exactly as the decode kernel does
    if (warp >= SOFTMAX_WARP0) {
        const int row = s_row_of(warp & 3, lane), half = lane >> 4;
        float p[8];
        for (int j = 0; j < 8; ++j) p[j] = p_in[row * 16 + half * 8 + j];
        write_p_hilo<C>(smem + C::OFF_P, row, half, p);
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (warp == 1) {
        ptx::mbar_wait(&bars[0], 0);
        __syncwarp();
        ptx::tc_fence_after();
        issue_gemm1_tile<C, 0, NCHUNK>(tmem_base + C::TCOL_S, ring_addr, q_addr, 0, 0);  // tile 0: chunk c in slot c
        for (int blk = 0; blk < 4; ++blk)
            issue_gemm2_block<C>(tmem_base + C::TCOL_O + C::OBLK * blk, ring_addr + (2 * blk) * SLOT_BYTES,
                              p_addr, true);
        ptx::umma_commit_elect(&bars[1]);
    }
    if (warp >= SOFTMAX_WARP0) {
        ptx::mbar_wait(&bars[1], 0);
        ptx::tc_fence_after();
        const int wq = warp & 3;
        const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(wq * 32) << 16);
        uint32_t r[32];
        {
            uint32_t sr[8];
            ptx::tmem_ld16x2<8>(t_lane + C::TCOL_S, sr);
            ptx::tmem_wait_ld();
            const int row = s_row_of(wq, lane), half = lane >> 4;
            for (int j = 0; j < 8; ++j) s_out[row * 16 + half * 8 + j] = __uint_as_float(sr[j]);
        }
        for (int blk = 0; blk < 4; ++blk) {
            ptx::tmem_ld32(t_lane + C::TCOL_O + C::OBLK * blk, r);
            ptx::tmem_wait_ld();
            for (int n = 0; n < 32; ++n)
                o_out[(blk * 128 + wq * 32 + lane) * 32 + n] = __uint_as_float(r[n]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
    }
}

// =============================================================================================
// host side
// =============================================================================================
thread_local std::string g_last_error = "ok";

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(ETAP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define ETAP_CUDA(call)                                        \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, #call);    \
    } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D bf16 tensor map over a row-major [rows][576] matrix, box {64 cols, box_rows}, SW128.
int make_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_rows) {
    auto enc = get_encode_fn();
    if (!enc) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return fail(ETAP_ERR_SHAPE, "tensor base address must be 16-byte aligned");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(D_QK), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(D_QK) * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return ETAP_OK;
}

// 3-D view of the same pool for whole-page boxes: {64 cols of a chunk, rows, chunk}, strides
// 1152 B (row) and 128 B (chunk), so a box {64, 64, nchunk} lands chunks c0.. c0+nchunk-1 of one
// page as consecutive 8 KB SW128 slots ([chunk][row][128 B]) with one TMA instruction.
int make_map_page3d(CUtensorMap* map, const void* base, uint64_t rows, uint32_t nchunk, uint32_t box_rows = PAGE) {
    auto enc = get_encode_fn();
    if (!enc) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return fail(ETAP_ERR_SHAPE, "tensor base address must be 16-byte aligned");
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(NCHUNK)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(D_QK) * 2, 128};
    cuuint32_t box[3] = {64, box_rows, nchunk};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled (page box) failed: " + std::to_string(r));
    return ETAP_OK;
}

void* g_trace_buf = nullptr;  // debug tracing target (etap_mla_debug_trace)
void* g_span_buf = nullptr;   // kernel-span stamps (etap_mla_debug_span)
void* g_state_buf = nullptr;  // debug softmax-state dump target (etap_mla_debug_state)
void* g_combine_trace_buf = nullptr;  // debug: [block][4] stamps of the combine kernel
int g_state_tiles = 0;

template <typename K>
int ensure_smem_attr(K kernel, int bytes) {
    ETAP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    return ETAP_OK;
}

int check_device() {
    int dev = 0;
    ETAP_CUDA(cudaGetDevice(&dev));
    // per-thread cache of verified devices (the attribute queries cost ~1 us per call)
    thread_local uint64_t verified = 0;
    if (dev < 64 && (verified >> dev & 1ull)) return ETAP_OK;
    int major = 0, minor = 0;
    ETAP_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    ETAP_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    if (major != 10 || minor != 0)
        return fail(ETAP_ERR_CUDA, "etap_mla requires an sm_100 (B200) device, found sm_" +
                                       std::to_string(major) + std::to_string(minor));
    if (dev < 64) verified |= 1ull << dev;
    return ETAP_OK;
}

// Tensor maps are pure functions of (base, rows, box rows); serving loops reuse the same
// buffers every call, so the last few encodings are cached per thread (encoding costs ~1-2 us).
struct MapCacheEntry {
    const void* base = nullptr;
    uint64_t rows = 0;
    uint32_t box_rows = 0;
    uint32_t box_chunks = 0;
    CUtensorMap map;
};

// box_chunks > 0: the 3-D page view (make_map_page3d), box {64, box_rows, box_chunks}
int cached_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_rows, uint32_t box_chunks = 0) {
    thread_local MapCacheEntry cache[8];
    thread_local unsigned next = 0;
    for (auto& e : cache)
        if (e.base == base && e.rows == rows && e.box_rows == box_rows && e.box_chunks == box_chunks) {
            *map = e.map;
            return ETAP_OK;
        }
    if (box_chunks > 0) {
        if (int rc = make_map_page3d(map, base, rows, box_chunks, box_rows)) return rc;
    } else if (int rc = make_map(map, base, rows, box_rows)) {
        return rc;
    }
    MapCacheEntry& e = cache[next++ % 8];
    e.base = base;
    e.rows = rows;
    e.box_rows = box_rows;
    e.box_chunks = box_chunks;
    e.map = *map;
    return ETAP_OK;
}

// 2-D uint8 tensor map over a row-major [rows][576] byte matrix (FP8 pool / three-term Q),
// box {box_cols, box_rows}, SW128 (box_cols 128) or SW64 (box_cols 64); cached
// box_chunks > 0: a 3-D view {128 B of a chunk, rows, chunk} (strides 576 B, 128 B) whose box
// {128, box_rows, box_chunks} lands box_chunks consecutive 128-column chunks of the rows as
// [chunk][row][128 B] SW128 tiles with ONE TMA instruction (each instruction costs the
// issuing thread ~115 cycles, so a page in two boxes instead of five shortens every tile's
// load chain and the start-of-step ring fill)
int cached_map_u8(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_cols, uint32_t box_rows,
                  uint32_t box_chunks = 0) {
    struct Entry {
        const void* base = nullptr;
        uint64_t rows = 0;
        uint32_t bc = 0, br = 0, bk = 0;
        CUtensorMap map;
    };
    thread_local Entry cache[8];
    thread_local unsigned next = 0;
    for (auto& e : cache)
        if (e.base == base && e.rows == rows && e.bc == box_cols && e.br == box_rows && e.bk == box_chunks) {
            *map = e.map;
            return ETAP_OK;
        }
    auto enc = get_encode_fn();
    if (!enc) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return fail(ETAP_ERR_SHAPE, "tensor base address must be 16-byte aligned");
    CUresult r;
    if (box_chunks > 0) {
        cuuint64_t dims[3] = {128, rows, static_cast<cuuint64_t>(D_V / 128)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(D_QK), 128};
        cuuint32_t box[3] = {128, box_rows, box_chunks};
        cuuint32_t estr[3] = {1, 1, 1};
        r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(D_QK), rows};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(D_QK)};
        cuuint32_t box[2] = {box_cols, box_rows};
        cuuint32_t estr[2] = {1, 1};
        r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE,
                box_cols == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled (u8) failed: " + std::to_string(r));
    Entry& e = cache[next++ % 8];
    e.base = base;
    e.rows = rows;
    e.bc = box_cols;
    e.br = box_rows;
    e.bk = box_chunks;
    e.map = *map;
    return ETAP_OK;
}

// Heads per CTA work unit: 32 when the head count allows it (N = 32 / 64 UMMAs halve the
// tensor-pipe issue count per KV byte, which is what bounds 64+ heads on one GPU), else 16.
// ETAP_HEAD_GROUP=16 in the environment forces 16 (A/B runs); read once per process.
int head_group_of(int heads) {
    static const int forced = [] {
        const char* e = std::getenv("ETAP_HEAD_GROUP");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 16) return 16;
    if (forced == 32) return heads % 32 == 0 ? 32 : 16;
    return heads % 64 == 0 ? 64 : (heads % 32 == 0 ? 32 : 16);
}

bool heads_ok(int heads) { return heads >= 16 && heads % 16 == 0; }

// The CTA-pair kernel (etap_mla_pair.cuh) takes 128-head work units when the head count allows
// it. ETAP_PAIR=0 or a forced ETAP_HEAD_GROUP in the environment keeps the single-CTA kernels
// (A/B runs); the debug instantiations (trace / BlockHook state dump) are single-CTA only, and so
// are external schedules and separate combines (their layouts follow etap_mla_head_group).
bool pair_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ETAP_PAIR");
        const char* f = std::getenv("ETAP_HEAD_GROUP");
        return !(e && e[0] == '0') && !(f && f[0] != '\0');
    }();
    return on;
}

// Work-unit layout of the split schedule, i.e. what sched / split_off entries mean: 128-head units
// over num_sm_parts / 2 CTA pairs when the pair kernel runs the head count, else head_group_of
// units over num_sm_parts CTAs. K1, the host restatement, the decode and the combine agree on it.
bool pair_used(int heads, int num_sm_parts) {
    return heads % pairk::UNIT == 0 && pair_enabled() && num_sm_parts >= 2;
}
void sched_layout(int heads, int num_sm_parts, int* unit, int* parts) {
    const bool p = pair_used(heads, num_sm_parts);
    *unit = p ? pairk::UNIT : head_group_of(heads);
    *parts = p ? num_sm_parts / 2 : num_sm_parts;
}

// Head-group lanes of the split schedule (line_shape); ETAP_GROUP_LANES=0 disables them (A/B).
bool lanes_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ETAP_GROUP_LANES");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Programmatic dependent launch on every launch of this library; ETAP_PDL=0 in the
// environment launches without it (A/B: stream launches vs CUDA graphs). Read once.
unsigned pdl_attrs() {
    static const unsigned n = [] {
        const char* e = std::getenv("ETAP_PDL");
        return (e && e[0] == '0') ? 0u : 1u;
    }();
    return n;
}

// ETAP_FLAG_INDEPENDENT_INPUTS (implies the early metadata read): the decode kernels wait for the
// grid dependency only before their first global write. Never with SKIP_COMBINE (K2 would then
// be the predecessor of the next call's K2, which writes the same workspace / FP8 Q scratch);
// ETAP_DEFER_DEP=0 in the environment ignores the flag (A/B runs).
int defer_dep_of(unsigned flags, int early_meta) {
    static const bool on = [] {
        const char* e = std::getenv("ETAP_DEFER_DEP");
        return !(e && e[0] == '0');
    }();
    return (on && early_meta && (flags & ETAP_FLAG_INDEPENDENT_INPUTS) && !(flags & ETAP_FLAG_SKIP_COMBINE)) ? 1 : 0;
}

// Schedule before the grid dependency (DecodeParams::early_meta, opt-in per call with
// ETAP_FLAG_EARLY_METADATA); ETAP_EARLY_META=0 in the environment ignores that flag (A/B runs).
bool early_meta_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ETAP_EARLY_META");
        return !(e && e[0] == '0');
    }();
    return on;
}

size_t max_partials(int batch, int heads, int num_sm_parts) {
    return static_cast<size_t>(num_sm_parts) + static_cast<size_t>(batch) * (heads / head_group_of(heads));
}

// workspace layout: partial O [np][hg][512] fp32, partial LSE [np][hg] fp32, then (1 KB
// aligned) the FP8 path's per-CTA scratch for the three fp8 terms of Q of later splits,
// [num_sm_parts][NSCR][48][576] bytes. A work unit of 16 heads needs no more partial space
// than one of 32 (np * hg grows with hg).
size_t q3_offset(int batch, int heads, int num_sm_parts) {
    const size_t np = max_partials(batch, heads, num_sm_parts);
    const size_t hg = head_group_of(heads);
    return (np * hg * D_V * sizeof(float) + np * hg * sizeof(float) + 1023) / 1024 * 1024;
}
size_t q3_bytes(int num_sm_parts) {
    return static_cast<size_t>(num_sm_parts) * kfp8::NSCR * fp8::NQ * D_QK;
}

}  // namespace

namespace etap_b200 {
// error reporting for the host-buffer entry points in etap_mla_host.cpp
int host_fail(int code, const char* msg) { return fail(code, msg); }

// 2-D bf16 tensor map over a row-major [rows][cols] matrix, box {64 cols, box_rows}, SW128
// (etap_proj.cu); cached per (base, shape) like the decode's maps.
int encode_bf16_sw128(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
    struct Entry {
        const void* base = nullptr;
        uint64_t cols = 0, rows = 0;
        uint32_t box_rows = 0;
        CUtensorMap map;
    };
    thread_local Entry cache[8];
    thread_local unsigned next = 0;
    for (auto& e : cache)
        if (e.base == base && e.cols == cols && e.rows == rows && e.box_rows == box_rows) {
            *map = e.map;
            return ETAP_OK;
        }
    auto enc = get_encode_fn();
    if (!enc) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (cols * 2) % 16 != 0)
        return fail(ETAP_ERR_SHAPE, "tensor base / row pitch must be 16-byte aligned");
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ETAP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    Entry& e = cache[next++ % 8];
    e.base = base;
    e.cols = cols;
    e.rows = rows;
    e.box_rows = box_rows;
    e.map = *map;
    return ETAP_OK;
}
// Launch of the serving-step ingest (etap_mla_host.cpp): q_src / rows / seqlens_src are
// device pointers of page-locked host memory.
int ingest_step(const void* q_src, void* q_dst, int nq_rows, const void* rows, void* pool, int64_t num_pages,
                const int32_t* block_table, int max_pages, const int32_t* seqlens_src, int32_t* seqlens_dst,
                int batch, int q_tokens, void* stream) {
    if ((reinterpret_cast<uintptr_t>(q_src) | reinterpret_cast<uintptr_t>(q_dst) | reinterpret_cast<uintptr_t>(rows) |
         reinterpret_cast<uintptr_t>(pool)) & 15)
        return fail(ETAP_ERR_SHAPE, "ingest: 16-byte alignment required");
    // a plain launch: no programmatic serialisation with the kernel before it either
    etap_mla_ingest_kernel<<<nq_rows + batch * q_tokens, D_QK * 2 / 16, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(q_src), static_cast<uint4*>(q_dst), nq_rows, static_cast<const uint4*>(rows),
        static_cast<uint4*>(pool), num_pages, block_table, max_pages, seqlens_src, seqlens_dst, batch, q_tokens);
    ETAP_CUDA(cudaGetLastError());
    return ETAP_OK;
}
}  // namespace etap_b200

extern "C" {

const char* etap_mla_last_error(void) { return g_last_error.c_str(); }

const char* etap_mla_version(void) { return ETAP_MLA_VERSION; }

int etap_mla_head_group(int heads, int* head_group) {
    if (!head_group) return fail(ETAP_ERR_SHAPE, "head_group is NULL");
    if (!heads_ok(heads)) return fail(ETAP_ERR_SHAPE, "heads must be a multiple of 16");
    *head_group = head_group_of(heads);
    return ETAP_OK;
}

int etap_mla_schedule_unit(int heads, int num_sm_parts, int* unit_heads, int* parts) {
    if (!unit_heads || !parts) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (!heads_ok(heads)) return fail(ETAP_ERR_SHAPE, "heads must be a positive multiple of 16");
    if (num_sm_parts < 1 || num_sm_parts > META_THREADS)
        return fail(ETAP_ERR_SHAPE, "num_sm_parts must be in [1, 1024]");
    sched_layout(heads, num_sm_parts, unit_heads, parts);
    return ETAP_OK;
}

int etap_mla_num_sm_parts(int device, int* num_sm_parts) {
    if (!num_sm_parts) return fail(ETAP_ERR_SHAPE, "num_sm_parts is NULL");
    int n = 0;
    ETAP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    *num_sm_parts = n;
    return ETAP_OK;
}

int etap_mla_sched_ints(int batch, int heads, int num_sm_parts, size_t* sched_ints,
                        size_t* split_off_ints) {
    if (batch < 1 || !heads_ok(heads) || num_sm_parts < 1)
        return fail(ETAP_ERR_SHAPE, "batch >= 1, heads a multiple of 16, num_sm_parts >= 1 required");
    if (sched_ints) *sched_ints = static_cast<size_t>(num_sm_parts) * SCHED_INTS;
    // sized for work units of 16 heads (the FP8 path), enough for 32 as well
    if (split_off_ints) *split_off_ints = static_cast<size_t>(batch) * (heads / 16) + 1;
    return ETAP_OK;
}

int etap_mla_workspace_bytes(int batch, int heads, int num_sm_parts, size_t* bytes) {
    if (batch < 1 || !heads_ok(heads) || num_sm_parts < 1 || !bytes)
        return fail(ETAP_ERR_SHAPE, "batch >= 1, heads a multiple of 16, num_sm_parts >= 1 required");
    *bytes = q3_offset(batch, heads, num_sm_parts) + q3_bytes(num_sm_parts);
    return ETAP_OK;
}

int etap_mla_metadata_host(const int32_t* seqlens, int batch, int heads, int num_sm_parts,
                           int32_t* sched, int32_t* split_off) {
    // Serial host restatement of etap_mla_metadata_kernel (same line, lanes and mapping);
    // used by tests to pin the device schedule and by callers that plan on the host.
    if (!seqlens || !sched || !split_off) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (batch < 1 || !heads_ok(heads))
        return fail(ETAP_ERR_SHAPE, "batch >= 1 and heads a multiple of 16 required");
    if (num_sm_parts < 1 || num_sm_parts > META_THREADS)
        return fail(ETAP_ERR_SHAPE, "num_sm_parts must be in [1, 1024]");
    int unit = 0, parts = 0;
    sched_layout(heads, num_sm_parts, &unit, &parts);
    const int groups = heads / unit;
    const int nvb = batch * groups;
    if (nvb > META_MAX_VB) return fail(ETAP_ERR_SHAPE, "batch * head groups too large");
    const LineShape ls = line_shape(batch, groups, parts, lanes_enabled());
    const int n = ls.line_n;
    std::vector<int> tiles(n), pref(n + 1, 0), ns(n, 0), first(n, 0x7fffffff), soff(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        const int len = std::max(0, seqlens[i % batch]);
        tiles[i] = (len + TILE - 1) / TILE;
        pref[i + 1] = pref[i] + (tiles[i] > 0 ? tiles[i] + META_FIXED_COST : 0);
    }
    const int total = pref[n];
    const int T = std::max(1, (total + ls.p_line - 1) / ls.p_line);
    auto map = [&](int x, int& vb, int& t) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pref[mid] <= x) lo = mid; else hi = mid - 1;
        }
        while (lo + 1 < n && pref[lo + 1] <= x) ++lo;
        vb = lo;
        t = std::min(std::max(0, x - pref[lo] - META_FIXED_COST), tiles[lo]);
    };
    std::vector<int> rb(ls.p_line), rt(ls.p_line), re(ls.p_line), rte(ls.p_line);
    for (int k = 0; k < ls.p_line; ++k) {
        const int x0 = k * T, x1 = std::min(total, (k + 1) * T);
        int b0 = 0, tb = 0, b1 = -1, te = 0;
        if (x0 < total) {
            map(x0, b0, tb);
            if (x1 >= total) { b1 = n - 1; te = tiles[n - 1]; }
            else map(x1, b1, te);
            for (int vb = b0; vb <= b1; ++vb) {
                const int t0 = vb == b0 ? tb : 0;
                const int t1 = vb == b1 ? te : tiles[vb];
                if (t0 < t1) { ++ns[vb]; first[vb] = std::min(first[vb], k); }
            }
        }
        rb[k] = b0; rt[k] = tb; re[k] = b1; rte[k] = te;
    }
    for (int i = 0; i < n; ++i) soff[i + 1] = soff[i] + ns[i];
    const int ns_line = soff[n];
    for (int v = 0; v <= nvb; ++v) split_off[v] = (v / n) * ns_line + soff[v % n];
    for (int kk = 0; kk < parts; ++kk) {
        const int lane = kk / ls.p_line, k = kk - lane * ls.p_line;
        int32_t* s = sched + kk * SCHED_INTS;
        const int lo = std::min(lane, ls.lanes - 1);
        if (lane >= ls.lanes) {
            s[0] = 0; s[1] = 0; s[2] = -1; s[3] = 0; s[4] = 0;
        } else {
            int first_idx = 0;
            if (re[k] >= rb[k] && rb[k] < n) first_idx = lane * ns_line + soff[rb[k]] + (k - std::min(first[rb[k]], k));
            s[0] = rb[k]; s[1] = rt[k]; s[2] = re[k]; s[3] = rte[k]; s[4] = first_idx;
        }
        s[5] = lo * n; s[6] = lo * ns_line; s[7] = 0;
    }
    return ETAP_OK;
}

int metadata_launch(const int32_t* seqlens, int batch, int groups, int num_sm_parts, int32_t* sched,
                    int32_t* split_off, void* stream, int fixed_cost = META_FIXED_COST);

int etap_mla_metadata(const int32_t* seqlens, int batch, int heads, int num_sm_parts,
                      int32_t* sched, int32_t* split_off, void* stream) {
    if (!seqlens || !sched || !split_off) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (batch < 1 || !heads_ok(heads))
        return fail(ETAP_ERR_SHAPE, "batch >= 1 and heads a multiple of 16 required");
    if (num_sm_parts < 1 || num_sm_parts > META_THREADS)
        return fail(ETAP_ERR_SHAPE, "num_sm_parts must be in [1, 1024]");
    int unit = 0, parts = 0;
    sched_layout(heads, num_sm_parts, &unit, &parts);
    return metadata_launch(seqlens, batch, heads / unit, parts, sched, split_off, stream);
}

int metadata_launch(const int32_t* seqlens, int batch, int groups, int num_sm_parts, int32_t* sched,
                    int32_t* split_off, void* stream, int fixed_cost) {
    if (batch * groups > META_MAX_VB)
        return fail(ETAP_ERR_SHAPE, "batch * head groups exceeds " + std::to_string(META_MAX_VB));
    if (num_sm_parts < 1 || num_sm_parts > META_THREADS)
        return fail(ETAP_ERR_SHAPE, "num_sm_parts must be in [1, 1024]");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(META_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_attrs();
    ETAP_CUDA(cudaLaunchKernelEx(&cfg, etap_mla_metadata_kernel, seqlens, batch, groups,
                                 num_sm_parts, lanes_enabled() ? 1 : 0, sched, split_off, fixed_cost));
    return ETAP_OK;
}

}  // extern "C"

namespace {

// O rows are stored (K3) and split partials loaded as float4
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

OutMap local_outmap(int heads, float* out, float* lse) {
    OutMap om = {};
    om.q_tokens = 1;
    om.heads_per_token = heads;  // tokens folded: [B][T][H] rows are [B][T*H] rows
    om.out_heads = heads;
    om.out_head0 = 0;
    om.n_out = 1;
    om.out[0] = out;
    om.lse[0] = lse;
    return om;
}

// seqlens != null: the split offsets follow in closed form from seqlens (the decode ran the
// in-kernel schedule on a line of <= 32 entries); otherwise K3 reads split_off
// hg_unit: heads per work unit of the decode that wrote the partials (the FP8 kernel uses 16
// whatever the head count); the partial / LSE areas keep the allocation layout of
// etap_mla_workspace_bytes either way
// sched_parts: parts of the decode's split schedule when they differ from the allocation's
// num_sm_parts (the CTA-pair kernel schedules pairs)
int combine_impl(const int32_t* split_off, int batch, int heads, int num_sm_parts, void* workspace,
                 const OutMap& om, void* stream, const int32_t* seqlens = nullptr, int hg_unit = 0,
                 int fixed_cost = META_FIXED_COST, int sched_parts = 0) {
    const int hg_alloc = head_group_of(heads);
    const int hg = hg_unit > 0 ? hg_unit : hg_alloc;
    const int groups = heads / hg;
    const size_t np = max_partials(batch, heads, num_sm_parts);
    float* ws_o = static_cast<float*>(workspace);
    float* ws_lse = ws_o + np * hg_alloc * D_V;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg2 = {};
    // (ETAP_COMBINE_NARROW=0 in the environment: HPB 1 / batch 16 for 16-head units too, A/B)
    static const bool narrow2 = [] {
        const char* e = std::getenv("ETAP_COMBINE_NARROW");
        return !(e && e[0] == '0');
    }();
    const int hpb = (hg == 16 && narrow2) ? 2 : 1;
    cfg2.gridDim = dim3(batch * groups * hg / hpb);
    cfg2.blockDim = dim3(128 * hpb);
    cfg2.dynamicSmemBytes = 0;
    cfg2.stream = static_cast<cudaStream_t>(stream);
    cfg2.attrs = attr;
    cfg2.numAttrs = pdl_attrs();
// 32 / 64-head units: the dense combine (64 registers, 8 CTAs per SM). Its CTAs take SMs as
// decode CTAs leave and hold them until the decode grid is done, and the next decode launches
// only once all of them are resident: packed 8 per SM they block 64 SMs at B = 16 x 32 heads
// instead of every SM (3 per SM at 139 registers); 0.5-1% per step at 32 / 64 heads, outputs
// bitwise unchanged (A/B: 0 batch 16, 1 batch 8)
#ifndef ETAP_COMBINE_WIDE
#define ETAP_COMBINE_WIDE 2
#endif
// 128-head (CTA-pair) units: 1 = the dense combine (64 registers, 8 CTAs per SM; 360.2 vs 361.6 us
// at 128 heads, same box, three interleaved repetitions, scripts/ab_combine_pair.sh), 0 = batch 8
// (72 registers), 2 = batch 16 (365.9 us)
#ifndef ETAP_COMBINE_PAIR
#define ETAP_COMBINE_PAIR 1
#endif
    auto kern = hpb == 2 ? etap_mla_combine2_kernel
                         : (hg >= 128 ? (ETAP_COMBINE_PAIR == 1 ? etap_mla_combine_dense_kernel
                                         : ETAP_COMBINE_PAIR == 2 ? etap_mla_combine_kernel<16>
                                                                  : etap_mla_combine_kernel<8>)
                                      : (hg >= 32 && ETAP_COMBINE_WIDE == 1 ? etap_mla_combine_kernel<8>
                                         : (hg >= 32 && ETAP_COMBINE_WIDE == 2 ? etap_mla_combine_dense_kernel
                                                                               : etap_mla_combine_kernel<16>)));
    ETAP_CUDA(cudaLaunchKernelEx(&cfg2, kern,
                                 static_cast<const float*>(ws_o),
                                 static_cast<const float*>(ws_lse), split_off, hg, batch, om,
                                 static_cast<unsigned long long*>(g_combine_trace_buf), seqlens,
                                 sched_parts > 0 ? sched_parts : num_sm_parts, lanes_enabled() ? 1 : 0, fixed_cost));
    return ETAP_OK;
}

// CTA pairs co-resident at once for the pair kernel (clusters of two must share a TPC; with
// 1 CTA per SM at most num_sms / 2), cached per device.
int pair_capacity(int* pairs) {
    int dev = 0;
    ETAP_CUDA(cudaGetDevice(&dev));
    static int cached[64] = {0};
    if (dev < 0 || dev >= 64) return fail(ETAP_ERR_CUDA, "device index out of range");
    if (cached[dev] == 0) {
        auto kern = etap_mla_decode_pair_kernel<false>;
        if (int rc = ensure_smem_attr(kern, pairk::SMEM)) return rc;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(pairk::THREADS);
        cfg.dynamicSmemBytes = pairk::SMEM;
        int n = 0;
        ETAP_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
        cached[dev] = n > 0 ? n : -1;
    }
    *pairs = cached[dev];
    return ETAP_OK;
}

// K2-pair (+ K3): 128-head work units on CTA pairs. Same contract as decode_impl; the split
// schedule is over pairs (num_sm_parts / 2, capped by the pairs that fit at once), partials are
// 128 heads wide inside the allocation layout of etap_mla_workspace_bytes.
int decode_pair(const void* q, const void* kv_pool, int64_t num_pages, const int32_t* block_table,
                int max_pages_per_seq, const int32_t* seqlens, int batch, int q_tokens, int heads_per_token,
                float scale, int causal, int32_t* sched, int32_t* split_off, int pairs, void* workspace,
                size_t ws_lse_off, const OutMap& om, unsigned flags, void* stream) {
    const int heads = q_tokens * heads_per_token;
    CUtensorMap tm_kv, tm_kv32, tm_q;
    // (ETAP_PAIR_BOX3D: 3-D page views, one box per GEMM1 half-page and per V chunk pair)
    if (int rc = cached_map(&tm_kv, kv_pool, static_cast<uint64_t>(num_pages) * PAGE, PAGE, ETAP_PAIR_BOX3D ? 2 : 0))
        return rc;
    if (int rc = cached_map(&tm_kv32, kv_pool, static_cast<uint64_t>(num_pages) * PAGE, 32,
                            ETAP_PAIR_BOX3D ? NCHUNK : 0))
        return rc;
    if (int rc = cached_map(&tm_q, q, static_cast<uint64_t>(batch) * heads, pairk::HPC)) return rc;
    const int groups = heads / pairk::UNIT;
    DecodeParams prm;
    prm.block_table = block_table;
    prm.seqlens = seqlens;
    prm.sched = sched;
    prm.split_off = split_off;
    prm.om = om;
    prm.ws_o = static_cast<float*>(workspace);
    prm.ws_lse = prm.ws_o + ws_lse_off;
    prm.kv_pool = kv_pool;
    prm.q = q;
    prm.num_pages = num_pages;
    prm.max_pages = max_pages_per_seq;
    prm.batch = batch;
    prm.heads = heads;
    prm.groups = groups;
    prm.q_tokens = q_tokens;
    prm.heads_per_token = heads_per_token;
    prm.causal = causal ? 1 : 0;
    prm.sched_out = sched;
    prm.split_off_out = split_off;
    prm.lanes_on = lanes_enabled() ? 1 : 0;
    prm.pair = 1;
    const LineShape ls = line_shape(batch, groups, pairs, prm.lanes_on != 0);
    const bool external = flags & ETAP_FLAG_EXTERNAL_SCHEDULE;
    prm.inkernel_sched = (ls.line_n <= pairk::MAX_VB && !external) ? 1 : 0;
    prm.early_meta = (early_meta_enabled() && (flags & (ETAP_FLAG_EARLY_METADATA | ETAP_FLAG_INDEPENDENT_INPUTS))) ? 1 : 0;
    prm.defer_dep = defer_dep_of(flags, prm.early_meta);
    prm.fixed_cost = META_FIXED_COST;
    if (!prm.inkernel_sched && !external) {
        if (int rc = metadata_launch(seqlens, batch, groups, pairs, sched, split_off, stream)) return rc;
    }
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.flags = flags;
    prm.trace = static_cast<unsigned long long*>(g_trace_buf);
    prm.span = static_cast<unsigned long long*>(g_span_buf);
    prm.state = nullptr;
    prm.state_tiles = 0;

    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(pairk::THREADS);
    cfg.dynamicSmemBytes = pairk::SMEM;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = pdl_attrs();
    if (prm.trace != nullptr) {
        static int attr_rc = ensure_smem_attr(etap_mla_decode_pair_kernel<true>, pairk::SMEM);
        if (attr_rc) return attr_rc;
        ETAP_CUDA(cudaLaunchKernelEx(&cfg, etap_mla_decode_pair_kernel<true>, tm_kv, tm_kv32, tm_q, prm));
    } else {
        ETAP_CUDA(cudaLaunchKernelEx(&cfg, etap_mla_decode_pair_kernel<false>, tm_kv, tm_kv32, tm_q, prm));
    }
    return ETAP_OK;
}

// K2 (+ K3 unless SKIP_COMBINE) for one call; final rows go wherever `om` says.
int decode_impl(const void* q, const void* kv_pool, int64_t num_pages, const int32_t* block_table,
                int max_pages_per_seq, const int32_t* seqlens, int batch, int q_tokens,
                int heads_per_token, float scale, int causal, const int32_t* sched,
                const int32_t* split_off, int num_sm_parts, void* workspace, const OutMap& om,
                unsigned flags, void* stream) {
    if (!q || !kv_pool || !block_table || !seqlens || !sched || !split_off || !workspace)
        return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (q_tokens < 1 || q_tokens > ETAP_MLA_MAX_Q_TOKENS)
        return fail(ETAP_ERR_SHAPE, "q_tokens must be in [1, " + std::to_string(ETAP_MLA_MAX_Q_TOKENS) + "]");
    if (heads_per_token < 1) return fail(ETAP_ERR_SHAPE, "heads must be >= 1");
    // the q_tokens query tokens of a sequence are folded into its head axis (rows of Q / O)
    const int heads = q_tokens * heads_per_token;
    if (batch < 1 || !heads_ok(heads))
        return fail(ETAP_ERR_SHAPE, "batch >= 1 and q_tokens * heads a multiple of 16 required");
    if (num_pages < 1 || max_pages_per_seq < 1)
        return fail(ETAP_ERR_SHAPE, "num_pages and max_pages_per_seq must be >= 1");
    if (num_pages * PAGE > (int64_t)0x7fffffff)
        return fail(ETAP_ERR_SHAPE, "kv pool exceeds 2^31 rows");
    if (!(scale >= 0.f) || !std::isfinite(scale))
        return fail(ETAP_ERR_SHAPE, "scale must be finite and >= 0");
    if (num_sm_parts < 1 || num_sm_parts > META_THREADS)
        return fail(ETAP_ERR_SHAPE, "num_sm_parts must be in [1, 1024]");
    if (int rc = check_device()) return rc;

    if (pair_used(heads, num_sm_parts) && g_state_buf == nullptr) {
        int cap = 0;
        if (int rc = pair_capacity(&cap)) return rc;
        const int pairs = num_sm_parts / 2;
        if (cap < pairs && (flags & ETAP_FLAG_EXTERNAL_SCHEDULE))
            return fail(ETAP_ERR_SHAPE, "external schedule for " + std::to_string(pairs) + " CTA pairs, but only " +
                                            std::to_string(cap) + " fit on the device at once");
        if (cap >= pairs) {  // (else: the single-CTA kernels with their own schedule)
            // partial LSEs sit where the allocation layout (head_group_of units) puts them
            const size_t ws_lse_off = max_partials(batch, heads, num_sm_parts) * head_group_of(heads) * D_V;
            if (int rc = decode_pair(q, kv_pool, num_pages, block_table, max_pages_per_seq, seqlens, batch, q_tokens,
                                     heads_per_token, scale, causal, const_cast<int32_t*>(sched),
                                     const_cast<int32_t*>(split_off), pairs, workspace, ws_lse_off, om, flags, stream))
                return rc;
            if (flags & ETAP_FLAG_SKIP_COMBINE) return ETAP_OK;
            const bool closed_form = !(flags & ETAP_FLAG_EXTERNAL_SCHEDULE) &&
                                     line_shape(batch, heads / pairk::UNIT, pairs, lanes_enabled()).line_n <= 32;
            return combine_impl(split_off, batch, heads, num_sm_parts, workspace, om, stream,
                                closed_form ? seqlens : nullptr, pairk::UNIT, META_FIXED_COST, pairs);
        }
    }

    CUtensorMap tm_kv, tm_q;
    if (int rc = cached_map(&tm_kv, kv_pool, static_cast<uint64_t>(num_pages) * PAGE, PAGE)) return rc;
    const int hg = head_group_of(heads);
    if (int rc = cached_map(&tm_q, q, static_cast<uint64_t>(batch) * heads, hg)) return rc;

    const int groups = heads / hg;
    const size_t np = max_partials(batch, heads, num_sm_parts);
    DecodeParams prm;
    prm.block_table = block_table;
    prm.seqlens = seqlens;
    prm.sched = sched;
    prm.split_off = split_off;
    prm.om = om;
    prm.ws_o = static_cast<float*>(workspace);
    prm.ws_lse = prm.ws_o + np * hg * D_V;
    prm.kv_pool = kv_pool;
    prm.q = q;
    prm.num_pages = num_pages;
    prm.max_pages = max_pages_per_seq;
    prm.batch = batch;
    prm.heads = heads;
    prm.groups = groups;
    prm.q_tokens = q_tokens;
    prm.heads_per_token = heads_per_token;
    prm.causal = causal ? 1 : 0;
    prm.sched_out = const_cast<int32_t*>(sched);
    prm.split_off_out = const_cast<int32_t*>(split_off);
    prm.lanes_on = lanes_enabled() ? 1 : 0;
    prm.pair = 0;
    const LineShape ls = line_shape(batch, groups, num_sm_parts, prm.lanes_on != 0);
    const int max_vb = hg == 64 ? Cfg<64>::MAX_VB : (hg == 32 ? Cfg<32>::MAX_VB : Cfg<16>::MAX_VB);
    prm.inkernel_sched = (ls.line_n <= max_vb && !(flags & ETAP_FLAG_EXTERNAL_SCHEDULE)) ? 1 : 0;
    prm.early_meta = (early_meta_enabled() && (flags & (ETAP_FLAG_EARLY_METADATA | ETAP_FLAG_INDEPENDENT_INPUTS))) ? 1 : 0;
    prm.defer_dep = defer_dep_of(flags, prm.early_meta);
    prm.fixed_cost = META_FIXED_COST;
    if (!prm.inkernel_sched && !(flags & ETAP_FLAG_EXTERNAL_SCHEDULE)) {
        // too many virtual sequences for the fused prologue: run K1 first on the same stream
        if (int rc = metadata_launch(seqlens, batch, groups, num_sm_parts, const_cast<int32_t*>(sched),
                                     const_cast<int32_t*>(split_off), stream))
            return rc;
    }
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.flags = flags;
    prm.trace = static_cast<unsigned long long*>(g_trace_buf);
    prm.span = static_cast<unsigned long long*>(g_span_buf);
    prm.state = static_cast<float*>(g_state_buf);
    prm.state_tiles = g_state_tiles;
    const bool dbg = prm.trace != nullptr || prm.state != nullptr;  // debug instantiation

    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sm_parts);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_attrs();
    if (hg == 64) {
        cfg.dynamicSmemBytes = Cfg<64>::SMEM_ALLOC;
        cfg.blockDim = dim3(Cfg<64>::THREADS);
        auto kern = dbg ? etap_mla_decode_kernel<64, true> : etap_mla_decode_kernel<64, false>;
        static int attr_rc = ensure_smem_attr(etap_mla_decode_kernel<64, false>, Cfg<64>::SMEM_ALLOC) |
                             ensure_smem_attr(etap_mla_decode_kernel<64, true>, Cfg<64>::SMEM_ALLOC);
        if (attr_rc) return attr_rc;
        ETAP_CUDA(cudaLaunchKernelEx(&cfg, kern, tm_kv, tm_q, prm));
    } else if (hg == 32) {
        cfg.dynamicSmemBytes = Cfg<32>::SMEM_ALLOC;
        cfg.blockDim = dim3(Cfg<32>::THREADS);
        auto kern = dbg ? etap_mla_decode_kernel<32, true> : etap_mla_decode_kernel<32, false>;
        static int attr_rc = ensure_smem_attr(etap_mla_decode_kernel<32, false>, Cfg<32>::SMEM_ALLOC) |
                             ensure_smem_attr(etap_mla_decode_kernel<32, true>, Cfg<32>::SMEM_ALLOC);
        if (attr_rc) return attr_rc;
        ETAP_CUDA(cudaLaunchKernelEx(&cfg, kern, tm_kv, tm_q, prm));
    } else {
        cfg.dynamicSmemBytes = Cfg<16>::SMEM_ALLOC;
        cfg.blockDim = dim3(Cfg<16>::THREADS);
        auto kern = dbg ? etap_mla_decode_kernel<16, true> : etap_mla_decode_kernel<16, false>;
        static int attr_rc = ensure_smem_attr(etap_mla_decode_kernel<16, false>, Cfg<16>::SMEM_ALLOC) |
                             ensure_smem_attr(etap_mla_decode_kernel<16, true>, Cfg<16>::SMEM_ALLOC);
        if (attr_rc) return attr_rc;
        ETAP_CUDA(cudaLaunchKernelEx(&cfg, kern, tm_kv, tm_q, prm));
    }

    if (flags & ETAP_FLAG_SKIP_COMBINE) return ETAP_OK;
    const bool closed_form = prm.inkernel_sched && ls.line_n <= 32;
    return combine_impl(split_off, batch, heads, num_sm_parts, workspace, om, stream,
                        closed_form ? seqlens : nullptr);
}

}  // namespace

namespace etap_b200 {
int peer_signal_wait(const etap_mla_peer_gather* pg, uint32_t epoch, void* stream);  // etap_peer.cu
}

extern "C" {

// FP8 (e4m3) latent cache: quantise Q into three fp8 terms (workspace), K2-FP8, K3 (16 heads
// per work unit). kv_scale: the per-tensor dequantisation scale of the cache.
int decode_impl_fp8(const void* q, const void* kv_pool8, float kv_scale, int64_t num_pages, const int32_t* block_table,
                    int max_pages_per_seq, const int32_t* seqlens, int batch, int q_tokens, int heads_per_token,
                    float scale, int causal, const int32_t* sched, const int32_t* split_off, int num_sm_parts,
                    void* workspace, const OutMap& om, unsigned flags, void* stream) {
    if (!q || !kv_pool8 || !block_table || !seqlens || !sched || !split_off || !workspace)
        return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (q_tokens < 1 || q_tokens > ETAP_MLA_MAX_Q_TOKENS)
        return fail(ETAP_ERR_SHAPE, "q_tokens must be in [1, " + std::to_string(ETAP_MLA_MAX_Q_TOKENS) + "]");
    if (heads_per_token < 1) return fail(ETAP_ERR_SHAPE, "heads must be >= 1");
    const int heads = q_tokens * heads_per_token;
    if (batch < 1 || !heads_ok(heads))
        return fail(ETAP_ERR_SHAPE, "batch >= 1 and q_tokens * heads a multiple of 16 required");
    if (num_pages < 1 || max_pages_per_seq < 1 || num_pages * PAGE > (int64_t)0x7fffffff)
        return fail(ETAP_ERR_SHAPE, "num_pages and max_pages_per_seq must be >= 1, pool below 2^31 rows");
    if (!(scale >= 0.f) || !std::isfinite(scale) || !(kv_scale > 0.f) || !std::isfinite(kv_scale))
        return fail(ETAP_ERR_SHAPE, "scale must be finite and >= 0, kv_scale finite and > 0");
    if (num_sm_parts < 1 || num_sm_parts > META_THREADS)
        return fail(ETAP_ERR_SHAPE, "num_sm_parts must be in [1, 1024]");
    if (flags & (ETAP_FLAG_EXTERNAL_SCHEDULE | ETAP_FLAG_NEGATE_RESCALE))
        return fail(ETAP_ERR_SHAPE, "FP8 path: external schedules and the rescale fault are not supported");
    // the FP8 kernel leaves partials in 16-head units; etap_mla_combine assumes the bf16
    // kernel's head group, which is 32 for these head counts
    if ((flags & ETAP_FLAG_SKIP_COMBINE) && head_group_of(heads) != fp8::HGF)
        return fail(ETAP_ERR_SHAPE, "FP8 path: SKIP_COMBINE needs a head count whose work unit is 16 heads "
                                    "(heads not a multiple of 32)");
    if (g_state_buf) return fail(ETAP_ERR_SHAPE, "FP8 path: the softmax-state dump is not supported");
    if (int rc = check_device()) return rc;

    constexpr int hg = fp8::HGF;
    const int groups = heads / hg;
    const size_t np = max_partials(batch, heads, num_sm_parts);
    uint8_t* q3 = static_cast<uint8_t*>(workspace) + q3_offset(batch, heads, num_sm_parts);
    CUtensorMap tm_kv128, tm_kv64, tm_q128, tm_q64;
    const uint64_t pool_rows = static_cast<uint64_t>(num_pages) * PAGE;
    const uint64_t q3_rows = static_cast<uint64_t>(num_sm_parts) * kfp8::NSCR * fp8::NQ;
    if (int rc = cached_map_u8(&tm_kv128, kv_pool8, pool_rows, 128, PAGE, ETAP_FP8_PAGE3D ? fp8::VCH : 0)) return rc;
    if (int rc = cached_map_u8(&tm_kv64, kv_pool8, pool_rows, 64, PAGE)) return rc;
    if (int rc = cached_map_u8(&tm_q128, q3, q3_rows, 128, fp8::NQ)) return rc;
    if (int rc = cached_map_u8(&tm_q64, q3, q3_rows, 64, fp8::NQ)) return rc;

    DecodeParams prm;
    prm.block_table = block_table;
    prm.seqlens = seqlens;
    prm.sched = sched;
    prm.split_off = split_off;
    prm.om = om;
    prm.ws_o = static_cast<float*>(workspace);
    prm.ws_lse = prm.ws_o + np * head_group_of(heads) * D_V;  // allocation layout
    prm.kv_pool = kv_pool8;
    prm.q = q;
    prm.num_pages = num_pages;
    prm.max_pages = max_pages_per_seq;
    prm.batch = batch;
    prm.heads = heads;
    prm.groups = groups;
    prm.q_tokens = q_tokens;
    prm.heads_per_token = heads_per_token;
    prm.causal = causal ? 1 : 0;
    prm.sched_out = const_cast<int32_t*>(sched);
    prm.split_off_out = const_cast<int32_t*>(split_off);
    prm.lanes_on = lanes_enabled() ? 1 : 0;
    prm.pair = 0;
    const LineShape ls = line_shape(batch, groups, num_sm_parts, prm.lanes_on != 0);
    prm.inkernel_sched = ls.line_n <= MAX_FUSED_VB ? 1 : 0;
    prm.early_meta = (early_meta_enabled() && (flags & (ETAP_FLAG_EARLY_METADATA | ETAP_FLAG_INDEPENDENT_INPUTS))) ? 1 : 0;
    prm.defer_dep = defer_dep_of(flags, prm.early_meta);
    prm.fixed_cost = FP8_FIXED_COST;
    prm.scale_log2 = scale * kv_scale * 1.4426950408889634f;
    prm.flags = flags;
    prm.trace = static_cast<unsigned long long*>(g_trace_buf);
    prm.span = static_cast<unsigned long long*>(g_span_buf);
    prm.state = nullptr;
    prm.state_tiles = 0;

    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    if (!prm.inkernel_sched)
        if (int rc = metadata_launch(seqlens, batch, groups, num_sm_parts, const_cast<int32_t*>(sched),
                                     const_cast<int32_t*>(split_off), stream, FP8_FIXED_COST))
            return rc;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(num_sm_parts);
        cfg.blockDim = dim3(NUM_THREADS);
        cfg.dynamicSmemBytes = kfp8::SMEM_ALLOC;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_attrs();
        const bool dbg = prm.trace != nullptr;
        auto kern = dbg ? etap_mla_decode_fp8_kernel<true> : etap_mla_decode_fp8_kernel<false>;
        static int attr_rc = ensure_smem_attr(etap_mla_decode_fp8_kernel<false>, kfp8::SMEM_ALLOC) |
                             ensure_smem_attr(etap_mla_decode_fp8_kernel<true>, kfp8::SMEM_ALLOC);
        if (attr_rc) return attr_rc;
        ETAP_CUDA(cudaLaunchKernelEx(&cfg, kern, tm_kv128, tm_kv64, tm_q128, tm_q64, prm, kv_scale, q3));
    }
    if (flags & ETAP_FLAG_SKIP_COMBINE) return ETAP_OK;
    const bool closed_form = prm.inkernel_sched && ls.line_n <= 32;
    return combine_impl(split_off, batch, heads, num_sm_parts, workspace, om, stream, closed_form ? seqlens : nullptr,
                        hg, FP8_FIXED_COST);
}

int etap_mla_decode_fp8(const void* q, const void* kv_pool8, float kv_scale, int64_t num_pages,
                        const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens, int batch,
                        int q_tokens, int heads_per_token, float scale, int causal, const int32_t* sched,
                        const int32_t* split_off, int num_sm_parts, void* workspace, float* out, float* lse,
                        unsigned flags, void* stream) {
    if (!out || !lse) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (!aligned16(out) || !aligned16(workspace)) return fail(ETAP_ERR_SHAPE, "out / workspace must be 16-byte aligned");
    const OutMap om = local_outmap(q_tokens * heads_per_token, out, lse);
    return decode_impl_fp8(q, kv_pool8, kv_scale, num_pages, block_table, max_pages_per_seq, seqlens, batch, q_tokens,
                           heads_per_token, scale, causal, sched, split_off, num_sm_parts, workspace, om, flags, stream);
}

int etap_mla_decode(const void* q, const void* kv_pool, int64_t num_pages,
                    const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens,
                    int batch, int q_tokens, int heads_per_token, float scale, int causal,
                    const int32_t* sched, const int32_t* split_off, int num_sm_parts,
                    void* workspace, float* out, float* lse, unsigned flags, void* stream) {
    if (!out || !lse) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (!aligned16(out) || !aligned16(workspace)) return fail(ETAP_ERR_SHAPE, "out / workspace must be 16-byte aligned");
    const OutMap om = local_outmap(q_tokens * heads_per_token, out, lse);
    return decode_impl(q, kv_pool, num_pages, block_table, max_pages_per_seq, seqlens, batch, q_tokens,
                       heads_per_token, scale, causal, sched, split_off, num_sm_parts, workspace, om,
                       flags, stream);
}

int etap_mla_decode_peer(const void* q, const void* kv_pool, int64_t num_pages,
                         const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens,
                         int batch, int q_tokens, int heads_per_token, float scale, int causal,
                         const int32_t* sched, const int32_t* split_off, int num_sm_parts,
                         void* workspace, const etap_mla_peer_gather* pg, uint32_t epoch,
                         unsigned flags, void* stream) {
    if (!pg) return fail(ETAP_ERR_SHAPE, "peer gather descriptor is NULL");
    if (pg->world < 1 || pg->world > ETAP_MLA_MAX_PEERS || pg->rank < 0 || pg->rank >= pg->world)
        return fail(ETAP_ERR_SHAPE, "peer gather: world must be in [1, 8] and 0 <= rank < world");
    if (pg->head_offset < 0 || pg->head_offset + heads_per_token > pg->heads_total)
        return fail(ETAP_ERR_SHAPE, "peer gather: head_offset + heads exceeds heads_total");
    if (flags & ETAP_FLAG_SKIP_COMBINE) return fail(ETAP_ERR_SHAPE, "peer gather: SKIP_COMBINE not allowed");
    if (epoch == 0) return fail(ETAP_ERR_SHAPE, "peer gather: epoch must be nonzero");
    if (!aligned16(workspace)) return fail(ETAP_ERR_SHAPE, "workspace must be 16-byte aligned");
    OutMap om = {};
    om.q_tokens = q_tokens;
    om.heads_per_token = heads_per_token;
    om.out_heads = pg->heads_total;
    om.out_head0 = pg->head_offset;
    om.n_out = pg->world;
    for (int r = 0; r < pg->world; ++r) {
        if (!pg->out[r] || !pg->lse[r] || !pg->flags[r])
            return fail(ETAP_ERR_SHAPE, "peer gather: NULL output / flag pointer");
        if (!aligned16(pg->out[r])) return fail(ETAP_ERR_SHAPE, "peer gather: output buffers must be 16-byte aligned");
        // own copy first: the local rows are written before the remote ones
        const int src = (pg->rank + r) % pg->world;
        om.out[r] = pg->out[src];
        om.lse[r] = pg->lse[src];
    }
    if (int rc = decode_impl(q, kv_pool, num_pages, block_table, max_pages_per_seq, seqlens, batch,
                             q_tokens, heads_per_token, scale, causal, sched, split_off, num_sm_parts,
                             workspace, om, flags, stream))
        return rc;
    return etap_b200::peer_signal_wait(pg, epoch, stream);
}

int etap_mla_append_kv(const void* kv_rows, void* kv_pool, int64_t num_pages, const int32_t* block_table,
                       int max_pages_per_seq, const int32_t* seqlens, int batch, int q_tokens, void* stream) {
    if (!kv_rows || !kv_pool || !block_table || !seqlens) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (batch < 1 || q_tokens < 1 || q_tokens > ETAP_MLA_MAX_Q_TOKENS || num_pages < 1 || max_pages_per_seq < 1)
        return fail(ETAP_ERR_SHAPE, "batch, num_pages, max_pages_per_seq >= 1 and q_tokens in [1, 8] required");
    if ((reinterpret_cast<uintptr_t>(kv_rows) | reinterpret_cast<uintptr_t>(kv_pool)) & 15)
        return fail(ETAP_ERR_SHAPE, "kv_rows / kv_pool must be 16-byte aligned");
    if (int rc = check_device()) return rc;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(batch * q_tokens);
    cfg.blockDim = dim3(D_QK * 2 / 16);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = pdl_attrs();
    ETAP_CUDA(cudaLaunchKernelEx(&cfg, etap_mla_append_kv_kernel, static_cast<const uint4*>(kv_rows),
                                 static_cast<uint4*>(kv_pool), num_pages, block_table, max_pages_per_seq,
                                 seqlens, q_tokens));
    return ETAP_OK;
}

int etap_mla_combine(const int32_t* split_off, int batch, int heads, int num_sm_parts,
                     void* workspace, float* out, float* lse, void* stream) {
    if (!split_off || !workspace || !out || !lse) return fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (!aligned16(out) || !aligned16(workspace)) return fail(ETAP_ERR_SHAPE, "out / workspace must be 16-byte aligned");
    if (batch < 1 || !heads_ok(heads) || num_sm_parts < 1)
        return fail(ETAP_ERR_SHAPE, "batch >= 1, heads a multiple of 16, num_sm_parts >= 1 required");
    int unit = 0, parts = 0;
    sched_layout(heads, num_sm_parts, &unit, &parts);
    return combine_impl(split_off, batch, heads, num_sm_parts, workspace, local_outmap(heads, out, lse), stream,
                        nullptr, unit, META_FIXED_COST, parts);
}

int etap_mla_debug_state(void* device_buf, int max_tiles) {
    g_state_buf = device_buf;
    g_state_tiles = device_buf ? max_tiles : 0;
    return ETAP_OK;
}

int etap_mla_debug_trace(void* device_buf) {
    g_trace_buf = device_buf;
    return ETAP_OK;
}

int etap_mla_debug_span(void* device_buf) {
    g_span_buf = device_buf;
    return ETAP_OK;
}

int etap_mla_debug_trace_combine(void* device_buf) {
    g_combine_trace_buf = device_buf;
    return ETAP_OK;
}

int etap_mla_selftest_umma(const void* k, const void* q, const float* p, float* s_t, float* o_t,
                           void* stream) {
    if (int rc = check_device()) return rc;
    CUtensorMap tm_k, tm_q;
    if (int rc = make_map(&tm_k, k, TILE, PAGE)) return rc;  // one 64-row page
    if (int rc = make_map(&tm_q, q, 16, 16)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static int attr_rc = ensure_smem_attr(etap_mla_selftest_kernel, Cfg<16>::SMEM_ALLOC);
    if (attr_rc) return attr_rc;
    etap_mla_selftest_kernel<<<1, NUM_THREADS, Cfg<16>::SMEM_ALLOC, st>>>(tm_k, tm_q, p, s_t, o_t);
    ETAP_CUDA(cudaGetLastError());
    return ETAP_OK;
}

}  // extern "C"

// =============================================================================================
// Tensor-pipe microbenchmark (debug): cycles for n back-to-back tcgen05.mma of one variant.
//   0: M128 N16 A K-major SW128      1: M128 N16 A MN-major SW128 (GEMM2 style)
//   2: M128 N32 A MN-major SW128     3: M64  N16 A K-major SW128
//   4: M128 N64 A K-major SW128      5: M128 N16 A MN-major, B K-major SW128
// =============================================================================================
namespace {
__global__ void __launch_bounds__(128, 1) etap_umma_bench_kernel(int variant, int n, long long* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 65536 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = tslot;
    const int mode = variant / 10;   // 0: lane-0 divergent issue, 1: warp-uniform elect in asm
    const int shape = variant % 10;
    if (threadIdx.x < 32 && (mode == 1 || threadIdx.x == 0)) {
        const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
        uint32_t idesc;
        uint64_t bd = ptx::smem_desc(b, 16, 1024, ptx::LAYOUT_SW128);
        const bool mn = (shape == 1 || shape == 2 || shape == 5);
        switch (shape) {
            case 1: idesc = ptx::idesc_bf16_f32(128, 16, 1, 1); bd = ptx::smem_desc(b, 256, 128, ptx::LAYOUT_NONE); break;
            case 2: idesc = ptx::idesc_bf16_f32(128, 32, 1, 1); bd = ptx::smem_desc(b, 512, 128, ptx::LAYOUT_NONE); break;
            case 3: idesc = ptx::idesc_bf16_f32(64, 16, 0, 0); break;
            case 4: idesc = ptx::idesc_bf16_f32(128, 64, 0, 0); break;
            case 5: idesc = ptx::idesc_bf16_f32(128, 16, 1, 0); break;
            case 6: idesc = ptx::idesc_bf16_f32(128, 256, 0, 0); break;
            default: idesc = ptx::idesc_bf16_f32(128, 16, 0, 0); break;
        }
        const uint64_t ad0 = mn ? ptx::smem_desc(a, 16384, 1024, ptx::LAYOUT_SW128)
                                : ptx::smem_desc(a, 16, 1024, ptx::LAYOUT_SW128);
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 1) __syncwarp();
            const long long t0 = clock64();
            if (mode == 0) {
                for (int i = 0; i < n; ++i) {
                    const uint64_t ad = ad0 + (mn ? (uint64_t)((i & 7) * 128) : (uint64_t)((i & 3) * 2));
                    ptx::umma_f16(tbase, ad, bd, idesc, i > 0);
                }
            } else {
                for (int i = 0; i < n; i += 4) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t ad = ad0 + (mn ? (uint64_t)(j * 128) : (uint64_t)(j * 2));
                        ptx::umma_f16_elect(tbase, ad, bd, idesc, (i + j) > 0);
                    }
                }
            }
            const long long t1 = clock64();
            if (mode == 0) ptx::umma_commit(&bar); else ptx::umma_commit_elect(&bar);
            ptx::mbar_wait(&bar, rep & 1);
            const long long t2 = clock64();
            if (rep == 1 && (threadIdx.x == 0)) { out[0] = t1 - t0; out[1] = t2 - t0; }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}
}  // namespace

extern "C" int etap_mla_umma_bench(int variant, int n, long long* out_dev, int grid) {
    cudaFuncSetAttribute(etap_umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    etap_umma_bench_kernel<<<grid, 128, 66 * 1024>>>(variant, n, out_dev);
    ETAP_CUDA(cudaGetLastError());
    return ETAP_OK;
}

// =============================================================================================
// PDL producer (tests): triggers its dependents at entry, then writes dst after a delay — the
// shape of a serving-stack kernel that updates seqlens / block_table right before the decode.
// =============================================================================================
namespace {
__global__ void etap_pdl_writer_kernel(int32_t* dst, const int32_t* src, int n, int delay_ns) {
    ptx::grid_dep_wait();    // ordered after the kernel before it
    ptx::grid_dep_launch();  // ... and lets the next kernel (the decode) start right away
    const uint64_t t0 = ptx::global_timer_ns();
    while (ptx::global_timer_ns() - t0 < static_cast<uint64_t>(delay_ns)) __nanosleep(500);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
}  // namespace

extern "C" int etap_mla_debug_pdl_write(int32_t* dst, const int32_t* src, int n, int delay_ns, void* stream) {
    if (!dst || !src || n < 0 || delay_ns < 0) return fail(ETAP_ERR_SHAPE, "bad argument");
    if (int rc = check_device()) return rc;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(128);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ETAP_CUDA(cudaLaunchKernelEx(&cfg, etap_pdl_writer_kernel, dst, src, n, delay_ns));
    return ETAP_OK;
}

// =============================================================================================
// Streaming microbenchmark (debug): the decode kernel's TMA access pattern (9 boxes of
// 64 rows x 64 cols per page, tile-level full barriers, 24-slot ring) with no compute, to
// measure the attainable HBM read rate. Each CTA streams pages [cta*ppc, (cta+1)*ppc).
// =============================================================================================
namespace {
__global__ void __launch_bounds__(64, 1) etap_stream_bench_kernel(const __grid_constant__ CUtensorMap tm_kv,
                                                                   int pages_per_cta, int nslot) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
    uint64_t* done = full + NTB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NTB; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&done[i], 1); }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int p0 = blockIdx.x * pages_per_cta;
    const uint32_t tiles_in_ring = (uint32_t)nslot / NCHUNK;  // whole tiles that fit
    if (warp == 0) {
        const uint64_t pol = ptx::policy_evict_first();
        for (uint32_t gt = 0; gt < (uint32_t)pages_per_cta; ++gt) {
            if (gt >= tiles_in_ring)
                ptx::mbar_wait(&done[(gt - tiles_in_ring) % NTB], ((gt - tiles_in_ring) / NTB) & 1);
            if (lane == 0) {
                ptx::mbar_arrive_expect_tx(&full[gt % NTB], NCHUNK * SLOT_BYTES);
                const uint32_t base = (gt % tiles_in_ring) * NCHUNK;
                for (int c = 0; c < NCHUNK; ++c)
                    ptx::tma_load_2d(smem + (base + c) * SLOT_BYTES, &tm_kv, &full[gt % NTB], c * 64,
                                     (p0 + gt) * PAGE, pol);
            }
            __syncwarp();
        }
    } else {
        for (uint32_t gt = 0; gt < (uint32_t)pages_per_cta; ++gt) {
            ptx::mbar_wait(&full[gt % NTB], (gt / NTB) & 1);
            if (lane == 0) ptx::mbar_arrive(&done[gt % NTB]);
            __syncwarp();
        }
    }
}
}  // namespace

namespace {
// Cluster-of-two variant: both CTAs stream the same pages (as the two head-group lanes of a
// 128-head decode do); each issues every other box with .multicast::cluster into both CTAs, so
// every SM still receives whole pages but generates half the requests. A slot is reloaded once
// both CTAs released it (remote arrive on the peer's `done`).
__global__ void __launch_bounds__(64, 1) etap_stream_bench_mc_kernel(const __grid_constant__ CUtensorMap tm_kv,
                                                                      int pages_per_cta, int nslot) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
    uint64_t* done = full + NTB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NTB; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&done[i], 2); }
        ptx::fence_mbar_init();
    }
    ptx::cluster_sync_all();
    const int p0 = (blockIdx.x >> 1) * pages_per_cta;
    const uint32_t tiles_in_ring = (uint32_t)nslot / NCHUNK;
    if (warp == 0) {
        const uint64_t pol = ptx::policy_evict_first();
        for (uint32_t gt = 0; gt < (uint32_t)pages_per_cta; ++gt) {
            if (gt >= tiles_in_ring)
                ptx::mbar_wait(&done[(gt - tiles_in_ring) % NTB], ((gt - tiles_in_ring) / NTB) & 1);
            if (lane == 0) {
                ptx::mbar_arrive_expect_tx(&full[gt % NTB], NCHUNK * SLOT_BYTES);
                const uint32_t base = (gt % tiles_in_ring) * NCHUNK;
                for (int c = static_cast<int>(rank); c < NCHUNK; c += 2)
                    ptx::tma_load_2d_mc(smem + (base + c) * SLOT_BYTES, &tm_kv, &full[gt % NTB], c * 64,
                                        (p0 + gt) * PAGE, 0x3, pol);
            }
            __syncwarp();
        }
    } else {
        for (uint32_t gt = 0; gt < (uint32_t)pages_per_cta; ++gt) {
            ptx::mbar_wait(&full[gt % NTB], (gt / NTB) & 1);
            if (lane == 0) {
                ptx::mbar_arrive(&done[gt % NTB]);
                ptx::mbar_arrive_cluster(&done[gt % NTB], rank ^ 1u);
            }
            __syncwarp();
        }
    }
    ptx::cluster_sync_all();  // no remote arrive may target an exited CTA
}
}  // namespace

extern "C" int etap_mla_stream_bench_mc(const void* kv_pool, int64_t num_pages, int pages_per_cta,
                                        int grid, int nslot, void* stream) {
    if (nslot < NCHUNK || nslot * SLOT_BYTES > 200 * 1024 || grid % 2) return fail(ETAP_ERR_SHAPE, "bad nslot/grid");
    CUtensorMap tm;
    if (int rc = make_map(&tm, kv_pool, static_cast<uint64_t>(num_pages) * PAGE, PAGE)) return rc;
    cudaFuncSetAttribute(etap_stream_bench_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 202 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = 202 * 1024;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ETAP_CUDA(cudaLaunchKernelEx(&cfg, etap_stream_bench_mc_kernel, tm, pages_per_cta, nslot));
    return ETAP_OK;
}

namespace {
// Whole-page boxes: one 3-D TMA instruction per page instead of nine 2-D chunk boxes.
__global__ void __launch_bounds__(64, 1) etap_stream_bench_page_kernel(const __grid_constant__ CUtensorMap tm_pg,
                                                                        int pages_per_cta, int nslot, int box_chunks) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
    uint64_t* done = full + NTB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NTB; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&done[i], 1); }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int p0 = blockIdx.x * pages_per_cta;
    const uint32_t tiles_in_ring = (uint32_t)nslot / NCHUNK;
    if (warp == 0) {
        const uint64_t pol = ptx::policy_evict_first();
        for (uint32_t gt = 0; gt < (uint32_t)pages_per_cta; ++gt) {
            if (gt >= tiles_in_ring)
                ptx::mbar_wait(&done[(gt - tiles_in_ring) % NTB], ((gt - tiles_in_ring) / NTB) & 1);
            if (lane == 0) {
                ptx::mbar_arrive_expect_tx(&full[gt % NTB], NCHUNK * SLOT_BYTES);
                const uint32_t base = (gt % tiles_in_ring) * NCHUNK;
                for (int c = 0; c < NCHUNK; c += box_chunks)
                    ptx::tma_load_3d(smem + (base + c) * SLOT_BYTES, &tm_pg, &full[gt % NTB], 0, (p0 + gt) * PAGE, c, pol);
            }
            __syncwarp();
        }
    } else {
        for (uint32_t gt = 0; gt < (uint32_t)pages_per_cta; ++gt) {
            ptx::mbar_wait(&full[gt % NTB], (gt / NTB) & 1);
            if (lane == 0) ptx::mbar_arrive(&done[gt % NTB]);
            __syncwarp();
        }
    }
}
}  // namespace

extern "C" int etap_mla_stream_bench_page(const void* kv_pool, int64_t num_pages, int pages_per_cta,
                                          int grid, int nslot, int box_chunks, void* stream) {
    if (nslot < NCHUNK || nslot * SLOT_BYTES > 200 * 1024 || box_chunks < 1 || NCHUNK % box_chunks)
        return fail(ETAP_ERR_SHAPE, "bad nslot / box_chunks");
    CUtensorMap tm;
    if (int rc = make_map_page3d(&tm, kv_pool, static_cast<uint64_t>(num_pages) * PAGE, box_chunks)) return rc;
    cudaFuncSetAttribute(etap_stream_bench_page_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 202 * 1024);
    etap_stream_bench_page_kernel<<<grid, 64, 202 * 1024, static_cast<cudaStream_t>(stream)>>>(tm, pages_per_cta, nslot,
                                                                                                   box_chunks);
    ETAP_CUDA(cudaGetLastError());
    return ETAP_OK;
}

extern "C" int etap_mla_stream_bench(const void* kv_pool, int64_t num_pages, int pages_per_cta,
                                     int grid, int nslot, void* stream) {
    if (nslot < NCHUNK || nslot * SLOT_BYTES > 200 * 1024) return fail(ETAP_ERR_SHAPE, "bad nslot");
    CUtensorMap tm;
    if (int rc = make_map(&tm, kv_pool, static_cast<uint64_t>(num_pages) * PAGE, PAGE)) return rc;
    cudaFuncSetAttribute(etap_stream_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 202 * 1024);
    etap_stream_bench_kernel<<<grid, 64, 202 * 1024, static_cast<cudaStream_t>(stream)>>>(tm, pages_per_cta, nslot);
    ETAP_CUDA(cudaGetLastError());
    return ETAP_OK;
}
