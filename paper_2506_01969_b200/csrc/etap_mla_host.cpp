// SPDX-License-Identifier: Apache-2.0
// Host-buffer entry points of the C-ABI (include/etap_mla.h):
//   * etap_mla_host_ctx_* / etap_mla_host_decode — end-to-end call with host buffers
//     (H2D copies, K1/K2/K3, D2H copies), the path the `e2e` bench number measures;
//   * etap_mla_run_etap_f64 — binary64 row-major matrices exactly as stored in
//     etaplab::AttentionProblem (/root/reference/proj/include/etaplab/attention.hpp:15-25),
//     mirroring run_etap's argument meaning and error behaviour (etap.cpp:102-106).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/etap_mla.h"

namespace etap_b200 {
int host_fail(int code, const char* msg);  // etap_mla.cu: sets etap_mla_last_error()
int ingest_step(const void* q_src, void* q_dst, int nq_rows, const void* rows, void* pool, int64_t num_pages,
                const int32_t* block_table, int max_pages, const int32_t* seqlens_src, int32_t* seqlens_dst,
                int batch, int q_tokens, void* stream);  // etap_mla.cu
}
using etap_b200::host_fail;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t bytes) {
        n = bytes;
        return cudaMalloc(&p, bytes > 0 ? bytes : 16);
    }
};

// Round a binary64 value to the nearest bfloat16 (ties to even) directly, without the
// double -> float -> bf16 double rounding; returns the 16-bit pattern. Reference form, used for
// the bf16 subnormal range only (frexp / nearbyint / ldexp cost ~40 ns per element).
uint16_t bf16_bits_rne_slow(double x) {
    if (std::isnan(x)) return 0x7FC0;
    const double ax = std::fabs(x);
    float f;
    if (ax == 0.0) {
        f = static_cast<float>(x);
    } else {
        int e = 0;
        std::frexp(ax, &e);              // ax = m * 2^e, m in [0.5, 1)
        int q = e - 8;                   // 8 significant bits
        if (q < -133) q = -133;          // bf16 subnormal quantum
        const double r = std::nearbyint(std::ldexp(ax, -q));  // ties-to-even
        const double v = std::ldexp(r, q);
        // largest finite bf16 = (2 - 2^-7) * 2^127
        f = v > 3.3895313892515355e38 ? INFINITY : static_cast<float>(v);
        if (x < 0) f = -f;
    }
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return static_cast<uint16_t>(u >> 16);
}

// The same rounding on the bit pattern: for |x| >= 2^-126 (bf16 normal range) rebias the
// exponent, add the ties-to-even increment at bit 45 and shift; a carry out of the mantissa
// bumps the exponent (to infinity past the largest finite bf16). Bit-identical to the reference
// form (CPU test against it over random, boundary and tie values).
inline uint16_t bf16_bits_rne(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    const uint16_t sign = static_cast<uint16_t>((u >> 48) & 0x8000u);
    const uint64_t m = u & 0x7FFFFFFFFFFFFFFFull;
    if (m > 0x7FF0000000000000ull) return 0x7FC0;  // NaN
    const int64_t e = static_cast<int64_t>(m >> 52) - 1023;
    if (e < -126) return bf16_bits_rne_slow(x);    // zero and the bf16 subnormal range
    if (e > 127) return sign | 0x7F80;             // overflow and infinity
    uint64_t t = m - (static_cast<uint64_t>(1023 - 127) << 52);
    t += (1ull << 44) - 1 + ((t >> 45) & 1);
    const uint64_t r = t >> 45;
    return sign | static_cast<uint16_t>(r >= 0x7F80 ? 0x7F80 : r);
}

// for (i in [0, n)) f(i) over up to 16 host threads (large problems only)
template <class F>
void parallel_for(int64_t n, const F& f) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int64_t nt = n < (1 << 16) ? 1 : static_cast<int64_t>(hw);
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) f(i);
        });
    for (auto& x : th) x.join();
}

// Device address of page-locked (cudaHostAlloc / cudaHostRegister) host memory, or nullptr
// for pageable memory: the serving step then reads / writes it directly over PCIe.
void* mapped(const void* host) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    // page-locked memory of another device's context may not be mapped here: copy path then
    return (a.type == cudaMemoryTypeHost && a.devicePointer && a.device == dev) ? a.devicePointer : nullptr;
}

}  // namespace

struct etap_mla_host_ctx {
    int batch = 0, heads = 0, max_pages = 0, num_sm_parts = 0;
    int64_t num_pages = 0;
    cudaStream_t stream = nullptr;
    DevBuf q, kv, bt, sl, out, lse, sched, split_off, ws, rows;
};

extern "C" {

int etap_mla_host_ctx_create(int batch, int heads, int64_t num_pages, int max_pages_per_seq,
                             etap_mla_host_ctx** ctx) {
    if (!ctx) return host_fail(ETAP_ERR_SHAPE, "ctx is NULL");
    *ctx = nullptr;
    if (batch < 1 || heads < ETAP_MLA_HEAD_GROUP || heads % ETAP_MLA_HEAD_GROUP != 0 ||
        num_pages < 1 || max_pages_per_seq < 1)
        return host_fail(ETAP_ERR_SHAPE, "batch >= 1, heads a multiple of 16, pages >= 1 required");
    auto* c = new etap_mla_host_ctx();
    c->batch = batch;
    c->heads = heads;
    c->num_pages = num_pages;
    c->max_pages = max_pages_per_seq;
    int dev = 0;
    size_t sched_n = 0, so_n = 0, ws_n = 0;
    cudaError_t e = cudaGetDevice(&dev);
    int rc = e == cudaSuccess ? etap_mla_num_sm_parts(dev, &c->num_sm_parts)
                              : host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    if (!rc) rc = etap_mla_sched_ints(batch, heads, c->num_sm_parts, &sched_n, &so_n);
    if (!rc) rc = etap_mla_workspace_bytes(batch, heads, c->num_sm_parts, &ws_n);
    if (!rc) {
        const size_t rows = static_cast<size_t>(batch) * heads;
        if (c->q.alloc(rows * ETAP_MLA_D_QK * 2) ||
            c->kv.alloc(static_cast<size_t>(num_pages) * ETAP_MLA_PAGE_ROWS * ETAP_MLA_D_QK * 2) ||
            c->bt.alloc(static_cast<size_t>(batch) * max_pages_per_seq * 4) ||
            c->sl.alloc(static_cast<size_t>(batch) * 4) || c->out.alloc(rows * ETAP_MLA_D_V * 4) ||
            c->lse.alloc(rows * 4) || c->sched.alloc(sched_n * 4) ||
            c->split_off.alloc(so_n * 4) || c->ws.alloc(ws_n) ||
            c->rows.alloc(static_cast<size_t>(batch) * ETAP_MLA_D_QK * 2) ||
            cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) ||
            cudaMemset(c->ws.p, 0, c->ws.n) ||  // combine flags / counters start at zero
            cudaMemset(c->sched.p, 0, c->sched.n))  // read as a prefetch hint before the first decode
            rc = host_fail(ETAP_ERR_CUDA, "device allocation failed");
    }
    if (rc) {
        delete c;
        return rc;
    }
    *ctx = c;
    return ETAP_OK;
}

int etap_mla_host_decode(etap_mla_host_ctx* c, const void* q_host, const void* kv_pool_host,
                         const int32_t* block_table_host, const int32_t* seqlens_host,
                         float scale, unsigned flags, float* out_host, float* lse_host) {
    if (!c || !q_host || !kv_pool_host || !block_table_host || !seqlens_host || !out_host ||
        !lse_host)
        return host_fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    cudaStream_t s = c->stream;
    if (cudaMemcpyAsync(c->q.p, q_host, c->q.n, cudaMemcpyHostToDevice, s) ||
        cudaMemcpyAsync(c->kv.p, kv_pool_host, c->kv.n, cudaMemcpyHostToDevice, s) ||
        cudaMemcpyAsync(c->bt.p, block_table_host, c->bt.n, cudaMemcpyHostToDevice, s) ||
        cudaMemcpyAsync(c->sl.p, seqlens_host, c->sl.n, cudaMemcpyHostToDevice, s))
        return host_fail(ETAP_ERR_CUDA, "host->device copy failed");
    int rc = etap_mla_metadata(static_cast<int32_t*>(c->sl.p), c->batch, c->heads,
                               c->num_sm_parts, static_cast<int32_t*>(c->sched.p),
                               static_cast<int32_t*>(c->split_off.p), s);
    if (rc) return rc;
    rc = etap_mla_decode(c->q.p, c->kv.p, c->num_pages, static_cast<int32_t*>(c->bt.p),
                         c->max_pages, static_cast<int32_t*>(c->sl.p), c->batch, 1, c->heads,
                         scale, 1, static_cast<int32_t*>(c->sched.p),
                         static_cast<int32_t*>(c->split_off.p), c->num_sm_parts, c->ws.p,
                         static_cast<float*>(c->out.p), static_cast<float*>(c->lse.p), flags, s);
    if (rc) return rc;
    if (cudaMemcpyAsync(out_host, c->out.p, c->out.n, cudaMemcpyDeviceToHost, s) ||
        cudaMemcpyAsync(lse_host, c->lse.p, c->lse.n, cudaMemcpyDeviceToHost, s) ||
        cudaStreamSynchronize(s))
        return host_fail(ETAP_ERR_CUDA, "device->host copy / synchronize failed");
    return ETAP_OK;
}

int etap_mla_host_ctx_load(etap_mla_host_ctx* c, const void* kv_pool_host, const int32_t* block_table_host) {
    if (!c || !kv_pool_host || !block_table_host) return host_fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (cudaMemcpyAsync(c->kv.p, kv_pool_host, c->kv.n, cudaMemcpyHostToDevice, c->stream) ||
        cudaMemcpyAsync(c->bt.p, block_table_host, c->bt.n, cudaMemcpyHostToDevice, c->stream) ||
        cudaStreamSynchronize(c->stream))
        return host_fail(ETAP_ERR_CUDA, "host->device copy of the cache failed");
    return ETAP_OK;
}

// One serving decode step against the resident cache: the per-step inputs cross PCIe (Q, the
// new latent row of every sequence, seqlens), the cache does not.
int etap_mla_host_decode_step(etap_mla_host_ctx* c, const void* q_host, const void* kv_rows_host,
                              const int32_t* seqlens_host, float scale, unsigned flags, float* out_host,
                              float* lse_host) {
    if (!c || !q_host || !kv_rows_host || !seqlens_host || !out_host || !lse_host)
        return host_fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    cudaStream_t s = c->stream;
    int rc;
    // Page-locked host buffers are read / written in place over PCIe: one ingest kernel for Q,
    // the new rows and seqlens, and the decode's O / LSE stores go straight to host memory
    // (no copy engine round trips). Pageable buffers take the copy path.
    const void* q_m = mapped(q_host);
    const void* rows_m = mapped(kv_rows_host);
    const void* sl_m = mapped(seqlens_host);
    float* out_m = static_cast<float*>(mapped(out_host));
    float* lse_m = static_cast<float*>(mapped(lse_host));
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (q_m && rows_m && sl_m && al16(q_m) && al16(rows_m)) {
        rc = etap_b200::ingest_step(q_m, c->q.p, c->batch * c->heads, rows_m, c->kv.p, c->num_pages,
                                    static_cast<int32_t*>(c->bt.p), c->max_pages, static_cast<const int32_t*>(sl_m),
                                    static_cast<int32_t*>(c->sl.p), c->batch, 1, s);
        if (rc) return rc;
    } else {
        if (cudaMemcpyAsync(c->q.p, q_host, c->q.n, cudaMemcpyHostToDevice, s) ||
            cudaMemcpyAsync(c->rows.p, kv_rows_host, c->rows.n, cudaMemcpyHostToDevice, s) ||
            cudaMemcpyAsync(c->sl.p, seqlens_host, c->sl.n, cudaMemcpyHostToDevice, s))
            return host_fail(ETAP_ERR_CUDA, "host->device copy failed");
        rc = etap_mla_append_kv(c->rows.p, c->kv.p, c->num_pages, static_cast<int32_t*>(c->bt.p), c->max_pages,
                                static_cast<int32_t*>(c->sl.p), c->batch, 1, s);
        if (rc) return rc;
    }
    const bool direct_out = out_m && lse_m && al16(out_m);
    // the schedule is computed inside the decode kernel (no K1 launch)
    rc = etap_mla_decode(c->q.p, c->kv.p, c->num_pages, static_cast<int32_t*>(c->bt.p), c->max_pages,
                         static_cast<int32_t*>(c->sl.p), c->batch, 1, c->heads, scale, 1,
                         static_cast<int32_t*>(c->sched.p), static_cast<int32_t*>(c->split_off.p),
                         c->num_sm_parts, c->ws.p, direct_out ? out_m : static_cast<float*>(c->out.p),
                         direct_out ? lse_m : static_cast<float*>(c->lse.p), flags, s);
    if (rc) return rc;
    if (!direct_out && (cudaMemcpyAsync(out_host, c->out.p, c->out.n, cudaMemcpyDeviceToHost, s) ||
                        cudaMemcpyAsync(lse_host, c->lse.p, c->lse.n, cudaMemcpyDeviceToHost, s)))
        return host_fail(ETAP_ERR_CUDA, "device->host copy failed");
    if (cudaStreamSynchronize(s)) return host_fail(ETAP_ERR_CUDA, "synchronize failed");
    return ETAP_OK;
}

void etap_mla_host_ctx_destroy(etap_mla_host_ctx* c) {
    if (!c) return;
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// The reference's BlockHook stream (tiled_standard.hpp:32-40, called per (query block, KV
// block) at etap.cpp:128) reconstructed from the device's softmax-state dump. One decode of a
// batch of "prefix sequences" that share the KV pages through the block table: sequence j
// sees rows [0, R_j), R_j = min((j+1) b_c, n_kv), and its last tile's state IS the state after
// KV block j (the running max / sum over exactly those rows). When b_c is a multiple of 64
// every R_j is a tile boundary of the full problem and one sequence suffices (its per-tile
// states at the boundaries). num_sm_parts = 1: every sequence is one split, the reference's
// serial chain of blocks.
static int run_etap_f64_impl(const double* q, int64_t n_q, const double* k, int64_t n_kv,
                             int64_t d_qk, const double* v, int64_t d_v, double scale, int precision,
                             int64_t b_r, int64_t b_c, int64_t stages, unsigned flags, double* o,
                             double* l, double* state) {
    // argument validation mirrors run_etap / make_problem (etap.cpp:104-106,
    // attention.cpp:11-19): these are the cases the reference rejects with invalid_argument
    if (b_r < 1 || b_c < 1 || stages < 1)
        return host_fail(ETAP_ERR_SHAPE, "tile config fields must be >= 1");
    if (!q || !k || !v || !o || !l || n_q < 1 || n_kv < 1)
        return host_fail(ETAP_ERR_SHAPE, "matrix dimensions must be >= 1");
    if (precision != ETAP_PRECISION_EXACT64)
        return host_fail(ETAP_ERR_SHAPE,
                         "GPU ETAP path computes bf16 x bf16 -> fp32 on exact64-stored operands; the fp32 / "
                         "fp16emu emulation modes (Precision, matrix.hpp:22) are not mapped");
    if (d_qk != ETAP_MLA_D_QK || d_v != ETAP_MLA_D_V)
        return host_fail(ETAP_ERR_SHAPE, "GPU ETAP path is MLA decode: d_qk=576, d_v=512");
    if (!(scale >= 0.0) || !std::isfinite(scale))
        return host_fail(ETAP_ERR_SHAPE, "scale must be finite and >= 0");
    if (n_kv > (int64_t)1 << 30) return host_fail(ETAP_ERR_SHAPE, "n_kv too large");
    // MLA aliasing: V must be the first 512 columns of the latent KV rows
    std::vector<uint8_t> v_ok(static_cast<size_t>(n_kv));
    parallel_for(n_kv, [&](int64_t i) { v_ok[i] = std::memcmp(v + i * d_v, k + i * d_qk, sizeof(double) * d_v) == 0; });
    if (std::find(v_ok.begin(), v_ok.end(), uint8_t{0}) != v_ok.end())
        return host_fail(ETAP_ERR_SHAPE, "V must be the first 512 columns of K (MLA aliasing)");

    const int heads = static_cast<int>((n_q + ETAP_MLA_HEAD_GROUP - 1) / ETAP_MLA_HEAD_GROUP) *
                      ETAP_MLA_HEAD_GROUP;
    const int64_t pages = (n_kv + ETAP_MLA_PAGE_ROWS - 1) / ETAP_MLA_PAGE_ROWS;
    if (pages > 0x7fffffff) return host_fail(ETAP_ERR_SHAPE, "too many pages");
    const int64_t t_c = (n_kv + b_c - 1) / b_c;
    // hook replay: prefix sequences unless every block boundary is a tile boundary
    const bool prefixes = state && (b_c % ETAP_MLA_PAGE_ROWS) != 0 && t_c > 1;
    const int64_t batch = prefixes ? t_c : 1;
    if (prefixes && (batch * (heads / ETAP_MLA_HEAD_GROUP) > 2048 || batch * pages > ((int64_t)1 << 26)))
        return host_fail(ETAP_ERR_SHAPE, "BlockHook replay with b_c not a multiple of 64 is limited to "
                                         "2048 (KV blocks x 16-head groups) and 2^26 prefix tiles");
    std::vector<uint16_t> qb(static_cast<size_t>(batch) * heads * d_qk, 0);
    std::vector<uint16_t> kvb(static_cast<size_t>(pages) * ETAP_MLA_PAGE_ROWS * d_qk, 0);
    for (int64_t i = 0; i < n_q * d_qk; ++i) qb[i] = bf16_bits_rne(q[i]);
    for (int64_t b = 1; b < batch; ++b)
        std::memcpy(qb.data() + b * heads * d_qk, qb.data(), sizeof(uint16_t) * heads * d_qk);
    parallel_for(n_kv, [&](int64_t r) {
        for (int64_t c = 0; c < d_qk; ++c) kvb[r * d_qk + c] = bf16_bits_rne(k[r * d_qk + c]);
    });
    std::vector<int32_t> bt(static_cast<size_t>(batch) * pages), sl(batch);
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t i = 0; i < pages; ++i) bt[b * pages + i] = static_cast<int32_t>(i);
        sl[b] = static_cast<int32_t>(prefixes ? std::min((b + 1) * b_c, n_kv) : n_kv);
    }
    std::vector<float> of(static_cast<size_t>(batch) * heads * d_v), lf(static_cast<size_t>(batch) * heads);

    // one cached context per host thread and device, rebuilt when the shape changes: a
    // reference harness calls run_etap once per problem, and per-call cudaMalloc / cudaFree /
    // stream creation would dominate a decode that takes microseconds
    thread_local struct CtxCache {
        etap_mla_host_ctx* ctx = nullptr;
        int dev = -1, batch = 0, heads = 0;
        int64_t pages = 0;
        ~CtxCache() { etap_mla_host_ctx_destroy(ctx); }
    } cache;
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return host_fail(ETAP_ERR_CUDA, "no CUDA device");
    int rc = ETAP_OK;
    if (!cache.ctx || cache.dev != dev || cache.batch != batch || cache.heads != heads || cache.pages != pages) {
        etap_mla_host_ctx_destroy(cache.ctx);
        cache.ctx = nullptr;
        rc = etap_mla_host_ctx_create(static_cast<int>(batch), heads, pages, static_cast<int>(pages), &cache.ctx);
        if (rc) return rc;
        cache.dev = dev;
        cache.batch = static_cast<int>(batch);
        cache.heads = heads;
        cache.pages = pages;
    }
    etap_mla_host_ctx* ctx = cache.ctx;
    int full_parts = 0;
    if (int e = etap_mla_num_sm_parts(dev, &full_parts)) return e;
    ctx->num_sm_parts = full_parts;
    float* st_dev = nullptr;
    int hg = ETAP_MLA_HEAD_GROUP;
    if (int e = etap_mla_head_group(heads, &hg)) return e;
    const int groups = heads / hg;
    const size_t st_n = static_cast<size_t>(groups) * batch * pages * 4 * hg;
    if (state) {
        ctx->num_sm_parts = 1;  // one split per sequence: the reference's serial chain of KV blocks
        if (cudaMalloc(&st_dev, st_n * sizeof(float)) != cudaSuccess)
            return host_fail(ETAP_ERR_CUDA, "state buffer allocation failed");
        cudaMemset(st_dev, 0, st_n * sizeof(float));
        etap_mla_debug_state(st_dev, static_cast<int>(pages));
    }
    rc = etap_mla_host_decode(ctx, qb.data(), kvb.data(), bt.data(), sl.data(), static_cast<float>(scale), flags,
                              of.data(), lf.data());
    if (state) {
        etap_mla_debug_state(nullptr, 0);
        std::vector<float> sf(st_n);
        if (!rc && cudaMemcpy(sf.data(), st_dev, st_n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = host_fail(ETAP_ERR_CUDA, "state copy failed");
        cudaFree(st_dev);
        // dump [vb = g * batch + b][tile][4][hg] (m_old, m, rescale, l; natural-log units) ->
        // state[j][4][n_q] after KV block j: m and l from the tile that ends block j; m_old is
        // the previous block's m and the block's rescale exp(m_old - m) (0 on the first block,
        // m_old = -inf), as block_update_impl reports them (etap.cpp:40-47)
        if (!rc)
            for (int64_t j = 0; j < t_c; ++j) {
                const int64_t rows_j = std::min((j + 1) * b_c, n_kv);
                const int64_t seq = prefixes ? j : 0;
                const int64_t tile = (rows_j + ETAP_MLA_PAGE_ROWS - 1) / ETAP_MLA_PAGE_ROWS - 1;
                for (int64_t i = 0; i < n_q; ++i) {
                    const int g = static_cast<int>(i / hg), h = static_cast<int>(i % hg);
                    const float* st = sf.data() + ((static_cast<size_t>(g) * batch + seq) * pages + tile) * 4 * hg;
                    const double m_old = j == 0 ? -INFINITY : state[((j - 1) * 4 + 1) * n_q + i];
                    double m = st[hg + h], lsum = st[3 * hg + h];
                    // prefix sequences are separate runs: a tile's S^T may differ in the last fp32
                    // bit with the tile's ring parity (GEMM1 chunk order), so the running max is
                    // carried over explicitly (m = max(m_old, max over block j), the definition)
                    // and l re-expressed relative to it
                    if (m_old > m) {
                        lsum *= std::exp(m - m_old);
                        m = m_old;
                    }
                    state[(j * 4 + 0) * n_q + i] = m_old;
                    state[(j * 4 + 1) * n_q + i] = m;
                    state[(j * 4 + 2) * n_q + i] = j == 0 ? 0.0 : std::exp(m_old - m);
                    state[(j * 4 + 3) * n_q + i] = lsum;
                }
            }
    }
    ctx->num_sm_parts = full_parts;
    if (rc) return rc;
    // the full problem is the last prefix sequence
    const size_t last = static_cast<size_t>(batch - 1) * heads;
    for (int64_t i = 0; i < n_q * d_v; ++i) o[i] = static_cast<double>(of[last * d_v + i]);
    for (int64_t i = 0; i < n_q; ++i) l[i] = static_cast<double>(lf[last + i]);
    return ETAP_OK;
}

int etap_mla_debug_bf16_rne(const double* x, int64_t n, uint16_t* out, int reference_form) {
    if ((!x || !out) && n > 0) return host_fail(ETAP_ERR_SHAPE, "NULL buffer");
    for (int64_t i = 0; i < n; ++i) out[i] = reference_form ? bf16_bits_rne_slow(x[i]) : bf16_bits_rne(x[i]);
    return ETAP_OK;
}

int etap_mla_run_etap_f64(const double* q, int64_t n_q, const double* k, int64_t n_kv, int64_t d_qk,
                          const double* v, int64_t d_v, double scale, int precision, int64_t b_r, int64_t b_c,
                          int64_t stages, unsigned flags, double* o, double* l) {
    return run_etap_f64_impl(q, n_q, k, n_kv, d_qk, v, d_v, scale, precision, b_r, b_c, stages, flags, o, l,
                             nullptr);
}

int etap_mla_run_etap_f64_state(const double* q, int64_t n_q, const double* k, int64_t n_kv, int64_t d_qk,
                                const double* v, int64_t d_v, double scale, int precision, int64_t b_c,
                                unsigned flags, double* o, double* l, double* state) {
    if (!state) return host_fail(ETAP_ERR_SHAPE, "state is NULL");
    return run_etap_f64_impl(q, n_q, k, n_kv, d_qk, v, d_v, scale, precision, 1, b_c, 1, flags, o, l, state);
}

}  // extern "C"
