/* SPDX-License-Identifier: Apache-2.0
 *
 * etap_mla.h — C-ABI of the B200 (sm_100a) ETAP MLA decode path.
 *
 * This is the drop-in boundary under the reference's hot path
 *   etaplab::run_etap(const AttentionProblem&, const TileConfig&, const BlockHook&,
 *                     const EtapFaults&)          (reference: proj/include/etaplab/etap.hpp:47-48,
 *                                                   proj/src/etap.cpp:102-148)
 * The reference has no C-ABI and no device boundary; each entry point below
 * names the reference interface whose work it takes over.
 *
 * Conventions
 *   - Plain pointers and sizes only. "device" pointers are CUDA device pointers; "host"
 *     pointers are host memory (pinned recommended). The caller owns every buffer.
 *   - The device entry points allocate nothing and are stream-ordered on `stream`
 *     (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - Return codes: 0 ok, ETAP_ERR_SHAPE for shape/argument problems (the reference throws
 *     std::invalid_argument there: etap.cpp:24-32,104-106, attention.cpp:11-19), ETAP_ERR_CUDA
 *     for CUDA failures. etap_mla_last_error() returns a thread-local message.
 *   - There is no CPU fallback: without a usable sm_100 device every compute entry point
 *     returns ETAP_ERR_CUDA.
 *
 * Layouts (MLA latent attention, DeepSeek shapes)
 *   q          [batch][q_tokens][heads][576]    bf16, row-major (heads folded into n_q as in
 *              the reference bench harness, cli.cpp:214)
 *   kv_pool    [num_pages][64][576]             bf16, the latent KV cache; V is the first 512
 *              columns of every row (MLA aliasing; the reference keeps V separate,
 *              attention.cpp:38-40, and callers build V = K[:, :512] with col_block)
 *   block_table[batch][max_pages]               int32 page ids
 *   seqlens    [batch]                          int32 context lengths (varlen; 0 allowed)
 *   out        [batch][q_tokens][heads][512]    fp32  O = softmax(scale * Q K^T) V (16-byte
 *              aligned, like q, kv_pool and the workspace; ETAP_ERR_SHAPE otherwise)
 *   lse        [batch][q_tokens][heads]         fp32  L = m + log l, natural log (etap.cpp:144)
 *   q_tokens > 1 (multi-token / MTP decode, no reference analog: SPEC.md:12,146,249 put it out
 *   of scope) folds the tokens into the head axis, n_q = q_tokens * heads rows per sequence
 *   (the reference bench's own folding, cli.cpp:214); with `causal` token j sees KV rows
 *   [0, seqlen - q_tokens + j]. The sizing and metadata entry points below take that folded
 *   row count as `heads`. A query row that sees no KV row gets O = 0, L = -inf.
 */
#ifndef ETAP_MLA_H
#define ETAP_MLA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ETAP_MLA_D_QK 576
#define ETAP_MLA_D_V 512
#define ETAP_MLA_PAGE_ROWS 64
#define ETAP_MLA_TILE_ROWS 64      /* KV rows per pipeline tile (M of S^T = K Q^T) */
#define ETAP_MLA_HEAD_GROUP 16     /* minimum heads per CTA work unit (see etap_mla_head_group) */
#define ETAP_MLA_SCHED_INTS 8      /* int32 per CTA in the schedule */
#define ETAP_MLA_MAX_Q_TOKENS 8    /* query tokens per sequence (multi-token / MTP decode) */

#define ETAP_OK 0
#define ETAP_ERR_SHAPE 1
#define ETAP_ERR_CUDA 2

/* flags for etap_mla_decode */
#define ETAP_FLAG_NEGATE_RESCALE 1u /* fault injection, mirrors EtapFaults::negate_rescale
                                       (etap.hpp:39-41, etap.cpp:62): flips the sign of the
                                       accumulator rescale factor; implies EAGER_RESCALE */
#define ETAP_FLAG_EAGER_RESCALE 2u  /* rescale O^T whenever the running max grows (the
                                       reference's per-block order, etap.cpp:40-47,62-70)
                                       instead of the default thresholded lazy rescale */
#define ETAP_FLAG_SKIP_COMBINE 4u   /* launch K2 only; the caller runs etap_mla_combine (used to
                                       time K2 alone) */
#define ETAP_FLAG_EXTERNAL_SCHEDULE 8u /* read sched / split_off produced by etap_mla_metadata.
                                       Without it K2 computes the same schedule in its
                                       prologue and writes it to sched / split_off when
                                       the line (batch * head groups) has <= 256 entries:
                                       K1 off the per-step critical path; longer lines make
                                       etap_mla_decode launch K1 itself first. */
#define ETAP_FLAG_DEP_METADATA 16u  /* the default since round 2, kept as a no-op for callers
                                       that pass it: seqlens / block_table are read only after
                                       the grid dependency on the preceding kernel resolved */
#define ETAP_FLAG_EARLY_METADATA 32u /* opt-in fast path (~1-2 us per call): the decode kernels
                                       launch with programmatic dependent launch and read
                                       seqlens and block_table (never KV or Q) BEFORE the
                                       kernel immediately before them on the stream has
                                       finished, so the split schedule and the first page ids
                                       are ready when it does. The caller guarantees that this
                                       preceding kernel does not write seqlens / block_table
                                       (host copies and this library's decode / combine kernels
                                       satisfy this; a PDL producer kernel that writes them
                                       and triggers its dependents early does not). Without
                                       the flag (default) both are read after the dependency
                                       resolves, which is safe whoever wrote them. */
#define ETAP_FLAG_INDEPENDENT_INPUTS 64u /* opt-in, implies EARLY_METADATA: the kernel launched
                                       immediately before the decode on the stream writes none
                                       of its inputs (q, kv_pool, block_table, seqlens) and is
                                       not a decode launched with SKIP_COMBINE. The decode then
                                       streams KV and Q while that kernel still runs and waits
                                       for it only before its first global write (schedule
                                       publish, split partials, outputs): back-to-back decode
                                       steps overlap the next step's start with the previous
                                       step's combine. Ignored with ETAP_FLAG_SKIP_COMBINE. */

/* Thread-local description of the last error. Never NULL. */
const char* etap_mla_last_error(void);

/* Library build identification (for the driver's "which .so was loaded" evidence). */
const char* etap_mla_version(void);

/* Heads per CTA work unit the library uses for `heads` query heads: 32 when heads is a
 * multiple of 32 (N = 32 / 64 UMMAs), else 16 (ETAP_HEAD_GROUP=16 in the environment forces
 * 16). Sizes below, the split_off layout and the debug state dump follow it. */
int etap_mla_head_group(int heads, int* head_group);

/* Work unit of the split schedule for `heads` query rows and num_sm_parts: what the entries of
 * sched / split_off refer to. 128 heads per unit over num_sm_parts / 2 CTA pairs when the
 * CTA-pair kernel runs the head count (heads a multiple of 128, num_sm_parts >= 2; ETAP_PAIR=0 or
 * a forced ETAP_HEAD_GROUP in the environment turns it off), else etap_mla_head_group units over
 * num_sm_parts CTAs. K1, etap_mla_metadata_host, the decode and etap_mla_combine follow it; the
 * buffer sizes below (head_group units) bound either layout.
 * Replaces nothing in the reference: its run_etap is one serial loop (etap.cpp:122-129). */
int etap_mla_schedule_unit(int heads, int num_sm_parts, int* unit_heads, int* parts);

/* Number of persistent CTAs the decode kernel uses on `device` (= its SM count). */
int etap_mla_num_sm_parts(int device, int* num_sm_parts);

/* Sizes of the caller-owned scratch buffers.
 *   sched     : num_sm_parts * ETAP_MLA_SCHED_INTS int32 (zero it once after allocation: the
 *               decode reads the previous call's ranges from it as an L2 prefetch hint)
 *   split_off : batch * heads/head_group + 1 int32
 *   workspace : bytes for split-KV partial O / LSE (zero it once after allocation) */
int etap_mla_sched_ints(int batch, int heads, int num_sm_parts, size_t* sched_ints,
                        size_t* split_off_ints);
int etap_mla_workspace_bytes(int batch, int heads, int num_sm_parts, size_t* bytes);

/* K1 — split-KV work scheduler (no reference analog: run_etap streams every KV block in one
 * serial loop, etap.cpp:122-129, kv_block_count tiled_standard.cpp:21-23). Integer partition
 * of the (sequence, head-group, 64-row tile) space over num_sm_parts persistent CTAs. */
int etap_mla_metadata(const int32_t* seqlens /*device [batch]*/, int batch, int heads,
                      int num_sm_parts, int32_t* sched /*device*/, int32_t* split_off /*device*/,
                      void* stream);

/* Host restatement of K1 (same partition, computed serially on the CPU from host seqlens);
 * sched / split_off are host arrays of the sizes given by etap_mla_sched_ints. */
int etap_mla_metadata_host(const int32_t* seqlens /*host [batch]*/, int batch, int heads,
                           int num_sm_parts, int32_t* sched, int32_t* split_off);

/* K2 + K3 — the transposed pipeline (run_etap + block_update_impl, etap.cpp:15-148) on
 * tcgen05/TMEM/TMA, followed by the log-sum-exp combine of split partials.
 * All pointers are device pointers. 1 <= q_tokens <= ETAP_MLA_MAX_Q_TOKENS; heads is per
 * token and q_tokens * heads must be a multiple of 16 (the value to pass as `heads` to the
 * sizing / metadata / combine entry points). `causal` masks the trailing rows per token
 * (a no-op for q_tokens = 1). */
int etap_mla_decode(const void* q, const void* kv_pool, int64_t num_pages,
                    const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens,
                    int batch, int q_tokens, int heads, float scale, int causal,
                    const int32_t* sched, const int32_t* split_off, int num_sm_parts,
                    void* workspace, float* out, float* lse, unsigned flags, void* stream);

/* K2-FP8 + K3 — the same decode on an FP8 (e4m3) latent cache: kv_pool8 [pages][64][576]
 * e4m3 bytes, dequantised value = kv_scale * e4m3 (per-tensor scale > 0). q stays bf16; the
 * kernel itself splits it into three fp8 terms (exact for bf16 values in the normal range)
 * and P into three fp8 terms (about 12 significant bits), so both contractions run as
 * kind::f8f6f4 UMMAs straight on the fp8 page (no dequantising pass, no extra kernel); fp32
 * accumulation, fp32 O / LSE. Same sizing, schedule and workspace as etap_mla_decode (16 heads
 * per work unit; the workspace also holds per-CTA scratch for the fp8 terms of later splits'
 * Q). External schedules (ETAP_FLAG_EXTERNAL_SCHEDULE) and the rescale fault flag are not
 * supported here. */
int etap_mla_decode_fp8(const void* q, const void* kv_pool8, float kv_scale, int64_t num_pages,
                        const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens,
                        int batch, int q_tokens, int heads, float scale, int causal,
                        const int32_t* sched, const int32_t* split_off, int num_sm_parts,
                        void* workspace, float* out, float* lse, unsigned flags, void* stream);

/* ---------------------------------------------------------------------------------------
 * Head-sharded decode with a fused all-gather over NVLink peer memory (each
 * rank owns heads [head_offset, head_offset + heads) against the replicated latent KV; the
 * only exchange is the all-gather of O / LSE, which the reference lacks: single process).
 * Instead of a decode followed by ncclAllGather, K2's epilogue and K3 store every finished
 * O / LSE row straight into every rank's full-head output buffer (peer-mapped through CUDA
 * IPC), then a one-warp kernel publishes `epoch` into every rank's arrival words (release,
 * system scope) and waits until every rank's word in its own array reached `epoch` (acquire).
 * On return (stream order) this rank's out[rank] / lse[rank] hold all heads_total heads.
 * Buffers: out [batch][q_tokens][heads_total][512] fp32, lse [batch][q_tokens][heads_total]
 * fp32, flags ETAP_MLA_MAX_PEERS uint32 zero-initialised; epochs are nonzero and increase
 * per call. A caller that reuses one output buffer must not start call k+1 on any rank before
 * every rank consumed call k (alternate two buffer sets by epoch parity to avoid that).
 * ------------------------------------------------------------------------------------- */
#define ETAP_MLA_MAX_PEERS 8
#define ETAP_MLA_IPC_HANDLE_BYTES 64

typedef struct etap_mla_peer_gather {
    int world;        /* ranks sharing the output, 1..ETAP_MLA_MAX_PEERS */
    int rank;         /* this rank */
    int heads_total;  /* heads per token over all ranks */
    int head_offset;  /* first head of this rank */
    float* out[ETAP_MLA_MAX_PEERS];     /* rank r's full output, mapped in this process */
    float* lse[ETAP_MLA_MAX_PEERS];
    uint32_t* flags[ETAP_MLA_MAX_PEERS]; /* rank r's arrival words */
} etap_mla_peer_gather;

/* etap_mla_decode + fused all-gather (see above); out / lse come from `pg`. */
int etap_mla_decode_peer(const void* q, const void* kv_pool, int64_t num_pages,
                         const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens,
                         int batch, int q_tokens, int heads, float scale, int causal,
                         const int32_t* sched, const int32_t* split_off, int num_sm_parts,
                         void* workspace, const etap_mla_peer_gather* pg, uint32_t epoch,
                         unsigned flags, void* stream);

/* CUDA IPC plumbing for the peer buffers: allocate a zeroed device buffer on the current
 * device and export its handle (ETAP_MLA_IPC_HANDLE_BYTES bytes); map a peer's handle into
 * this process (peer access enabled lazily); unmap; free. */
int etap_mla_ipc_alloc(size_t bytes, void** dev_ptr, void* handle);
int etap_mla_ipc_open(const void* handle, void** dev_ptr);
int etap_mla_ipc_close(void* dev_ptr);
int etap_mla_ipc_free(void* dev_ptr);

/* K3 alone — log-sum-exp merge of the split partials left in `workspace` by a decode call
 * made with ETAP_FLAG_SKIP_COMBINE (same batch/heads/num_sm_parts/split_off). */
int etap_mla_combine(const int32_t* split_off, int batch, int heads, int num_sm_parts,
                     void* workspace, float* out, float* lse, void* stream);

/* End-to-end call with HOST buffers (the reference-facing path: run_etap receives host
 * matrices): host->device copies, K1, K2, K3, device->host copies, synchronize.
 * A context caches the device buffers for one (batch, heads, pages) shape. */
typedef struct etap_mla_host_ctx etap_mla_host_ctx;
int etap_mla_host_ctx_create(int batch, int heads, int64_t num_pages, int max_pages_per_seq,
                             etap_mla_host_ctx** ctx);
int etap_mla_host_decode(etap_mla_host_ctx* ctx, const void* q_host, const void* kv_pool_host,
                         const int32_t* block_table_host, const int32_t* seqlens_host,
                         float scale, unsigned flags, float* out_host, float* lse_host);
void etap_mla_host_ctx_destroy(etap_mla_host_ctx* ctx);

/* ---------------------------------------------------------------------------------------
 * Serving-style decode steps (the caller side of the path: a paged latent-KV cache that
 * stays resident in HBM, and one new latent row per sequence per step).
 *
 * etap_mla_append_kv: write the q_tokens new latent rows of every sequence into the paged
 *   pool — row j of sequence b lands at token position seqlens[b] - q_tokens + j (seqlens
 *   are the lengths AFTER the append), page block_table[b][pos / 64], row pos % 64. Device
 *   pointers, stream-ordered; rows whose position or page is out of range are skipped.
 *   kv_rows: [batch][q_tokens][576] bf16.
 * etap_mla_host_ctx_load: upload the resident cache state (pool + block table) once.
 * etap_mla_host_decode_step: one decode step from HOST buffers against the resident cache:
 *   Q, the new rows and seqlens in; append (above); K2 + K3; O / LSE out; synchronize. With
 *   page-locked buffers (cudaHostAlloc / cudaHostRegister) the inputs are read in place over
 *   PCIe by one ingest kernel and O / LSE are stored straight into the host buffers; pageable
 *   buffers go through H2D / D2H staging copies. What `bench.py` reports as e2e_serving. */
/* ---------------------------------------------------------------------------------------
 * The steps on either side of the kernel in an absorbed-MLA (DeepSeek) decode layer
 * (not in the reference). Per-head GEMMs with only B token rows, run
 * transposed like the decode itself (weights on the UMMA M axis, tokens on N), bf16
 * operands, fp32 accumulation. Device pointers, stream-ordered.
 *
 * etap_mla_head_proj: y[b,h,:n_out] = x[b,h,:k_dim] . w[h] with w [heads][k_dim][n_out] bf16;
 *   x bf16 (x_fp32 = 0) or fp32 (rounded to bf16 on load); y bf16 or fp32; strides in elements.
 *   1 <= batch <= 256, k_dim % 64 == 0, n_out % 128 == 0.
 * etap_mla_absorb_q: Q[b,t,h,0:512] = q_nope[b,t,h,:128] . W_UK[h] ([heads][128][512]) and
 *   Q[b,t,h,512:576] = RoPE(q_pe[b,t,h,:64]) with per-token cos/sin [batch*q_tokens][32]
 *   (half rotation: out_i = x_i cos_i - x_{i+32} sin_i, out_{i+32} = x_{i+32} cos_i + x_i sin_i).
 *   Q is the decode's bf16 [batch][q_tokens][heads][576] input.
 * etap_mla_up_proj: out[b,t,h,:128] = O[b,t,h,:512] . W_UV[h] ([heads][512][128]) from the
 *   decode's fp32 O; out bf16 or fp32. */
int etap_mla_head_proj(const void* x, int x_fp32, int64_t x_stride_b, int64_t x_stride_h, const void* w,
                       int batch, int heads, int k_dim, int n_out, void* y, int y_fp32, int64_t y_stride_b,
                       int64_t y_stride_h, void* stream);
int etap_mla_absorb_q(const void* q_nope, const void* q_pe, const float* cos_t, const float* sin_t,
                      const void* w_uk, int batch, int q_tokens, int heads, void* q, void* stream);
int etap_mla_up_proj(const float* o, const void* w_uv, int batch, int q_tokens, int heads, void* out,
                     int out_fp32, void* stream);

int etap_mla_append_kv(const void* kv_rows, void* kv_pool, int64_t num_pages,
                       const int32_t* block_table, int max_pages_per_seq, const int32_t* seqlens,
                       int batch, int q_tokens, void* stream);
int etap_mla_host_ctx_load(etap_mla_host_ctx* ctx, const void* kv_pool_host,
                           const int32_t* block_table_host);
int etap_mla_host_decode_step(etap_mla_host_ctx* ctx, const void* q_host, const void* kv_rows_host,
                              const int32_t* seqlens_host, float scale, unsigned flags,
                              float* out_host, float* lse_host);

/* Precision of the reference's AttentionProblem (etaplab::Precision, matrix.hpp:22). The GPU
 * path computes bf16 x bf16 -> fp32 on the stored operands, which is a mapping of exact64
 * storage only; the fp32 / fp16emu emulation modes are rejected with ETAP_ERR_SHAPE (the
 * adapter throws std::invalid_argument) rather than silently computed differently. */
#define ETAP_PRECISION_EXACT64 0
#define ETAP_PRECISION_FP32 1
#define ETAP_PRECISION_FP16EMU 2

/* Reference-shaped entry (binary64 row-major matrices, exactly the storage of
 * etaplab::AttentionProblem, attention.hpp:15-25): rounds Q/K to bf16, checks the MLA
 * aliasing V == K[:, :512], runs the GPU path, widens O and L back to binary64.
 * d_qk must be 576, d_v 512 and precision ETAP_PRECISION_EXACT64; n_q is padded to a multiple
 * of 16 heads internally. b_r/b_c/stages mirror TileConfig (tiled_standard.hpp:11-15):
 * validated (>= 1, as run_etap does at etap.cpp:104-106) and otherwise without numeric effect
 * — the GPU tiling is fixed and the result is partition invariant (acceptance.cpp:209-229). */
int etap_mla_run_etap_f64(const double* q, int64_t n_q, const double* k, int64_t n_kv,
                          int64_t d_qk, const double* v, int64_t d_v, double scale, int precision,
                          int64_t b_r, int64_t b_c, int64_t stages, unsigned flags, double* o,
                          double* l);

/* Reference-shaped entry with the BlockHook stream (tiled_standard.hpp:32-40; run_etap calls
 * the hook after every KV block of b_c rows, etap.cpp:122-129): state [t_c][4][n_q] host
 * binary64, t_c = ceil(n_kv / b_c), holding after KV block j for every query row i
 *   state[(j*4 + 0)*n_q + i] = m_old (-inf before the first block), [1] = m (running max of
 *   scale*q.k), [2] = rescale exp(m_old - m) (0 on the first block), [3] = running sum l
 * — the device's softmax state over exactly rows [0, min((j+1) b_c, n_kv)) with one split (the
 * reference's serial block order), for any b_c: every block boundary that is not a 64-row tile
 * boundary is observed as the final state of a prefix sequence sharing the same KV pages. */
int etap_mla_run_etap_f64_state(const double* q, int64_t n_q, const double* k, int64_t n_kv,
                                int64_t d_qk, const double* v, int64_t d_v, double scale,
                                int precision, int64_t b_c, unsigned flags, double* o, double* l,
                                double* state);

/* UMMA descriptor self-test (one CTA, one tile): S^T = K Q^T and O^T = V^T P^T through the
 * same smem layouts as the 16-head decode kernel. Device pointers: k [64][576] bf16,
 * q [16][576] bf16, p [64][16] fp32; outputs s_t [64][16] fp32, o_t [512][32] fp32 (columns
 * 0-15 = V^T P_hi, 16-31 = V^T P_lo). */
int etap_mla_selftest_umma(const void* k, const void* q, const float* p, float* s_t, float* o_t,
                           void* stream);

/* FP8 (e4m3) UMMA self-test (kind::f8f6f4), the FP8 latent-KV layouts: k8 [64][576], q8 [48][576]
 * (three fp8 terms x 16 heads), p8 [64][48] e4m3 bytes; outputs s_t [64][48] = k8 q8^T and
 * o_t [512][48] = k8[:, :512]^T p8, fp32. */
int etap_mla_selftest_fp8(const void* k8, const void* q8, const void* p8, float* s_t, float* o_t, void* stream);

/* Debug: when device_buf is non-NULL, subsequent decode launches (bf16 and FP8) run the
 * debug instantiation of the decode kernel, which records per-tile %clock64 stamps of the
 * pipeline events into it: [cta][256][16] uint64, row = tile (< 255): 0/1 first / last chunk
 * TMA issued, 2 last chunk landed, 3 S^T committed, 4 softmax saw S^T, 5 P^T written, 6 MMA saw
 * P^T, 7 O^T update committed, 8 softmax exp done, 9 P buffer free (FP8: 10/11 split epilogue
 * start / end on a split's last tile). Row 255: %globaltimer ns at 0 entry, 1 schedule done,
 * 2 exit; 3 SM id; %clock64 at 5 entry, 6 exit. NULL disables (the default, and the product
 * instantiation carries no stamps at all). */
int etap_mla_debug_trace(void* device_buf);

/* Kernel span (bench timing that keeps programmatic dependent launch intact): when device_buf
 * is non-NULL, the product decode kernels (bf16 and FP8) record per CTA [cta][2] uint64
 * %globaltimer ns: 0 = its grid dependency resolved (the earliest moment it may read KV), 1 =
 * exit. The launch reads the pointer at launch time, so a caller may point successive launches
 * at successive rows. NULL (default) disables; two stores per CTA outside every loop. */
int etap_mla_debug_span(void* device_buf);

/* Debug: combine-kernel stamps [block][4] (entry, after grid-dependency wait, exit) or NULL. */
int etap_mla_debug_trace_combine(void* device_buf);

/* Debug (BlockHook replay, the reference's per-KV-block observer tiled_standard.hpp:32-40):
 * when device_buf is non-NULL, decode launches record for every (virtual sequence vb,
 * 64-row tile t < max_tiles) the softmax state after the tile:
 *   device_buf[((vb * max_tiles) + t) * 4 * hg + {0, hg, 2 hg, 3 hg} + h] = m_old, m_new
 *   (natural log units of scale*q.k), rescale exp(m_old - m_new) (0 on the first tile of a
 *   split), running l
 * for head h of the head group (hg = etap_mla_head_group(heads), vb head-group major). Per-split state: run with one split per sequence
 * (num_sm_parts = 1 or a single sequence) to observe the reference's single chain. */
int etap_mla_debug_state(void* device_buf, int max_tiles);

/* Debug: tensor-pipe microbenchmark — `grid` CTAs each issue n tcgen05.mma of one operand
 * layout variant; out_dev[0..1] (device, int64) = issue cycles, issue+completion cycles. */
int etap_mla_umma_bench(int variant, int n, long long* out_dev, int grid);

/* Debug: stream the KV pool with the decode kernel's TMA access pattern and no compute
 * (grid CTAs x pages_per_cta pages, ring of nslot 8 KB slots) — the attainable read rate. */
int etap_mla_stream_bench(const void* kv_pool, int64_t num_pages, int pages_per_cta, int grid,
                          int nslot, void* stream);
/* Debug: the same with clusters of two CTAs that stream the same pages, each issuing every
 * other box as a cluster multicast into both (grid even; grid / 2 page ranges). */
int etap_mla_stream_bench_mc(const void* kv_pool, int64_t num_pages, int pages_per_cta, int grid,
                             int nslot, void* stream);
/* Debug: the same with 3-D TMA boxes of box_chunks chunks (1, 3 or 9: one box per page)
 * instead of nine 2-D chunk boxes. */
int etap_mla_stream_bench_page(const void* kv_pool, int64_t num_pages, int pages_per_cta, int grid,
                               int nslot, int box_chunks, void* stream);

/* Debug / tests (host only): the binary64 -> bfloat16 round-to-nearest-even that
 * etap_mla_run_etap_f64 applies to AttentionProblem operands, as the bit-level fast form or
 * (reference_form != 0) the frexp / nearbyint form it must equal. out: n bf16 bit patterns. */
int etap_mla_debug_bf16_rne(const double* x, int64_t n, uint16_t* out, int reference_form);

/* Debug / tests: a one-CTA kernel launched with programmatic dependent launch that triggers
 * its dependents at entry, sleeps delay_ns, then copies n int32 from src to dst (device
 * pointers) — a PDL producer writing seqlens or block_table right before a decode. */
int etap_mla_debug_pdl_write(int32_t* dst, const int32_t* src, int n, int delay_ns, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ETAP_MLA_H */
