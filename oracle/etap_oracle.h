/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
 * CPU restatement (plain C, binary64) of the reference's algorithm for the ETAP MLA decode
 * hot path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it, and only as the checker. Every function cites the reference lines it
 * restates (paths relative to /root/reference/proj).
 *
 * Parity pinning: the restatement is checked against (a) the reference's own inline golden
 * values (tests/test_oracle.cpp:24-45, tests/test_etap.cpp:127-146) and (b) the reference
 * itself, compiled from its sources into oracle/_ref/ by oracle/Makefile, through fixtures
 * committed under tests/golden/ (tests/golden/make_golden.py).
 */
#ifndef ETAP_ORACLE_H
#define ETAP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* matrix_from_seed (src/matrix.cpp:23-48,153-165): splitmix64 stream; dist 0 = normal
 * (Box-Muller, one element per pair of draws), 1 = uniform(-1,1). */
void oracle_matrix_from_seed(int64_t rows, int64_t cols, uint64_t seed, int dist, double* out);

/* binary64 -> bfloat16, round to nearest even, widened back (the GPU path's input rounding;
 * the reference has no bf16 mode, include/etaplab/matrix.hpp:22). */
double oracle_bf16_round(double x);
void oracle_bf16_round_array(const double* in, double* out, int64_t n);
void oracle_bf16_bits(const double* in, uint16_t* out, int64_t n);
void oracle_bf16_widen(const uint16_t* in, double* out, int64_t n);

/* round_half (src/matrix.cpp:167-184): IEEE binary16 RNE widened to binary64. */
double oracle_round_half(double x);

/* attention_ref (src/attention.cpp:44-77): row-wise binary64 softmax with max subtraction.
 * V rows are read with stride ldv (ldv = d_qk gives the MLA aliasing V = K[:, :d_v]). */
void oracle_attention_ref(const double* q, int64_t n_q, const double* k, int64_t n_kv,
                          int64_t d_qk, const double* v, int64_t ldv, int64_t d_v, double scale,
                          double* o, double* l);

/* run_etap in exact64 (src/etap.cpp:15-148): KV-major transposed pipeline with b_r x b_c
 * tiles, two d_v-half accumulators sharing the softmax state, one transpose per query block,
 * L = m + log l. negate_rescale mirrors EtapFaults (etap.hpp:39-41, etap.cpp:62). */
int oracle_run_etap(const double* q, int64_t n_q, const double* k, int64_t n_kv, int64_t d_qk,
                    const double* v, int64_t ldv, int64_t d_v, double scale, int64_t b_r,
                    int64_t b_c, int negate_rescale, double* o, double* l);

/* Batched paged MLA decode on bf16 inputs: for every sequence b and head h,
 * attention_ref(q[b][h], K_b, V_b = K_b[:, :512]) where K_b is gathered from the page pool
 * through block_table. q [B][H][576] bf16 bits, kv_pool [pages][64][576] bf16 bits,
 * o [B][H][512], l [B][H] (binary64). Threads split the (b, h-group) work. */
int oracle_mla_decode_bf16(const uint16_t* q, const uint16_t* kv_pool, int64_t num_pages,
                           const int32_t* block_table, int64_t max_pages,
                           const int32_t* seqlens, int64_t batch, int64_t heads, double scale,
                           int nthreads, double* o, double* l);

#ifdef __cplusplus
}
#endif
#endif
