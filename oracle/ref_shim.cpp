// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
// extern "C" shim over the UNMODIFIED reference library (etaplab, compiled from the sources
// under /root/reference/proj/src by oracle/Makefile into oracle/_ref/libetaplab_ref.so).
// It only marshals plain arrays into etaplab::Matrix / AttentionProblem and calls the
// reference's own functions; no reference code is copied here.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "etaplab/attention.hpp"
#include "etaplab/etap.hpp"
#include "etaplab/matrix.hpp"
#include "etaplab/matrix_io.hpp"
#include "etaplab/tiled_standard.hpp"
#include "etaplab/wgmma_model.hpp"

using namespace etaplab;

namespace {

Matrix from_ptr(const double* p, std::int64_t rows, std::int64_t cols) {
    return Matrix(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols),
                  std::vector<double>(p, p + rows * cols));
}

void to_ptr(const AttentionOutput& out, double* o, double* l) {
    std::memcpy(o, out.o.data(), sizeof(double) * out.o.size());
    std::memcpy(l, out.l.data(), sizeof(double) * out.l.size());
}

Precision prec_of(int p) {
    return p == 1 ? Precision::fp32 : p == 2 ? Precision::fp16emu : Precision::exact64;
}

}  // namespace

extern "C" {

// matrix_from_seed (src/matrix.cpp:153-165)
void ref_matrix_from_seed(std::int64_t rows, std::int64_t cols, std::uint64_t seed, int dist,
                          double* out) {
    const Matrix m = matrix_from_seed(rows, cols, seed, dist == 1 ? Dist::uniform : Dist::normal);
    std::memcpy(out, m.data(), sizeof(double) * m.size());
}

double ref_round_half(double x) { return round_half(x); }

// make_problem(seed, ...) (src/attention.cpp:33-42): returns the stored (rounded) operands
int ref_make_problem_seeded(std::uint64_t seed, std::int64_t n_q, std::int64_t n_kv,
                            std::int64_t d_qk, std::int64_t d_v, double scale, int precision,
                            double* q, double* k, double* v, double* scale_out) {
    try {
        const AttentionProblem p = make_problem(seed, n_q, n_kv, d_qk, d_v, scale, prec_of(precision));
        std::memcpy(q, p.q.data(), sizeof(double) * p.q.size());
        std::memcpy(k, p.k.data(), sizeof(double) * p.k.size());
        std::memcpy(v, p.v.data(), sizeof(double) * p.v.size());
        *scale_out = p.scale;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// mode 0: attention_ref (attention.cpp:44-77); 1: run_etap (etap.cpp:102-148);
// 2: run_standard (tiled_standard.cpp:32-101). Returns 1 on std::invalid_argument.
int ref_run(int mode, const double* q, std::int64_t n_q, const double* k, std::int64_t n_kv,
            std::int64_t d_qk, const double* v, std::int64_t d_v, double scale, int precision,
            std::int64_t b_r, std::int64_t b_c, std::int64_t stages, int negate_rescale, double* o,
            double* l) {
    try {
        const AttentionProblem p = make_problem(from_ptr(q, n_q, d_qk), from_ptr(k, n_kv, d_qk),
                                                from_ptr(v, n_kv, d_v), scale, prec_of(precision));
        const TileConfig tiles{static_cast<std::size_t>(b_r), static_cast<std::size_t>(b_c),
                               static_cast<std::size_t>(stages)};
        AttentionOutput out;
        if (mode == 0) {
            out = attention_ref(p);
        } else if (mode == 1) {
            EtapFaults f;
            f.negate_rescale = negate_rescale != 0;
            out = run_etap(p, tiles, {}, f);
        } else {
            out = run_standard(p, tiles);
        }
        to_ptr(out, o, l);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// run_etap exact64 with a BlockHook (tiled_standard.hpp:32-40, called at etap.cpp:128) that
// records, per (query block qb, kv block j), m_old / m / rescale / l for the block's queries:
// state[((qb * t_c) + j) * 4 * b_r + f * b_r + i]. Returns the number of hook calls.
long ref_run_etap_state(const double* q, std::int64_t n_q, const double* k, std::int64_t n_kv,
                        std::int64_t d_qk, const double* v, std::int64_t d_v, double scale,
                        std::int64_t b_r, std::int64_t b_c, double* o, double* l, double* state) {
    try {
        const AttentionProblem p = make_problem(from_ptr(q, n_q, d_qk), from_ptr(k, n_kv, d_qk),
                                                from_ptr(v, n_kv, d_v), scale, Precision::exact64);
        const TileConfig tiles{static_cast<std::size_t>(b_r), static_cast<std::size_t>(b_c), 2};
        const std::int64_t t_c = (n_kv + b_c - 1) / b_c;
        long calls = 0;
        BlockHook hook = [&](const BlockStepInfo& info) {
            ++calls;
            double* st = state + (static_cast<std::int64_t>(info.query_block) * t_c +
                                  static_cast<std::int64_t>(info.kv_block)) * 4 * b_r;
            for (std::size_t i = 0; i < info.m_old.size(); ++i) {
                st[0 * b_r + i] = info.m_old[i];
                st[1 * b_r + i] = info.state.m[i];
                st[2 * b_r + i] = info.rescale[i];
                st[3 * b_r + i] = info.state.l[i];
            }
        };
        to_ptr(run_etap(p, tiles, hook), o, l);
        return calls;
    } catch (const std::exception&) {
        return -1;
    }
}

// matrix_io (ATNM): save from / load into plain arrays. Returns 0, or 1 on std::runtime_error.
int ref_save_matrix(const char* path, const double* data, std::int64_t rows, std::int64_t cols) {
    try {
        save_matrix(std::string(path), from_ptr(data, rows, cols));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

int ref_load_matrix(const char* path, double* out, std::int64_t cap, std::int64_t* rows,
                    std::int64_t* cols) {
    try {
        const Matrix m = load_matrix(std::string(path));
        *rows = static_cast<std::int64_t>(m.rows());
        *cols = static_cast<std::int64_t>(m.cols());
        if (static_cast<std::int64_t>(m.size()) > cap) return 2;
        std::memcpy(out, m.data(), sizeof(double) * m.size());
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

std::uint64_t ref_transpose_count() { return transpose_count(); }
void ref_reset_transpose_count() { reset_transpose_count(); }

// CPU baseline: run_etap (exact64) over B MLA problems (V = K[:, :512] via col_block), one
// std::thread per worker over the batch. Problems are built outside the timed region, like
// cmd_bench (cli.cpp:236-283). q [B][H][576], kv [B][ctx][576] as binary64.
// Returns the wall time of the run_etap calls in seconds (or -1 on error).
double ref_mla_run_etap_batch(const double* q, const double* kv, std::int64_t batch,
                              std::int64_t heads, std::int64_t ctx, double scale, int nthreads,
                              double* o, double* l) {
    try {
        std::vector<AttentionProblem> probs;
        probs.reserve(batch);
        for (std::int64_t b = 0; b < batch; ++b) {
            Matrix k = from_ptr(kv + b * ctx * 576, ctx, 576);
            Matrix v = k.col_block(0, 512);
            probs.push_back(make_problem(from_ptr(q + b * heads * 576, heads, 576), std::move(k),
                                         std::move(v), scale, Precision::exact64));
        }
        const TileConfig tiles{64, 64, 2};  // cmd_bench defaults (cli.hpp:30-63)
        std::vector<AttentionOutput> outs(batch);
        if (nthreads < 1) nthreads = 1;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int w = 0; w < nthreads; ++w)
            th.emplace_back([&, w] {
                for (std::int64_t b = w; b < batch; b += nthreads) outs[b] = run_etap(probs[b], tiles);
            });
        for (auto& t : th) t.join();
        const auto t1 = std::chrono::steady_clock::now();
        for (std::int64_t b = 0; b < batch; ++b) {
            std::memcpy(o + b * heads * 512, outs[b].o.data(), sizeof(double) * heads * 512);
            std::memcpy(l + b * heads, outs[b].l.data(), sizeof(double) * heads);
        }
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception&) {
        return -1.0;
    }
}

// Full-size CPU workload of the bench (BASELINE.json configs[1]: B sequences x ctx rows x H
// heads): the B MLA problems are generated ONCE with the reference's own generator
// (matrix_from_seed, seeds s_b = seed0 + 7919 b as cmd_bench, cli.cpp:239; Q from s*3+1, latent
// KV from s*3+2, attention.cpp:38-39), rounded to bf16 (the operands the GPU reads, i.e. the
// device inputs of inputs.make_mla_inputs, pinned equal by the tests), V = KV.col_block(0, 512).
// Generation runs in parallel and outside every timed region; each step then times run_etap
// (exact64, cmd_bench's TileConfig{64,64,2}) on all B problems, one std::thread per worker over
// the batch, like ref_mla_run_etap_batch. Returns an opaque handle (nullptr on error).
struct RefBench {
    std::vector<AttentionProblem> probs;
    std::vector<AttentionOutput> outs;
};

static double bf16_round_rne(double x) {
    const double ax = std::fabs(x);
    if (ax == 0.0 || !std::isfinite(x)) return x;
    int e;
    std::frexp(ax, &e);
    return std::copysign(std::ldexp(std::nearbyint(std::ldexp(ax, 8 - e)), e - 8), x);
}

void* ref_mla_bench_create(std::int64_t batch, std::int64_t heads, std::int64_t ctx, std::uint64_t seed0,
                           double scale, int nthreads) {
    try {
        auto* rb = new RefBench();
        rb->probs.resize(batch);
        rb->outs.resize(batch);
        if (nthreads < 1) nthreads = 1;
        std::vector<std::thread> th;
        for (int w = 0; w < nthreads; ++w)
            th.emplace_back([&, w] {
                for (std::int64_t b = w; b < batch; b += nthreads) {
                    const std::uint64_t s = seed0 + 7919ull * static_cast<std::uint64_t>(b);
                    Matrix q = matrix_from_seed(heads, 576, s * 3 + 1, Dist::normal);
                    Matrix kv = matrix_from_seed(ctx, 576, s * 3 + 2, Dist::normal);
                    for (std::size_t i = 0; i < q.size(); ++i) q.data()[i] = bf16_round_rne(q.data()[i]);
                    for (std::size_t i = 0; i < kv.size(); ++i) kv.data()[i] = bf16_round_rne(kv.data()[i]);
                    Matrix v = kv.col_block(0, 512);
                    rb->probs[b] = make_problem(std::move(q), std::move(kv), std::move(v), scale, Precision::exact64);
                }
            });
        for (auto& t : th) t.join();
        return rb;
    } catch (const std::exception&) {
        return nullptr;
    }
}

// One timed step: run_etap on every problem (nthreads workers); seconds, or -1 on error.
// o / l (optional, [B][H][512] / [B][H]) receive the outputs.
double ref_mla_bench_step(void* h, int nthreads, double* o, double* l) {
    auto* rb = static_cast<RefBench*>(h);
    if (!rb) return -1.0;
    try {
        const std::int64_t batch = static_cast<std::int64_t>(rb->probs.size());
        const TileConfig tiles{64, 64, 2};  // cmd_bench defaults (cli.hpp:30-63)
        if (nthreads < 1) nthreads = 1;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int w = 0; w < nthreads; ++w)
            th.emplace_back([&, w] {
                for (std::int64_t b = w; b < batch; b += nthreads) rb->outs[b] = run_etap(rb->probs[b], tiles);
            });
        for (auto& t : th) t.join();
        const auto t1 = std::chrono::steady_clock::now();
        if (o && l)
            for (std::int64_t b = 0; b < batch; ++b) {
                const std::size_t H = rb->outs[b].l.size();
                std::memcpy(o + b * H * 512, rb->outs[b].o.data(), sizeof(double) * H * 512);
                std::memcpy(l + b * H, rb->outs[b].l.data(), sizeof(double) * H);
            }
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception&) {
        return -1.0;
    }
}

void ref_mla_bench_destroy(void* h) { delete static_cast<RefBench*>(h); }

// utilization / predicted_speedup (wgmma_model.cpp:54-86) with the given WgmmaSpec.
// out = {useful_macs, issued_macs, utilization, qk m-axis util, pv m-axis util, speedup}
int ref_wgmma_model(int mode, std::int64_t heads, std::int64_t q_tokens, std::int64_t kv_len,
                    std::int64_t d_qk, std::int64_t d_v, std::int64_t batch, std::int64_t m_min,
                    std::int64_t n_step, std::int64_t k_step, double* out) {
    try {
        DecodeShape s;
        s.heads = heads; s.q_tokens = q_tokens; s.kv_len = kv_len; s.d_qk = d_qk; s.d_v = d_v; s.batch = batch;
        WgmmaSpec w;
        w.m_min = m_min; w.n_step = n_step; w.k_step = k_step;
        const UtilizationReport r = utilization(mode == 1 ? ComputeMode::etap : ComputeMode::original, s, w);
        out[0] = static_cast<double>(r.useful_macs);
        out[1] = static_cast<double>(r.issued_macs);
        out[2] = r.utilization;
        out[3] = r.qk.m_axis_utilization();
        out[4] = r.pv.m_axis_utilization();
        out[5] = predicted_speedup(s, w);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

}  // extern "C"
