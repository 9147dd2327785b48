// SPDX-License-Identifier: Apache-2.0
// Native decode-step benchmark through the C-ABI (no Python in the launch path): the GPU-side
// step time of K2 (+in-kernel schedule) + K3 for a config, with stream launches (programmatic
// dependent launch between steps) and optionally a captured CUDA graph of `per_graph` steps.
// The reference's analog is cmd_bench's timed loop (cli.cpp:277-283).
//   etap_bench --batch 16 --ctx 65536 --heads 16 --iters 200 [--graph 20] [--contiguous]
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "../../include/etap_mla.h"

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
            std::exit(2);                                                              \
        }                                                                              \
    } while (0)
#define EK(x)                                                                          \
    do {                                                                               \
        if ((x) != ETAP_OK) {                                                          \
            std::fprintf(stderr, "%s: %s\n", #x, etap_mla_last_error());               \
            std::exit(2);                                                              \
        }                                                                              \
    } while (0)

int main(int argc, char** argv) {
    int B = 16, ctx = 65536, H = 16, iters = 200, per_graph = 0;
    bool contiguous = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto next = [&] { return std::atoi(argv[++i]); };
        if (a == "--batch") B = next();
        else if (a == "--ctx") ctx = next();
        else if (a == "--heads") H = next();
        else if (a == "--iters") iters = next();
        else if (a == "--graph") per_graph = next();
        else if (a == "--contiguous") contiguous = true;
    }
    const int pages_per_seq = (ctx + 63) / 64;
    const int64_t num_pages = static_cast<int64_t>(B) * pages_per_seq;
    int dev = 0, parts = 0;
    CK(cudaGetDevice(&dev));
    EK(etap_mla_num_sm_parts(dev, &parts));
    size_t n_sched, n_so, ws;
    EK(etap_mla_sched_ints(B, H, parts, &n_sched, &n_so));
    EK(etap_mla_workspace_bytes(B, H, parts, &ws));
    void *q, *kv, *work;
    int32_t *bt, *sl, *sched, *so;
    float *out, *lse;
    CK(cudaMalloc(&q, static_cast<size_t>(B) * H * ETAP_MLA_D_QK * 2));
    CK(cudaMalloc(&kv, static_cast<size_t>(num_pages) * 64 * ETAP_MLA_D_QK * 2));
    CK(cudaMalloc(&bt, static_cast<size_t>(num_pages) * 4));
    CK(cudaMalloc(&sl, B * 4));
    CK(cudaMalloc(&sched, n_sched * 4));
    CK(cudaMalloc(&so, n_so * 4));
    CK(cudaMalloc(&work, ws));
    CK(cudaMalloc(&out, static_cast<size_t>(B) * H * ETAP_MLA_D_V * 4));
    CK(cudaMalloc(&lse, static_cast<size_t>(B) * H * 4));
    CK(cudaMemset(q, 0x3c, static_cast<size_t>(B) * H * ETAP_MLA_D_QK * 2));        // bf16 0.0115
    CK(cudaMemset(kv, 0x3c, static_cast<size_t>(num_pages) * 64 * ETAP_MLA_D_QK * 2));
    std::vector<int32_t> pages(num_pages);
    std::iota(pages.begin(), pages.end(), 0);
    if (!contiguous) std::shuffle(pages.begin(), pages.end(), std::mt19937(2506));
    std::vector<int32_t> seqlens(B, ctx);
    CK(cudaMemcpy(bt, pages.data(), num_pages * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(sl, seqlens.data(), B * 4, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const float scale = 1.f / 24.f;
    auto step = [&] {
        EK(etap_mla_decode(q, kv, num_pages, bt, pages_per_seq, sl, B, 1, H, scale, 1, sched, so, parts,
                           work, out, lse, 0, st));
    };
    for (int i = 0; i < 10; ++i) step();
    CK(cudaStreamSynchronize(st));
    // host cost of one decode call (C-ABI entry + K2/K3 launches), enqueue only
    const auto h0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) step();
    const double us_host = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count() / iters;
    CK(cudaStreamSynchronize(st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) step();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us_stream = ms * 1e3 / iters;
    double us_graph = -1;
    if (per_graph > 0) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
        for (int i = 0; i < per_graph; ++i) step();
        CK(cudaStreamEndCapture(st, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, st));
        CK(cudaStreamSynchronize(st));
        const int reps = std::max(1, iters / per_graph);
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        us_graph = ms * 1e3 / (reps * per_graph);
        CK(cudaGraphExecDestroy(ge));
        CK(cudaGraphDestroy(g));
    }
    const double kv_bytes = static_cast<double>(B) * ctx * ETAP_MLA_D_QK * 2;
    const double best = us_graph > 0 ? std::min(us_stream, us_graph) : us_stream;
    std::printf("{\"batch\": %d, \"ctx\": %d, \"heads\": %d, \"us_per_step_stream\": %.2f, "
                "\"us_per_step_graph\": %.2f, \"host_enqueue_us\": %.2f, \"kv_gbs_best\": %.1f, \"pages\": \"%s\"}\n",
                B, ctx, H, us_stream, us_graph, us_host, kv_bytes / best / 1e3, contiguous ? "contiguous" : "shuffled");
    return 0;
}
