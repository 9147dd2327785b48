// SPDX-License-Identifier: Apache-2.0
// Probe (experiment, not product): (1) does tcgen05.mma kind::f16 accept mixed operand formats
// (A = bf16 V^T, B = fp16 P) — the instruction descriptor has separate A / B format fields;
// (2) issue cost of back-to-back MMAs for the GEMM1 / GEMM2 shapes of wider head groups.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/probe_umma.cu -o /tmp/probe && /tmp/probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2506_01969_b200/csrc/sm100_ptx.cuh"

using namespace etap_b200;

__host__ __device__ constexpr uint32_t idesc(uint32_t m, uint32_t n, uint32_t afmt, uint32_t bfmt, uint32_t amn,
                                            uint32_t bmn) {
    return (1u << 4) | (afmt << 7) | (bfmt << 10) | (amn << 15) | (bmn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// ---- (1) O^T[128 x 16] = V^T[128 x 64] . P[64 x 16]; V two SW128 K-major chunks [64 rows][64 cols]
// bf16 (as TMA writes them), P MN-major no swizzle (the decode's P^T layout), fmt selectable.
__global__ void mixed_kernel(const uint16_t* v /*[64][128] bf16 bits*/, const uint16_t* p /*[64][16] bits*/,
                             int bfmt, float* o /*[128][16]*/) {
    __shared__ __align__(1024) uint8_t sm[2 * 8192 + 64 * 16 * 2 + 1024];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    uint8_t* a = sm;
    uint8_t* b = sm + 16384;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 64 * 128; i += blockDim.x) {
        const int r = i / 128, c = i % 128, chunk = c / 64, cc = c % 64;
        const int byte = r * 128 + ((((cc * 2) >> 4) ^ (r & 7)) << 4) + ((cc * 2) & 15);
        *reinterpret_cast<uint16_t*>(a + chunk * 8192 + byte) = v[r * 128 + c];
    }
    constexpr int ROWGRP = 16 * 16;  // P_ROWGRP for N = 16
    for (int i = tid; i < 64 * 16; i += blockDim.x) {
        const int r = i / 16, n = i % 16;
        *reinterpret_cast<uint16_t*>(b + (r >> 3) * ROWGRP + (n >> 3) * 128 + (r & 7) * 16 + (n & 7) * 2) = p[i];
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(&tslot, 32);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t t = tslot;
    if (warp == 0) {
        const uint64_t a0 = ptx::smem_desc(ptx::smem_u32(a), 8192, 1024, ptx::LAYOUT_SW128);
        const uint64_t b0 = ptx::smem_desc(ptx::smem_u32(b), ROWGRP, 128, ptx::LAYOUT_NONE);
        const uint32_t id = idesc(128, 16, 1, bfmt, 1, 1);
        for (int kk = 0; kk < 4; ++kk)
            ptx::umma_f16_elect(t, a0 + kk * (2048 >> 4), b0 + kk * ((2 * ROWGRP) >> 4), id, kk > 0);
        ptx::umma_commit_elect(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    uint32_t r[16];
    ptx::tmem_ld16(t + (static_cast<uint32_t>(warp * 32) << 16), r);
    ptx::tmem_wait_ld();
    for (int n = 0; n < 16; ++n) o[(warp * 32 + (tid & 31)) * 16 + n] = __uint_as_float(r[n]);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(t, 32); }
}

// ---- (2) issue cost: n back-to-back MMAs of one shape; A K-major SW128 (GEMM1) or MN-major
// SW128 (GEMM2), B K-major SW128 or MN-major none.
__global__ void cost_kernel(int m, int n, int gemm2, int count, long long* out) {
    extern __shared__ uint8_t dsm[];
    uint8_t* smem = ptx::align_smem_1024(dsm);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t t = tslot;
    if (threadIdx.x < 32) {
        const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
        uint64_t ad, bd;
        uint32_t id;
        if (gemm2) {
            ad = ptx::smem_desc(a, 8192, 1024, ptx::LAYOUT_SW128);
            bd = ptx::smem_desc(b, n * 16, 128, ptx::LAYOUT_NONE);
            id = idesc(m, n, 1, gemm2 == 2 ? 0 : 1, 1, 1);
        } else {
            ad = ptx::smem_desc(a, 16, 1024, ptx::LAYOUT_SW128);
            bd = ptx::smem_desc(b, 16, 1024, ptx::LAYOUT_SW128);
            id = idesc(m, n, 1, 1, 0, 0);
        }
        for (int rep = 0; rep < 2; ++rep) {
            __syncwarp();
            const long long t0 = clock64();
            for (int i = 0; i < count; i += 4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) ptx::umma_f16_elect(t, ad + j * 2, bd + j * 2, id, (i + j) > 0);
            }
            ptx::umma_commit_elect(&bar);
            ptx::mbar_wait(&bar, rep & 1);
            const long long t1 = clock64();
            if (rep == 1 && threadIdx.x == 0) out[0] = t1 - t0;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(t, 512); }
}

static uint16_t bf16_bits(float x) { __nv_bfloat16 h = __float2bfloat16_rn(x); return *reinterpret_cast<uint16_t*>(&h); }
static uint16_t f16_bits(float x) { __half h = __float2half_rn(x); return *reinterpret_cast<uint16_t*>(&h); }
static float bf16_val(uint16_t b) { uint32_t u = static_cast<uint32_t>(b) << 16; float f; memcpy(&f, &u, 4); return f; }

int main(int argc, char** argv) {
    const bool mixed = argc > 1 && argv[1][0] == 'm';
    // (1) mixed formats (an illegal instruction poisons the context: run it alone)
    if (mixed) {
    std::vector<uint16_t> v(64 * 128), p(64 * 16);
    std::vector<double> vd(64 * 128), pd(64 * 16);
    srand(1);
    for (int i = 0; i < 64 * 128; ++i) { v[i] = bf16_bits((rand() / (float)RAND_MAX - 0.5f) * 4); vd[i] = bf16_val(v[i]); }
    for (int i = 0; i < 64 * 16; ++i) {
        // values with > 8 significant bits: fp16 keeps them, bf16 would not
        const float x = 1.0f + (rand() % 1024) / 1024.0f;
        p[i] = f16_bits(x);
        pd[i] = __half2float(*reinterpret_cast<__half*>(&p[i]));
    }
    uint16_t *dv, *dp; float* dout;
    cudaMalloc(&dv, v.size() * 2); cudaMalloc(&dp, p.size() * 2); cudaMalloc(&dout, 128 * 16 * 4);
    cudaMemcpy(dv, v.data(), v.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, p.data(), p.size() * 2, cudaMemcpyHostToDevice);
    mixed_kernel<<<1, 128>>>(dv, dp, 0 /*F16*/, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(128 * 16);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int d = 0; d < 128; ++d)
        for (int n = 0; n < 16; ++n) {
            double ref = 0;
            for (int r = 0; r < 64; ++r) ref += vd[r * 128 + d] * pd[r * 16 + n];
            maxerr = std::fmax(maxerr, std::fabs(ref - o[d * 16 + n]));
            maxref = std::fmax(maxref, std::fabs(ref));
        }
    printf("{\"probe\": \"mixed bf16 A x f16 B kind::f16\", \"cuda\": \"%s\", \"max_abs_err\": %.3e, \"max_ref\": %.3e}\n",
           cudaGetErrorString(e), maxerr, maxref);
    return 0;
    }
    // (2) issue costs
    long long* dc; cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 129 * 1024);
    const int shapes[][3] = {{64, 16, 0}, {64, 32, 0}, {64, 64, 0}, {64, 128, 0}, {128, 32, 0}, {128, 64, 0},
                             {128, 128, 0}, {128, 256, 0}, {128, 32, 1}, {128, 64, 1}, {128, 128, 1},
                             {128, 256, 1}};
    for (auto& s : shapes) {
        cost_kernel<<<1, 128, 129 * 1024>>>(s[0], s[1], s[2], 256, dc);
        cudaError_t e2 = cudaDeviceSynchronize();
        long long cyc = 0;
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"mma cost\", \"m\": %d, \"n\": %d, \"gemm\": \"%s\", \"cycles_per_mma\": %.1f, \"cuda\": \"%s\"}\n",
               s[0], s[1], s[2] == 0 ? "K-major SW128 A/B (GEMM1)" : (s[2] == 1 ? "MN-major A SW128, B none bf16 (GEMM2)" : "GEMM2 with f16 B"),
               cyc / 256.0, cudaGetErrorString(e2));
    }
    // 148 CTAs at once (one per SM): same per-SM cost?
    return 0;
}
