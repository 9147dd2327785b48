// SPDX-License-Identifier: Apache-2.0
// Probe (experiment, not product): the CTA-pair output GEMM with P in tensor memory,
// O[64 heads x 256 d] += P[64 x 16] . V[16 x 256] per CTA (tcgen05.mma.cta_group::2, A from TMEM,
// B = V MN-major SW128 split by N between the two CTAs), for the 128-head pair decode:
//   (1) the A layout in TMEM (K packing, whether lanes 64-127 must duplicate lanes 0-63),
//   (2) cycles per MMA for the TS shapes vs the SS ones.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/probe_pair_ts.cu -o /tmp/pts && /tmp/pts
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2506_01969_b200/csrc/sm100_ptx.cuh"

using namespace etap_b200;

__device__ __forceinline__ void umma_pair_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_pair_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_pair_mc(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            ptx::smem_u32(bar)), "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void alloc_pair(uint32_t* dst, uint32_t n) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(dst)), "r"(n)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc_pair(uint32_t t, uint32_t n) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(n) : "memory");
}

__host__ __device__ constexpr uint32_t idesc(uint32_t m, uint32_t n, uint32_t amn, uint32_t bmn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (amn << 15) | (bmn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__host__ __device__ inline int sw128(int r, int c) { return r * 128 + ((((c * 2) >> 4) ^ (r & 7)) << 4) + ((c * 2) & 15); }

// a[cta][64][64] (heads x K) bf16, b[cta][64 K][128 N] bf16 (this CTA's N half), out[cta][128][128]
// dup: 1 = lanes 64-127 duplicate lanes 0-63, 0 = lanes 64-127 zero
__global__ void __cluster_dims__(2, 1, 1) ts_layout_kernel(int dup, const uint16_t* a, const uint16_t* b, float* out) {
    extern __shared__ uint8_t dsm[];
    uint8_t* sm = ptx::align_smem_1024(dsm);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int cta = ptx::cluster_ctarank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 64 * 128; i += blockDim.x) {
        const int k = i / 128, n = i % 128;
        *reinterpret_cast<uint16_t*>(sm + (n / 64) * 8192 + sw128(k, n % 64)) = b[(cta * 64 + k) * 128 + n];
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) alloc_pair(&tslot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    ptx::tc_fence_after();
    const uint32_t t = tslot;
    // A into TMEM columns [256, 288): lane m: column c = (A[m][2c], A[m][2c+1])
    {
        const int L = warp * 32 + lane;
        const int m = L & 63;
        uint32_t r[32];
        for (int c = 0; c < 32; ++c) {
            const uint32_t lo = a[(cta * 64 + m) * 64 + 2 * c], hi = a[(cta * 64 + m) * 64 + 2 * c + 1];
            r[c] = (L < 64 || dup) ? (lo | (hi << 16)) : 0u;
        }
        ptx::tmem_st32(t + (static_cast<uint32_t>(warp * 32) << 16) + 256, r);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    ptx::tc_fence_after();
    if (cta == 0 && warp == 0) {
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(sm), 8192, 1024, ptx::LAYOUT_SW128);
        const uint32_t id = idesc(128, 256, 0, 1);
        for (int kk = 0; kk < 4; ++kk) umma_pair_ts(t, t + 256 + 8 * kk, bd + kk * (2048 >> 4), id, kk > 0);
        commit_pair_mc(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    for (int c = 0; c < 128; c += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(t + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
        ptx::tmem_wait_ld();
        for (int j = 0; j < 32; ++j) out[(cta * 128 + warp * 32 + lane) * 128 + c + j] = __uint_as_float(r[j]);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    if (warp == 0) { ptx::tc_fence_after(); dealloc_pair(t, 512); }
}

// kind 0: TS (A = TMEM col 256), B MN-major SW128; kind 1: SS, A K-major SW128, B MN-major SW128
__global__ void __cluster_dims__(2, 1, 1) cost_kernel(int kind, int m, int n, int count, long long* out) {
    extern __shared__ uint8_t dsm[];
    uint8_t* smem = ptx::align_smem_1024(dsm);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) alloc_pair(&tslot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    ptx::tc_fence_after();
    const uint32_t t = tslot;
    const bool leader = ptx::cluster_ctarank() == 0;
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    const uint64_t ad = ptx::smem_desc(a, 16, 1024, ptx::LAYOUT_SW128);
    const uint64_t bd = ptx::smem_desc(b, 8192, 1024, ptx::LAYOUT_SW128);
    const uint32_t id = idesc(m, n, 0, 1);
    for (int rep = 0; rep < 2; ++rep) {
        long long t0 = 0;
        if (threadIdx.x < 32 && leader) {
            __syncwarp();
            t0 = clock64();
            for (int i = 0; i < count; i += 4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (kind == 0) umma_pair_ts(t, t + 384 + 8 * j, bd + j * 128, id, (i + j) > 0);
                    else umma_pair_ss(t, ad + j * 2, bd + j * 128, id, (i + j) > 0);
                }
            }
            commit_pair_mc(&bar);
        }
        if (threadIdx.x < 32) {
            ptx::mbar_wait(&bar, rep & 1);
            const long long t1 = clock64();
            if (rep == 1 && threadIdx.x == 0 && leader) out[blockIdx.x] = t1 - t0;
        }
        ptx::cluster_sync_all();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    if (threadIdx.x < 32) { ptx::tc_fence_after(); dealloc_pair(t, 512); }
}

static uint16_t bf16_bits(float x) { __nv_bfloat16 h = __float2bfloat16_rn(x); return *reinterpret_cast<uint16_t*>(&h); }
static float bf16_val(uint16_t bb) { uint32_t u = static_cast<uint32_t>(bb) << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
    srand(11);
    std::vector<uint16_t> a(2 * 64 * 64), b(2 * 64 * 128);
    for (auto& x : a) x = bf16_bits((rand() % 17 - 8) / 8.0f);
    for (auto& x : b) x = bf16_bits((rand() % 17 - 8) / 8.0f);
    uint16_t *da, *db; float* dout;
    cudaMalloc(&da, a.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dout, 2 * 128 * 128 * 4);
    cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(ts_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    for (int dup = 1; dup >= 0; --dup) {
        cudaMemset(dout, 0xff, 2 * 128 * 128 * 4);
        ts_layout_kernel<<<2, 128, 40 * 1024>>>(dup, da, db, dout);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> o(2 * 128 * 128);
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        // expected (2x2 layout): CTA c, lane m < 64, col j: D[m][j] (N 0..127, B of CTA 0);
        // lane 64 + m, col j: D[m][128 + j] (B of CTA 1); D = A_c . [B_0 | B_1]
        double maxerr = 0;
        for (int c = 0; c < 2; ++c)
            for (int L = 0; L < 128; ++L)
                for (int j = 0; j < 128; ++j) {
                    const int m = L & 63, nb = L >> 6;
                    double s = 0;
                    for (int k = 0; k < 64; ++k)
                        s += (double)bf16_val(a[(c * 64 + m) * 64 + k]) * bf16_val(b[(nb * 64 + k) * 128 + j]);
                    maxerr = std::fmax(maxerr, std::fabs(s - o[(c * 128 + L) * 128 + j]));
                }
        printf("{\"probe\": \"pair TS layout\", \"dup\": %d, \"cuda\": \"%s\", \"max_abs_err_vs_2x2\": %.3e}\n", dup,
               cudaGetErrorString(e), maxerr);
        if (e != cudaSuccess) return 1;
    }
    long long* dc; cudaMalloc(&dc, 148 * 8);
    cudaFuncSetAttribute(cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 129 * 1024);
    const int shapes[][3] = {{0, 128, 256}, {0, 128, 128}, {0, 128, 64}, {1, 128, 256}, {1, 128, 128}, {0, 256, 256}, {0, 256, 128}};
    for (int grid : {2, 148})
        for (auto& s : shapes) {
            cudaMemset(dc, 0, 148 * 8);
            cost_kernel<<<grid, 128, 129 * 1024>>>(s[0], s[1], s[2], 256, dc);
            cudaError_t e2 = cudaDeviceSynchronize();
            std::vector<long long> cyc(148);
            cudaMemcpy(cyc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
            long long mx = 0; for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
            printf("{\"probe\": \"pair mma cost\", \"grid\": %d, \"a\": \"%s\", \"m\": %d, \"n\": %d, \"cycles_per_mma\": %.1f, \"cuda\": \"%s\"}\n",
                   grid, s[0] == 0 ? "TMEM" : "smem K-major", s[1], s[2], mx / 256.0, cudaGetErrorString(e2));
            if (e2 != cudaSuccess) return 1;
        }
    return 0;
}
