// SPDX-License-Identifier: Apache-2.0
// Probe (experiment, not product): tcgen05 cta_group::2 (CTA pair) semantics and cost for the
// 128-head pair decode.
//   (1) layout: where D rows land in each CTA's TMEM for M = 128 and M = 256 pair MMAs, and how
//       the B operand is split between the two CTAs' shared memory;
//   (2) cost: cycles per back-to-back MMA, pair shapes vs the 1-CTA shapes the HG = 64 kernel uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/probe_pair.cu -o /tmp/probe_pair && /tmp/probe_pair
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

__device__ __forceinline__ void umma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
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
__device__ __forceinline__ void fence_after_pair() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__host__ __device__ constexpr uint32_t idesc(uint32_t m, uint32_t n, uint32_t amn, uint32_t bmn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (amn << 15) | (bmn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// byte offset of element (row r, col c) of a [rows][64] bf16 SW128 tile (TMA layout)
__host__ __device__ inline int sw128(int r, int c) { return r * 128 + ((((c * 2) >> 4) ^ (r & 7)) << 4) + ((c * 2) & 15); }

// mode 0: GEMM1 shape, M = 128 pair (64 A rows per CTA, K-major), B K-major: per CTA nb rows x 64 K
// mode 1: GEMM2 shape, M = 256 pair (128 A rows per CTA, MN-major: two [64 K][64 M] atoms 8 KB apart), B K-major
// A / B per CTA come from global: a[cta][rows_a][64] (logical M x K), b[cta][nb][64] (logical N x K)
// out[cta][128 lanes][ncol]
__global__ void __cluster_dims__(2, 1, 1) layout_kernel(int mode, int n, const uint16_t* a, const uint16_t* b, float* out) {
    extern __shared__ uint8_t dsm[];
    uint8_t* sm = ptx::align_smem_1024(dsm);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int cta = ptx::cluster_ctarank();
    const int tid = threadIdx.x, warp = tid >> 5;
    const int arows = mode == 0 ? 64 : 128, nb = n / 2;
    uint8_t* sa = sm;
    uint8_t* sb = sm + 32768;
    for (int i = tid; i < arows * 64; i += blockDim.x) {
        const int m = i / 64, k = i % 64;
        const uint16_t v = a[(cta * arows + m) * 64 + k];
        if (mode == 0) *reinterpret_cast<uint16_t*>(sa + sw128(m, k)) = v;            // [M rows][64 K]
        else *reinterpret_cast<uint16_t*>(sa + (m / 64) * 8192 + sw128(k, m % 64)) = v;  // [64 K rows][64 M] atoms
    }
    for (int i = tid; i < nb * 64; i += blockDim.x) {
        const int nn = i / 64, k = i % 64;
        *reinterpret_cast<uint16_t*>(sb + sw128(nn, k)) = b[(cta * nb + nn) * 64 + k];
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) alloc_pair(&tslot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    fence_after_pair();
    const uint32_t t = tslot;
    if (cta == 0 && warp == 0) {
        uint64_t ad, bd;
        uint32_t id;
        const uint32_t a0 = ptx::smem_u32(sa), b0 = ptx::smem_u32(sb);
        bd = ptx::smem_desc(b0, 16, 1024, ptx::LAYOUT_SW128);
        if (mode == 0) {
            ad = ptx::smem_desc(a0, 16, 1024, ptx::LAYOUT_SW128);
            id = idesc(128, n, 0, 0);
            for (int kk = 0; kk < 4; ++kk) umma_pair(t, ad + 2 * kk, bd + 2 * kk, id, kk > 0);
        } else {
            ad = ptx::smem_desc(a0, 8192, 1024, ptx::LAYOUT_SW128);
            id = idesc(256, n, 1, 0);
            for (int kk = 0; kk < 4; ++kk) umma_pair(t, ad + kk * (2048 >> 4), bd + 2 * kk, id, kk > 0);
        }
        commit_pair_mc(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    if (warp < 4) {
        for (int c = 0; c < n; c += 16) {
            uint32_t r[16];
            ptx::tmem_ld16(t + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
            ptx::tmem_wait_ld();
            for (int j = 0; j < 16; ++j) out[(cta * 128 + warp * 32 + (tid & 31)) * n + c + j] = __uint_as_float(r[j]);
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    if (warp == 0) { fence_after_pair(); dealloc_pair(t, 512); }
}

// cost: `count` back-to-back MMAs of one pair (or single) shape; zeros in smem
// kind 0: pair GEMM1 (A K-major), 1: pair GEMM2 (A MN-major), 2: single GEMM1, 3: single GEMM2
template <bool PAIR>
__device__ void cost_body(int kind, int m, int n, int count, long long* out) {
    extern __shared__ uint8_t dsm[];
    uint8_t* smem = ptx::align_smem_1024(dsm);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) {
        if (PAIR) alloc_pair(&tslot, 512);
        else ptx::tmem_alloc(&tslot, 512);
    }
    ptx::tc_fence_before();
    if (PAIR) ptx::cluster_sync_all(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t t = tslot;
    const bool leader = PAIR ? ptx::cluster_ctarank() == 0 : true;
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    const bool g2 = (kind & 1) != 0;
    const uint64_t ad = g2 ? ptx::smem_desc(a, 8192, 1024, ptx::LAYOUT_SW128) : ptx::smem_desc(a, 16, 1024, ptx::LAYOUT_SW128);
    const uint64_t bd = ptx::smem_desc(b, 16, 1024, ptx::LAYOUT_SW128);
    const uint32_t id = idesc(m, n, g2 ? 1 : 0, 0);
    for (int rep = 0; rep < 2; ++rep) {
        long long t0 = 0;
        if (threadIdx.x < 32 && leader) {
            __syncwarp();
            t0 = clock64();
            for (int i = 0; i < count; i += 4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (PAIR) umma_pair(t, ad + j * 2, bd + j * 2, id, (i + j) > 0);
                    else ptx::umma_f16_elect(t, ad + j * 2, bd + j * 2, id, (i + j) > 0);
                }
            }
            if (PAIR) commit_pair_mc(&bar); else ptx::umma_commit_elect(&bar);
        }
        if (threadIdx.x < 32) {
            ptx::mbar_wait(&bar, rep & 1);
            const long long t1 = clock64();
            if (rep == 1 && threadIdx.x == 0 && leader) out[blockIdx.x] = t1 - t0;
        }
        if (PAIR) ptx::cluster_sync_all(); else __syncthreads();
    }
    ptx::tc_fence_before();
    if (PAIR) ptx::cluster_sync_all(); else __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        if (PAIR) dealloc_pair(t, 512); else ptx::tmem_dealloc(t, 512);
    }
}

__global__ void __cluster_dims__(2, 1, 1) cost_pair(int kind, int m, int n, int count, long long* out) {
    cost_body<true>(kind, m, n, count, out);
}
__global__ void cost_single(int kind, int m, int n, int count, long long* out) { cost_body<false>(kind, m, n, count, out); }

static uint16_t bf16_bits(float x) { __nv_bfloat16 h = __float2bfloat16_rn(x); return *reinterpret_cast<uint16_t*>(&h); }
static float bf16_val(uint16_t bb) { uint32_t u = static_cast<uint32_t>(bb) << 16; float f; memcpy(&f, &u, 4); return f; }

static void layout_test(int mode, int n) {
    const int arows = mode == 0 ? 64 : 128, nb = n / 2;
    std::vector<uint16_t> a(2 * arows * 64), b(2 * nb * 64);
    for (auto& x : a) x = bf16_bits((rand() % 17 - 8) / 8.0f);
    for (auto& x : b) x = bf16_bits((rand() % 17 - 8) / 8.0f);
    uint16_t *da, *db; float* dout;
    cudaMalloc(&da, a.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dout, 2 * 128 * n * 4);
    cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0xff, 2 * 128 * n * 4);
    cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    layout_kernel<<<2, 128, 80 * 1024>>>(mode, n, da, db, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(2 * 128 * n);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    {
        char fn[128];
        snprintf(fn, sizeof fn, "gpurun_out/pair_layout_m%d_n%d.bin", mode, n);
        FILE* f = fopen(fn, "wb");
        if (f) { fwrite(a.data(), 2, a.size(), f); fwrite(b.data(), 2, b.size(), f); fwrite(o.data(), 4, o.size(), f); fclose(f); }
    }
    // candidate: D_cta[i][j] = sum_k A_cta[i][k] * Bcat[j][k], Bcat = [B_0 ; B_1] (N rows)
    int found = 0, total = 0, lane_match_ident = 0;
    std::vector<int> lane_of(2 * arows, -1);
    for (int cta = 0; cta < 2; ++cta)
        for (int i = 0; i < arows; ++i) {
            std::vector<double> ref(n);
            for (int j = 0; j < n; ++j) {
                double s = 0;
                for (int k = 0; k < 64; ++k) s += (double)bf16_val(a[(cta * arows + i) * 64 + k]) * bf16_val(b[j * 64 + k]);
                ref[j] = s;
            }
            ++total;
            for (int lane = 0; lane < 128; ++lane) {
                bool ok = true;
                for (int j = 0; j < n && ok; ++j) ok = std::fabs(o[(cta * 128 + lane) * n + j] - ref[j]) < 1e-3;
                if (ok) { lane_of[cta * arows + i] = lane; ++found; break; }
            }
        }
    for (int cta = 0; cta < 2; ++cta)
        for (int i = 0; i < arows; ++i) lane_match_ident += lane_of[cta * arows + i] == i;
    printf("{\"probe\": \"pair layout\", \"mode\": \"%s\", \"n\": %d, \"cuda\": \"%s\", \"rows_found\": %d, \"rows\": %d, "
           "\"lane_eq_row\": %d, \"lanes_cta0\": [",
           mode == 0 ? "M128 pair K-major A" : "M256 pair MN-major A", n, cudaGetErrorString(e), found, total, lane_match_ident);
    for (int i = 0; i < arows; ++i) printf("%d%s", lane_of[i], i + 1 < arows ? "," : "");
    printf("], \"lanes_cta1\": [");
    for (int i = 0; i < arows; ++i) printf("%d%s", lane_of[arows + i], i + 1 < arows ? "," : "");
    printf("]}\n");
    cudaFree(da); cudaFree(db); cudaFree(dout);
}

int main(int argc, char** argv) {
    srand(7);
    layout_test(0, 64);
    layout_test(0, 128);
    layout_test(1, 128);
    layout_test(1, 64);
    long long* dc; cudaMalloc(&dc, 148 * 8);
    cudaFuncSetAttribute(cost_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 129 * 1024);
    cudaFuncSetAttribute(cost_single, cudaFuncAttributeMaxDynamicSharedMemorySize, 129 * 1024);
    struct S { int pair, kind, m, n; };
    const S shapes[] = {{0, 2, 64, 64}, {0, 3, 128, 64}, {0, 3, 128, 128}, {1, 0, 128, 32}, {1, 0, 128, 64}, {1, 0, 128, 128},
                        {1, 0, 256, 64}, {1, 1, 256, 64}, {1, 1, 256, 128}, {1, 1, 256, 256}, {1, 1, 128, 128}};
    for (int grid : {2, 148}) {
        for (auto& s : shapes) {
            cudaMemset(dc, 0, 148 * 8);
            if (s.pair) cost_pair<<<grid, 128, 129 * 1024>>>(s.kind, s.m, s.n, 256, dc);
            else cost_single<<<grid, 128, 129 * 1024>>>(s.kind, s.m, s.n, 256, dc);
            cudaError_t e2 = cudaDeviceSynchronize();
            std::vector<long long> cyc(148);
            cudaMemcpy(cyc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
            long long mx = 0; for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
            printf("{\"probe\": \"mma cost\", \"grid\": %d, \"pair\": %d, \"a\": \"%s\", \"m\": %d, \"n\": %d, \"cycles_per_mma\": %.1f, \"cuda\": \"%s\"}\n",
                   grid, s.pair, (s.kind & 1) ? "MN-major" : "K-major", s.m, s.n, mx / 256.0, cudaGetErrorString(e2));
            if (e2 != cudaSuccess) return 1;
        }
    }
    return 0;
}
