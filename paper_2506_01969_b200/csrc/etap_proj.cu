// SPDX-License-Identifier: Apache-2.0
// The steps on either side of the decode kernel in an absorbed-MLA (DeepSeek) decode layer
// (out of scope in the reference):
//
//   before:  q_latent[b,h,:] = q_nope[b,h,:] . W_UK[h]    (128 -> 512, per head)
//            q_rope[b,h,:]   = RoPE(q_pe[b,h,:], cos[b], sin[b])
//            -> Q[b,0,h,:] = [q_latent | q_rope] bf16, the decode kernel's input
//   after:   o_head[b,h,:]   = O[b,h,:] . W_UV[h]          (512 -> 128, per head, fp32 O in)
//
// Both projections are per-head GEMMs with only B (tokens) rows. They use the same
// transposition as the decode kernel (ETAP): y^T[n_out x B] = W[h]^T[n_out x K] . x^T[K x B],
// so the wide weight dimension sits on the UMMA M axis (M = 128 per CTA) and the B tokens on
// N (16..256): no padding of 16 tokens up to M = 64 / 128. W[h] is read MN-major straight from
// its [K][n_out] row-major storage (like V^T in GEMM2), x K-major. bf16 operands, fp32
// accumulation in TMEM; x may be fp32 (the decode output), converted to bf16 on the way into
// shared memory.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/etap_mla.h"
#include "sm100_ptx.cuh"

namespace etap_b200 {
int host_fail(int code, const char* msg);  // etap_mla.cu
int encode_bf16_sw128(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows);
}

namespace {

using namespace etap_b200;

constexpr int PJ_THREADS = 128;
constexpr int PJ_KC = 64;                       // K rows per pipeline stage (one SW128 atom row)
constexpr int PJ_W_BYTES = PJ_KC * 128 * 2;     // W^T stage: 64 k x 128 n_out bf16 = 2 x 8 KB slots
constexpr int PJ_MAX_ST = 8;                    // stages in flight (all of K = 512 for <= 64 tokens)
constexpr int PJ_RING = 200 * 1024;             // stage ring budget
constexpr int PJ_SMEM = PJ_RING + 192 + 1024;

// stage = W^T chunk + x^T chunk (n_pad rows x 128 B), 1 KB aligned
__host__ __device__ inline int pj_stage_bytes(int n_pad) { return (PJ_W_BYTES + n_pad * 128 + 1023) / 1024 * 1024; }
__host__ __device__ inline int pj_stages(int n_pad, int nk) {
    int st = PJ_RING / pj_stage_bytes(n_pad);
    st = st < PJ_MAX_ST ? st : PJ_MAX_ST;
    return st < nk ? st : nk;
}

struct ProjParams {
    const void* x;        // [B][H][K] (strides in elements), bf16 or fp32
    int x_fp32;
    int64_t x_sb, x_sh;
    const __nv_bfloat16* w;  // [H][K][N_out] bf16
    int batch, heads, k_dim, n_out, n_pad;
    void* y;              // [B][H][N_out] (strides in elements), bf16 or fp32
    int y_fp32;
    int64_t y_sb, y_sh;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// SW128: 16-byte unit u of row r (128 B rows, 8-row atoms) lives at unit u ^ (r & 7)
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t unit) {
    return row * 128 + ((unit ^ (row & 7)) << 4);
}

// Stages for chunks [kc0, kc1) of K (stage i at st0 + (kc % NST) * SB): the W^T block
// (MN-major: 64 k-rows x 64 n per 8 KB slot, two slots) and x^T (K-major: one 128 B row of
// 64 k per token, rows >= batch zero). W and bf16 x go through cp.async, one commit group per
// chunk; fp32 x is loaded 4 units per thread at a time across all the chunks (independent
// loads in flight) and converted to bf16 on the way into shared memory.
__device__ void load_stages(const ProjParams& p, const CUtensorMap* tm_w, uint64_t* full, int h, int n0, int kc0,
                            int kc1, uint8_t* st0, int SB, int NST) {
    if (p.x_fp32) {
        const int per = p.n_pad * 8, total = (kc1 - kc0) * per;
        for (int base = threadIdx.x; base < total; base += 4 * PJ_THREADS) {
            float4 a[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = base + j * PJ_THREADS;
                const int kc = kc0 + i / per, rem = i % per, r = rem >> 3, u = rem & 7;
                if (i < total && r < p.batch) {
                    const float4* src = reinterpret_cast<const float4*>(
                        static_cast<const float*>(p.x) + r * p.x_sb + h * p.x_sh + kc * PJ_KC + u * 8);
                    a[j][0] = __ldg(src);
                    a[j][1] = __ldg(src + 1);
                } else {
                    a[j][0] = a[j][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = base + j * PJ_THREADS;
                if (i >= total) break;
                const int kc = kc0 + i / per, rem = i % per, r = rem >> 3, u = rem & 7;
                const uint32_t dst = ptx::smem_u32(st0 + (kc % NST) * SB + PJ_W_BYTES) + sw128(r, u);
                __nv_bfloat162 v0 = __floats2bfloat162_rn(a[j][0].x, a[j][0].y);
                __nv_bfloat162 v1 = __floats2bfloat162_rn(a[j][0].z, a[j][0].w);
                __nv_bfloat162 v2 = __floats2bfloat162_rn(a[j][1].x, a[j][1].y);
                __nv_bfloat162 v3 = __floats2bfloat162_rn(a[j][1].z, a[j][1].w);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst),
                             "r"(*reinterpret_cast<uint32_t*>(&v0)), "r"(*reinterpret_cast<uint32_t*>(&v1)),
                             "r"(*reinterpret_cast<uint32_t*>(&v2)), "r"(*reinterpret_cast<uint32_t*>(&v3))
                             : "memory");
            }
        }
    }
    for (int kc = kc0; kc < kc1; ++kc) {
        uint8_t* st = st0 + (kc % NST) * SB;
        const uint32_t x_s = ptx::smem_u32(st) + PJ_W_BYTES;
        // W: two TMA boxes of 64 k-rows x 64 n (8 KB, SW128) per chunk, on the stage's barrier
        if (threadIdx.x == 0) {
            ptx::mbar_arrive_expect_tx(&full[kc % NST], PJ_W_BYTES);
            const int row = h * p.k_dim + kc * PJ_KC;
            ptx::tma_load_2d(st, tm_w, &full[kc % NST], n0, row, ptx::policy_evict_first());
            ptx::tma_load_2d(st + 8192, tm_w, &full[kc % NST], n0 + 64, row, ptx::policy_evict_first());
        }
        if (!p.x_fp32) {
            for (int i = threadIdx.x; i < p.n_pad * 8; i += PJ_THREADS) {
                const int r = i >> 3, u = i & 7;
                const uint32_t dst = x_s + sw128(r, u);
                if (r >= p.batch)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0u) : "memory");
                else
                    cp_async16(dst, static_cast<const __nv_bfloat16*>(p.x) + r * p.x_sb + h * p.x_sh + kc * PJ_KC + u * 8);
            }
        }
        cp_async_commit();
    }
}

__device__ __forceinline__ void cp_async_wait_pending(int pending) {
    switch (pending) {  // wait_group takes an immediate
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
}

// grid (heads, n_out / 128), 128 threads: y[b, h, n0 .. n0+128) for all b. A ring of NST
// stages: every chunk's loads are in flight before the first MMA when K fits (<= 8 chunks),
// so the kernel costs about one global round trip instead of one per chunk.
__global__ void __launch_bounds__(PJ_THREADS, 1)
    etap_head_proj_kernel(const __grid_constant__ CUtensorMap tm_w, const ProjParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + PJ_RING);  // [PJ_MAX_ST] stage consumed
    uint64_t* full = bar + PJ_MAX_ST;                                // [PJ_MAX_ST] W chunk landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + PJ_RING + 16 * PJ_MAX_ST);
    const int h = blockIdx.x, n0 = blockIdx.y * 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = p.k_dim / PJ_KC;
    const int SB = pj_stage_bytes(p.n_pad), NST = pj_stages(p.n_pad, nk);
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tm_w);
        for (int i = 0; i < PJ_MAX_ST; ++i) {
            ptx::mbar_init(&bar[i], 1);
            ptx::mbar_init(&full[i], 1);
        }
        ptx::fence_mbar_init();
    }
    const uint32_t tcols = p.n_pad <= 32 ? 32 : p.n_pad <= 64 ? 64 : p.n_pad <= 128 ? 128 : 256;
    if (warp == 0) ptx::tmem_alloc(tmem_slot, tcols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();

    const uint32_t idesc = ptx::idesc_bf16_f32(128, p.n_pad, 1, 0);
    load_stages(p, &tm_w, full, h, n0, 0, NST, smem, SB, NST);
    for (int kc = 0; kc < nk; ++kc) {
        const int slot = kc % NST;
        uint8_t* st = smem + slot * SB;
        // chunks 0 .. min(nk, kc + NST) - 1 have been issued (chunk j + NST refills slot j after
        // iteration j): wait until only the groups after chunk kc's are pending
        cp_async_wait_pending(min(NST - 1, nk - 1 - kc));
        ptx::fence_proxy_async_smem();  // cp.async / st.shared writes -> tensor core reads
        __syncthreads();
        ptx::mbar_wait(&full[slot], (kc / NST) & 1);
        if (warp == 0) {
            ptx::tc_fence_after();
            const uint32_t w_s = ptx::smem_u32(st), x_s = w_s + PJ_W_BYTES;
            const uint64_t a0 = ptx::smem_desc(w_s, 8192, 1024, ptx::LAYOUT_SW128);   // MN-major W^T
            const uint64_t b0 = ptx::smem_desc(x_s, 16, 1024, ptx::LAYOUT_SW128);     // K-major x^T
#pragma unroll
            for (int kk = 0; kk < PJ_KC / 16; ++kk)
                ptx::umma_f16_elect(tmem, a0 + kk * (2048 >> 4), b0 + 2 * kk, idesc, (kc == 0 && kk == 0) ? 0u : 1u);
            ptx::umma_commit_elect(&bar[slot]);
        }
        if (kc + NST < nk) {
            // refill this slot with chunk kc + NST once the MMAs above have read it
            ptx::mbar_wait(&bar[slot], (kc / NST) & 1);
            load_stages(p, &tm_w, full, h, n0, kc + NST, kc + NST + 1, smem, SB, NST);
        }
    }
    // all MMAs complete: the last commit covers every earlier tcgen05 op of the issuing thread
    ptx::mbar_wait(&bar[(nk - 1) % NST], ((nk - 1) / NST) & 1);
    ptx::tc_fence_after();
    // epilogue: TMEM lane = output feature n0 + 32*warp + lane, column = token
    const int n = n0 + warp * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    for (int c0 = 0; c0 < p.n_pad; c0 += 32) {
        uint32_t v[32];
        ptx::tmem_ld32(t_lane + c0, v);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int b = c0 + j;
            if (b >= p.batch) break;
            const int64_t off = b * p.y_sb + h * p.y_sh + n;
            const float f = __uint_as_float(v[j]);
            if (p.y_fp32) static_cast<float*>(p.y)[off] = f;
            else static_cast<__nv_bfloat16*>(p.y)[off] = __float2bfloat16_rn(f);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, tcols);
    }
}

// RoPE on the rope part of Q (NeoX half rotation over the 64 rope dims, fp32 math):
// Q[b,0,h,512+i] = x_i cos_i - x_{i+32} sin_i, Q[b,0,h,544+i] = x_{i+32} cos_i + x_i sin_i
__global__ void __launch_bounds__(128) etap_rope_q_kernel(const __nv_bfloat16* __restrict__ q_pe,
                                                         const float* __restrict__ cos_t,
                                                         const float* __restrict__ sin_t,
                                                         __nv_bfloat16* __restrict__ q, int batch, int heads,
                                                         int q_tokens) {
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (bt, h, i)
    const int64_t total = static_cast<int64_t>(batch) * q_tokens * heads * 32;
    if (idx >= total) return;
    const int i = static_cast<int>(idx % 32);
    const int64_t row = idx / 32;                   // (b * q_tokens + t) * heads + h
    const int64_t bt = row / heads;
    const float c = cos_t[bt * 32 + i], s = sin_t[bt * 32 + i];
    const float x0 = __bfloat162float(q_pe[row * 64 + i]), x1 = __bfloat162float(q_pe[row * 64 + 32 + i]);
    q[row * 576 + 512 + i] = __float2bfloat16_rn(x0 * c - x1 * s);
    q[row * 576 + 544 + i] = __float2bfloat16_rn(x1 * c + x0 * s);
}

int launch_attr(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr, void* stream) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return 0;
}

}  // namespace

extern "C" {

int etap_mla_head_proj(const void* x, int x_fp32, int64_t x_stride_b, int64_t x_stride_h, const void* w,
                       int batch, int heads, int k_dim, int n_out, void* y, int y_fp32, int64_t y_stride_b,
                       int64_t y_stride_h, void* stream) {
    using etap_b200::host_fail;
    if (!x || !w || !y) return host_fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (batch < 1 || batch > 256 || heads < 1 || k_dim < 64 || k_dim % 64 != 0 || n_out < 128 || n_out % 128 != 0)
        return host_fail(ETAP_ERR_SHAPE, "head_proj: 1 <= batch <= 256, k_dim a multiple of 64, n_out of 128");
    if (x_stride_h % 8 != 0 || x_stride_b % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) ||
        (reinterpret_cast<uintptr_t>(w) & 15))
        return host_fail(ETAP_ERR_SHAPE, "head_proj: x / w must be 16-byte aligned with strides multiple of 8");
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        major != 10)
        return host_fail(ETAP_ERR_CUDA, "head_proj: needs an sm_100 device");
    if (pj_stage_bytes((batch + 15) / 16 * 16) > PJ_RING) return host_fail(ETAP_ERR_SHAPE, "head_proj: stage too large");
    static const cudaError_t attr_rc =
        cudaFuncSetAttribute(etap_head_proj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PJ_SMEM);
    if (attr_rc != cudaSuccess) return host_fail(ETAP_ERR_CUDA, cudaGetErrorString(attr_rc));
    ProjParams p;
    p.x = x;
    p.x_fp32 = x_fp32 ? 1 : 0;
    p.x_sb = x_stride_b;
    p.x_sh = x_stride_h;
    p.w = static_cast<const __nv_bfloat16*>(w);
    p.batch = batch;
    p.heads = heads;
    p.k_dim = k_dim;
    p.n_out = n_out;
    p.n_pad = (batch + 15) / 16 * 16;
    p.y = y;
    p.y_fp32 = y_fp32 ? 1 : 0;
    p.y_sb = y_stride_b;
    p.y_sh = y_stride_h;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(heads, n_out / 128);
    cfg.blockDim = dim3(PJ_THREADS);
    cfg.dynamicSmemBytes = PJ_SMEM;
    launch_attr(cfg, attr, stream);
    CUtensorMap tm_w;
    if (int rc = etap_b200::encode_bf16_sw128(&tm_w, w, static_cast<uint64_t>(n_out),
                                              static_cast<uint64_t>(heads) * k_dim, PJ_KC))
        return rc;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, etap_head_proj_kernel, tm_w, p);
    if (e != cudaSuccess) return host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}

int etap_mla_absorb_q(const void* q_nope, const void* q_pe, const float* cos_t, const float* sin_t,
                      const void* w_uk, int batch, int q_tokens, int heads, void* q, void* stream) {
    using etap_b200::host_fail;
    if (!q_nope || !q_pe || !cos_t || !sin_t || !w_uk || !q) return host_fail(ETAP_ERR_SHAPE, "NULL pointer argument");
    if (q_tokens < 1 || q_tokens > ETAP_MLA_MAX_Q_TOKENS) return host_fail(ETAP_ERR_SHAPE, "q_tokens must be in [1, 8]");
    const int rows = batch * q_tokens;  // token rows of the projection
    // q_latent = q_nope . W_UK (128 -> 512) into Q[..., 0:512]
    if (int rc = etap_mla_head_proj(q_nope, 0, static_cast<int64_t>(heads) * 128, 128, w_uk, rows, heads, 128,
                                    ETAP_MLA_D_V, q, 0, static_cast<int64_t>(heads) * ETAP_MLA_D_QK, ETAP_MLA_D_QK,
                                    stream))
        return rc;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = {};
    const int64_t total = static_cast<int64_t>(rows) * heads * 32;
    cfg.gridDim = dim3(static_cast<unsigned>((total + 127) / 128));
    cfg.blockDim = dim3(128);
    launch_attr(cfg, attr, stream);
    const cudaError_t e = cudaLaunchKernelEx(&cfg, etap_rope_q_kernel, static_cast<const __nv_bfloat16*>(q_pe), cos_t,
                                             sin_t, static_cast<__nv_bfloat16*>(q), batch, heads, q_tokens);
    if (e != cudaSuccess) return host_fail(ETAP_ERR_CUDA, cudaGetErrorString(e));
    return ETAP_OK;
}

int etap_mla_up_proj(const float* o, const void* w_uv, int batch, int q_tokens, int heads, void* out, int out_fp32,
                     void* stream) {
    using etap_b200::host_fail;
    if (q_tokens < 1 || q_tokens > ETAP_MLA_MAX_Q_TOKENS) return host_fail(ETAP_ERR_SHAPE, "q_tokens must be in [1, 8]");
    // out[b,t,h,:] = O[b,t,h,:] . W_UV[h]  (512 -> 128)
    return etap_mla_head_proj(o, 1, static_cast<int64_t>(heads) * ETAP_MLA_D_V, ETAP_MLA_D_V, w_uv,
                              batch * q_tokens, heads, ETAP_MLA_D_V, 128, out, out_fp32,
                              static_cast<int64_t>(heads) * 128, 128, stream);
}

}  // extern "C"
