// Kernel 3: block-sparse FlashAttention prefill for sm_100a.
//
// One CTA computes one 128-row query tile of one head over that tile's
// selected key blocks (ascending block ids from kernel 2). Per selected block
// j (128 keys):  S = Q K_j^T (tcgen05, fp32 in TMEM) -> online softmax in
// registers -> P (bf16, shared memory) -> O += P V_j (tcgen05, fp32 in TMEM).
// The reference semantics it realises are softmax_weighted_sum over the kept
// set (proj/src/attention.cpp:35-49) with the causal mask of :28-30; rows with
// no visible kept key produce zeros (:40-41).
//
// Warp roles (192 threads):
//   warps 0-3  softmax / correction / epilogue; thread t owns query row t
//              (TMEM lane t), 128 fp32 scores per block.
//   warp 4     TMA producer: Q once, then K_j / V_j tiles into 2-stage rings.
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer.
// Pipelines (mbarriers): K/V full/empty rings (TMA <-> MMA), S full/empty
// double buffer in TMEM (MMA <-> softmax), P full (softmax -> MMA) and
// per-P-buffer "PV done" (MMA -> softmax, gates P reuse, O rescale, epilogue).
// The MMA warp issues S_{j+1} before O += P_j V_j, so the tensor core computes
// the next score tile while the softmax warps exponentiate the current one.
// The running max is rescaled lazily (only when it grows by > 2^8), so most
// blocks need no O correction.
//
// Shared memory (1024-aligned, 128B-swizzled, UMMA K-major unless noted):
//   Q  [2 d-chunks][128 rows][64 bf16]                 32 KB
//   K  [2 stages][2 d-chunks][128 keys][64 bf16]       64 KB
//   V  [2 stages][2 d-chunks][128 keys][64 bf16]       64 KB (MN-major B operand)
//   P  [2 bufs][2 key-chunks][128 rows][64 bf16]       64 KB
// TMEM (512 columns): S0 [0,128), S1 [128,256), O [256,384).
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace shplb::kern {
namespace {

using namespace shplb::ptx;

constexpr int kThreads = 192;
constexpr int kTileBytes = kBlock * kHeadDim * 2;  // 32 KB: one 128x128 bf16 tile
constexpr int kChunkBytes = kTileBytes / 2;        // 16 KB: 128 rows x 128 B
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale when max grows by > 2^8

constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, 0, 0);  // A=Q K-major, B=K K-major
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, 0, 1);  // A=P K-major, B=V MN-major

struct __align__(8) Barriers {
    uint64_t q_full;
    uint64_t k_full[2], k_empty[2];
    uint64_t v_full[2], v_empty[2];
    uint64_t s_full[2], s_empty[2];
    uint64_t p_full[2];
    uint64_t pv_done[2];
    uint32_t tmem_base;
};

constexpr size_t kSmemQ = 0;
constexpr size_t kSmemK = kSmemQ + kTileBytes;
constexpr size_t kSmemV = kSmemK + 2 * kTileBytes;
constexpr size_t kSmemP = kSmemV + 2 * kTileBytes;
constexpr size_t kSmemBar = kSmemP + 2 * kTileBytes;
constexpr size_t kSmemTotal = kSmemBar + sizeof(Barriers) + 1024;  // + alignment slack

// K-major SW128 operand (Q, K, P): k-step kk (16 elements) lives in d/key
// chunk kk/4 at byte offset (kk%4)*32 within each 128-byte row; 8-row groups
// are 1024 B apart (SBO); LBO is unused for swizzled K-major.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile_addr, int kk) {
    return umma_desc_sw128(tile_addr + (kk >> 2) * kChunkBytes + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 operand (V as B of P.V): N = d spans the two 64-wide d
// chunks (LBO = 16 KB apart); K = keys, 8-key groups 1024 B apart (SBO);
// k-step kk starts 16 keys = 2 KB further.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile_addr, int kk) {
    return umma_desc_sw128(tile_addr + kk * 2048, kChunkBytes, 1024);
}

__global__ void __launch_bounds__(kThreads, 1) fa_sparse_kernel(const __grid_constant__ FaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bar = reinterpret_cast<Barriers*>(smem + kSmemBar);
    const uint32_t sQ = smem_u32(smem + kSmemQ);
    const uint32_t sK = smem_u32(smem + kSmemK);
    const uint32_t sV = smem_u32(smem + kSmemV);
    const uint32_t sP = smem_u32(smem + kSmemP);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const int32_t tile = p.tiles[blockIdx.x];
    const int h = tile >> 20;
    const int qb = tile & 0xFFFFF;
    const int g = p.heads.kv[h];
    const int64_t row_id = static_cast<int64_t>(h) * p.nqb + qb;
    const int nsel = p.cnt[row_id];
    const int32_t* sel = p.idx + row_id * p.kmax;

    if (threadIdx.x == 0) {
        mbar_init(&bar->q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->k_full[i], 1);
            mbar_init(&bar->k_empty[i], 1);
            mbar_init(&bar->v_full[i], 1);
            mbar_init(&bar->v_empty[i], 1);
            mbar_init(&bar->s_full[i], 1);
            mbar_init(&bar->s_empty[i], 128);
            mbar_init(&bar->p_full[i], 128);
            mbar_init(&bar->pv_done[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 5) tmem_alloc<kTmemCols>(&bar->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == 4) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0 && nsel > 0) {
            prefetch_tmap(&p.tm_q);
            prefetch_tmap(&p.tm_k);
            prefetch_tmap(&p.tm_v);
            mbar_arrive_expect_tx(&bar->q_full, kTileBytes);
            tma_load_3d(smem + kSmemQ, &p.tm_q, &bar->q_full, 0, qb * kBlock, h);
            tma_load_3d(smem + kSmemQ + kChunkBytes, &p.tm_q, &bar->q_full, 64, qb * kBlock, h);
            for (int j = 0; j < nsel; ++j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                const int key0 = sel[j] * kBlock;
                uint8_t* kdst = smem + kSmemK + st * kTileBytes;
                uint8_t* vdst = smem + kSmemV + st * kTileBytes;
                mbar_wait(&bar->k_empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&bar->k_full[st], kTileBytes);
                tma_load_3d(kdst, &p.tm_k, &bar->k_full[st], 0, key0, g);
                tma_load_3d(kdst + kChunkBytes, &p.tm_k, &bar->k_full[st], 64, key0, g);
                mbar_wait(&bar->v_empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&bar->v_full[st], kTileBytes);
                tma_load_3d(vdst, &p.tm_v, &bar->v_full[st], 0, key0, g);
                tma_load_3d(vdst + kChunkBytes, &p.tm_v, &bar->v_full[st], 64, key0, g);
            }
        }
    } else if (warp == 5) {
        // -------------------------------------------------------- MMA issuer
        if (lane == 0 && nsel > 0) {
            mbar_wait(&bar->q_full, 0);
            auto issue_pv = [&](int j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                mbar_wait(&bar->v_full[st], ph);
                mbar_wait(&bar->p_full[st], ph);
                tc_fence_after();
                const uint32_t pa = sP + st * kTileBytes;
                const uint32_t va = sV + st * kTileBytes;
#pragma unroll
                for (int kk = 0; kk < kBlock / 16; ++kk)
                    mma_bf16_ss(tmem + kColO, desc_kmajor(pa, kk), desc_mnmajor(va, kk), kIdescPV,
                                (j > 0 || kk > 0) ? 1u : 0u);
                mma_commit(&bar->v_empty[st]);
                mma_commit(&bar->pv_done[st]);
            };
            for (int j = 0; j < nsel; ++j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                mbar_wait(&bar->k_full[st], ph);
                mbar_wait(&bar->s_empty[st], ph ^ 1);
                tc_fence_after();
                const uint32_t ka = sK + st * kTileBytes;
                const uint32_t s_col = st ? kColS1 : kColS0;
#pragma unroll
                for (int kk = 0; kk < kHeadDim / 16; ++kk)
                    mma_bf16_ss(tmem + s_col, desc_kmajor(sQ, kk), desc_kmajor(ka, kk), kIdescQK,
                                kk > 0 ? 1u : 0u);
                mma_commit(&bar->k_empty[st]);
                mma_commit(&bar->s_full[st]);
                if (j > 0) issue_pv(j - 1);
            }
            issue_pv(nsel - 1);
        }
    } else {
        // ------------------------------------------------- softmax warpgroup
        const int r = threadIdx.x;  // query row within the tile == TMEM lane
        const int64_t qrow = static_cast<int64_t>(qb) * kBlock + r;
        const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
        float m = -INFINITY;  // running max (log2 domain, possibly stale by < 2^8)
        float l = 0.0f;       // running denominator relative to m
        for (int j = 0; j < nsel; ++j) {
            const int st = j & 1;
            const uint32_t ph = (j >> 1) & 1;
            const int64_t key0 = static_cast<int64_t>(sel[j]) * kBlock;
            mbar_wait(&bar->s_full[st], ph);
            tc_fence_after();
            float s[kBlock];
            const uint32_t s_addr = tmem + lane_base + (st ? kColS1 : kColS0);
#pragma unroll
            for (int c = 0; c < kBlock / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(s_addr + c * 32, v);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(v[e]);
            }
            tc_fence_before();
            mbar_arrive(&bar->s_empty[st]);

            // Mask keys past the query (causal) or past the sequence end.
            const bool need_mask = (p.causal && key0 + kBlock - 1 > static_cast<int64_t>(qb) * kBlock) ||
                                   key0 + kBlock > p.n;
            float mx = -INFINITY;
            if (need_mask) {
                const int64_t lim = p.causal ? min(qrow, p.n - 1) : p.n - 1;
#pragma unroll
                for (int c = 0; c < kBlock; ++c) {
                    s[c] = (key0 + c <= lim) ? s[c] * p.scale_log2 : -INFINITY;
                    mx = fmaxf(mx, s[c]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < kBlock; ++c) {
                    s[c] = s[c] * p.scale_log2;
                    mx = fmaxf(mx, s[c]);
                }
            }
            float alpha = 1.0f;
            if (mx > m + kRescaleThreshold || (m == -INFINITY && mx > -INFINITY)) {
                alpha = (m == -INFINITY) ? 0.0f : ex2(m - mx);
                m = mx;
            }
            const float msub = (m == -INFINITY) ? 0.0f : m;
            float rowsum = 0.0f;
            uint32_t pk[kBlock / 2];
#pragma unroll
            for (int c = 0; c < kBlock; c += 2) {
                const float p0 = ex2(s[c] - msub);
                const float p1 = ex2(s[c + 1] - msub);
                rowsum += p0 + p1;
                pk[c / 2] = pack_bf16x2(p0, p1);
            }
            l = l * alpha + rowsum;

            // P buffer `st` is free once O += P_{j-2} V_{j-2} has completed.
            if (j >= 2) mbar_wait(&bar->pv_done[st], ((j - 2) >> 1) & 1);
            uint8_t* prow = smem + kSmemP + st * kTileBytes + r * 128;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint4 w = make_uint4(pk[c * 32 + u * 4 + 0], pk[c * 32 + u * 4 + 1],
                                               pk[c * 32 + u * 4 + 2], pk[c * 32 + u * 4 + 3]);
                    *reinterpret_cast<uint4*>(prow + c * kChunkBytes + ((u ^ (r & 7)) << 4)) = w;
                }
            }
            fence_proxy_async_smem();

            // Rescale O (in TMEM) when the running max moved: needs O += P_{j-1} V_{j-1} done.
            if (j >= 1 && __any_sync(0xffffffffu, alpha != 1.0f)) {
                mbar_wait(&bar->pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
                const uint32_t o_addr = tmem + lane_base + kColO;
#pragma unroll
                for (int c = 0; c < kHeadDim / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(o_addr + c * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
                    tmem_st32(o_addr + c * 32, v);
                }
                tmem_wait_st();
            }
            tc_fence_before();
            mbar_arrive(&bar->p_full[st]);
        }

        // ------------------------------------------------------- epilogue
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) + (static_cast<int64_t>(h) * p.n + qrow) * kHeadDim;
        const bool live = qrow < p.n;
        if (nsel > 0) {
            const int jl = nsel - 1;
            mbar_wait(&bar->pv_done[jl & 1], (jl >> 1) & 1);
            tc_fence_after();
            const float inv = l > 0.0f ? 1.0f / l : 0.0f;
            const uint32_t o_addr = tmem + lane_base + kColO;
#pragma unroll
            for (int c = 0; c < kHeadDim / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(o_addr + c * 32, v);
                tmem_wait_ld();
                if (live) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        uint4 w;
                        w.x = pack_bf16x2(__uint_as_float(v[u * 8 + 0]) * inv, __uint_as_float(v[u * 8 + 1]) * inv);
                        w.y = pack_bf16x2(__uint_as_float(v[u * 8 + 2]) * inv, __uint_as_float(v[u * 8 + 3]) * inv);
                        w.z = pack_bf16x2(__uint_as_float(v[u * 8 + 4]) * inv, __uint_as_float(v[u * 8 + 5]) * inv);
                        w.w = pack_bf16x2(__uint_as_float(v[u * 8 + 6]) * inv, __uint_as_float(v[u * 8 + 7]) * inv);
                        *reinterpret_cast<uint4*>(out + c * 32 + u * 8) = w;
                    }
                }
            }
        } else if (live) {
#pragma unroll
            for (int u = 0; u < kHeadDim / 8; ++u) *reinterpret_cast<uint4*>(out + u * 8) = make_uint4(0, 0, 0, 0);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

}  // namespace

void launch_fa(const FaParams& p, int num_tiles, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(fa_sparse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemTotal));
        configured = true;
    }
    fa_sparse_kernel<<<num_tiles, kThreads, kSmemTotal, s>>>(p);
}

}  // namespace shplb::kern
