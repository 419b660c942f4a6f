// Kernel 3: block-sparse FlashAttention prefill for sm_100a.
//
// One CTA computes one 128-row query tile of one head over that tile's
// selected key blocks (ascending block ids from kernel 2). Per selected block
// j (128 keys):  S = Q K_j^T (tcgen05, fp32 in TMEM) -> online softmax in
// registers -> P (bf16, written back into TMEM over S) -> O += P V_j
// (tcgen05 with the A operand read from TMEM). The reference semantics it
// realises are softmax_weighted_sum over the kept set
// (proj/src/attention.cpp:35-49) with the causal mask of :28-30; rows with no
// visible kept key produce zeros (:40-41).
//
// Two softmax warpgroups split the key blocks: group 0 takes even j, group 1
// odd j. Each keeps its own running max / denominator and its own O
// accumulator in TMEM (two independent online softmaxes over disjoint key
// sets, merged exactly in the epilogue). While group 0 exponentiates block j
// the tensor core runs S_{j+1} for group 1, and each group has two blocks of
// MMA time to finish its softmax, which hides the MUFU (ex2) and TMEM latency
// that a single group exposes.
//
// Warp roles (384 threads, registers rebalanced with setmaxnreg):
//   warps 0-3  softmax group 0 (thread t owns query row t = TMEM lane t)
//   warps 4-7  softmax group 1 (same rows, lanes 32*(w%4)..)
//   warp 8     TMA producer: Q once, then K_j / V_j into 2-stage rings
//   warp 9     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 10-11 idle (complete the control warpgroup for setmaxnreg)
// MMA issue order: S0, S1, PV0, S2, PV1, S3, ... (S_{j+2} right after PV_j,
// so the WAR on the aliased S/P columns is ordered by the tensor pipe).
//
// Shared memory (1024-aligned, 128B-swizzled UMMA operands):
//   Q  [2 d-chunks][128 rows][64 bf16]                   32 KB (K-major A)
//   K  [2 stages][2 d-chunks][128 keys][64 bf16]         64 KB (K-major B)
//   V  [2 stages][2 d-chunks][128 keys][64 bf16]         64 KB (MN-major B)
//   selected block ids, softmax statistics, mbarriers
// TMEM (512 columns): S/P group 0 [0,128), S/P group 1 [128,256),
//                     O group 0 [256,384), O group 1 [384,512).
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace shplb::kern {
namespace {

using namespace shplb::ptx;

constexpr int kThreads = 384;  // 3 warpgroups
constexpr uint32_t kRegsSoftmax = 224, kRegsControl = 56;  // 2*128*224 + 128*56 = 64K
constexpr int kTileBytes = kBlock * kHeadDim * 2;  // 32 KB: one 128x128 bf16 tile
constexpr int kChunkBytes = kTileBytes / 2;        // 16 KB: 128 rows x 128 B
constexpr int kMaxSel = kMaxSelected;              // selected blocks staged in smem
constexpr uint32_t kTmemCols = 512;
// TMEM column of group g's S/P and O accumulators.
__host__ __device__ constexpr uint32_t col_s(int g) { return static_cast<uint32_t>(g) * 128u; }
__host__ __device__ constexpr uint32_t col_o(int g) { return 256u + static_cast<uint32_t>(g) * 128u; }
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale when max grows by > 2^8

constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, 0, 0);  // A=Q K-major, B=K K-major
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, 0, 1);  // A=P (TMEM), B=V MN-major

struct __align__(8) Barriers {
    uint64_t q_full;
    uint64_t k_full[2], k_empty[2];
    uint64_t v_full[2], v_empty[2];
    uint64_t s_full[2];   // per softmax group: S of its next block is in TMEM
    uint64_t p_full[2];   // per group: P written (and O rescaled) -> PV may run
    uint64_t pv_done[2];  // per group: its last issued PV has completed
    uint32_t tmem_base;
};

constexpr size_t kSmemQ = 0;
constexpr size_t kSmemK = kSmemQ + kTileBytes;
constexpr size_t kSmemV = kSmemK + 2 * kTileBytes;
constexpr size_t kSmemSel = kSmemV + 2 * kTileBytes;
constexpr size_t kSmemStats = kSmemSel + kMaxSel * sizeof(int32_t);
constexpr size_t kSmemBar = kSmemStats + 2 * 2 * 128 * sizeof(float);
constexpr size_t kSmemTotal = kSmemBar + sizeof(Barriers) + 1024;  // + alignment slack

// K-major SW128 operand (Q, K): k-step kk (16 elements) lives in d chunk kk/4
// at byte offset (kk%4)*32 within each 128-byte row; 8-row groups are 1024 B
// apart (SBO); LBO is unused for swizzled K-major.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile_addr, int kk) {
    return umma_desc_sw128(tile_addr + (kk >> 2) * kChunkBytes + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 operand (V as B of P.V): N = d spans the two 64-wide d
// chunks (LBO = 16 KB apart); K = keys, 8-key groups 1024 B apart (SBO);
// k-step kk starts 16 keys = 2 KB further.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile_addr, int kk) {
    return umma_desc_sw128(tile_addr + kk * 2048, kChunkBytes, 1024);
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) fa_sparse_kernel(const __grid_constant__ FaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bar = reinterpret_cast<Barriers*>(smem + kSmemBar);
    int32_t* sel = reinterpret_cast<int32_t*>(smem + kSmemSel);
    float* stats = reinterpret_cast<float*>(smem + kSmemStats);  // [group][m|l][128]
    const uint32_t sQ = smem_u32(smem + kSmemQ);
    const uint32_t sK = smem_u32(smem + kSmemK);
    const uint32_t sV = smem_u32(smem + kSmemV);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const int32_t tile = p.tiles[blockIdx.x];
    const int h = tile >> 20;
    const int qb = tile & 0xFFFFF;
    const int g = p.heads.kv[h];
    const int64_t row_id = static_cast<int64_t>(h) * p.nqb + qb;
    const int nsel = p.cnt[row_id];
    {
        const int32_t* gsel = p.idx + row_id * p.kmax;
        for (int j = threadIdx.x; j < nsel; j += kThreads) sel[j] = gsel[j];
    }

    if (threadIdx.x == 0) {
        mbar_init(&bar->q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->k_full[i], 1);
            mbar_init(&bar->k_empty[i], 1);
            mbar_init(&bar->v_full[i], 1);
            mbar_init(&bar->v_empty[i], 1);
            mbar_init(&bar->s_full[i], 1);
            mbar_init(&bar->p_full[i], 128);
            mbar_init(&bar->pv_done[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 9) tmem_alloc<kTmemCols>(&bar->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp >= 8) {
      setmaxnreg_dec<kRegsControl>();
      if (warp == 8) {
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
    } else if (warp == 9) {
        // -------------------------------------------------------- MMA issuer
        if (lane == 0 && nsel > 0) {
            mbar_wait(&bar->q_full, 0);
            auto issue_s = [&](int j) {  // S_j = Q K_j^T into group (j&1)'s S columns
                const int st = j & 1;
                mbar_wait(&bar->k_full[st], (j >> 1) & 1);
                tc_fence_after();
                const uint32_t ka = sK + st * kTileBytes;
#pragma unroll
                for (int kk = 0; kk < kHeadDim / 16; ++kk)
                    mma_bf16_ss(tmem + col_s(j & 1), desc_kmajor(sQ, kk), desc_kmajor(ka, kk), kIdescQK,
                                kk > 0 ? 1u : 0u);
                mma_commit(&bar->k_empty[st]);
                mma_commit(&bar->s_full[j & 1]);
            };
            issue_s(0);
            if (nsel > 1) issue_s(1);
            for (int j = 0; j < nsel; ++j) {
                // O_grp += P_j V_j, P_j read from TMEM (bf16 pairs over S_grp).
                const int grp = j & 1;
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                mbar_wait(&bar->v_full[st], ph);
                mbar_wait(&bar->p_full[grp], ph);
                tc_fence_after();
                const uint32_t va = sV + st * kTileBytes;
#pragma unroll
                for (int kk = 0; kk < kBlock / 16; ++kk)
                    mma_bf16_ts(tmem + col_o(grp), tmem + col_s(grp) + kk * 8, desc_mnmajor(va, kk),
                                kIdescPV, (j >= 2 || kk > 0) ? 1u : 0u);
                mma_commit(&bar->v_empty[st]);
                mma_commit(&bar->pv_done[grp]);
                if (j + 2 < nsel) issue_s(j + 2);
            }
        }
      }
    } else {
        setmaxnreg_inc<kRegsSoftmax>();
        // ------------------------------------------------ softmax warpgroups
        const int grp = warp >> 2;            // 0: even blocks, 1: odd blocks
        const int r = threadIdx.x & 127;      // query row within the tile == TMEM lane
        const int64_t qrow = static_cast<int64_t>(qb) * kBlock + r;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t s_addr = tmem + lane_base + col_s(grp);
        const uint32_t o_addr = tmem + lane_base + col_o(grp);
        const float sl2 = p.scale_log2;
        const int64_t lim = p.causal ? min(qrow, p.n - 1) : p.n - 1;  // last visible key
        float m = -INFINITY;  // running max, log2 domain (stale by < 2^8)
        float l = 0.0f;       // running denominator relative to m
        int it = 0;
        for (int j = grp; j < nsel; j += 2, ++it) {
            const int64_t key0 = static_cast<int64_t>(sel[j]) * kBlock;
            mbar_wait(&bar->s_full[grp], it & 1);
            tc_fence_after();
            uint32_t sv[kBlock];
            {
                uint32_t(&c0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[0]);
                uint32_t(&c1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[32]);
                uint32_t(&c2)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[64]);
                uint32_t(&c3)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[96]);
                tmem_ld32(s_addr + 0, c0);
                tmem_ld32(s_addr + 32, c1);
                tmem_ld32(s_addr + 64, c2);
                tmem_ld32(s_addr + 96, c3);
                tmem_wait_ld();
            }
            float* s = reinterpret_cast<float*>(sv);
            // Mask keys past the query (causal) or past the sequence end; row max
            // with 8 independent chains.
            const bool need_mask = key0 + kBlock - 1 > lim || key0 + kBlock > p.n;
            if (need_mask) {
#pragma unroll
                for (int c = 0; c < kBlock; ++c)
                    if (key0 + c > lim) s[c] = -INFINITY;
            }
            float mx8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx8[e] = s[e];
#pragma unroll
            for (int c = 8; c < kBlock; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
            const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
            const float mx = mraw * sl2;  // scale > 0 commutes with max
            float alpha = 1.0f;
            if (mx > m + kRescaleThreshold || (m == -INFINITY && mx > -INFINITY)) {
                alpha = (m == -INFINITY) ? 0.0f : ex2(m - mx);
                m = mx;
            }
            // Rescale O_grp (needs the group's previous PV complete) when the max moved.
            if (it >= 1 && __any_sync(0xffffffffu, alpha != 1.0f)) {
                mbar_wait(&bar->pv_done[grp], (it - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < kHeadDim / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(o_addr + c * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
                    tmem_st32(o_addr + c * 32, v);
                }
            }
            const float msub = (m == -INFINITY) ? 0.0f : m;
            float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // four 32-key quarters -> 16 packed columns each
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float p0 = ex2(fmaf(s[c * 32 + 2 * e], sl2, -msub));
                    const float p1 = ex2(fmaf(s[c * 32 + 2 * e + 1], sl2, -msub));
                    sum4[e & 3] += p0 + p1;
                    pk[e] = pack_bf16x2(p0, p1);
                }
                tmem_st16(s_addr + c * 16, pk);
            }
            l = l * alpha + ((sum4[0] + sum4[1]) + (sum4[2] + sum4[3]));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bar->p_full[grp]);
        }

        // -------------------------------------------------------- epilogue
        // Merge the two groups' (m, l, O): m* = max, O = sum_g O_g 2^(m_g - m*)
        // / sum_g l_g 2^(m_g - m*). Group g writes output columns [64g, 64g+64).
        stats[(grp * 2 + 0) * 128 + r] = m;
        stats[(grp * 2 + 1) * 128 + r] = l;
        named_bar_sync(1, 256);
        const float m0 = stats[0 * 128 + r], l0 = stats[1 * 128 + r];
        const float m1 = stats[2 * 128 + r], l1 = stats[3 * 128 + r];
        const float mm = fmaxf(m0, m1);
        const float a0 = (l0 > 0.0f) ? ex2(m0 - mm) : 0.0f;
        const float a1 = (l1 > 0.0f) ? ex2(m1 - mm) : 0.0f;
        const float den = l0 * a0 + l1 * a1;
        const float inv = den > 0.0f ? 1.0f / den : 0.0f;
        const int n0 = (nsel + 1) >> 1, n1 = nsel >> 1;  // blocks per group
        if (n0 > 0) mbar_wait(&bar->pv_done[0], (n0 - 1) & 1);
        if (n1 > 0) mbar_wait(&bar->pv_done[1], (n1 - 1) & 1);
        tc_fence_after();
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) +
                             (static_cast<int64_t>(h) * p.n + qrow) * kHeadDim + grp * 64;
        const bool live = qrow < p.n;
        const uint32_t oa0 = tmem + lane_base + col_o(0) + grp * 64;
        const uint32_t oa1 = tmem + lane_base + col_o(1) + grp * 64;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t v0[16], v1[16];
            if (n0 > 0) tmem_ld16(oa0 + c * 16, v0);
            if (n1 > 0) tmem_ld16(oa1 + c * 16, v1);
            tmem_wait_ld();
            if (live) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    float f[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float x0 = n0 > 0 ? __uint_as_float(v0[u * 8 + e]) * a0 : 0.0f;
                        const float x1 = n1 > 0 ? __uint_as_float(v1[u * 8 + e]) * a1 : 0.0f;
                        f[e] = (x0 + x1) * inv;
                    }
                    uint4 w;
                    w.x = pack_bf16x2(f[0], f[1]);
                    w.y = pack_bf16x2(f[2], f[3]);
                    w.z = pack_bf16x2(f[4], f[5]);
                    w.w = pack_bf16x2(f[6], f[7]);
                    *reinterpret_cast<uint4*>(out + c * 16 + u * 8) = w;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
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
