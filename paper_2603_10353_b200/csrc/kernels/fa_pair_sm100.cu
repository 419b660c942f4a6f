// Kernel 3, CTA-pair variant (cta_group::2): block-sparse FlashAttention
// prefill with the two 128-row halves of a 256-row query block on the two SMs
// of a cluster, so that S(j+1) = Q K(j+1)^T is computed WHILE the softmax of
// block j runs (the single-CTA kernel, fa_sm100.cu, has to wait for P(j)·V(j)
// before S(j+1) can reuse the TMEM columns P(j) occupies).
//
// Per selected key block j (ascending ids from kernel 2), the leader CTA's
// single MMA thread issues M = 256 products over both SMs:
//   S    = Q K_j^T   SS: A = each CTA's 128 Q rows, B = K_j split by keys
//                    (64 keys in each CTA's shared memory)
//   O   += P V_j     TS: A = P from each CTA's TMEM, B = V_j split by d
//                    (64 d-columns in each CTA's shared memory)
// and each CTA's softmax warpgroup (thread = query row = TMEM lane) reads S,
// tells the leader S may be overwritten (s_free), exponentiates into one of two
// P buffers in TMEM, and hands P over (p_full). Same semantics as fa_sm100.cu:
// softmax_weighted_sum over the kept set (proj/src/attention.cpp:35-49), causal
// mask (:28-30), zero row when nothing is visible (:40-41), lazy rescale.
//
// Per CTA: warps 0-7 softmax (two warpgroups splitting each row's 128 keys,
// row max exchanged through shared memory), warp 8 TMA producer (its own halves
// of Q, K, V; completion bytes on the leader's barriers), warp 9 TMEM allocator
// and (in the leader) MMA issuer. Shared memory: Q 32 KB, K 4 x 16 KB, V 4 x 16 KB.
// TMEM (512 columns allocated): S [0,128), P buffers [128,192) and
// [192,256), O [256,384).
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace shplb::kern {
namespace {

using namespace shplb::ptx;

constexpr int kPThreads = 320;  // warps 0-7 softmax (2 groups), 8 TMA, 9 TMEM + MMA
constexpr int kPStages = 4;
constexpr int kQHalfBytes = 32768;  // [2 d-chunks][128 rows][128 B]
constexpr int kKHalfBytes = 16384;  // [2 d-chunks][64 keys][128 B]
constexpr int kVHalfBytes = 16384;  // [128 keys][64 d = 128 B]
constexpr uint32_t kPairTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 128, kColO = 256;  // P buffer b at kColP + 64 b
constexpr uint32_t kIdescPairS = idesc_bf16_f32(256, 128, 0, 0);   // Q K-major, K K-major
constexpr uint32_t kIdescPairPV = idesc_bf16_f32(256, 128, 0, 1);  // P (TMEM), V MN-major
constexpr float kPairRescaleThreshold = 8.0f;

struct __align__(8) PairBarriers {
    uint64_t q_full;                                  // leader: both CTAs' Q landed
    uint64_t k_full[kPStages], v_full[kPStages];      // leader: both halves of the stage landed
    uint64_t k_empty[kPStages], v_empty[kPStages];    // each CTA: the stage's MMAs completed
    uint64_t s_full;                                  // each CTA: S(j) is in TMEM
    uint64_t s_free;                                  // leader: both softmaxes loaded S(j) (8 warps)
    // leader: CTA r's P(j) stored and O rescaled (4 warp arrivals), one barrier
    // per CTA and per block parity: a CTA can finish softmax(j+1) before the
    // MMA thread has waited for its P(j), and a single barrier per CTA would
    // then be two phases ahead of that wait (parity aliasing, a deadlock).
    uint64_t p_full[2][2];
    uint64_t pv_done[2];                              // each CTA: P.V of P buffer b's last use completed
    uint32_t tmem_base;
};

constexpr size_t kPSmemQ = 0;
constexpr size_t kPSmemK = kPSmemQ + kQHalfBytes;
constexpr size_t kPSmemV = kPSmemK + kPStages * kKHalfBytes;
constexpr size_t kPSmemSel = kPSmemV + kPStages * kVHalfBytes;
constexpr size_t kPSmemBar = kPSmemSel + kMaxSelected * sizeof(int32_t);
constexpr size_t kPSmemX = kPSmemBar + ((sizeof(PairBarriers) + 15) / 16) * 16;  // row max / sum exchange
constexpr size_t kPSmemTotal = kPSmemX + 3 * 256 * sizeof(float) + 1024;

#ifdef SHPLB_PTRACE  // dev-only: per-block clock64 timeline of cluster SHPLB_PTRACE, printed at exit
constexpr int kPTraceBlocks = 24;
#define PTRACE(j, e, cond) \
    do { if ((cond) && (j) >= 0 && (j) < kPTraceBlocks) ptrace[(j)][(e)] = clock64(); } while (0)
#else
#define PTRACE(j, e, cond) do { } while (0)
#endif

__global__ void __launch_bounds__(kPThreads, 1) fa_pair_kernel(const __grid_constant__ FaParams p) {
#ifdef SHPLB_PTRACE
    __shared__ long long ptrace[kPTraceBlocks][12];
    for (int i = threadIdx.x; i < kPTraceBlocks * 12; i += kPThreads) ptrace[i / 12][i % 12] = 0;
#endif
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    PairBarriers* bar = reinterpret_cast<PairBarriers*>(smem + kPSmemBar);
    int32_t* sel = reinterpret_cast<int32_t*>(smem + kPSmemSel);
    const uint32_t sSel = smem_u32(sel);
    auto sel_at = [&](int j) { return lds_s32(sSel + 4u * static_cast<uint32_t>(j)); };

    const uint32_t rank = cluster_ctarank();
    const int warp = warp_index_uniform();
    const int32_t tile = p.tiles[blockIdx.x >> 1];
    const int h = tile >> 20;
    const int qb = tile & 0xFFFFF;
    const int g = p.heads.kv[h];
    const int64_t row_id = static_cast<int64_t>(h) * p.nqb + qb;
    const int nsel = p.cnt[row_id];
    const int64_t row0 = static_cast<int64_t>(qb) * 256;
    {
        const int32_t* gsel = p.idx + row_id * p.kmax;
        for (int j = threadIdx.x; j < nsel; j += kPThreads) sel[j] = gsel[j];
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar->q_full, 1);
        for (int i = 0; i < kPStages; ++i) {
            mbar_init(&bar->k_full[i], 1);
            mbar_init(&bar->v_full[i], 1);
            mbar_init(&bar->k_empty[i], 1);
            mbar_init(&bar->v_empty[i], 1);
        }
        mbar_init(&bar->s_full, 1);
        mbar_init(&bar->s_free, 16);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->p_full[i][0], 8);
            mbar_init(&bar->p_full[i][1], 8);
            mbar_init(&bar->pv_done[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 9) tmem_alloc_pair<kPairTmemCols>(&bar->tmem_base);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem = bar->tmem_base;
    auto leader = [&](const uint64_t* b) { return mapa_shared(smem_u32(b), 0); };

    if (warp == 8) {
        // ------------------------------------------------------ TMA producer
        if (nsel > 0) {
            if (rank == 0) mbar_expect_tx_warp(&bar->q_full, 2 * kQHalfBytes);
            tma_load_pair_warp(smem + kPSmemQ, &p.tm_q, leader(&bar->q_full), 0,
                               static_cast<int>(row0) + 128 * static_cast<int>(rank), h, 2, 16384);
            for (int j = 0; j < nsel; ++j) {
                const int st = j % kPStages;
                const uint32_t ph = (j / kPStages) & 1;
                const int key0 = sel_at(j) * kBlock;
                mbar_wait(&bar->k_empty[st], ph ^ 1);
                if (rank == 0) mbar_expect_tx_warp(&bar->k_full[st], 2 * kKHalfBytes);
                tma_load_pair_warp(smem + kPSmemK + st * kKHalfBytes, &p.tm_k_half, leader(&bar->k_full[st]), 0,
                                   key0 + 64 * static_cast<int>(rank), g, 2, 8192);
                mbar_wait(&bar->v_empty[st], ph ^ 1);
                if (rank == 0) mbar_expect_tx_warp(&bar->v_full[st], 2 * kVHalfBytes);
                tma_load_pair_warp(smem + kPSmemV + st * kVHalfBytes, &p.tm_v, leader(&bar->v_full[st]),
                                   64 * static_cast<int>(rank), key0, g, 1, 0);
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------- MMA issuer (leader only)
        if (rank == 0 && nsel > 0) {
            const uint32_t tm = __shfl_sync(0xffffffffu, static_cast<uint32_t>(lds_s32(smem_u32(&bar->tmem_base))), 0);
            const uint64_t qd = umma_desc_sw128(smem_u32(smem + kPSmemQ), 16, 1024);
            const uint64_t kd0 = umma_desc_sw128(smem_u32(smem + kPSmemK), 16, 1024);
            const uint64_t vd0 = umma_desc_sw128(smem_u32(smem + kPSmemV), 16384, 1024);
            auto kdesc = [&](int st) { return kd0 + static_cast<uint64_t>(st) * (kKHalfBytes >> 4); };
            auto vdesc = [&](int st) { return vd0 + static_cast<uint64_t>(st) * (kVHalfBytes >> 4); };
            auto issue_s = [&](int j) {
                const int st = j % kPStages;
                mbar_wait(&bar->k_full[st], (j / kPStages) & 1);
                tc_fence_after();
                mma_pair_ss(tm + kColS, qd, kdesc(st), kIdescPairS, 0u);
                mma_commit_pair_warp(&bar->s_full);
                mma_commit_pair_warp(&bar->k_empty[st]);
            };
            mbar_wait(&bar->q_full, 0);
            issue_s(0);
            for (int j = 0; j < nsel; ++j) {
                if (j + 1 < nsel) {
                    mbar_wait_cluster(&bar->s_free, j & 1);  // both softmaxes hold S(j) in registers
                    PTRACE(j, 0, (threadIdx.x & 31) == 0);
                    issue_s(j + 1);
                    PTRACE(j, 1, (threadIdx.x & 31) == 0);
                }
                mbar_wait_cluster(&bar->p_full[0][j & 1], (j >> 1) & 1);
                mbar_wait_cluster(&bar->p_full[1][j & 1], (j >> 1) & 1);
                PTRACE(j, 2, (threadIdx.x & 31) == 0);
                const int st = j % kPStages;
                mbar_wait(&bar->v_full[st], (j / kPStages) & 1);
                PTRACE(j, 3, (threadIdx.x & 31) == 0);
                tc_fence_after();
                mma_pair_ts(tm + kColO, tm + kColP + 64u * static_cast<uint32_t>(j & 1), vdesc(st), kIdescPairPV,
                            j > 0 ? 1u : 0u);
                mma_commit_pair_warp(&bar->pv_done[j & 1]);
                mma_commit_pair_warp(&bar->v_empty[st]);
            }
        }
    } else {
        // ------------------------------------------- softmax (warps 0-7)
        // Two warpgroups per CTA share each row (thread = query row = TMEM
        // lane): warpgroup ch takes keys [64 ch, 64 ch + 64) of S, the
        // matching 32 packed columns of P and d-columns [64 ch, 64 ch + 64)
        // of O; the row max is exchanged through shared memory once per block.
        const int ch = warp >> 2;
        const int r = threadIdx.x & 127;
        const int64_t qrow = row0 + 128 * static_cast<int64_t>(rank) + r;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t c0 = 64u * static_cast<uint32_t>(ch);
        const uint32_t s_addr = tmem + lane_base + kColS + c0;
        const uint32_t o_addr = tmem + lane_base + kColO + c0;
        const float sl2 = p.scale_log2;
        const int64_t lim = p.causal ? min(qrow, p.n - 1) : p.n - 1;
        const uint32_t s_free_l = leader(&bar->s_free);
        const uint32_t p_full_l = leader(&bar->p_full[rank][0]);  // [rank][1] is 8 bytes further
        const float2 sc2 = make_float2(sl2, sl2);
        float* xmax = reinterpret_cast<float*>(smem + kPSmemX);  // [2 parities][2 groups][128 rows]
        float m = -INFINITY, l = 0.0f;  // l: this group's part of the row sum
        for (int j = 0; j < nsel; ++j) {
            const int64_t key0 = static_cast<int64_t>(sel_at(j)) * kBlock + c0;
            const bool need_mask = key0 + 63 > lim;
            uint32_t sv[64];
            float* s = reinterpret_cast<float*>(sv);
            mbar_wait(&bar->s_full, j & 1);
            PTRACE(j, 4 + 3 * rank, r == 0 && ch == 0);
            tc_fence_after();
#ifdef SHPLB_PDIAG_SKIP_SOFTMAX  // dev-only diagnostic (wrong results): the MMA/TMA pipeline alone
            tc_fence_before();
            mbar_arrive_cluster_warp(s_free_l);
            mbar_arrive_cluster_warp(p_full_l + 8u * static_cast<uint32_t>(j & 1));
            continue;
#endif
            tmem_ld32(s_addr + 0, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
            tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive_cluster_warp(s_free_l);  // the leader may now compute S(j+1) over it
            PTRACE(j, 5 + 3 * rank, r == 0 && ch == 0);
            if (need_mask) {
#pragma unroll
                for (int c = 0; c < 64; ++c)
                    if (key0 + c > lim) s[c] = -INFINITY;
            }
            float mx8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
#pragma unroll
            for (int c = 0; c < 64; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
            float mine = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
            float* xm = xmax + (j & 1) * 256;  // parity-buffered: the other group may still read j-1's
            xm[ch * 128 + r] = mine;
            named_bar_sync(1, 256);
            const float mraw = fmaxf(mine, xm[(ch ^ 1) * 128 + r]);
            PTRACE(j, 10, r == 0 && ch == 0 && rank == 0);
            const float mx = mraw * sl2;
            float alpha = 1.0f;
            if (mx > m + kPairRescaleThreshold || (m == -INFINITY && mx > -INFINITY)) {
                alpha = (m == -INFINITY) ? 0.0f : ex2(m - mx);
                m = mx;
            }
            if (j >= 1 && __any_sync(0xffffffffu, alpha != 1.0f)) {
                // this group's half of O *= alpha once P(j-1).V(j-1) has landed
                mbar_wait(&bar->pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t v[32];
                    tmem_ld32(o_addr + c * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
                    tmem_st32(o_addr + c * 32, v);
                }
            }
            if (j >= 2) {  // P buffer j & 1 was last read by P(j-2).V(j-2)
                mbar_wait(&bar->pv_done[j & 1], ((j - 2) >> 1) & 1);
                tc_fence_after();
            }
            const float msub = (m == -INFINITY) ? 0.0f : m;
            const float2 nm2 = make_float2(-msub, -msub);
            const uint32_t p_addr = tmem + lane_base + kColP + 64u * static_cast<uint32_t>(j & 1) + c0 / 2;
            float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float2 x = ffma2(make_float2(s[c * 32 + 2 * e], s[c * 32 + 2 * e + 1]), sc2, nm2);
                    float2 pe;
                    pe.x = ex2(x.x);
                    pe.y = ex2(x.y);
                    sum2[e & 1] = fadd2(sum2[e & 1], pe);
                    pk[e] = pack_bf16x2(pe.x, pe.y);
                }
                tmem_st16(p_addr + c * 16, pk);
            }
            const float2 sum = fadd2(sum2[0], sum2[1]);
            l = l * alpha + (sum.x + sum.y);
            PTRACE(j, 11, r == 0 && ch == 0 && rank == 0);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive_cluster_warp(p_full_l + 8u * static_cast<uint32_t>(j & 1));
            PTRACE(j, 6 + 3 * rank, r == 0 && ch == 0);
        }

        // -------------------------------------------------------- epilogue
        // Row sum = group 0's part + group 1's part (the same order in both).
        float* lsum = xmax + 512;
        lsum[ch * 128 + r] = l;
        named_bar_sync(2, 256);
        const float ltot = lsum[r] + lsum[128 + r];
        const bool live = qrow < p.n;
        const int ndst = p.n_out_peers > 0 ? p.n_out_peers : 1;
        auto dst_row = [&](int i) -> __nv_bfloat16* {
            if (p.n_out_peers == 0)
                return static_cast<__nv_bfloat16*>(p.out) + (static_cast<int64_t>(h) * p.n + qrow) * kHeadDim + c0;
            return static_cast<__nv_bfloat16*>(p.out_peers[i]) +
                   (static_cast<int64_t>(p.heads.k[h]) * p.n + qrow) * kHeadDim + c0;
        };
        if (nsel > 0) {
            mbar_wait(&bar->pv_done[(nsel - 1) & 1], ((nsel - 1) >> 1) & 1);
            tc_fence_after();
            const float inv = ltot > 0.0f ? 1.0f / ltot : 0.0f;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                uint32_t v[32];
                tmem_ld32(o_addr + c * 32, v);
                tmem_wait_ld();
                if (live) {
                    uint4 w[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        w[u].x = pack_bf16x2(__uint_as_float(v[u * 8 + 0]) * inv, __uint_as_float(v[u * 8 + 1]) * inv);
                        w[u].y = pack_bf16x2(__uint_as_float(v[u * 8 + 2]) * inv, __uint_as_float(v[u * 8 + 3]) * inv);
                        w[u].z = pack_bf16x2(__uint_as_float(v[u * 8 + 4]) * inv, __uint_as_float(v[u * 8 + 5]) * inv);
                        w[u].w = pack_bf16x2(__uint_as_float(v[u * 8 + 6]) * inv, __uint_as_float(v[u * 8 + 7]) * inv);
                    }
#pragma unroll 1
                    for (int i = 0; i < ndst; ++i) {
                        __nv_bfloat16* out = dst_row(i);
#pragma unroll
                        for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(out + c * 32 + u * 8) = w[u];
                    }
                }
            }
        } else if (live) {
#pragma unroll 1
            for (int i = 0; i < ndst; ++i) {
                __nv_bfloat16* out = dst_row(i);
#pragma unroll
                for (int u = 0; u < 8; ++u) *reinterpret_cast<uint4*>(out + u * 8) = make_uint4(0, 0, 0, 0);
            }
        }
        if (p.n_out_peers > 1) __threadfence_system();
    }

#ifdef SHPLB_PTRACE
    __syncthreads();
    if ((blockIdx.x >> 1) == SHPLB_PTRACE && threadIdx.x == 0) {
        const long long t0 = ptrace[0][rank == 0 ? 4 : 7];
        for (int j = 0; j < kPTraceBlocks && j < nsel; ++j)
            printf("PTRACE r%u j %d mma %lld %lld %lld %lld sm0 %lld %lld %lld sm1 %lld %lld %lld x %lld %lld\n", rank,
                   j, ptrace[j][0] - t0, ptrace[j][1] - t0, ptrace[j][2] - t0, ptrace[j][3] - t0,
                   ptrace[j][4] - t0, ptrace[j][5] - t0, ptrace[j][6] - t0, ptrace[j][7] - t0,
                   ptrace[j][8] - t0, ptrace[j][9] - t0, ptrace[j][10] - t0, ptrace[j][11] - t0);
    }
#endif
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer is done with this CTA's barriers and operands
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc_pair<kPairTmemCols>(tmem);
    }
}

}  // namespace

cudaError_t launch_fa_pair(const FaParams& p, int num_tiles, cudaStream_t s) {
    set_max_dynamic_smem(reinterpret_cast<const void*>(fa_pair_kernel), static_cast<int>(kPSmemTotal));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * static_cast<unsigned>(num_tiles));
    cfg.blockDim = dim3(kPThreads);
    cfg.dynamicSmemBytes = kPSmemTotal;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fa_pair_kernel, p);
}

}  // namespace shplb::kern
