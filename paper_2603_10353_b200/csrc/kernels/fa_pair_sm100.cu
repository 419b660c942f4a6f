// Kernel 3, CTA-pair variant (block_q = 256): block-sparse FlashAttention
// prefill with the two 128-row halves of a 256-row query block on the two SMs
// of a cluster and, in each SM, two softmax warpgroups that take ALTERNATE
// selected key blocks of the same 128 rows.
//
// Why: in the single-CTA kernel (fa_sm100.cu) each query half's
// P(j) overwrites its S(j) in TMEM, so S(j+1) waits for P(j)·V(j), and the
// chain S -> softmax -> P·V -> S leaves the tensor pipe ~31% idle even though
// the two halves ping-pong. Here P has its own TMEM buffers, so S(j+1) is
// computed as soon as S(j) has been read into registers, and while warpgroup A
// exponentiates block j, warpgroup B loads and reduces block j+1: the MUFU
// (16 ex2 / clk / SM, exactly the tensor pipe's pace for one 128 x 128 tile)
// and the tensor pipe both stay busy.
//
// Per selected key block j the leader CTA's single MMA thread issues M = 256
// products over both SMs (cta_group::2):
//   S    = Q K_j^T   SS: A = each CTA's 128 Q rows, B = K_j split by keys
//                    (64 keys in each CTA's shared memory)
//   O   += P_j V_j   TS: A = P from each CTA's TMEM, B = V_j split by d
//                    (64 d-columns in each CTA's shared memory)
// so each 64 KB K/V tile still feeds 256 query rows (the reuse of the
// single-CTA kernel's two halves) while each SM reads only half of it.
//
// Online softmax per warpgroup (same semantics as fa_sm100.cu:
// softmax_weighted_sum over the kept set, proj/src/attention.cpp:35-49; causal
// mask :28-30; zero row when nothing is visible :40-41). Each warpgroup keeps
// its own running max (lazy rule: raised only when a block max exceeds it by
// > 2^8), row sum and accumulator O_w in TMEM — P(j)·V(j) accumulates into
// O_(j mod 2) — so the two never wait on each other; when m rises the
// warpgroup rescales its O_w after its previous P·V has landed and before its
// next is issued. The epilogue merges (O_0, l_0, m_0) and (O_1, l_1, m_1).
// (Round-2 history: one shared O with the max chained between the warpgroups
// through shared memory cost every block a cross-warpgroup wait.)
//
// Warps (384 threads, registers rebalanced with setmaxnreg as fa_sm100.cu):
//   0-3 softmax A (even blocks), 4-7 softmax B (odd blocks), 8 TMA producer of
//   this CTA's halves of Q and K, 10 of V (completion bytes on the leader's
//   barriers), 9 TMEM allocator and (leader) S issuer, 11 (leader) P·V issuer.
// Shared memory: Q 32 KB, K 4 x 16 KB, V 4 x 16 KB, selection, barriers, (l, m).
// TMEM (512 columns): S [0,128), P_A [128,192), P_B [192,256), O_A [256,384), O_B [384,512).
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

constexpr int kPThreads = 384;
constexpr uint32_t kPRegsLaunch = 168, kPRegsSoftmax = 216, kPRegsControl = 72;
static_assert(2 * kPRegsSoftmax + kPRegsControl <= 3 * kPRegsLaunch, "setmaxnreg budget exceeds the launch grant");
constexpr int kPStages = 4;
constexpr int kQHalfBytes = 32768;  // [2 d-chunks][128 rows][128 B]
constexpr int kKHalfBytes = 16384;  // [2 d-chunks][64 keys][128 B]
constexpr int kVHalfBytes = 16384;  // [128 keys][64 d = 128 B]
constexpr uint32_t kPairTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 128, kColO = 256;  // P_w at kColP + 64 w, O_w at kColO + 128 w
constexpr uint32_t kIdescPairS = idesc_bf16_f32(256, 128, 0, 0);   // Q K-major, K K-major
constexpr uint32_t kIdescPairPV = idesc_bf16_f32(256, 128, 0, 1);  // P (TMEM), V MN-major
constexpr float kPairRescaleThreshold = 8.0f;
// Control warp roles (warp index; SMSP = warp % 4). A warp blocked issuing
// tcgen05.mma slows the softmax warps of its SMSP (~300 cycles per block on
// the leader CTA, measured with SHPLB_PTRACE); moving the issuers to other
// SMSPs only moves the lag (profiles/r02/k3_pair_tuning.txt).
constexpr int kWarpQK = 8, kWarpS = 9, kWarpV = 10, kWarpPV = 11;

struct __align__(8) PairBarriers {
    uint64_t q_full;                                // leader: both CTAs' Q landed
    uint64_t k_full[kPStages], v_full[kPStages];    // leader: both halves of the stage landed
    uint64_t k_empty[kPStages], v_empty[kPStages];  // each CTA: the stage's MMAs completed
    uint64_t s_full[2];   // each CTA: S(j) in TMEM, one barrier per warpgroup (j mod 2)
    uint64_t s_free;      // leader: the owning warpgroups of both CTAs loaded S(j) (8 warps)
    uint64_t p_full[2][2];  // leader: CTA r's P(j) stored (and O rescaled), [r][j mod 2], 4 warps
    uint64_t pv_done[4];  // each CTA: P(j)·V(j) completed, [j mod 4] (4 slots: see the rescale wait)
    uint32_t tmem_base;
};

constexpr size_t kPSmemQ = 0;
constexpr size_t kPSmemK = kPSmemQ + kQHalfBytes;
constexpr size_t kPSmemV = kPSmemK + kPStages * kKHalfBytes;
constexpr size_t kPSmemSel = kPSmemV + kPStages * kVHalfBytes;
constexpr size_t kPSmemBar = kPSmemSel + kMaxSelected * sizeof(int32_t);
constexpr size_t kPSmemX = kPSmemBar + ((sizeof(PairBarriers) + 15) / 16) * 16;  // l / m [2][2][128]
constexpr size_t kPSmemTotal = kPSmemX + 4 * 128 * sizeof(float) + 1024;

#ifdef SHPLB_TILETRACE  // dev-only: per-CTA timestamps of every tile (tools/tile_trace.py)
constexpr int kTTraceCtas = 1 << 16;
// [cta][0 entry globaltimer, 1 smid | nsel << 32, 2 entry clock64, 3 setup done, 4 first S landed
//       (warpgroup A), 5 last P·V landed (epilogue), 6 output stored, 7 exit clock64]
__device__ unsigned long long g_tiletrace[kTTraceCtas][8];
#define TTRACE(e, v) do { if (blockIdx.x < kTTraceCtas) g_tiletrace[blockIdx.x][(e)] = (v); } while (0)
#else
#define TTRACE(e, v) do { } while (0)
#endif

#ifdef SHPLB_PTRACE  // dev-only: per-block clock64 timeline of cluster SHPLB_PTRACE (leader CTA), printed at exit
constexpr int kPTraceBlocks = 32;
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
#ifdef SHPLB_TILETRACE
    if (threadIdx.x == 0) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        TTRACE(0, gt);
        TTRACE(2, clock64());
        const int32_t t = p.tiles[blockIdx.x >> 1];
        TTRACE(1, smid | (static_cast<unsigned long long>(p.cnt[static_cast<int64_t>(t >> 20) * p.nqb + (t & 0xFFFFF)]) << 32));
    }
#endif
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    PairBarriers* bar = reinterpret_cast<PairBarriers*>(smem + kPSmemBar);
    int32_t* sel = reinterpret_cast<int32_t*>(smem + kPSmemSel);
    const uint32_t sSel = smem_u32(sel);
    auto sel_at = [&](int j) { return lds_s32(sSel + 4u * static_cast<uint32_t>(j)); };
    float* lfin = reinterpret_cast<float*>(smem + kPSmemX);  // [2 warpgroups][2 (l, m)][128]

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
        mbar_init(&bar->s_full[0], 1);
        mbar_init(&bar->s_full[1], 1);
        mbar_init(&bar->s_free, 8);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->p_full[i][0], 4);
            mbar_init(&bar->p_full[i][1], 4);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&bar->pv_done[i], 1);
        fence_mbar_init();
    }
    if (warp == 9) tmem_alloc_pair<kPairTmemCols>(&bar->tmem_base);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / TMA
    tc_fence_after();
    if (threadIdx.x == 0) TTRACE(3, clock64());
    const uint32_t tmem = bar->tmem_base;
    auto leader = [&](const uint64_t* b) { return mapa_shared(smem_u32(b), 0); };

    // Tile scalars are re-read after setmaxnreg (values live across it are
    // kept on the stack by ptxas and reloaded inside the loops).
    auto tile_scalars = [&](int& nsel_o, int64_t& row0_o, int& h_o, int& g_o) {
        const int32_t t = p.tiles[blockIdx.x >> 1];
        h_o = t >> 20;
        g_o = p.heads.kv[h_o];
        row0_o = static_cast<int64_t>(t & 0xFFFFF) * 256;
        nsel_o = p.cnt[static_cast<int64_t>(h_o) * p.nqb + (t & 0xFFFFF)];
    };
    if (warp >= 8) {
        setmaxnreg_dec<kPRegsControl>();
        int nsel, h, g;
        int64_t row0;
        tile_scalars(nsel, row0, h, g);
        if (warp == kWarpQK) {
            // ---------------------------------------- TMA producer: Q and K
            // (K and V have separate producers: a V load waits for the P·V four
            // blocks back, which must not hold up the K loads S runs on.)
            if (nsel > 0) {
                if (rank == 0) mbar_expect_tx_warp(&bar->q_full, 2 * kQHalfBytes);
                tma_load_pair_warp(smem + kPSmemQ, &p.tm_q, leader(&bar->q_full), 0,
                                   static_cast<int>(row0) + 128 * static_cast<int>(rank), h, 2, 16384);
                for (int j = 0; j < nsel; ++j) {
                    const int st = j % kPStages;
                    const uint32_t ph = (j / kPStages) & 1;
                    mbar_wait(&bar->k_empty[st], ph ^ 1);
                    if (rank == 0) mbar_expect_tx_warp(&bar->k_full[st], 2 * kKHalfBytes);
                    tma_load_pair_warp(smem + kPSmemK + st * kKHalfBytes, &p.tm_k_half, leader(&bar->k_full[st]), 0,
                                       sel_at(j) * kBlock + 64 * static_cast<int>(rank), g, 2, 8192);
                }
            }
        } else if (warp == kWarpV) {
            // ----------------------------------------------- TMA producer: V
            for (int j = 0; j < nsel; ++j) {
                const int st = j % kPStages;
                const uint32_t ph = (j / kPStages) & 1;
                mbar_wait(&bar->v_empty[st], ph ^ 1);
                if (rank == 0) mbar_expect_tx_warp(&bar->v_full[st], 2 * kVHalfBytes);
                tma_load_pair_warp(smem + kPSmemV + st * kVHalfBytes, &p.tm_v, leader(&bar->v_full[st]),
                                   64 * static_cast<int>(rank), sel_at(j) * kBlock, g, 1, 0);
            }
        } else if (warp == kWarpS || warp == kWarpPV) {
            // ----------------------------- MMA issuers (leader only): warp 9 issues
            // the S stream, warp 11 the P·V stream. tcgen05.mma issue blocks while
            // the tensor pipe is full, so one thread issuing both streams in a fixed
            // order idles on whichever event comes later; two issuers each wait
            // only for their own operands. The streams share no TMEM or shared
            // memory (S buffer vs P buffers / O; K vs V), and each commits its own
            // barriers (a commit tracks the committing thread's MMAs).
            if (rank == 0 && nsel > 0) {
                const uint32_t tm = __shfl_sync(0xffffffffu, static_cast<uint32_t>(lds_s32(smem_u32(&bar->tmem_base))), 0);
                if (warp == kWarpS) {
                    const uint64_t qd = umma_desc_sw128(smem_u32(smem + kPSmemQ), 16, 1024);
                    const uint64_t kd0 = umma_desc_sw128(smem_u32(smem + kPSmemK), 16, 1024);
                    mbar_wait(&bar->q_full, 0);
                    for (int j = 0; j < nsel; ++j) {
                        if (j > 0) mbar_wait(&bar->s_free, (j - 1) & 1);  // S(j-1) is in registers
                        PTRACE(j - 1, 0, (threadIdx.x & 31) == 0);
                        const int st = j % kPStages;
                        mbar_wait(&bar->k_full[st], (j / kPStages) & 1);
                        tc_fence_after();
                        mma_pair_ss(tm + kColS, qd, kd0 + static_cast<uint64_t>(st) * (kKHalfBytes >> 4), kIdescPairS, 0u);
                        mma_commit_pair_warp(&bar->s_full[j & 1]);
                        mma_commit_pair_warp(&bar->k_empty[st]);
                        PTRACE(j - 1, 1, (threadIdx.x & 31) == 0);
                    }
                } else {
                    const uint64_t vd0 = umma_desc_sw128(smem_u32(smem + kPSmemV), 16384, 1024);
                    for (int j = 0; j < nsel; ++j) {
                        const int st = j % kPStages;
                        mbar_wait(&bar->p_full[0][j & 1], (j >> 1) & 1);
                        mbar_wait(&bar->p_full[1][j & 1], (j >> 1) & 1);
                        PTRACE(j, 2, (threadIdx.x & 31) == 0);
                        mbar_wait(&bar->v_full[st], (j / kPStages) & 1);
                        tc_fence_after();
                        mma_pair_ts(tm + kColO + 128u * static_cast<uint32_t>(j & 1),
                                    tm + kColP + 64u * static_cast<uint32_t>(j & 1),
                                    vd0 + static_cast<uint64_t>(st) * (kVHalfBytes >> 4), kIdescPairPV, j > 1 ? 1u : 0u);
                        mma_commit_pair_warp(&bar->pv_done[j & 3]);
                        mma_commit_pair_warp(&bar->v_empty[st]);
                        PTRACE(j, 3, (threadIdx.x & 31) == 0);
                    }
                }
            }
        }
    } else {
        setmaxnreg_inc<kPRegsSoftmax>();
        int nsel, h, g;
        int64_t row0;
        tile_scalars(nsel, row0, h, g);
        (void)g;
        // ------------------------------------------------ softmax warpgroups
        // Each warpgroup runs its own online softmax over its blocks (its own
        // running max m, row sum l and accumulator O_wg in TMEM), so neither
        // waits on the other; the epilogue merges the two.
        const int wg = warp >> 2;          // takes blocks j = wg, wg + 2, ...
        const int r = threadIdx.x & 127;   // row within this CTA's half == TMEM lane
        const int64_t qrow = row0 + 128 * static_cast<int64_t>(rank) + r;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t s_addr = tmem + lane_base + kColS;
        const uint32_t p_addr = tmem + lane_base + kColP + 64u * static_cast<uint32_t>(wg);
        const uint32_t o_addr = tmem + lane_base + kColO + 128u * static_cast<uint32_t>(wg);
        const float sl2 = p.scale_log2;
        const int64_t lim = p.causal ? min(qrow, p.n - 1) : p.n - 1;  // last visible key
        const uint32_t s_free_l = leader(&bar->s_free);
        const uint32_t p_full_l = leader(&bar->p_full[rank][wg]);
        const float2 sc2 = make_float2(sl2, sl2);
        float m = -INFINITY;  // this warpgroup's reference max (log2 domain)
        float l = 0.0f;       // its row sum, relative to m
        int mine = 0;         // blocks this warpgroup has processed
        for (int j = wg; j < nsel; j += 2, ++mine) {
            const int64_t key0 = static_cast<int64_t>(sel_at(j)) * kBlock;
            const bool need_mask = key0 + kBlock - 1 > lim;
            uint32_t sv[kBlock];
            float* s = reinterpret_cast<float*>(sv);
            mbar_wait(&bar->s_full[wg], mine & 1);
            PTRACE(j, 4, r == 0);
            if (j == 0 && threadIdx.x == 0) TTRACE(4, clock64());
            tc_fence_after();
            tmem_ld32(s_addr + 0, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
            tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
            tmem_ld32(s_addr + 64, *reinterpret_cast<uint32_t(*)[32]>(&sv[64]));
            tmem_ld32(s_addr + 96, *reinterpret_cast<uint32_t(*)[32]>(&sv[96]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive_cluster_warp(s_free_l);  // the leader may now compute S(j+1) over it
            if (need_mask) {
#pragma unroll
                for (int c = 0; c < kBlock; ++c)
                    if (key0 + c > lim) s[c] = -INFINITY;
            }
            float mx8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
#pragma unroll
            for (int c = 0; c < kBlock; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
            PTRACE(j, 5, r == 0);
            // Lazy rule: raise m only when the block max exceeds it by > 2^8.
            const float mprev = m;
            if (mx > m + kPairRescaleThreshold || (m == -INFINITY && mx > -INFINITY)) m = mx;
            const bool rose = m != mprev && mprev != -INFINITY;
            const float msub = (m == -INFINITY) ? 0.0f : m;
            const float2 nm2 = make_float2(-msub, -msub);
            float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            PTRACE(j, 6, r == 0);
            // All 128 exponentials first (packed bf16 pairs; the S registers die
            // as they are consumed), then wait for this warpgroup's last P·V —
            // P(j-2)·V(j-2), which read its P buffer and accumulated into its O —
            // while this block exponentiated.
            uint32_t pk[4][16];
#pragma unroll
            for (int e = 0; e < kBlock / 2; ++e) {
                const float2 x = ffma2(make_float2(s[2 * e], s[2 * e + 1]), sc2, nm2);
                float2 pe;
                pe.x = ex2(x.x);
                pe.y = ex2(x.y);
                sum2[e & 1] = fadd2(sum2[e & 1], pe);
                pk[e >> 4][e & 15] = pack_bf16x2(pe.x, pe.y);
            }
            PTRACE(j, 7, r == 0);
            if (mine >= 1) {
                mbar_wait(&bar->pv_done[(j - 2) & 3], ((j - 2) >> 2) & 1);
                tc_fence_after();
            }
            // O_wg holds this warpgroup's P·V relative to mprev: rescale it before
            // P(j)·V(j) accumulates when m rose (rare; branches, not selects: an
            // ex2 per row per block would queue on the MUFU).
            if (__any_sync(0xffffffffu, rose)) {
                const float alpha = rose ? ex2(mprev - m) : 1.0f;
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
            if (rose) l *= ex2(mprev - m);
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_st16(p_addr + c * 16, pk[c]);
            const float2 sum = fadd2(sum2[0], sum2[1]);
            l += sum.x + sum.y;
            tmem_wait_st();
            PTRACE(j, 8 + (warp & 3), (threadIdx.x & 31) == 0);  // P stored, per warp
            tc_fence_before();
            mbar_arrive_cluster_warp(p_full_l);
        }

        // -------------------------------------------------------- epilogue
        // O = (O_0 2^(m_0 - m_f) + O_1 2^(m_1 - m_f)) / (l_0 2^(m_0 - m_f) +
        // l_1 2^(m_1 - m_f)), m_f = max(m_0, m_1); a warpgroup that had no
        // block (nsel = 1) or only masked ones (m = -inf) contributes nothing
        // (its O is never read). Staged in this CTA's Q buffer (free once the
        // last P·V, which follows every S, has completed) — warpgroup w writes
        // d-chunk w — then stored with bulk tensor copies.
        lfin[(wg * 2 + 0) * 128 + r] = l;
        lfin[(wg * 2 + 1) * 128 + r] = m;
        named_bar_sync(1, 256);
        const float m0 = lfin[1 * 128 + r], m1 = (nsel > 1) ? lfin[3 * 128 + r] : -INFINITY;
        const float mf = fmaxf(m0, m1);
        const float f0 = m0 != -INFINITY ? ex2(m0 - mf) : 0.0f;
        const float f1 = m1 != -INFINITY ? ex2(m1 - mf) : 0.0f;
        const float lt = lfin[0 * 128 + r] * f0 + (nsel > 1 ? lfin[2 * 128 + r] * f1 : 0.0f);
        const float inv = lt > 0.0f ? 1.0f / lt : 0.0f;
        const float g0 = f0 * inv, g1 = f1 * inv;
        const bool live = row0 + 128 * static_cast<int64_t>(rank) < p.n;
        if (nsel > 0) {
            mbar_wait(&bar->pv_done[(nsel - 1) & 3], ((nsel - 1) >> 2) & 1);
            tc_fence_after();
        }
        if (threadIdx.x == 0) TTRACE(5, clock64());
        if (live) {
            const uint32_t tile_s = smem_u32(smem + kPSmemQ);
            const uint32_t o0 = tmem + lane_base + kColO, o1 = o0 + 128u;
#pragma unroll 1
            for (int cc = 0; cc < 2; ++cc) {
                const int c = wg * 2 + cc;  // 32-column group of d (warpgroup w: d-chunk w)
                float v[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.0f;
                if (nsel > 0 && m0 != -INFINITY) {
                    uint32_t t[32];
                    tmem_ld32(o0 + c * 32, t);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(t[e]) * g0;
                }
                if (nsel > 1 && m1 != -INFINITY) {
                    uint32_t t[32];
                    tmem_ld32(o1 + c * 32, t);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = fmaf(__uint_as_float(t[e]), g1, v[e]);
                }
                const uint32_t row_s = tile_s + static_cast<uint32_t>(wg) * 16384u + static_cast<uint32_t>(r) * 128u;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t chunk = static_cast<uint32_t>(cc * 4 + u) ^ static_cast<uint32_t>(r & 7);
                    sts128(row_s + chunk * 16u, pack_bf16x2(v[u * 8 + 0], v[u * 8 + 1]),
                           pack_bf16x2(v[u * 8 + 2], v[u * 8 + 3]), pack_bf16x2(v[u * 8 + 4], v[u * 8 + 5]),
                           pack_bf16x2(v[u * 8 + 6], v[u * 8 + 7]));
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(2, 256);
            if (threadIdx.x == 0) {
                const int ndst = p.n_out_peers > 0 ? p.n_out_peers : 1;
                const int plane = p.n_out_peers > 0 ? p.heads.k[h] : h;
                const int32_t rowg = static_cast<int32_t>(row0) + 128 * static_cast<int32_t>(rank);
                for (int i = 0; i < ndst; ++i) tma_store_tile(&p.tm_out[i], tile_s, rowg, plane);
                bulk_commit_group();
                if (p.n_out_peers > 1) {
                    bulk_wait_group0();
                    __threadfence_system();
                } else {
                    bulk_wait_group_read0();
                }
            }
        }
        if (threadIdx.x == 0) TTRACE(6, clock64());
    }

#ifdef SHPLB_PTRACE
    __syncthreads();
    for (int rr = 0; rr < 2; ++rr) {
    cluster_sync_all();
    if ((blockIdx.x >> 1) == SHPLB_PTRACE && rank == rr && threadIdx.x == 0) {
        const long long t0 = ptrace[0][4];
        printf("PTRACE rank %d\n", rr);
        printf("PTRACE nsel %d\n", p.cnt[(p.tiles[blockIdx.x >> 1] >> 20) * (int64_t)p.nqb + (p.tiles[blockIdx.x >> 1] & 0xFFFFF)]);
        for (int j = 0; j < kPTraceBlocks; ++j)
            printf("PTRACE j %d mma sfree %lld s_iss %lld pfull %lld vfull %lld | sm sfull %lld max %lld mdec %lld expd %lld pst %lld %lld %lld %lld\n", j,
                   ptrace[j][0] - t0, ptrace[j][1] - t0, ptrace[j][2] - t0, ptrace[j][3] - t0, ptrace[j][4] - t0,
                   ptrace[j][5] - t0, ptrace[j][6] - t0, ptrace[j][7] - t0, ptrace[j][8] - t0,
                   ptrace[j][9] - t0, ptrace[j][10] - t0, ptrace[j][11] - t0);
    }
    }
#endif
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer is done with this CTA's barriers and operands
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc_pair<kPairTmemCols>(tmem);
    }
    if (threadIdx.x == 0) TTRACE(7, clock64());
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

#ifdef SHPLB_TILETRACE
extern "C" int shplb_debug_tiletrace(void* host, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, shplb::kern::g_tiletrace, bytes));
}
#endif
