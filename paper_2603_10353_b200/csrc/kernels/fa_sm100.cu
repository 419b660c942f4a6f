// Kernel 3: block-sparse FlashAttention prefill for sm_100a.
//
// One CTA computes one query block (bq = 256 rows, or 128) of one head over
// that block's selected 128-key blocks (ascending ids from kernel 2). The
// query block is split into two 128-row halves, each owned by one softmax
// warpgroup with its own S/P and O accumulators in TMEM; every K/V tile that
// TMA stages in shared memory is consumed by both halves, so each 64 KB of
// K/V pulled from L2 feeds 2 x 8.4 MFLOP of tensor work. (With one 128-row
// tile per K/V load the kernel was bound by L2->SM bandwidth.)
//
// Per selected block j and half h (skipped when block j is entirely in the
// causal future of half h):
//   S_h = Q_h K_j^T        tcgen05.mma, A = Q_h (smem), B = K_j (smem), fp32 in TMEM
//   P_h = exp2(S_h*c - m_h) online softmax in registers (thread = query row =
//                          TMEM lane), bf16 P written back over S_h in TMEM
//   O_h += P_h V_j          tcgen05.mma with A read from TMEM, B = V_j (MN-major)
// The reference semantics are softmax_weighted_sum over the kept set
// (proj/src/attention.cpp:35-49) with the causal mask of :28-30; a row with no
// visible kept key is zero (:40-41). The running max is rescaled lazily (only
// when it grows by > 2^8); the O correction is an in-place TMEM ld/st.
//
// Warp roles (384 threads, registers rebalanced with setmaxnreg):
//   warps 0-3   softmax, query half 0 (rows 0..127 of the block)
//   warps 4-7   softmax, query half 1 (rows 128..255)
//   warp 8      TMA producer: Q once, then K_j / V_j into 2-stage rings
//   warp 9      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 10-11 idle (complete the control warpgroup for setmaxnreg)
// MMA issue order per block j: PV_0(j), S_0(j+1), PV_1(j), S_1(j+1): while
// half 0 exponentiates block j the tensor core runs half 1's PV/S, and the
// S/P aliasing WAR is ordered by the in-order tensor pipe.
//
// Shared memory (1024-aligned, 128B-swizzled UMMA operands):
//   Q  [2 halves][2 d-chunks][128 rows][64 bf16]         64 KB (K-major A)
//   K  [2 stages][2 d-chunks][128 keys][64 bf16]         64 KB (K-major B)
//   V  [2 stages][2 d-chunks][128 keys][64 bf16]         64 KB (MN-major B)
//   selected block ids, mbarriers
// TMEM (512 columns): S/P half 0 [0,128), S/P half 1 [128,256),
//                     O half 0 [256,384), O half 1 [384,512).
#include <cstdint>
#include <cstdio>
#include <type_traits>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace shplb::kern {
namespace {

using namespace shplb::ptx;

#ifndef SHPLB_THREADS
#define SHPLB_THREADS 384
#endif
// 384: 3 warpgroups, registers rebalanced with setmaxnreg (softmax 216 / control 72).
// 320: 10 warps (no idle warps), no setmaxnreg; every thread gets the 200-register launch grant.
constexpr int kThreads = SHPLB_THREADS;
constexpr bool kRebalance = kThreads == 384;
// Register split. The CTA is granted 384 x 168 registers at launch (65536/384
// rounded down to a multiple of 8); setmaxnreg.inc blocks until the pool can
// cover it, so 2*softmax + control must not exceed 3*168 or the kernel hangs.
constexpr uint32_t kRegsLaunch = 168;
constexpr uint32_t kRegsSoftmax = 216, kRegsControl = 72;
static_assert(2 * kRegsSoftmax + kRegsControl <= 3 * kRegsLaunch, "setmaxnreg budget exceeds the launch grant");
constexpr int kTileBytes = kBlock * kHeadDim * 2;  // 32 KB: one 128x128 bf16 tile
constexpr int kChunkBytes = kTileBytes / 2;        // 16 KB: 128 rows x 128 B
constexpr uint32_t kTmemCols = 512;
// TMEM column of half h's S/P and O accumulators.
__host__ __device__ constexpr uint32_t col_s(int h) { return static_cast<uint32_t>(h) * 128u; }
__host__ __device__ constexpr uint32_t col_o(int h) { return 256u + static_cast<uint32_t>(h) * 128u; }
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale when max grows by > 2^8
#ifndef SHPLB_EMU_PAIRS
#define SHPLB_EMU_PAIRS 0
#endif
// Exponential pairs (of every 16) computed by the FMA-pipe polynomial instead
// of MUFU ex2, in blocks without masked keys (0 = all on MUFU).
constexpr int kEmuPairs = SHPLB_EMU_PAIRS;
static_assert(kEmuPairs >= 0 && kEmuPairs <= 16, "SHPLB_EMU_PAIRS out of range");

constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, 0, 0);   // A=Q K-major, B=K K-major
#ifndef SHPLB_WARP_ARRIVE
#define SHPLB_WARP_ARRIVE 1
#endif
// P handoff arrivals: one elected lane per softmax warp (4 per half) after the
// warp-collective tcgen05.wait::st, instead of all 128 threads.
constexpr uint32_t kPArrivals = SHPLB_WARP_ARRIVE ? 4u : 128u;
__device__ __forceinline__ void p_arrive(uint64_t* bar) {
    if (SHPLB_WARP_ARRIVE) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
    } else {
        mbar_arrive(bar);
    }
}
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, 0, 1);  // A=P (TMEM), B=V MN-major

struct __align__(8) Barriers {
    uint64_t q_full;
    uint64_t k_full[2], k_empty[2];
    uint64_t v_full[2], v_empty[2];
    uint64_t s_full[2];   // per half: S of its next block is in TMEM
    uint64_t p_full[2];   // per half: P written (and O rescaled) -> PV may run
    uint64_t pv_done[2];  // per half: its last issued PV has completed
    uint32_t tmem_base;
};

constexpr size_t kSmemQ = 0;
constexpr size_t kSmemK = kSmemQ + 2 * kTileBytes;
constexpr size_t kSmemV = kSmemK + 2 * kTileBytes;
constexpr size_t kSmemSel = kSmemV + 2 * kTileBytes;
constexpr size_t kSmemBar = kSmemSel + 2 * kMaxSelected * sizeof(int32_t);  // one list per half (dual)
constexpr size_t kSmemTotal = kSmemBar + sizeof(Barriers) + 1024;  // + alignment slack

// Operand layouts (the descriptor walk per k-step is in ptx.cuh's mma_tile_*):
// K-major SW128 Q / K — k-step kk (16 elements) lives in d chunk kk/4 at byte
// offset (kk%4)*32 within each 128-byte row, 8-row groups 1024 B apart (SBO);
// MN-major SW128 V as B of P.V — N = d spans the two 64-wide d chunks (LBO =
// 16 KB apart), K = keys, 8-key groups 1024 B apart, k-step kk 2 KB further.

#ifdef SHPLB_TRACE  // dev-only: per-block clock64 timeline of one CTA, printed at exit
constexpr int kTraceBlocks = 48;
#define TRACE(j, e, cond) \
    do { if ((cond) && (j) >= 0 && (j) < kTraceBlocks) trace[(j)][(e)] = clock64(); } while (0)
#else
#define TRACE(j, e, cond) do { } while (0)
#endif

// kDual (block_q = 128): the two halves are two consecutive 128-row query
// blocks of one head, each with its OWN selection and its own single-stage
// K / V buffers (the "stage" index of the shared-tile kernel becomes the half),
// fed by its own producer warp (8 or 10); the work list packs the pair as
// (h << 20) | (pair << 2) | (mask of live halves). Without it (block_q = 256)
// both halves read the same selection and share 2-stage K / V rings.
template <bool kDual>
__global__ void __launch_bounds__(kThreads, 1) fa_sparse_kernel(const __grid_constant__ FaParams p) {
#ifdef SHPLB_TRACE
    __shared__ long long trace[kTraceBlocks][16];
    for (int i = threadIdx.x; i < kTraceBlocks * 16; i += kThreads) trace[i / 16][i % 16] = 0;
#endif
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bar = reinterpret_cast<Barriers*>(smem + kSmemBar);
    int32_t* sel = reinterpret_cast<int32_t*>(smem + kSmemSel);
    const uint32_t sSel = smem_u32(sel);
    auto sel_at = [&](int j) { return lds_s32(sSel + 4u * static_cast<uint32_t>(j)); };
    // half hf's list (dual: its own, 2048 entries further for half 1)
    auto sel_at_h = [&](int hf, int j) {
        return lds_s32(sSel + 4u * static_cast<uint32_t>(j + (kDual ? hf * kMaxSelected : 0)));
    };
    const uint32_t sQ = smem_u32(smem + kSmemQ);
    const uint32_t sK = smem_u32(smem + kSmemK);
    const uint32_t sV = smem_u32(smem + kSmemV);

    const int warp = warp_index_uniform();

    const int32_t tile = p.tiles[blockIdx.x];
    const int h = tile >> 20;
    const int qb = kDual ? ((tile >> 2) & 0x3FFFF) : (tile & 0xFFFFF);  // dual: the pair index
    const int g = p.heads.kv[h];
    const int64_t row_id = static_cast<int64_t>(h) * p.nqb + (kDual ? 2 * qb : qb);
    // dual: per-half counts (a half outside the tile's mask or past nqb is empty)
    const int nsel0 = kDual ? ((tile & 1) ? p.cnt[row_id] : 0) : p.cnt[row_id];
    const int nsel1 = kDual ? (((tile & 2) && 2 * qb + 1 < p.nqb) ? p.cnt[row_id + 1] : 0) : nsel0;
    const int nsel = nsel0 > nsel1 ? nsel0 : nsel1;
    auto nsel_h = [&](int hf) { return hf == 0 ? nsel0 : nsel1; };
    const int64_t row0 = static_cast<int64_t>(qb) * (kDual ? 2 * kBlock : p.bq);  // first query row
    const int halves = kDual ? 2 : p.bq / kBlock;  // 2 (bq = 256 or dual) or 1 (bq = 128, not dual)
    {
        const int32_t* gsel = p.idx + row_id * p.kmax;
        for (int j = threadIdx.x; j < nsel0; j += kThreads) sel[j] = gsel[j];
        if (kDual) {
            for (int j = threadIdx.x; j < nsel1; j += kThreads) sel[kMaxSelected + j] = gsel[p.kmax + j];
        }
    }
    // Does half hf compute key block j? It must hold rows (< n) and, under the
    // causal mask, see at least the block's first key. (Dual: every entry of a
    // 128-row block's own list is visible to it.)
    auto active = [&](int hf, int j) -> bool {
        const int64_t first = row0 + hf * kBlock;
        if (hf >= halves || first >= p.n) return false;
        if (kDual) return j < nsel_h(hf);
        return !p.causal || static_cast<int64_t>(sel_at(j)) * kBlock <= first + kBlock - 1;
    };

    if (threadIdx.x == 0) {
        mbar_init(&bar->q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->k_full[i], 1);
            mbar_init(&bar->k_empty[i], 1);
            mbar_init(&bar->v_full[i], 1);
            mbar_init(&bar->v_empty[i], 1);
            mbar_init(&bar->s_full[i], 1);
            mbar_init(&bar->p_full[i], kPArrivals);
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
      if constexpr (kRebalance) setmaxnreg_dec<kRegsControl>();
      // The control warps run their loops with all 32 lanes (warp-uniform
      // control flow); one elected lane issues each TMA / MMA / commit inside
      // the same asm statement, so ptxas emits plain uniform-datapath issue.
      if (kDual && warp == 10) {
        // ---------------------------- TMA producer of half 1's K / V (dual)
        for (int j = 0; j < nsel1; ++j) {
            const uint32_t ph = j & 1;
            const int key0 = sel_at_h(1, j) * kBlock;
            mbar_wait(&bar->k_empty[1], ph ^ 1);
            tma_load_tile_warp(smem + kSmemK + kTileBytes, &p.tm_k, &bar->k_full[1], kTileBytes, key0, g);
            mbar_wait(&bar->v_empty[1], ph ^ 1);
            tma_load_tile_warp(smem + kSmemV + kTileBytes, &p.tm_v, &bar->v_full[1], kTileBytes, key0, g);
        }
      } else if (warp == 8) {
        // ------------------------------------------------------ TMA producer
        if (nsel > 0) {
            tma_load_tile_warp(smem + kSmemQ, &p.tm_q, &bar->q_full, halves * kTileBytes,
                               static_cast<int>(row0), h);
            if (halves == 2)
                tma_load_tile_noarm_warp(smem + kSmemQ + kTileBytes, &p.tm_q, &bar->q_full,
                                         static_cast<int>(row0) + kBlock, h);
            // dual: this warp streams half 0's own K / V through single stages
            if constexpr (kDual) {
                for (int j = 0; j < nsel0; ++j) {
                    const uint32_t ph = j & 1;
                    const int key0 = sel_at_h(0, j) * kBlock;
                    mbar_wait(&bar->k_empty[0], ph ^ 1);
                    tma_load_tile_warp(smem + kSmemK, &p.tm_k, &bar->k_full[0], kTileBytes, key0, g);
                    mbar_wait(&bar->v_empty[0], ph ^ 1);
                    tma_load_tile_warp(smem + kSmemV, &p.tm_v, &bar->v_full[0], kTileBytes, key0, g);
                }
            }
            for (int j = 0; j < (kDual ? 0 : nsel); ++j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                const int key0 = sel_at(j) * kBlock;
                mbar_wait(&bar->k_empty[st], ph ^ 1);
#ifdef SHPLB_DIAG_NO_KV_TMA  // dev-only diagnostic: K/V tiles loaded once, then reused (stale data)
                if (j >= 2) {
                    TRACE(j, 11, (threadIdx.x & 31) == 0);
                    if ((threadIdx.x & 31) == 0) mbar_arrive(&bar->k_full[st]);
                    mbar_wait(&bar->v_empty[st], ph ^ 1);
                    TRACE(j, 12, (threadIdx.x & 31) == 0);
                    if ((threadIdx.x & 31) == 0) mbar_arrive(&bar->v_full[st]);
                    continue;
                }
#endif
                tma_load_tile_warp(smem + kSmemK + st * kTileBytes, &p.tm_k, &bar->k_full[st],
                                   kTileBytes, key0, g);
                TRACE(j, 11, (threadIdx.x & 31) == 0);
                mbar_wait(&bar->v_empty[st], ph ^ 1);
                tma_load_tile_warp(smem + kSmemV + st * kTileBytes, &p.tm_v, &bar->v_full[st],
                                   kTileBytes, key0, g);
                TRACE(j, 12, (threadIdx.x & 31) == 0);
            }
        }
      } else if (warp == 9) {
        // -------------------------------------------------------- MMA issuer
        if (nsel > 0) {
            // TMEM base re-read here (warp-uniform) so no register has to
            // survive the setmaxnreg.dec above (it was spilled to the stack
            // and reloaded before every MMA group).
            const uint32_t tmem = __shfl_sync(0xffffffffu, static_cast<uint32_t>(lds_s32(smem_u32(&bar->tmem_base))), 0);
            // Operand descriptors of stage / half s: the base descriptor plus the
            // tile offset in the 16-byte start-address field (plain adds; an
            // array indexed by j & 1 would live in local memory and put an
            // LDL on the issue path).
            const uint64_t qd0 = umma_desc_sw128(sQ, 16, 1024);
            const uint64_t kd0 = umma_desc_sw128(sK, 16, 1024);
            const uint64_t vd0 = umma_desc_sw128(sV, kChunkBytes, 1024);
            constexpr uint64_t kTileDesc = kTileBytes >> 4;
            auto qdesc = [&](int hf) { return qd0 + static_cast<uint64_t>(hf) * kTileDesc; };
            auto kdesc = [&](int st) { return kd0 + static_cast<uint64_t>(st) * kTileDesc; };
            auto vdesc = [&](int st) { return vd0 + static_cast<uint64_t>(st) * kTileDesc; };
            mbar_wait(&bar->q_full, 0);
            int done[2] = {0, 0};  // blocks each half has issued PV for
            // K / V buffer and phase of (half, block): shared 2-stage rings, or
            // (dual) the half's own single stage.
            auto stage = [&](int hf, int j) { return kDual ? hf : (j & 1); };
            auto phase = [&](int j) { return kDual ? static_cast<uint32_t>(j & 1) : static_cast<uint32_t>((j >> 1) & 1); };
            auto issue_s = [&](int hf, int j) {  // S_hf = Q_hf K_j^T
                mbar_wait(&bar->k_full[stage(hf, j)], phase(j));
                TRACE(j - 1, 9, hf == 0 && (threadIdx.x & 31) == 0);
                tc_fence_after();
                mma_tile_ss_kmajor(tmem + col_s(hf), qdesc(hf), kdesc(stage(hf, j)), kIdescQK, 0u);
                TRACE(j - 1, hf == 0 ? 10 : 14, (threadIdx.x & 31) == 0);
                mma_commit_warp(&bar->s_full[hf]);
                if (kDual) mma_commit_warp(&bar->k_empty[hf]);
            };
            auto issue_pv = [&](int hf, int j) {  // O_hf += P_hf V_j
                mbar_wait(&bar->v_full[stage(hf, j)], phase(j));
                TRACE(j, 6, hf == 0 && (threadIdx.x & 31) == 0);
                mbar_wait(&bar->p_full[hf], done[hf] & 1);
                TRACE(j, 7, hf == 0 && (threadIdx.x & 31) == 0);
                tc_fence_after();
                mma_tile_ts_mnmajor(tmem + col_o(hf), tmem + col_s(hf), vdesc(stage(hf, j)), kIdescPV,
                                    done[hf] > 0 ? 1u : 0u);
                TRACE(j, hf == 0 ? 8 : 13, (threadIdx.x & 31) == 0);
                mma_commit_warp(&bar->pv_done[hf]);
                if (kDual) mma_commit_warp(&bar->v_empty[hf]);
                ++done[hf];
            };
            for (int hf = 0; hf < 2; ++hf)
                if (active(hf, 0)) issue_s(hf, 0);
            if (!kDual) mma_commit_warp(&bar->k_empty[0]);
            for (int j = 0; j < nsel; ++j) {
                const bool next = j + 1 < nsel;
                for (int hf = 0; hf < 2; ++hf) {
                    if (active(hf, j)) issue_pv(hf, j);
                    if (next && active(hf, j + 1)) issue_s(hf, j + 1);
                }
                if (!kDual) {
                    mma_commit_warp(&bar->v_empty[j & 1]);
                    if (next) mma_commit_warp(&bar->k_empty[(j + 1) & 1]);
                }
                TRACE(j, 15, (threadIdx.x & 31) == 0);
            }
        }
      }
    } else {
        if constexpr (kRebalance) setmaxnreg_inc<kRegsSoftmax>();
        // ------------------------------------------------ softmax warpgroups
        const int hf = warp >> 2;             // query half
        const int r = threadIdx.x & 127;      // row within the half == TMEM lane
        const int64_t qrow = row0 + hf * kBlock + r;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t s_addr = tmem + lane_base + col_s(hf);
        const uint32_t o_addr = tmem + lane_base + col_o(hf);
        const float sl2 = p.scale_log2;
        const int64_t lim = p.causal ? min(qrow, p.n - 1) : p.n - 1;  // last visible key
        float m = -INFINITY;  // running max, log2 domain (stale by < 2^8)
        float l = 0.0f;       // running denominator relative to m
        int it = 0;           // blocks this half has processed
        const float2 sc2 = make_float2(sl2, sl2);
        // One 32-key quarter of P = 2^(S*scale_log2 - msub): packed-pair
        // FFMA2 / MUFU ex2 (or, for kEmuPairs of every 16 pairs in unmasked
        // blocks, the FMA-pipe polynomial) / FADD2 row sum, bf16 pairs stored
        // back over S's first columns (tcgen05.st). With track, the raw row
        // max of the quarter is folded into mx8 on the ALU pipe meanwhile.
        auto exp_quarter = [&](const float* s, int c, float msub, float2 (&sum2)[2], auto emu_tag) {
            constexpr bool kEmu = decltype(emu_tag)::value;
            const float2 nm2 = make_float2(-msub, -msub);
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const float2 x = ffma2(make_float2(s[c * 32 + 2 * e], s[c * 32 + 2 * e + 1]), sc2, nm2);
                float2 pe;
                if constexpr (kEmu) {
                    if (((e * kEmuPairs) & 15) < kEmuPairs) {
                        pe = ex2_poly2(x);
                    } else {
                        pe.x = ex2(x.x);
                        pe.y = ex2(x.y);
                    }
                } else {
#ifdef SHPLB_DIAG_NO_EX2  // dev-only diagnostic (wrong results): no MUFU, for energy accounting
                    pe = x;
#else
                    pe.x = ex2(x.x);
                    pe.y = ex2(x.y);
#endif
                }
                sum2[e & 1] = fadd2(sum2[e & 1], pe);
                pk[e] = pack_bf16x2(pe.x, pe.y);
            }
#ifdef SHPLB_DIAG_NO_PST  // dev-only diagnostic (wrong results): P not written back to TMEM
            if (__float_as_uint(sum2[0].x) == 0x7fc00001u) tmem_st16(s_addr + c * 16, pk);
#else
            tmem_st16(s_addr + c * 16, pk);
#endif
        };
        // O_hf *= alpha (this half's previous P.V must have completed).
        auto rescale_o = [&](float alpha) {
            mbar_wait(&bar->pv_done[hf], (it - 1) & 1);
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
        };
        for (int j = 0; j < nsel; ++j) {
            if (!active(hf, j)) continue;
            const int64_t key0 = static_cast<int64_t>(sel_at_h(hf, j)) * kBlock;
            const bool need_mask = key0 + kBlock - 1 > lim;  // keys past the query / sequence end
            uint32_t sv[kBlock];
            float* s = reinterpret_cast<float*>(sv);
            uint32_t(&lo0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[0]);
            uint32_t(&lo1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[32]);
            uint32_t(&hi0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[64]);
            uint32_t(&hi1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[96]);
            mbar_wait(&bar->s_full[hf], it & 1);
            tc_fence_after();
            TRACE(j, 3 * hf + 0, r == 0);
#ifdef SHPLB_DIAG_SKIP_ALL  // dev-only diagnostic: no TMEM reads either (pure MMA/TMA pipeline)
            tc_fence_before();
            p_arrive(&bar->p_full[hf]);
            ++it;
            continue;
#endif
            tmem_ld32(s_addr + 0, lo0);
            tmem_ld32(s_addr + 32, lo1);
            tmem_ld32(s_addr + 64, hi0);
            tmem_ld32(s_addr + 96, hi1);
            tmem_wait_ld();
#ifdef SHPLB_DIAG_SKIP_SOFTMAX  // dev-only diagnostic: MMA/TMA pipeline alone
            tc_fence_before();
            p_arrive(&bar->p_full[hf]);
            ++it;
            continue;
#endif
            float mx8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
            float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float alpha = 1.0f;
            const bool emu_blk = kEmuPairs > 0 && !__any_sync(0xffffffffu, need_mask);
            {
                if (need_mask) {
#pragma unroll
                    for (int c = 0; c < kBlock; ++c)
                        if (key0 + c > lim) s[c] = -INFINITY;
                }
#pragma unroll
                for (int c = 0; c < kBlock; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
                const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                const float mx = mraw * sl2;
                if (mx > m + kRescaleThreshold || (m == -INFINITY && mx > -INFINITY)) {
                    alpha = (m == -INFINITY) ? 0.0f : ex2(m - mx);
                    m = mx;
                }
                if (it >= 1 && __any_sync(0xffffffffu, alpha != 1.0f)) rescale_o(alpha);
                const float msub = (m == -INFINITY) ? 0.0f : m;
                TRACE(j, 3 * hf + 1, r == 0);
                if (kEmuPairs > 0 && emu_blk) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) exp_quarter(s, c, msub, sum2, std::true_type{});
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) exp_quarter(s, c, msub, sum2, std::false_type{});
                }
            }
            const float2 sum = fadd2(sum2[0], sum2[1]);
            l = l * alpha + (sum.x + sum.y);
            tmem_wait_st();
            TRACE(j, 3 * hf + 2, r == 0);
            tc_fence_before();
            p_arrive(&bar->p_full[hf]);
            ++it;
        }

        // -------------------------------------------------------- epilogue
        // Row i of this half: O_hf / l (zero when no kept key was visible),
        // written to `out`, or — fused gather — to every listed output buffer
        // at the head's global index (peer buffers are written over NVLink).
        // (The head / row are re-derived from the work list here rather than kept
        // live across the block loop, which is register-bound.)
        const int32_t tile_e = p.tiles[blockIdx.x];
        const int h_e = tile_e >> 20;
        const int64_t row0_e = (kDual ? static_cast<int64_t>((tile_e >> 2) & 0x3FFFF) * (2 * kBlock)
                                      : static_cast<int64_t>(tile_e & 0xFFFFF) * p.bq) + hf * kBlock;
        const bool live_half = hf < halves && row0_e < p.n && (!kDual || ((tile_e >> hf) & 1));
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        if (it > 0) {
            mbar_wait(&bar->pv_done[hf], (it - 1) & 1);
            tc_fence_after();
        }
#ifndef SHPLB_STG_EPILOGUE
        // TMA-store epilogue: each thread writes its row, scaled and rounded to
        // bf16, into this half's Q tile in shared memory (free: the half's
        // last S MMA completed before its last P.V), in the 128B-swizzled
        // layout the Q loads use (16-byte chunk c of row r at c ^ (r mod 8));
        // then one thread stores the 128 x 128 tile with two bulk tensor copies
        // per destination — whole 128-byte row segments instead of one 16-byte
        // store per thread per row, and rows past n clipped by the tensor map.
        if (live_half) {
            const uint32_t tile_s = sQ + static_cast<uint32_t>(hf) * kTileBytes;
            // A half that computed nothing must still let the Q load (issued
            // whenever the tile has any block) land before reusing its buffer.
            if (it == 0 && nsel > 0) mbar_wait(&bar->q_full, 0);
#pragma unroll 1
            for (int c = 0; c < kHeadDim / 32; ++c) {
                uint32_t v[32];
                if (it > 0) {
                    tmem_ld32(o_addr + c * 32, v);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0u;
                }
                const uint32_t row_s = tile_s + static_cast<uint32_t>(c >> 1) * kChunkBytes + static_cast<uint32_t>(r) * 128u;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t chunk = static_cast<uint32_t>((c & 1) * 4 + u) ^ static_cast<uint32_t>(r & 7);
                    sts128(row_s + chunk * 16u,
                           pack_bf16x2(__uint_as_float(v[u * 8 + 0]) * inv, __uint_as_float(v[u * 8 + 1]) * inv),
                           pack_bf16x2(__uint_as_float(v[u * 8 + 2]) * inv, __uint_as_float(v[u * 8 + 3]) * inv),
                           pack_bf16x2(__uint_as_float(v[u * 8 + 4]) * inv, __uint_as_float(v[u * 8 + 5]) * inv),
                           pack_bf16x2(__uint_as_float(v[u * 8 + 6]) * inv, __uint_as_float(v[u * 8 + 7]) * inv));
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1 + hf, 128);  // the half's 4 warps wrote their rows
            if (r == 0) {
                const int ndst = p.n_out_peers > 0 ? p.n_out_peers : 1;
                const int plane = p.n_out_peers > 0 ? p.heads.k[h_e] : h_e;
                for (int i = 0; i < ndst; ++i) tma_store_tile(&p.tm_out[i], tile_s, static_cast<int32_t>(row0_e), plane);
                bulk_commit_group();
                // Peer stores must be performed (not just read out of shared
                // memory) before the system fence the cross-rank barrier relies on.
                if (p.n_out_peers > 1) {
                    bulk_wait_group0();
                    __threadfence_system();
                } else {
                    bulk_wait_group_read0();  // shared memory stays valid until read
                }
            }
        }
#else
        // Per-thread stores (dev-only A/B baseline of the TMA-store epilogue).
        const int64_t qrow_e = row0_e + r;
        const bool live = live_half && qrow_e < p.n;
        const int ndst = p.n_out_peers > 0 ? p.n_out_peers : 1;
        auto dst_row = [&](int i) -> __nv_bfloat16* {
            if (p.n_out_peers == 0)
                return static_cast<__nv_bfloat16*>(p.out) + (static_cast<int64_t>(h_e) * p.n + qrow_e) * kHeadDim;
            return static_cast<__nv_bfloat16*>(p.out_peers[i]) +
                   (static_cast<int64_t>(p.heads.k[h_e]) * p.n + qrow_e) * kHeadDim;
        };
#pragma unroll 1
        for (int c = 0; c < kHeadDim / 32; ++c) {
            uint32_t v[32];
            if (it > 0) {
                tmem_ld32(o_addr + c * 32, v);
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0u;
            }
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
        if (p.n_out_peers > 1) __threadfence_system();
#endif
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
#ifdef SHPLB_TRACE
    if (blockIdx.x == SHPLB_TRACE && threadIdx.x == 0) {
        const long long t0 = trace[0][0];
        printf("TRACE cta %d nsel %d\n", blockIdx.x, nsel);
        for (int j = 0; j < kTraceBlocks && j < nsel; ++j)
            printf("TRACE j %d v %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n", j,
                   trace[j][0] - t0, trace[j][1] - t0, trace[j][2] - t0, trace[j][3] - t0,
                   trace[j][4] - t0, trace[j][5] - t0, trace[j][6] - t0, trace[j][7] - t0,
                   trace[j][8] - t0, trace[j][9] - t0, trace[j][10] - t0, trace[j][11] - t0,
                   trace[j][12] - t0, trace[j][13] - t0, trace[j][14] - t0, trace[j][15] - t0);
    }
#endif
}

}  // namespace

void launch_fa(const FaParams& p, int num_tiles, bool dual, cudaStream_t s) {
    if (dual) {
        set_max_dynamic_smem(reinterpret_cast<const void*>(fa_sparse_kernel<true>), static_cast<int>(kSmemTotal));
        fa_sparse_kernel<true><<<num_tiles, kThreads, kSmemTotal, s>>>(p);
    } else {
        set_max_dynamic_smem(reinterpret_cast<const void*>(fa_sparse_kernel<false>), static_cast<int>(kSmemTotal));
        fa_sparse_kernel<false><<<num_tiles, kThreads, kSmemTotal, s>>>(p);
    }
}

}  // namespace shplb::kern
