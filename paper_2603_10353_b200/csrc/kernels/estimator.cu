// Kernels 1 and 2 of the hot path: the block-importance estimator (mean-pool
// Q/K blocks, score pooled Q.K^T) and the per-head top-k block selector.
//
// Reference semantics (proj/src/attention.cpp): scores are q.k * (1/sqrt(d))
// with the scale applied after the dot product (:20,26), causally masked
// entries are -inf (:28-30), the kept set is the k largest under (value desc,
// index asc), emitted in ascending index order (:53-64). The block
// generalisation and the fixed fp32 summation orders are DESIGN.md §3; the C
// oracle (oracle/shplb_oracle.c) restates them and the GPU output is
// bit-identical to it.
//
// Roofline: pooling streams Q and K once from HBM (2*n*d*(Hq+Hkv) bytes) and
// is HBM-bound. Scoring is an fp32 FFMA product of the pooled matrices (kept
// on CUDA cores so every score is bit-reproducible on the CPU), and selection
// is a warp-level radix (bisection) select on the order-preserving uint32
// image of each score; both work out of shared memory / L2.
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace shplb::kern {
namespace {

constexpr int kPoolThreads = 256;  // 16 row groups x 16 column groups of 8 columns

// One CTA pools kRows rows (128 or 256) of one head into kSub output blocks of
// kRows / kSub rows each. Thread (g, cg) sums rows g, g+16, ... (ascending) of
// columns 8cg..8cg+7 of each output block with 16-byte loads (all kRows/16 loads
// in flight); the 16 group partials per column are then added in ascending
// group order — per output block the same additions in the same order whatever
// kSub, so pooled values do not depend on how blocks are packed into CTAs.
template <int kRows, int kSub>
__device__ __forceinline__ void pool_rows(const __nv_bfloat16* __restrict__ x, int64_t n, int64_t head,
                                          int64_t b0, int64_t nb, float* __restrict__ out,
                                          float (&part)[kSub][kPoolSplit][kHeadDim + 4]) {
    constexpr int kLoads = kRows / kPoolSplit, kPerSub = kLoads / kSub, kSubRows = kRows / kSub;
    const int g = threadIdx.x >> 4;
    const int cg = threadIdx.x & 15;
    const int64_t t0 = b0 * kSubRows;  // b0: first output block of this CTA
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kRows), n - t0));
    const __nv_bfloat16* base = x + (head * n + t0) * kHeadDim + cg * 8;

    uint4 v[kLoads];
#pragma unroll
    for (int s = 0; s < kLoads; ++s) {
        const int t = g + s * kPoolSplit;
        v[s] = t < cnt ? __ldg(reinterpret_cast<const uint4*>(base + static_cast<int64_t>(t) * kHeadDim))
                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < kSub; ++j) {
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
#pragma unroll
        for (int s = j * kPerSub; s < (j + 1) * kPerSub; ++s) {
            if (g + s * kPoolSplit < cnt) {
                const uint32_t w[4] = {v[s].x, v[s].y, v[s].z, v[s].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    acc[2 * e] = __fadd_rn(acc[2 * e], __uint_as_float(w[e] << 16));
                    acc[2 * e + 1] = __fadd_rn(acc[2 * e + 1], __uint_as_float(w[e] & 0xFFFF0000u));
                }
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) part[j][g][cg * 8 + e] = acc[e];
    }
    __syncthreads();
    if (threadIdx.x < kSub * kHeadDim) {
        const int j = threadIdx.x / kHeadDim, c = threadIdx.x % kHeadDim;
        const int cj = min(kSubRows, cnt - j * kSubRows);  // rows of output block b0 + j
        if (cj > 0) {
            float total = 0.0f;
#pragma unroll
            for (int gg = 0; gg < kPoolSplit; ++gg) total = __fadd_rn(total, part[j][gg][c]);
            out[(head * nb + b0 + j) * kHeadDim + c] = __fdiv_rn(total, static_cast<float>(cj));
        }
    }
}

// Kernel 1: Q and K of a layer in one launch. The first nbq * hq CTAs pool Q
// (one kRowsQ-row block each), the rest K — at kRowsQ = 256 two 128-row key
// blocks per CTA, so both halves of the grid have the same shape and register
// footprint (a 128-row K CTA at the Q path's ~95 registers would run at half
// the occupancy it needs).
template <int kRowsQ>
__global__ void __launch_bounds__(kPoolThreads) pool_qk_kernel(const __nv_bfloat16* __restrict__ q, int64_t nbq,
                                                               int hq, const __nv_bfloat16* __restrict__ k,
                                                               int64_t nbk, int64_t n, float* __restrict__ qp,
                                                               float* __restrict__ kp) {
    constexpr int kSubK = kRowsQ / kBlock;
    __shared__ float part[kSubK][kPoolSplit][kHeadDim + 4];
    const int64_t id = blockIdx.x;
    const int64_t nq = nbq * hq;
    if (id < nq) {
        pool_rows<kRowsQ, 1>(q, n, id / nbq, id % nbq, nbq, qp,
                             *reinterpret_cast<float(*)[1][kPoolSplit][kHeadDim + 4]>(&part[0]));
    } else {
        const int64_t ck = (nbk + kSubK - 1) / kSubK;  // K CTAs per head
        pool_rows<kRowsQ, kSubK>(k, n, (id - nq) / ck, ((id - nq) % ck) * kSubK, nbk, kp, part);
    }
}

// Key blocks (of kBlock keys) visible to query block qb of bq rows.
__device__ __forceinline__ int64_t visible_blocks(int64_t qb, int64_t n, int64_t nkb, int bq,
                                                  bool causal) {
    if (!causal) return nkb;
    const int64_t last = min((qb + 1) * bq, n) - 1;
    return min(last / kBlock + 1, nkb);
}

// Order-preserving image of an fp32 score (larger float -> larger uint).
// -0.0 is folded onto +0.0 first so equal scores get equal keys.
__device__ __forceinline__ uint32_t order_key(float s) {
    const uint32_t u = __float_as_uint(__fadd_rn(s, 0.0f));
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Warp-level top-k over keys[0..vis) (order_key images): bisection on the key
// bits finds T, the kk-th largest key; keys > T are kept, plus the first
// (kk - #keys>T) keys == T in index order (index-ascending tie rule). Output
// is compacted in ascending index order with ballots. Rows of up to 1024
// candidates are held in registers (32 per lane) for the 33 counting passes.
template <typename KeyAt>
__device__ void warp_select_row(KeyAt key_at, int vis, int kk, int64_t kmax, int32_t* __restrict__ idx_row,
                                uint32_t* __restrict__ scratch) {
    const int lane = threadIdx.x & 31;
    if (kk >= vis) {  // every visible block is kept: no ranking needed
        for (int j = lane; j < vis; j += 32) idx_row[j] = j;
        for (int64_t p = vis + lane; p < kmax; p += 32) idx_row[p] = -1;
        return;
    }
    constexpr int kRegKeys = 32;  // rows of up to 1024 candidates (128K tokens) run from registers
    uint32_t kr[kRegKeys];
    const bool in_regs = vis <= 32 * kRegKeys;
    if (in_regs) {
#pragma unroll
        for (int t = 0; t < kRegKeys; ++t) {
            const int j = lane + 32 * t;
            kr[t] = j < vis ? key_at(j) : 0u;  // 0 is below every real key (order_key(-inf) > 0)
        }
    }
    auto count_ge = [&](uint32_t trial) {
        int c = 0;
        if (in_regs) {
#pragma unroll
            for (int t = 0; t < kRegKeys; ++t) c += kr[t] >= trial;
        } else {
            for (int j = lane; j < vis; j += 32) c += key_at(j) >= trial;
        }
        return __reduce_add_sync(0xffffffffu, c);
    };
    // T = the largest threshold with count(keys >= T) >= kk. Stop early when a
    // trial isolates exactly kk keys: they are then the unique top kk (no tie
    // straddles the boundary), the set the full bisection would keep.
    //
    // Narrowing: after the bits above `bit` are decided, every key is either
    // above the window [T, T + 2^bit) (counted in `hi`), below it, or inside
    // it (lo - hi keys, lo = count(keys >= T)). Once at most 32 keys are
    // inside, they are compacted into one register per lane (scratch: 32
    // words of shared memory per warp) and the remaining bits count only
    // those: hi0 + (inside keys >= trial), hi0 = the keys above the window at
    // narrowing time (later trials all fall inside it). Same counts, same T.
    uint32_t T = 0;
    int lo = vis, hi = 0, hi0 = 0;
    bool narrow = false;
    uint32_t cand = 0u;  // narrowed: this lane's window key (0 = none; trials are >= 1)
    auto count_ge_n = [&](uint32_t trial) {
        return narrow ? hi0 + __popc(__ballot_sync(0xffffffffu, cand >= trial)) : count_ge(trial);
    };
    for (int bit = 31; bit >= 0; --bit) {
        const uint32_t trial = T | (1u << bit);
        const int c = count_ge_n(trial);
        if (c >= kk) {
            T = trial;
            lo = c;
            if (c == kk) break;
        } else {
            hi = c;
        }
        if (!narrow && in_regs && bit > 0 && lo - hi <= 32) {
            // Window [T, T + 2^bit): T >= 1 here unless every trial so far failed,
            // in which case the window starts at 0 and padding (key 0, j >= vis) is excluded by j.
            const uint32_t span = 1u << bit;
            int pos = 0;
#pragma unroll
            for (int t = 0; t < kRegKeys; ++t) {
                const bool in = (lane + 32 * t) < vis && kr[t] >= T && kr[t] - T < span;
                const uint32_t m = __ballot_sync(0xffffffffu, in);
                if (in) scratch[pos + __popc(m & ((1u << lane) - 1u))] = kr[t];
                pos += __popc(m);
            }
            __syncwarp();
            cand = lane < pos ? scratch[lane] : 0u;
            __syncwarp();
            hi0 = hi;
            narrow = true;
        }
    }
    const int gt = T == 0xFFFFFFFFu ? 0 : count_ge_n(T + 1);  // keys > T
    const int need = kk - gt;
    const uint32_t lt_mask = (1u << lane) - 1u;
    int written = 0, ties = 0;
    // Ascending compaction of the kept indices, 32 candidates per step.
    auto emit = [&](int j, uint32_t key) {
        const bool valid = j < vis;
        const bool eq = valid && key == T;
        const uint32_t eq_mask = __ballot_sync(0xffffffffu, eq);
        const int tie_rank = ties + __popc(eq_mask & lt_mask);
        const bool sel = (valid && key > T) || (eq && tie_rank < need);
        const uint32_t sel_mask = __ballot_sync(0xffffffffu, sel);
        if (sel) idx_row[written + __popc(sel_mask & lt_mask)] = j;
        written += __popc(sel_mask);
        ties += __popc(eq_mask);
    };
    if (in_regs) {
#pragma unroll
        for (int t = 0; t < kRegKeys; ++t) {
            if (32 * t >= vis) break;  // warp-uniform
            emit(lane + 32 * t, kr[t]);
        }
    } else {
        for (int base = 0; base < vis; base += 32) {
            const int j = base + lane;
            emit(j, j < vis ? key_at(j) : 0u);
        }
    }
    for (int64_t p = kk + lane; p < kmax; p += 32) idx_row[p] = -1;
}

constexpr int kSelThreads = 256;  // standalone selector: 8 warps, one row each
constexpr int kPad = kHeadDim + 4;  // row stride (floats) of the Q / K tiles: 16-byte rows, no bank conflicts

// Kernel 2 (score + select). One CTA = one GROUP of up to 4 q heads that read
// the same kv head (GQA) x Q = 64, 32, 16, 16 consecutive query blocks for
// G = 1, 2, 3, 4 (powers of two: the slot -> (head, query block) map is
// shifts and masks; a group of 3 leaves 16 of the slots idle): 64 row slots
// share every pooled K chunk the CTA stages in shared memory (G x fewer K
// loads than one head per CTA). 512 threads; thread (rp, kq) holds an 8 x 4
// FFMA register tile: row slots rp + 8i, key blocks kq + 64j of the 256-block
// chunk (per 4 columns 8 + 4 float4 loads feed 128 FFMAs). Every dot product
// is one fmaf chain over c = 0..127 in order, then x (1/sqrt d), so no tiling
// choice changes a score. A thread computes only the key
// blocks of the chunk that exist (nj <= 4), so a partial last chunk costs its
// own size. Scores go to global memory (the caller's score matrix, or a
// workspace that stays in L2), then each warp selects 4 rows from there.
constexpr int kGrpThreads = 512;
constexpr int kGrpRows = 64;     // row slots per CTA
constexpr int kGrpRowStep = 8;   // threads along rows
constexpr int kGrpChunk = 256;   // key blocks per staged chunk
constexpr int kGrpKbStep = kGrpThreads / kGrpRowStep;  // 64 threads along key blocks
constexpr int kGrpRT = kGrpRows / kGrpRowStep;         // 8 rows per thread
constexpr int kGrpKT = kGrpChunk / kGrpKbStep;         // 4 key blocks per thread
constexpr size_t kGrpSmem = sizeof(float) * (kGrpRows + kGrpChunk) * kPad + sizeof(uint32_t) * 32 * (kGrpThreads / 32);

struct GrpCtx {
    float* scores;
    int64_t nqb, nkb, n, qb0;
    int bq, causal, Q, G, qshift;  // Q = 2^qshift query blocks per head
    uint32_t heads;  // 4 x 8-bit q head ids
    __device__ bool valid(int s) const { return (s >> qshift) < G && qb0 + (s & (Q - 1)) < nqb; }
    __device__ int head(int s) const { return static_cast<int>((heads >> (8 * (s >> qshift))) & 0xFFu); }
    __device__ int64_t qb(int s) const { return qb0 + (s & (Q - 1)); }
};

// One chunk's tile product for a thread computing NJ of its key blocks, and
// the store of those scores (-inf past the row's causally visible blocks).
template <int NJ>
__device__ __forceinline__ void grp_tile(const float* __restrict__ Qs, const float* __restrict__ Ks, int rp, int kq,
                                         int64_t kc, int kc_end, float scale, const GrpCtx& c) {
    float a[kGrpRT][NJ];
#pragma unroll
    for (int i = 0; i < kGrpRT; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[i][j] = 0.f;
    const float* q0p = Qs + rp * kPad;
    const float* k0p = Ks + kq * kPad;
#pragma unroll 2
    for (int c4 = 0; c4 < kHeadDim / 4; ++c4) {
        float4 qv[kGrpRT], kv[NJ];
#pragma unroll
        for (int i = 0; i < kGrpRT; ++i) qv[i] = *reinterpret_cast<const float4*>(q0p + i * kGrpRowStep * kPad + c4 * 4);
#pragma unroll
        for (int j = 0; j < NJ; ++j) kv[j] = *reinterpret_cast<const float4*>(k0p + j * kGrpKbStep * kPad + c4 * 4);
#pragma unroll
        for (int i = 0; i < kGrpRT; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                a[i][j] = __fmaf_rn(qv[i].x, kv[j].x, a[i][j]);
                a[i][j] = __fmaf_rn(qv[i].y, kv[j].y, a[i][j]);
                a[i][j] = __fmaf_rn(qv[i].z, kv[j].z, a[i][j]);
                a[i][j] = __fmaf_rn(qv[i].w, kv[j].w, a[i][j]);
            }
    }
#pragma unroll
    for (int i = 0; i < kGrpRT; ++i) {
        const int s = rp + kGrpRowStep * i;
        if (!c.valid(s)) continue;
        const int64_t qb = c.qb(s);
        const int64_t vis = visible_blocks(qb, c.n, c.nkb, c.bq, c.causal != 0);
        float* dst = c.scores + (static_cast<int64_t>(c.head(s)) * c.nqb + qb) * c.nkb + kc;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int kb = kq + kGrpKbStep * j;
            if (kb < kc_end) dst[kb] = kc + kb < vis ? __fmul_rn(a[i][j], scale) : -INFINITY;
        }
    }
}

__global__ void __launch_bounds__(kGrpThreads, 1)
    score_select_kernel(const float* __restrict__ qp, const float* __restrict__ kp, int64_t n, int64_t nqb,
                        int64_t nkb, int bq, int causal, float scale, HeadTable ht, GroupTable gt, int64_t kmax,
                        float* scores, int fill_tail, int select, int32_t* __restrict__ idx,
                        int32_t* __restrict__ cnt, int ksplit) {
    extern __shared__ __align__(16) float smem[];
    float* Qs = smem;                    // [64 row slots][kPad]
    float* Ks = Qs + kGrpRows * kPad;    // [256 key blocks][kPad]
    uint32_t* scratch = reinterpret_cast<uint32_t*>(Ks + kGrpChunk * kPad);  // [16 warps][32]

    GrpCtx c;
    c.scores = scores;
    c.nqb = nqb;
    c.nkb = nkb;
    c.n = n;
    c.bq = bq;
    c.causal = causal;
    c.G = gt.size[blockIdx.x];
    c.qshift = c.G == 1 ? 6 : (c.G == 2 ? 5 : 4);  // a group of 3 leaves 16 slots idle
    c.Q = 1 << c.qshift;
    c.heads = gt.heads[blockIdx.x];
    // Grid (groups, row chunks): the hardware hands out CTAs group-fastest, and
    // y = 0 is the LAST chunk of query blocks, so under the causal mask the
    // heaviest chunks (most visible key blocks) go first and the launch tail
    // is made of the lightest ones (LPT order). Groups with fewer heads have
    // fewer (longer) chunks; their surplus y exits.
    const int64_t nchunks = (nqb + c.Q - 1) / c.Q;
    if (static_cast<int64_t>(blockIdx.y) >= nchunks) return;
    c.qb0 = (nchunks - 1 - static_cast<int64_t>(blockIdx.y)) * c.Q;
    const int g = ht.kv[c.head(0)];
    const int tid = threadIdx.x;

    for (int f = tid; f < kGrpRows * (kHeadDim / 4); f += kGrpThreads) {
        const int s = f / (kHeadDim / 4), c4 = f % (kHeadDim / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c.valid(s))
            v = __ldg(reinterpret_cast<const float4*>(qp + (static_cast<int64_t>(c.head(s)) * nqb + c.qb(s)) * kHeadDim + c4 * 4));
        *reinterpret_cast<float4*>(Qs + s * kPad + c4 * 4) = v;
    }
    const int64_t vis_max = visible_blocks(min(c.qb0 + c.Q, nqb) - 1, n, nkb, bq, causal != 0);
    // Key split (small launches, select = 0): CTA z scores key chunk z only.
    const int64_t kc_begin = ksplit ? static_cast<int64_t>(blockIdx.z) * kGrpChunk : 0;
    const int64_t kc_stop = ksplit ? min(vis_max, kc_begin + kGrpChunk) : vis_max;
    if (kc_begin >= vis_max) return;
    // Thread (rp, kq): a warp spans 4 consecutive kq (K rows 132 floats = 4
    // banks apart: conflict-free 16-byte loads) and all 8 rp (Q rows, likewise).
    const int rp = tid % kGrpRowStep;
    const int kq = tid / kGrpRowStep;
    const float* kbase = kp + static_cast<int64_t>(g) * nkb * kHeadDim;
    for (int64_t kc = kc_begin; kc < kc_stop; kc += kGrpChunk) {
        const int kc_end = static_cast<int>(min(static_cast<int64_t>(kGrpChunk), vis_max - kc));
        __syncthreads();  // previous chunk consumed (and the Q tile visible)
        {
            const float4* src = reinterpret_cast<const float4*>(kbase + kc * kHeadDim);
            constexpr int kPer = kGrpChunk * (kHeadDim / 4) / kGrpThreads;  // 16 float4 per thread
            float4 t[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int f = tid + u * kGrpThreads;
                t[u] = f / (kHeadDim / 4) < kc_end ? __ldg(src + f) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int f = tid + u * kGrpThreads;
                *reinterpret_cast<float4*>(Ks + (f / (kHeadDim / 4)) * kPad + (f % (kHeadDim / 4)) * 4) = t[u];
            }
        }
        __syncthreads();
        const int nj = kq < kc_end ? min(kGrpKT, (kc_end - kq + kGrpKbStep - 1) / kGrpKbStep) : 0;
        switch (nj) {
            case 4: grp_tile<4>(Qs, Ks, rp, kq, kc, kc_end, scale, c); break;
            case 3: grp_tile<3>(Qs, Ks, rp, kq, kc, kc_end, scale, c); break;
            case 2: grp_tile<2>(Qs, Ks, rp, kq, kc, kc_end, scale, c); break;
            case 1: grp_tile<1>(Qs, Ks, rp, kq, kc, kc_end, scale, c); break;
            default: break;
        }
    }
    if (fill_tail) {  // score-matrix output: -inf past the CTA's last visible block
        for (int s = 0; s < kGrpRows; ++s) {
            if (!c.valid(s)) continue;
            float* dst = scores + (static_cast<int64_t>(c.head(s)) * nqb + c.qb(s)) * nkb;
            for (int64_t kb = vis_max + tid; kb < nkb; kb += kGrpThreads) dst[kb] = -INFINITY;
        }
    }
    if (!select) return;
    __syncthreads();  // this CTA's score rows are written (read back from L2 below)
    const int warp = tid >> 5;
    for (int s = warp; s < kGrpRows; s += kGrpThreads / 32) {
        if (!c.valid(s)) continue;
        const int h = c.head(s);
        const int64_t qb = c.qb(s);
        const int vis = static_cast<int>(visible_blocks(qb, n, nkb, bq, causal != 0));
        const int kk = min(ht.k[h], vis);
        const float* row = scores + (static_cast<int64_t>(h) * nqb + qb) * nkb;
        warp_select_row([row](int j) { return order_key(__ldcg(row + j)); }, vis, kk, kmax,
                        idx + (static_cast<int64_t>(h) * nqb + qb) * kmax, scratch + 32 * warp);
        if ((tid & 31) == 0) cnt[static_cast<int64_t>(h) * nqb + qb] = kk;
    }
}

// Standalone selector: one warp per (head, query block) row of a global score matrix.
__global__ void __launch_bounds__(kSelThreads)
    select_kernel(const float* __restrict__ scores, int hq, int64_t n, int64_t nqb, int64_t nkb,
                  int bq, int causal, HeadTable ht, int64_t kmax, int32_t* __restrict__ idx,
                  int32_t* __restrict__ cnt) {
    __shared__ uint32_t scratch[kSelThreads / 32][32];
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (kSelThreads / 32) + (threadIdx.x >> 5);
    if (row >= (int64_t)hq * nqb) return;
    const int h = static_cast<int>(row / nqb);
    const int64_t qb = row % nqb;
    const int vis = static_cast<int>(visible_blocks(qb, n, nkb, bq, causal != 0));
    const int kk = min(ht.k[h], vis);
    const float* srow = scores + row * nkb;
    warp_select_row([srow](int j) { return order_key(srow[j]); }, vis, kk, kmax, idx + row * kmax,
                    scratch[threadIdx.x >> 5]);
    if ((threadIdx.x & 31) == 0) cnt[row] = kk;
}

__global__ void check_finite_kernel(const uint16_t* __restrict__ x, int64_t count,
                                    int32_t* __restrict__ flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= (x[i] & 0x7F80u) == 0x7F80u;  // bf16 exponent all ones: Inf or NaN
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace

void launch_pool_qk(const void* q, int hq, int bq, const void* k, int hkv, int64_t n, float* qp, float* kp,
                    cudaStream_t s) {
    const int64_t nbq = (n + bq - 1) / bq, nbk = (n + kBlock - 1) / kBlock;
    const int64_t ck = (nbk + bq / kBlock - 1) / (bq / kBlock);  // K CTAs per head
    const unsigned grid = static_cast<unsigned>(nbq * hq + ck * hkv);
    const auto* qb = static_cast<const __nv_bfloat16*>(q);
    const auto* kb = static_cast<const __nv_bfloat16*>(k);
    if (bq == 256)
        pool_qk_kernel<256><<<grid, kPoolThreads, 0, s>>>(qb, nbq, hq, kb, nbk, n, qp, kp);
    else
        pool_qk_kernel<128><<<grid, kPoolThreads, 0, s>>>(qb, nbq, hq, kb, nbk, n, qp, kp);
}

int launch_score_select(const float* qp, const float* kp, int hq, int hkv, int64_t n, int bq,
                         bool causal, float scale, const HeadTable& ht, int64_t kmax,
                         float* scores_out, float* scores_ws, bool select, int32_t* idx, int32_t* cnt,
                         cudaStream_t s) {
    (void)hkv;
    const int64_t nqb = (n + bq - 1) / bq, nkb = (n + kBlock - 1) / kBlock;
    // Row groups: the q heads of each kv head in head order, up to
    // SHPLB_K2_GROUP (default 4; tests vary it) per group.
    static const int max_group = [] {
        const char* e = std::getenv("SHPLB_K2_GROUP");
        const int v = e ? std::atoi(e) : 4;
        return v < 1 ? 1 : (v > 4 ? 4 : v);
    }();
    GroupTable gt{};
    int groups = 0, min_q = kGrpRows;
    {
        int open_kv[kMaxHeads];
        int open_grp[kMaxHeads];
        for (int i = 0; i < kMaxHeads; ++i) open_kv[i] = -1;
        int n_open = 0;
        for (int h = 0; h < hq; ++h) {
            int slot = -1;
            for (int i = 0; i < n_open; ++i)
                if (open_kv[i] == ht.kv[h]) slot = i;
            if (slot < 0 || gt.size[open_grp[slot]] >= max_group) {
                if (slot < 0) slot = n_open++;
                open_kv[slot] = ht.kv[h];
                open_grp[slot] = groups++;
            }
            const int gi = open_grp[slot];
            gt.heads[gi] |= static_cast<uint32_t>(h) << (8 * gt.size[gi]);
            gt.size[gi] += 1;
        }
        for (int gi = 0; gi < groups; ++gi) min_q = std::min(min_q, gt.size[gi] == 1 ? 64 : (gt.size[gi] == 2 ? 32 : 16));
    }
    // The key chunks are split over grid.z and the rows selected by a second
    // kernel (one warp per row): a CTA that walked every visible key chunk made a
    // small launch (one GQA group: a KV-head chunk of the host entry, or one
    // rank's shard) latency-bound by its longest CTA — C3 one kv group 0.124 ->
    // 0.042 ms, a D = 8 rank 0.142 -> 0.046, the whole layer 0.194 -> 0.185
    // (tools/k2_probe.py). Scores are the same fmaf chains either way, so the
    // selection is unchanged. SHPLB_K2_SPLIT=0 keeps the fused single kernel.
    static const int split_env = [] {
        const char* e = std::getenv("SHPLB_K2_SPLIT");
        return e ? std::atoi(e) : -1;
    }();
    const int64_t key_chunks = (nkb + kGrpChunk - 1) / kGrpChunk;
    const bool split = select && !scores_out && key_chunks > 1 && split_env != 0;
    const dim3 grid(static_cast<unsigned>(groups), static_cast<unsigned>((nqb + min_q - 1) / min_q),
                    split ? static_cast<unsigned>(key_chunks) : 1u);
    set_max_dynamic_smem(reinterpret_cast<const void*>(score_select_kernel), static_cast<int>(kGrpSmem));
    score_select_kernel<<<grid, kGrpThreads, kGrpSmem, s>>>(qp, kp, n, nqb, nkb, bq, causal ? 1 : 0, scale, ht, gt,
                                                           kmax, scores_out ? scores_out : scores_ws,
                                                           scores_out ? 1 : 0, (select && !split) ? 1 : 0, idx, cnt,
                                                           split ? 1 : 0);
    if (split) launch_select_from_scores(scores_ws, hq, n, bq, causal, ht, kmax, idx, cnt, s);
    return split ? 2 : 1;  // kernels launched
}

void launch_select_from_scores(const float* scores, int hq, int64_t n, int bq, bool causal,
                               const HeadTable& ht, int64_t kmax, int32_t* idx, int32_t* cnt,
                               cudaStream_t s) {
    const int64_t nqb = (n + bq - 1) / bq, nkb = (n + kBlock - 1) / kBlock;
    const int64_t rows = (int64_t)hq * nqb;
    const unsigned grid = static_cast<unsigned>((rows + (kSelThreads / 32) - 1) / (kSelThreads / 32));
    select_kernel<<<grid, kSelThreads, 0, s>>>(scores, hq, n, nqb, nkb, bq, causal ? 1 : 0, ht, kmax,
                                               idx, cnt);
}

namespace {
// ---- ColumnAggregateTopK at block granularity (attention.cpp:136-148;
// restated in oracle/shplb_oracle.c orc_colagg_select with the same IEEE ops).

// 2^x, x <= 0, by a fixed fp32 polynomial (no MUFU: its result would differ
// from the CPU's), 0 below -126.
__device__ __forceinline__ float det_ex2(float x) {
    if (!(x > -126.0f)) return 0.0f;
    const float t = __fadd_rn(x, 12582912.0f);
    const float j = __fsub_rn(t, 12582912.0f);
    const float f = __fsub_rn(x, j);
    float p = __fmaf_rn(1.3333558e-3f, f, 9.6181291e-3f);
    p = __fmaf_rn(p, f, 5.5504109e-2f);
    p = __fmaf_rn(p, f, 2.4022651e-1f);
    p = __fmaf_rn(p, f, 6.9314718e-1f);
    p = __fmaf_rn(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + static_cast<int>(static_cast<uint32_t>(__float_as_int(t)) << 23));
}

constexpr float kLog2e = 1.44269504088896340736f;

// Per (head, query block), one warp: m = max visible score, z = sum of
// det_ex2((s - m) log2 e) as 32 lane-strided partial sums (coalesced reads)
// added in lane order — the order orc_colagg_select restates.
__global__ void colagg_rowstats_kernel(const float* __restrict__ scores, int hq, int64_t nqb, int64_t nkb,
                                       int64_t n, int bq, int causal, float* __restrict__ m_out,
                                       float* __restrict__ z_out) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= hq * nqb) return;
    const int64_t vis = visible_blocks(row % nqb, n, nkb, bq, causal != 0);
    const float* s = scores + row * nkb;
    float mx = -INFINITY;
    for (int64_t j = lane; j < vis; j += 32) mx = s[j] > mx ? s[j] : mx;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = o > mx ? o : mx;
    }
    float part = 0.0f;
    for (int64_t j = lane; j < vis; j += 32) part = __fadd_rn(part, det_ex2(__fmul_rn(__fsub_rn(s[j], mx), kLog2e)));
    float sum = 0.0f;
#pragma unroll
    for (int l = 0; l < 32; ++l) sum = __fadd_rn(sum, __shfl_sync(0xffffffffu, part, l));
    if (lane == 0) {
        m_out[row] = mx;
        z_out[row] = sum;
    }
}

// Per (head, key block): column sum of the block weights over query blocks, ascending.
__global__ void colagg_colsum_kernel(const float* __restrict__ scores, const float* __restrict__ m,
                                     const float* __restrict__ z, int hq, int64_t nqb, int64_t nkb, int64_t n,
                                     int bq, int causal, float* __restrict__ c_out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= hq * nkb) return;
    const int64_t h = t / nkb, kb = t % nkb;
    float acc = 0.0f;
    for (int64_t qb = 0; qb < nqb; ++qb) {
        if (kb >= visible_blocks(qb, n, nkb, bq, causal != 0)) continue;
        const int64_t row = h * nqb + qb;
        const float w = det_ex2(__fmul_rn(__fsub_rn(scores[row * nkb + kb], m[row]), kLog2e));
        acc = __fadd_rn(acc, __fdiv_rn(w, z[row]));
    }
    c_out[t] = acc;
}

// One warp per head: the k_h key blocks with the largest column sums, ascending.
__global__ void colagg_select_kernel(const float* __restrict__ c, int hq, int64_t nkb, HeadTable ht,
                                     int64_t kmax, int32_t* __restrict__ kept, int32_t* __restrict__ kk_out) {
    __shared__ uint32_t scratch[4][32];  // 128 threads
    const int h = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (h >= hq) return;
    const int kk = static_cast<int>(min(static_cast<int64_t>(ht.k[h]), nkb));
    const float* row = c + static_cast<int64_t>(h) * nkb;
    warp_select_row([row](int j) { return order_key(row[j]); }, static_cast<int>(nkb), kk, kmax,
                    kept + static_cast<int64_t>(h) * kmax, scratch[threadIdx.x >> 5]);
    if ((threadIdx.x & 31) == 0) kk_out[h] = kk;
}

// Per (head, query block): the head's kept blocks the query block can see.
__global__ void colagg_fill_kernel(const int32_t* __restrict__ kept, const int32_t* __restrict__ kk, int hq,
                                   int64_t nqb, int64_t nkb, int64_t kmax, int64_t n, int bq, int causal,
                                   int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= hq * nqb) return;
    const int64_t h = row / nqb;
    const int64_t vis = visible_blocks(row % nqb, n, nkb, bq, causal != 0);
    const int32_t* kr = kept + h * kmax;
    int32_t* out = idx + row * kmax;
    int64_t w = 0;
    for (int64_t j = 0; j < kk[h]; ++j)
        if (kr[j] < vis) out[w++] = kr[j];
    for (int64_t j = w; j < kmax; ++j) out[j] = -1;
    cnt[row] = static_cast<int32_t>(w);
}
}  // namespace

void launch_colagg_select(const float* scores, int hq, int64_t n, int bq, bool causal, const HeadTable& ht,
                          int64_t kmax, float* work, int32_t* kept, int32_t* idx, int32_t* cnt, cudaStream_t s) {
    const int64_t nqb = (n + bq - 1) / bq, nkb = (n + kBlock - 1) / kBlock;
    float* m = work;
    float* z = m + hq * nqb;
    float* c = z + hq * nqb;
    int32_t* kk = kept + hq * kmax;
    const int cz = causal ? 1 : 0;
    colagg_rowstats_kernel<<<static_cast<unsigned>((hq * nqb * 32 + 127) / 128), 128, 0, s>>>(scores, hq, nqb, nkb,
                                                                                              n, bq, cz, m, z);
    colagg_colsum_kernel<<<static_cast<unsigned>((hq * nkb + 127) / 128), 128, 0, s>>>(scores, m, z, hq, nqb,
                                                                                       nkb, n, bq, cz, c);
    colagg_select_kernel<<<static_cast<unsigned>((hq * 32 + 127) / 128), 128, 0, s>>>(c, hq, nkb, ht, kmax, kept,
                                                                                       kk);
    colagg_fill_kernel<<<static_cast<unsigned>((hq * nqb + 127) / 128), 128, 0, s>>>(kept, kk, hq, nqb, nkb, kmax,
                                                                                     n, bq, cz, idx, cnt);
}

size_t colagg_work_floats(int hq, int64_t n, int bq) {
    const int64_t nqb = (n + bq - 1) / bq, nkb = (n + kBlock - 1) / kBlock;
    return static_cast<size_t>(hq) * (2 * nqb + nkb);
}

namespace {
// Dense comparator selection: every causally visible key block, ascending.
__global__ void dense_selection_kernel(int32_t* idx, int32_t* cnt, int64_t rows, int64_t nqb, int64_t nkb,
                                       int bq, int64_t n, int causal) {
    const int64_t row = blockIdx.x;  // (head, query block)
    if (row >= rows) return;
    const int64_t qb = row % nqb;
    const int64_t last = min((qb + 1) * bq, n) - 1;
    const int64_t vis = causal ? min(last / kBlock + 1, nkb) : nkb;
    for (int64_t j = threadIdx.x; j < nkb; j += blockDim.x) idx[row * nkb + j] = j < vis ? static_cast<int32_t>(j) : -1;
    if (threadIdx.x == 0) cnt[row] = static_cast<int32_t>(vis);
}
}  // namespace

void launch_dense_selection(int32_t* idx, int32_t* cnt, int hq, int64_t n, int bq, bool causal, cudaStream_t s) {
    const int64_t nqb = (n + bq - 1) / bq, nkb = (n + kBlock - 1) / kBlock;
    dense_selection_kernel<<<static_cast<unsigned>(hq * nqb), 256, 0, s>>>(idx, cnt, hq * nqb, nqb, nkb, bq, n,
                                                                          causal ? 1 : 0);
}

void launch_check_finite(const void* x, int64_t count, int32_t* flag, cudaStream_t s) {
    check_finite_kernel<<<148 * 8, 256, 0, s>>>(static_cast<const uint16_t*>(x), count, flag);
}

void set_max_dynamic_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> set_to;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    int& cur = set_to[{func, dev}];
    if (bytes > cur && cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
        cur = bytes;
}

}  // namespace shplb::kern
