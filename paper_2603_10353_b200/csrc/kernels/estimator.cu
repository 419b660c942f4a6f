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

// One CTA pools one kRows-row block (128 or 256) of one head. Thread (g, cg)
// sums rows g, g+16, ... (ascending) of columns 8cg..8cg+7 with 16-byte loads
// (all kRows/16 loads in flight); the 16 group partials per column are then
// added in ascending group order.
template <int kRows>
__global__ void __launch_bounds__(kPoolThreads) pool_kernel(const __nv_bfloat16* __restrict__ x,
                                                            int64_t n, float* __restrict__ out) {
    __shared__ float part[kPoolSplit][kHeadDim + 4];
    const int64_t b = blockIdx.x;
    const int64_t head = blockIdx.y;
    const int64_t nb = gridDim.x;
    const int g = threadIdx.x >> 4;
    const int cg = threadIdx.x & 15;
    const int64_t t0 = b * kRows;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kRows), n - t0));
    const __nv_bfloat16* base = x + (head * n + t0) * kHeadDim + cg * 8;

    uint4 v[kRows / kPoolSplit];
#pragma unroll
    for (int s = 0; s < kRows / kPoolSplit; ++s) {
        const int t = g + s * kPoolSplit;
        v[s] = t < cnt ? __ldg(reinterpret_cast<const uint4*>(base + static_cast<int64_t>(t) * kHeadDim))
                       : make_uint4(0, 0, 0, 0);
    }
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
#pragma unroll
    for (int s = 0; s < kRows / kPoolSplit; ++s) {
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
    for (int e = 0; e < 8; ++e) part[g][cg * 8 + e] = acc[e];
    __syncthreads();
    if (threadIdx.x < kHeadDim) {
        const int c = threadIdx.x;
        float total = 0.0f;
#pragma unroll
        for (int gg = 0; gg < kPoolSplit; ++gg) total = __fadd_rn(total, part[gg][c]);
        out[(head * nb + b) * kHeadDim + c] = __fdiv_rn(total, static_cast<float>(cnt));
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
__device__ void warp_select_row(KeyAt key_at, int vis, int kk, int64_t kmax, int32_t* __restrict__ idx_row) {
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
    uint32_t T = 0;
    for (int bit = 31; bit >= 0; --bit) {
        const uint32_t trial = T | (1u << bit);
        const int c = count_ge(trial);
        if (c >= kk) {
            T = trial;
            if (c == kk) break;
        }
    }
    const int gt = T == 0xFFFFFFFFu ? 0 : count_ge(T + 1);  // keys > T
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

constexpr int kSelThreads = 256;  // 8 warps
constexpr int kRowsPerCta = 16;   // query blocks per CTA
constexpr int kPad = kHeadDim + 4;  // row stride (floats) of the Q / K tiles: 16-byte rows, no bank conflicts

// One CTA: head h, query blocks [qb0, qb0+16). Scores for all visible key
// blocks are built in shared memory with an FFMA register tile of kRT rows x
// kKT key blocks per thread (rows strided 16/kRT apart, key blocks kChunk/kKT
// apart; per 4 columns kRT + kKT float4 loads feed kRT*kKT*4 FFMAs; every dot
// product is one fmaf chain over c = 0..127 in order, so the tile shape never
// changes a score), then converted once to order keys, then each warp selects
// two rows. Two shapes: 4 x 4 over 256-block chunks (8 FFMA per float loaded
// from shared memory; needs the 135 KB chunk, so rows of up to 1390 key
// blocks), and 2 x 2 over 64-block chunks for longer rows.
template <int kRT, int kKT, int kChunk>
__global__ void __launch_bounds__(kSelThreads)
    score_select_kernel(const float* __restrict__ qp, const float* __restrict__ kp, int hq,
                        int hkv, int64_t n, int64_t nqb, int64_t nkb, int bq, int causal, float scale,
                        HeadTable ht, int64_t kmax, float* __restrict__ scores_out, int select,
                        int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
    static_assert((kRowsPerCta / kRT) * (kChunk / kKT) == kSelThreads, "one thread per register tile");
    constexpr int kRowStep = kRowsPerCta / kRT;  // threads along rows
    constexpr int kKbStep = kChunk / kKT;        // threads along key blocks
    extern __shared__ __align__(16) float smem[];
    float* Qs = smem;                     // [16 rows][kPad]
    float* Ks = Qs + kRowsPerCta * kPad;  // [kChunk key blocks][kPad]
    float* S = Ks + kChunk * kPad;        // [16 rows][nkb_pad]
    const int64_t nkb_pad = (nkb + 3) & ~int64_t(3);

    // Grid (heads, row chunks): the hardware hands out CTAs head-fastest, and
    // chunk y = 0 is the LAST chunk of query blocks, so under the causal mask
    // the heaviest chunks (most visible key blocks) of every head go first and
    // the launch tail is made of the lightest ones (LPT order).
    const int h = blockIdx.x;
    const int g = ht.kv[h];
    const int64_t qb0 = static_cast<int64_t>(gridDim.y - 1 - blockIdx.y) * kRowsPerCta;
    const int rows = static_cast<int>(min(static_cast<int64_t>(kRowsPerCta), nqb - qb0));
    const int tid = threadIdx.x;

    // Q tile (row-major, float4).
    for (int f = tid; f < kRowsPerCta * (kHeadDim / 4); f += kSelThreads) {
        const int r = f / (kHeadDim / 4), c4 = f % (kHeadDim / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < rows) v = *reinterpret_cast<const float4*>(qp + ((int64_t)h * nqb + qb0 + r) * kHeadDim + c4 * 4);
        *reinterpret_cast<float4*>(Qs + r * kPad + c4 * 4) = v;
    }
    const int64_t vis_max = visible_blocks(qb0 + rows - 1, n, nkb, bq, causal != 0);

    // Thread (rp, kq): rows rp + kRowStep*i, key blocks kq + kKbStep*j. A warp
    // spans 32/kRowStep consecutive kq, whose K rows (stride 132 floats = 4
    // banks) are conflict-free, and kRowStep rows of Q (broadcast).
    const int rp = tid % kRowStep;
    const int kq = tid / kRowStep;
    // The next chunk's pooled K rows are fetched into registers while the
    // current chunk is multiplied (one CTA per SM leaves few warps to hide the
    // L2 latency of a synchronous load), then stored to shared memory.
    constexpr int kLoads = kChunk * (kHeadDim / 4) / kSelThreads;  // float4 per thread per chunk
    float4 pre[kLoads];
    auto fetch = [&](int64_t kc) {
        const int64_t kc_end = min(static_cast<int64_t>(kChunk), vis_max - kc);
#pragma unroll
        for (int u = 0; u < kLoads; ++u) {
            const int f = tid + u * kSelThreads;
            const int kb = f / (kHeadDim / 4), c4 = f % (kHeadDim / 4);
            pre[u] = kb < kc_end ? __ldg(reinterpret_cast<const float4*>(kp + ((int64_t)g * nkb + kc + kb) * kHeadDim + c4 * 4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    if (vis_max > 0) fetch(0);
    for (int64_t kc = 0; kc < vis_max; kc += kChunk) {
        __syncthreads();  // previous chunk fully consumed (and Q tile visible)
        const int64_t kc_end = min(static_cast<int64_t>(kChunk), vis_max - kc);  // rows worth loading
#pragma unroll
        for (int u = 0; u < kLoads; ++u) {
            const int f = tid + u * kSelThreads;
            const int kb = f / (kHeadDim / 4), c4 = f % (kHeadDim / 4);
            *reinterpret_cast<float4*>(Ks + kb * kPad + c4 * 4) = pre[u];
        }
        __syncthreads();
        if (kc + kChunk < vis_max) fetch(kc + kChunk);
        if (kq >= kc_end) continue;  // none of this thread's key blocks is visible (kq is the smallest)
        float a[kRT][kKT];
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
            for (int j = 0; j < kKT; ++j) a[i][j] = 0.f;
        const float* q0p = Qs + rp * kPad;
        const float* k0p = Ks + kq * kPad;
#pragma unroll 2
        for (int c4 = 0; c4 < kHeadDim / 4; ++c4) {
            float4 qv[kRT], kv[kKT];
#pragma unroll
            for (int i = 0; i < kRT; ++i) qv[i] = *reinterpret_cast<const float4*>(q0p + i * kRowStep * kPad + c4 * 4);
#pragma unroll
            for (int j = 0; j < kKT; ++j) kv[j] = *reinterpret_cast<const float4*>(k0p + j * kKbStep * kPad + c4 * 4);
#pragma unroll
            for (int i = 0; i < kRT; ++i)
#pragma unroll
                for (int j = 0; j < kKT; ++j) {
                    a[i][j] = __fmaf_rn(qv[i].x, kv[j].x, a[i][j]);
                    a[i][j] = __fmaf_rn(qv[i].y, kv[j].y, a[i][j]);
                    a[i][j] = __fmaf_rn(qv[i].z, kv[j].z, a[i][j]);
                    a[i][j] = __fmaf_rn(qv[i].w, kv[j].w, a[i][j]);
                }
        }
#pragma unroll
        for (int i = 0; i < kRT; ++i) {
            const int r = rp + kRowStep * i;
            const int64_t vis = visible_blocks(qb0 + r, n, nkb, bq, causal != 0);
#pragma unroll
            for (int j = 0; j < kKT; ++j) {
                const int64_t kb = kc + kq + kKbStep * j;
                if (kb < nkb) S[r * nkb_pad + kb] = kb < vis ? __fmul_rn(a[i][j], scale) : -INFINITY;
            }
        }
    }
    __syncthreads();

    if (scores_out) {
        for (int r = 0; r < rows; ++r) {
            float* dst = scores_out + ((int64_t)h * nqb + qb0 + r) * nkb;
            for (int64_t kb = tid; kb < nkb; kb += kSelThreads)
                dst[kb] = kb < vis_max ? S[r * nkb_pad + kb] : -INFINITY;
        }
    }
    if (!select) return;
    // Scores -> order keys in place, once (the bisection reads each key 33 times).
    uint32_t* Kk = reinterpret_cast<uint32_t*>(S);
    for (int r = 0; r < rows; ++r)
        for (int64_t kb = tid; kb < vis_max; kb += kSelThreads) Kk[r * nkb_pad + kb] = order_key(S[r * nkb_pad + kb]);
    __syncthreads();
    const int warp = tid >> 5;
    for (int r = warp; r < rows; r += kSelThreads / 32) {
        const int64_t qb = qb0 + r;
        const int vis = static_cast<int>(visible_blocks(qb, n, nkb, bq, causal != 0));
        const int kk = min(ht.k[h], vis);
        const uint32_t* keys = Kk + r * nkb_pad;
        warp_select_row([keys](int j) { return keys[j]; }, vis, kk, kmax, idx + ((int64_t)h * nqb + qb) * kmax);
        if ((tid & 31) == 0) cnt[(int64_t)h * nqb + qb] = kk;
    }
}

// Standalone selector: one warp per (head, query block) row of a global score matrix.
__global__ void __launch_bounds__(kSelThreads)
    select_kernel(const float* __restrict__ scores, int hq, int64_t n, int64_t nqb, int64_t nkb,
                  int bq, int causal, HeadTable ht, int64_t kmax, int32_t* __restrict__ idx,
                  int32_t* __restrict__ cnt) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (kSelThreads / 32) + (threadIdx.x >> 5);
    if (row >= (int64_t)hq * nqb) return;
    const int h = static_cast<int>(row / nqb);
    const int64_t qb = row % nqb;
    const int vis = static_cast<int>(visible_blocks(qb, n, nkb, bq, causal != 0));
    const int kk = min(ht.k[h], vis);
    const float* srow = scores + row * nkb;
    warp_select_row([srow](int j) { return order_key(srow[j]); }, vis, kk, kmax, idx + row * kmax);
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

void launch_pool(const void* x, int heads, int64_t n, int rows, float* out, cudaStream_t s) {
    const int64_t nb = (n + rows - 1) / rows;
    const dim3 grid(static_cast<unsigned>(nb), heads);
    if (rows == 256)
        pool_kernel<256><<<grid, kPoolThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(x), n, out);
    else
        pool_kernel<128><<<grid, kPoolThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(x), n, out);
}

static size_t score_select_smem(int64_t nkb, int chunk) {
    const int64_t nkb_pad = (nkb + 3) & ~int64_t(3);
    return sizeof(float) * (kPad * kRowsPerCta + kPad * chunk + kRowsPerCta * nkb_pad);
}
constexpr size_t kSmemOptIn = 227 * 1024;

void launch_score_select(const float* qp, const float* kp, int hq, int hkv, int64_t n, int bq,
                         bool causal, float scale, const HeadTable& ht, int64_t kmax,
                         float* scores_out, bool select, int32_t* idx, int32_t* cnt,
                         cudaStream_t s) {
    const int64_t nqb = (n + bq - 1) / bq, nkb = (n + kBlock - 1) / kBlock;
    const dim3 grid(static_cast<unsigned>(hq), static_cast<unsigned>((nqb + kRowsPerCta - 1) / kRowsPerCta));
    const size_t wide = score_select_smem(nkb, 256);
    static const bool force_narrow = std::getenv("SHPLB_K2_NARROW") != nullptr;  // tests: exercise the 2 x 2 shape
    if (wide <= kSmemOptIn && !force_narrow) {  // 4 x 4 register tile over 256-block chunks
        auto* k = score_select_kernel<4, 4, 256>;
        set_max_dynamic_smem(reinterpret_cast<const void*>(k), static_cast<int>(wide));
        k<<<grid, kSelThreads, wide, s>>>(qp, kp, hq, hkv, n, nqb, nkb, bq, causal ? 1 : 0, scale, ht, kmax,
                                         scores_out, select ? 1 : 0, idx, cnt);
    } else {  // long rows: 2 x 2 over 64-block chunks leaves room for the score rows
        const size_t smem = score_select_smem(nkb, 64);
        auto* k = score_select_kernel<2, 2, 64>;
        set_max_dynamic_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
        k<<<grid, kSelThreads, smem, s>>>(qp, kp, hq, hkv, n, nqb, nkb, bq, causal ? 1 : 0, scale, ht, kmax,
                                         scores_out, select ? 1 : 0, idx, cnt);
    }
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
    const int h = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (h >= hq) return;
    const int kk = static_cast<int>(min(static_cast<int64_t>(ht.k[h]), nkb));
    const float* row = c + static_cast<int64_t>(h) * nkb;
    warp_select_row([row](int j) { return order_key(row[j]); }, static_cast<int>(nkb), kk, kmax,
                    kept + static_cast<int64_t>(h) * kmax);
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
