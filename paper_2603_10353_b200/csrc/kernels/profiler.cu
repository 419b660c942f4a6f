// GPU recovery-curve profiler: the offline input of the
// per-head budget table, moved from the host to the B200.
//
// Restates build_profiles + recovery_ratio for PerQueryTopK
// (proj/src/profiler.cpp:157-196, proj/src/attention.cpp:151-184): for every
// calibration row of every head, the dense softmax weights over all n_k keys
// (dense_attention, attention.cpp:84-114: max-subtracted, fp64), then at each
// grid budget k the mass of the k largest weights, averaged over rows.
//
//   P1 profile_scores_kernel  s[unit][j] = (q_i . k_j) / sqrt(d) in fp64. bf16
//      operands are exact in fp64 and each DFMA rounds once, so the dot is the
//      reference's fp64 dot up to summation order (exact for bf16 data whose
//      products span < 53 bits). A 128-key tile of K is staged transposed in
//      shared memory and reused by every calibration row of the GQA group.
//   P2 segmented radix sort of each unit's scores, descending (CUB, the one
//      library primitive here; the weights are a monotone map of the scores,
//      so sorting scores sorts weights).
//   P3 profile_prefix_kernel  one CTA per unit: Z = sum exp(s - s_max) and the
//      running top-k mass at every grid point (block scan in fp64).
//   P4 profile_rows_kernel    recovery[h][g] = sum over rows (ascending) / rows.
//
// Results agree with the host restatement and the reference to rounding
// (the reference itself sums the top-k in nth_element's arbitrary order).
#include <algorithm>
#include <cstdint>

#include <cub/device/device_segmented_radix_sort.cuh>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace shplb::kern {
namespace {

constexpr int kProfKeys = 128;     // keys per P1 tile
constexpr int kProfRows = 16;      // calibration rows per P1 pass over the tile
constexpr int kProfThreads = 256;  // P1: thread = key (t % 128), rows t/128 + 2i
constexpr int kPrefixThreads = 1024;

__global__ void __launch_bounds__(kProfThreads) profile_scores_kernel(
    const __nv_bfloat16* __restrict__ q_rows, const __nv_bfloat16* __restrict__ k, int hq, int hkv,
    int64_t n_rows, int64_t n_k, double scale, double* __restrict__ scores) {
    // Dynamic shared memory: K tile transposed kt[c][key] (padded rows), then
    // the current batch of query rows qs[row][c]; fp64 (bf16 is exact in it).
    extern __shared__ double prof_smem[];
    auto kt = reinterpret_cast<double(*)[kProfKeys + 1]>(prof_smem);
    auto qs = reinterpret_cast<double(*)[kHeadDim]>(prof_smem + kHeadDim * (kProfKeys + 1));
    const int g = blockIdx.y;
    const int64_t key0 = static_cast<int64_t>(blockIdx.x) * kProfKeys;
    const int group = hq / hkv;
    // Stage K[g][key0 .. key0+128) transposed (16-byte loads: 8 bf16 per thread step).
    for (int e = threadIdx.x; e < kProfKeys * (kHeadDim / 8); e += kProfThreads) {
        const int key = e / (kHeadDim / 8), c8 = (e % (kHeadDim / 8)) * 8;
        uint4 w = make_uint4(0, 0, 0, 0);
        if (key0 + key < n_k)
            w = *reinterpret_cast<const uint4*>(k + (static_cast<int64_t>(g) * n_k + key0 + key) * kHeadDim + c8);
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&w);
#pragma unroll
        for (int u = 0; u < 8; ++u) kt[c8 + u][key] = static_cast<double>(__bfloat162float(b[u]));
    }
    const int key = threadIdx.x % kProfKeys;
    const int64_t rows_total = static_cast<int64_t>(group) * n_rows;  // q heads g*group.. , all rows
    for (int64_t r0 = 0; r0 < rows_total; r0 += kProfRows) {
        __syncthreads();
        for (int e = threadIdx.x; e < kProfRows * kHeadDim; e += kProfThreads) {
            const int64_t r = r0 + e / kHeadDim;
            const int c = e % kHeadDim;
            double x = 0.0;
            if (r < rows_total) {
                const int64_t unit = static_cast<int64_t>(g) * group * n_rows + r;  // = h*n_rows + i
                x = static_cast<double>(__bfloat162float(q_rows[unit * kHeadDim + c]));
            }
            qs[e / kHeadDim][c] = x;
        }
        __syncthreads();
        if (key0 + key >= n_k) continue;
        for (int rr = threadIdx.x / kProfKeys; rr < kProfRows; rr += kProfThreads / kProfKeys) {
            const int64_t r = r0 + rr;
            if (r >= rows_total) break;
            double acc = 0.0;
#pragma unroll 16
            for (int c = 0; c < kHeadDim; ++c) acc = fma(qs[rr][c], kt[c][key], acc);
            const int64_t unit = static_cast<int64_t>(g) * group * n_rows + r;
            scores[unit * n_k + key0 + key] = acc * scale;
        }
    }
}

// Per unit (one CTA): sorted-descending scores s -> mass[unit][g] = (sum of the
// first grid[g] weights) where weight = exp(s - s[0]) / Z.
__global__ void __launch_bounds__(kPrefixThreads) profile_prefix_kernel(
    const double* __restrict__ sorted, int64_t n_k, const int64_t* __restrict__ grid, int64_t n_grid,
    double* __restrict__ mass) {
    __shared__ double part[kPrefixThreads];
    const int64_t unit = blockIdx.x;
    const double* s = sorted + unit * n_k;
    const double m = s[0];
    const int64_t per = (n_k + kPrefixThreads - 1) / kPrefixThreads;
    const int64_t lo = threadIdx.x * per, hi = min(lo + per, n_k);
    double local = 0.0;
    for (int64_t i = lo; i < hi; ++i) local += exp(s[i] - m);
    part[threadIdx.x] = local;
    __syncthreads();
    // Exclusive scan of the per-thread sums (Hillis-Steele on a copy; fp64).
    for (int off = 1; off < kPrefixThreads; off <<= 1) {
        const double add = threadIdx.x >= off ? part[threadIdx.x - off] : 0.0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    const double z = part[kPrefixThreads - 1];
    double run = part[threadIdx.x] - local;  // exclusive prefix
    const double inv = 1.0 / z;
    // First grid point past lo (grid is strictly increasing; entries are counts).
    int64_t a = 0, b = n_grid;
    while (a < b) {
        const int64_t mid = (a + b) / 2;
        if (grid[mid] <= lo) a = mid + 1; else b = mid;
    }
    int64_t gi = a;
    if (threadIdx.x == 0 && n_grid > 0 && grid[0] == 0) mass[unit * n_grid] = 0.0;
    for (int64_t i = lo; i < hi && gi < n_grid; ++i) {
        run += exp(s[i] - m);
        if (grid[gi] == i + 1) {
            mass[unit * n_grid + gi] = run * inv;
            ++gi;
        }
    }
}

// ColumnAggregateTopK: scores of each unit (row) -> softmax weights in place
// (one CTA per row: max, Z = sum exp(s - max), w = exp(s - max) / Z).
__global__ void __launch_bounds__(kPrefixThreads) profile_weights_kernel(double* __restrict__ scores, int64_t n_k) {
    __shared__ double red[kPrefixThreads];
    double* s = scores + static_cast<int64_t>(blockIdx.x) * n_k;
    double m = -INFINITY;
    for (int64_t j = threadIdx.x; j < n_k; j += kPrefixThreads) m = fmax(m, s[j]);
    red[threadIdx.x] = m;
    __syncthreads();
    for (int off = kPrefixThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + off]);
        __syncthreads();
    }
    m = red[0];
    __syncthreads();
    double z = 0.0;
    for (int64_t j = threadIdx.x; j < n_k; j += kPrefixThreads) z += exp(s[j] - m);
    red[threadIdx.x] = z;
    __syncthreads();
    for (int off = kPrefixThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
        __syncthreads();
    }
    const double inv = 1.0 / red[0];
    for (int64_t j = threadIdx.x; j < n_k; j += kPrefixThreads) s[j] = exp(s[j] - m) * inv;
}

// Column sums per head over its rows, rows ascending (column_sums, attention.cpp:66-73).
__global__ void profile_colsum_kernel(const double* __restrict__ w, int heads, int64_t n_rows, int64_t n_k,
                                      double* __restrict__ col) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(heads) * n_k) return;
    const int64_t h = t / n_k, j = t % n_k;
    double acc = 0.0;
    for (int64_t i = 0; i < n_rows; ++i) acc += w[(h * n_rows + i) * n_k + j];
    col[t] = acc;
}

// Per head (one CTA): sorted-descending column sums -> recovery at every grid
// point = prefix sum / rows.
__global__ void __launch_bounds__(kPrefixThreads) profile_colagg_prefix_kernel(
    const double* __restrict__ sorted, int64_t n_k, const int64_t* __restrict__ grid, int64_t n_grid,
    double inv_rows, double* __restrict__ recovery) {
    __shared__ double part[kPrefixThreads];
    const int64_t head = blockIdx.x;
    const double* s = sorted + head * n_k;
    const int64_t per = (n_k + kPrefixThreads - 1) / kPrefixThreads;
    const int64_t lo = threadIdx.x * per, hi = min(lo + per, n_k);
    double local = 0.0;
    for (int64_t i = lo; i < hi; ++i) local += s[i];
    part[threadIdx.x] = local;
    __syncthreads();
    for (int off = 1; off < kPrefixThreads; off <<= 1) {
        const double add = threadIdx.x >= off ? part[threadIdx.x - off] : 0.0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    double run = part[threadIdx.x] - local;
    int64_t a = 0, b = n_grid;
    while (a < b) {
        const int64_t mid = (a + b) / 2;
        if (grid[mid] <= lo) a = mid + 1; else b = mid;
    }
    int64_t gi = a;
    if (threadIdx.x == 0 && n_grid > 0 && grid[0] == 0) recovery[head * n_grid] = 0.0;
    for (int64_t i = lo; i < hi && gi < n_grid; ++i) {
        run += s[i];
        if (grid[gi] == i + 1) {
            recovery[head * n_grid + gi] = run * inv_rows;
            ++gi;
        }
    }
}

__global__ void profile_rows_kernel(const double* __restrict__ mass, int hq, int64_t n_rows,
                                    const int64_t* __restrict__ grid, int64_t n_grid,
                                    double* __restrict__ recovery) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(hq) * n_grid) return;
    const int64_t h = t / n_grid, gi = t % n_grid;
    double total = 0.0;
    for (int64_t i = 0; i < n_rows; ++i) total += mass[(h * n_rows + i) * n_grid + gi];
    recovery[t] = grid[gi] == 0 ? 0.0 : total / static_cast<double>(n_rows);
}

__global__ void segment_offsets_kernel(int64_t* off, int64_t units, int64_t n_k) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t <= units) off[t] = t * n_k;
}

// ---- Block-selection recovery (the kernels' own policy) --------------------
//
// The curve the layer actually realises: for calibration row i at position
// pos (causal: keys j <= pos), kernel 2 keeps the k highest-scoring 128-key
// blocks of i's query block (pooled fp32 scores, (score desc, index asc),
// among the blocks visible to the query block). recovery(k) = the fraction of
// row i's exact softmax mass (fp64, max-subtracted as attention.cpp:35-49)
// inside those k blocks — recovery_ratio's "mass of the kept set"
// (attention.cpp:151-184) with the kept set chosen by the block selector
// instead of per-token top-k. Budgets in tokens map to ceil(b / 128) blocks,
// as budgets_to_blocks does for the layer call.

constexpr int kBlockProfThreads = 1024;

__device__ __forceinline__ uint32_t prof_order_key(float s) {  // = estimator.cu order_key
    const uint32_t u = __float_as_uint(__fadd_rn(s, 0.0f));
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ double block_reduce_sum(double v, double* red) {
    // fixed order: warp xor-tree, then warp partials ascending by one thread
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kBlockProfThreads / 32; ++w) t += red[w];
        red[32] = t;
    }
    __syncthreads();
    return red[32];
}

__device__ __forceinline__ double block_reduce_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = -INFINITY;
        for (int w = 0; w < kBlockProfThreads / 32; ++w) t = fmax(t, red[w]);
        red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// One CTA per (head, calibration row) of a kv batch. scores: fp64 token scores
// of the batch's units [units][n] (unit = local head * n_rows + r); bscores:
// kernel 2's fp32 block-score matrix [hq][nqb][nkb] (-inf where invisible).
// Dynamic smem: keys u64[max(P, threads)] (reused as the scan scratch), mass
// double[P] (P = next power of two >= nkb).
__global__ void __launch_bounds__(kBlockProfThreads) profile_block_kernel(
    const double* __restrict__ scores, const float* __restrict__ bscores, const int64_t* __restrict__ rows,
    int h0, int64_t n_rows, int64_t n, int64_t nqb, int64_t nkb, int bq, int causal, int pow2,
    const int64_t* __restrict__ grid, int64_t n_grid, double* __restrict__ mass_out) {
    extern __shared__ __align__(16) unsigned char bp_smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(bp_smem);
    double* mass = reinterpret_cast<double*>(keys + max(pow2, kBlockProfThreads));
    __shared__ double red[33];
    const int64_t unit = blockIdx.x;
    const int h = h0 + static_cast<int>(unit / n_rows);
    const int64_t r = unit % n_rows;
    const int64_t pos = rows[r];
    const double* s = scores + unit * n;
    const int64_t tok_end = causal ? pos + 1 : n;
    const int64_t qb = pos / bq;
    const int64_t vis = causal ? min((min((qb + 1) * bq, n) - 1) / kBlock + 1, nkb) : nkb;

    double m = -INFINITY;
    for (int64_t j = threadIdx.x; j < tok_end; j += kBlockProfThreads) m = fmax(m, s[j]);
    m = block_reduce_max(m, red);
    // Unnormalised mass of every key block: warp w sums blocks w, w + 32, ...
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t b = warp; b < pow2; b += kBlockProfThreads / 32) {
        double e = 0.0;
        if (b < nkb) {
            for (int i = 0; i < kBlock / 32; ++i) {
                const int64_t j = b * kBlock + i * 32 + lane;
                if (j < tok_end) e += exp(s[j] - m);
            }
            for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        if (lane == 0) mass[b] = e;
    }
    __syncthreads();
    double zpart = 0.0;
    for (int64_t b = threadIdx.x; b < nkb; b += kBlockProfThreads) zpart += mass[b];
    const double inv_z = 1.0 / block_reduce_sum(zpart, red);
    // Rank keys of the row's query block: (order key << 32) | ~index, so a
    // descending sort is (score desc, index asc); invisible blocks sort last.
    const float* brow = bscores + (static_cast<int64_t>(h) * nqb + qb) * nkb;
    for (int64_t b = threadIdx.x; b < pow2; b += kBlockProfThreads) {
        keys[b] = b < vis ? (static_cast<uint64_t>(prof_order_key(brow[b])) << 32) |
                                static_cast<uint64_t>(0xFFFFFFFFu - static_cast<uint32_t>(b))
                          : 0ull;
    }
    __syncthreads();
    // Bitonic sort, descending by key, masses carried along.
    for (int size = 2; size <= pow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < pow2 / 2; t += kBlockProfThreads) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const uint64_t a = keys[lo], c = keys[hi];
                if ((a < c) == desc) {
                    keys[lo] = c;
                    keys[hi] = a;
                    const double x = mass[lo];
                    mass[lo] = mass[hi];
                    mass[hi] = x;
                }
            }
            __syncthreads();
        }
    }
    // Inclusive prefix of the ranked masses, serial per thread chunk then a
    // fixed-order scan of the chunk totals.
    const int per = (pow2 + kBlockProfThreads - 1) / kBlockProfThreads;
    const int lo = threadIdx.x * per, hi = min(lo + per, pow2);
    double local = 0.0;
    for (int i = lo; i < hi; ++i) local += mass[i];
    __syncthreads();
    double* part = reinterpret_cast<double*>(keys);  // keys are no longer needed
    part[threadIdx.x] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = 0.0;
        for (int t = 0; t < kBlockProfThreads; ++t) {
            const double x = part[t];
            part[t] = run;
            run += x;
        }
    }
    __syncthreads();
    double run = part[threadIdx.x];
    for (int i = lo; i < hi; ++i) {
        run += mass[i];
        mass[i] = run;
    }
    __syncthreads();
    for (int64_t gi = threadIdx.x; gi < n_grid; gi += kBlockProfThreads) {
        const int64_t kb = min((grid[gi] + kBlock - 1) / kBlock, vis);
        mass_out[(static_cast<int64_t>(h) * n_rows + r) * n_grid + gi] = kb == 0 ? 0.0 : fmin(mass[kb - 1] * inv_z, 1.0);
    }
}

__global__ void gather_rows_kernel(const uint4* __restrict__ q, const int64_t* __restrict__ rows, int hq,
                                   int64_t n, int64_t n_rows, uint4* __restrict__ out) {
    constexpr int kVec = kHeadDim * 2 / 16;  // 16-byte vectors per row
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(hq) * n_rows * kVec) return;
    const int64_t v = t % kVec, u = t / kVec, h = u / n_rows, r = u % n_rows;
    out[t] = q[(h * n + rows[r]) * kVec + v];
}

}  // namespace

void launch_gather_rows(const void* q, const int64_t* rows, int hq, int64_t n, int64_t n_rows, void* out,
                        cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(hq) * n_rows * (kHeadDim * 2 / 16);
    gather_rows_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        static_cast<const uint4*>(q), rows, hq, n, n_rows, static_cast<uint4*>(out));
}

void launch_profile_block(const double* scores, const float* bscores, const int64_t* rows, int h0, int heads,
                          int64_t n_rows, int64_t n, int bq, bool causal, const int64_t* grid, int64_t n_grid,
                          double* mass, cudaStream_t s) {
    const int64_t nkb = (n + kBlock - 1) / kBlock, nqb = (n + bq - 1) / bq;
    int pow2 = 1;
    while (pow2 < nkb) pow2 <<= 1;
    pow2 = max(pow2, 2);
    const size_t smem = static_cast<size_t>(std::max(pow2, kBlockProfThreads)) * sizeof(uint64_t) +
                        static_cast<size_t>(pow2) * sizeof(double);
    set_max_dynamic_smem(reinterpret_cast<const void*>(profile_block_kernel), static_cast<int>(smem));
    profile_block_kernel<<<static_cast<unsigned>(static_cast<int64_t>(heads) * n_rows), kBlockProfThreads, smem, s>>>(
        scores, bscores, rows, h0, n_rows, n, nqb, nkb, bq, causal ? 1 : 0, pow2, grid, n_grid, mass);
}

void launch_profile_scores(const void* q_rows, const void* k, int hq, int hkv, int64_t n_rows,
                           int64_t n_k, double scale, double* scores, cudaStream_t s) {
    constexpr size_t smem = sizeof(double) * (kHeadDim * (kProfKeys + 1) + kProfRows * kHeadDim);
    set_max_dynamic_smem(reinterpret_cast<const void*>(profile_scores_kernel), static_cast<int>(smem));
    const dim3 grid(static_cast<unsigned>((n_k + kProfKeys - 1) / kProfKeys), static_cast<unsigned>(hkv));
    profile_scores_kernel<<<grid, kProfThreads, smem, s>>>(static_cast<const __nv_bfloat16*>(q_rows),
                                                        static_cast<const __nv_bfloat16*>(k), hq, hkv, n_rows,
                                                        n_k, scale, scores);
}

size_t profile_sort_temp_bytes(int64_t units, int64_t n_k) {
    size_t bytes = 0;
    cub::DeviceSegmentedRadixSort::SortKeysDescending(nullptr, bytes, static_cast<const double*>(nullptr),
                                                      static_cast<double*>(nullptr), units * n_k,
                                                      static_cast<int64_t>(units),
                                                      static_cast<const int64_t*>(nullptr),
                                                      static_cast<const int64_t*>(nullptr));
    return bytes;
}

void launch_profile_sort(const double* in, double* out, int64_t units, int64_t n_k, int64_t* offsets,
                         void* temp, size_t temp_bytes, cudaStream_t s) {
    segment_offsets_kernel<<<static_cast<unsigned>((units + 256) / 256), 256, 0, s>>>(offsets, units, n_k);
    cub::DeviceSegmentedRadixSort::SortKeysDescending(temp, temp_bytes, in, out, units * n_k,
                                                      static_cast<int64_t>(units), offsets, offsets + 1, 0,
                                                      64, s);
}

void launch_profile_prefix(const double* sorted, int64_t units, int64_t n_k, const int64_t* grid,
                           int64_t n_grid, double* mass, cudaStream_t s) {
    profile_prefix_kernel<<<static_cast<unsigned>(units), kPrefixThreads, 0, s>>>(sorted, n_k, grid, n_grid,
                                                                                  mass);
}

void launch_profile_rows(const double* mass, int hq, int64_t n_rows, const int64_t* grid, int64_t n_grid,
                         double* recovery, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(hq) * n_grid;
    profile_rows_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(mass, hq, n_rows, grid, n_grid,
                                                                              recovery);
}

}  // namespace shplb::kern

namespace shplb::kern {

void launch_profile_colagg(double* scores, int heads, int64_t n_rows, int64_t n_k, double* col, double* sorted,
                           int64_t* offsets, void* temp, size_t temp_bytes, const int64_t* grid, int64_t n_grid,
                           double* recovery, cudaStream_t s) {
    profile_weights_kernel<<<static_cast<unsigned>(heads * n_rows), kPrefixThreads, 0, s>>>(scores, n_k);
    const int64_t cols = static_cast<int64_t>(heads) * n_k;
    profile_colsum_kernel<<<static_cast<unsigned>((cols + 255) / 256), 256, 0, s>>>(scores, heads, n_rows, n_k, col);
    launch_profile_sort(col, sorted, heads, n_k, offsets, temp, temp_bytes, s);
    profile_colagg_prefix_kernel<<<static_cast<unsigned>(heads), kPrefixThreads, 0, s>>>(
        sorted, n_k, grid, n_grid, 1.0 / static_cast<double>(n_rows), recovery);
}

}  // namespace shplb::kern
