// Internal launch interface between the C ABI (shplb_api.cpp) and the sm_100a
// kernels. Host-callable, CUDA-runtime types only.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace shplb::kern {

constexpr int kHeadDim = 128;   // d
constexpr int kBlock = 128;     // bq = bk
constexpr int kPoolSplit = 16;  // interleaved row groups of the pooled sum
constexpr int kMaxHeads = 256;  // per-launch k-block table lives in the kernel parameters
constexpr int kMaxSelected = 2048;  // selected key blocks per query tile staged in smem (256K tokens)
constexpr int kMaxPeers = 8;        // output buffers kernel 3 can write each row to (fused gather)
// Supported sequence range (key blocks per row): the round-1 selector kept 16
// score rows in shared memory (41.25 KB of tiles + 64 B per key block within
// 227 KB); kernel 2 now writes scores to L2 and has no such limit, but the
// range the parity tests cover stays the documented one.
constexpr int kMaxKeyBlocks = (227 * 1024 - 42240) / 64;  // 2972 -> 380,416 tokens

// Per-q-head table passed in kernel parameters.
struct HeadTable {
    int32_t k[kMaxHeads];   // key blocks to keep
    int32_t kv[kMaxHeads];  // kv head read by this q head
};

// Kernel 2 row groups: up to 4 q heads that read the same kv head.
struct GroupTable {
    uint32_t heads[kMaxHeads];  // q head ids, 8 bits each
    uint8_t size[kMaxHeads];    // heads in the group (1..4)
};

// Kernel 2 (fused score + select): pooled q [hq][nqb][128], pooled k
// [hkv][nkb][128]; q head h scores against pooled kv head ht.kv[h]. scores_out (nullable) receives the full score matrix
// [hq][nqb][nkb] (-inf where causally invisible); otherwise the scores go to
// scores_ws (hq*nqb*nkb floats, contents undefined after). With select=true,
// idx/cnt receive the per-(head, q block) top-k block lists.
// Kernel 1: Q [hq][n][128] and K [hkv][n][128] bf16 -> qp [hq][ceil(n/bq)][128] and
// kp [hkv][ceil(n/128)][128] fp32 block means (bq = 128 or 256), one launch.
void launch_pool_qk(const void* q, int hq, int bq, const void* k, int hkv, int64_t n, float* qp, float* kp,
                    cudaStream_t s);
int launch_score_select(const float* qp, const float* kp, int hq, int hkv, int64_t n, int bq,
                         bool causal, float scale, const HeadTable& ht, int64_t kmax,
                         float* scores_out, float* scores_ws, bool select, int32_t* idx, int32_t* cnt,
                         cudaStream_t s);

// Kernel 2 (standalone): selection from a precomputed score matrix.
void launch_select_from_scores(const float* scores, int hq, int64_t n, int bq, bool causal,
                               const HeadTable& ht, int64_t kmax, int32_t* idx, int32_t* cnt,
                               cudaStream_t s);

// Kernel 3: block-sparse FlashAttention prefill (tcgen05/TMEM/TMA).
struct FaParams {
    CUtensorMap tm_q;  // [hq][n][128] bf16, box {64,128,1}, 128B swizzle
    CUtensorMap tm_k;  // [hkv][n][128]
    CUtensorMap tm_v;  // [hkv][n][128]
    CUtensorMap tm_k_half;  // K again with a {64,64,1} box (CTA-pair kernel: 64 keys per CTA)
    void* out;         // [hq][n][128] bf16
    const int32_t* idx;
    const int32_t* cnt;
    const int32_t* tiles;  // work list: tile t -> (h << 20) | qb, heaviest first
    // Persistent kernel only: tile ticket counter (zero at launch) and list length.
    int32_t* counter;
    int32_t num_tiles;
    int64_t kmax;
    int64_t n;
    int32_t hq, hkv, nqb;
    int32_t bq;  // query block rows: 256 (two 128-row halves share each K/V tile) or 128
    int32_t causal;
    float scale_log2;  // (1/sqrt(d)) * log2(e)
    HeadTable heads;   // kv head of each q head; k = global output head index (fused gather)
    // Fused output gather: with n_out_peers > 0 every output row of local head h
    // is stored to out_peers[i] + (heads.k[h] * n + row) * 128 for every i (this
    // GPU's full output and its peers' over NVLink) instead of to `out`.
    void* out_peers[kMaxPeers];
    int32_t n_out_peers;
    // Output tensor maps of the TMA-store epilogue ([heads][n][128] bf16, box
    // {64,128,1}, 128B swizzle): tm_out[0] over `out` (heads = hq), or with the
    // fused gather tm_out[i] over out_peers[i] (heads = the global head count).
    CUtensorMap tm_out[kMaxPeers];
};
// dual: block_q = 128 with two query blocks per CTA (tiles packed as pairs, see
// fa_sm100.cu); otherwise one tile per query block.
void launch_fa(const FaParams& p, int num_tiles, bool dual, cudaStream_t s);
// The persistent CTA-pair kernel (fa_persist_sm100.cu; bq = 256): num_clusters resident
// clusters taking tiles of p.tiles in order through the ticket counter p.counter.
cudaError_t launch_fa_persist(const FaParams& p, int num_clusters, cudaStream_t s);
// Clusters of the persistent kernel that fit on the device at once (0 if the
// occupancy query fails).
int fa_persist_max_clusters();

// GPU recovery-curve profiler (profiler.cu). q_rows bf16 [hq][n_rows][128],
// k bf16 [hkv][n_k][128]; units = hq * n_rows.
void launch_profile_scores(const void* q_rows, const void* k, int hq, int hkv, int64_t n_rows,
                           int64_t n_k, double scale, double* scores, cudaStream_t s);
size_t profile_sort_temp_bytes(int64_t units, int64_t n_k);
void launch_profile_sort(const double* in, double* out, int64_t units, int64_t n_k, int64_t* offsets,
                         void* temp, size_t temp_bytes, cudaStream_t s);
void launch_profile_prefix(const double* sorted, int64_t units, int64_t n_k, const int64_t* grid,
                           int64_t n_grid, double* mass, cudaStream_t s);
// ColumnAggregateTopK profile of `heads` heads whose scores [heads*n_rows][n_k]
// are in `scores` (overwritten with weights): col / sorted [heads][n_k] scratch,
// recovery [heads][n_grid] out (launch_profile_sort's offsets / temp reused).
void launch_profile_colagg(double* scores, int heads, int64_t n_rows, int64_t n_k, double* col, double* sorted,
                           int64_t* offsets, void* temp, size_t temp_bytes, const int64_t* grid, int64_t n_grid,
                           double* recovery, cudaStream_t s);
void launch_profile_rows(const double* mass, int hq, int64_t n_rows, const int64_t* grid, int64_t n_grid,
                         double* recovery, cudaStream_t s);

// Block-selection recovery (profiler.cu): scores = fp64 token scores of the
// units of q heads [h0, h0 + heads) x calibration rows [units][n]; bscores =
// kernel 2's block-score matrix [hq][nqb][nkb]; rows = device positions;
// mass [hq*n_rows][n_grid] (rows of heads h0.. written).
void launch_profile_block(const double* scores, const float* bscores, const int64_t* rows, int h0, int heads,
                          int64_t n_rows, int64_t n, int bq, bool causal, const int64_t* grid, int64_t n_grid,
                          double* mass, cudaStream_t s);
// out [hq][n_rows][128] bf16 = q[h][rows[r]][:].
void launch_gather_rows(const void* q, const int64_t* rows, int hq, int64_t n, int64_t n_rows, void* out,
                        cudaStream_t s);

// Block-level ColumnAggregateTopK from a score matrix [hq][nqb][nkb]: one kept
// key-block set per head (largest block-weight column sums), each query block
// gets its visible part. work: colagg_work_floats(...) floats; kept: hq*(kmax+1) int32.
void launch_colagg_select(const float* scores, int hq, int64_t n, int bq, bool causal, const HeadTable& ht,
                          int64_t kmax, float* work, int32_t* kept, int32_t* idx, int32_t* cnt, cudaStream_t s);
size_t colagg_work_floats(int hq, int64_t n, int bq);

// Dense comparator: idx [hq][nqb][nkb] = every visible key block ascending
// (tail -1), cnt [hq][nqb] = visible count.
void launch_dense_selection(int32_t* idx, int32_t* cnt, int hq, int64_t n, int bq, bool causal, cudaStream_t s);

// cudaFuncSetAttribute(func, MaxDynamicSharedMemorySize, bytes) once per
// (kernel, device, larger size): the attribute belongs to the device's context,
// so it is set the first time a kernel runs on a device (or needs more).
void set_max_dynamic_smem(const void* func, int bytes);

// Validation: sets *flag to 1 if any element of x (count elements, bf16) is not finite.
void launch_check_finite(const void* x, int64_t count, int32_t* flag, cudaStream_t s);

}  // namespace shplb::kern
