/*
 * shplb.h — C ABI of the B200-native S-HPLB sparse-attention hot path.
 *
 * This is the drop-in boundary. Each entry point replaces one function of the
 * reference operator API (C++ namespace `headbal`, /root/reference/proj); the
 * reference interface it stands in for is cited on every declaration. Plain
 * pointers and sizes only: no C++ or torch types. Device pointers are caller-
 * owned; the opaque shplb_ctx owns all device workspace (one per device/rank).
 * Device calls are asynchronous on the caller's CUDA stream (passed as void*,
 * a cudaStream_t; NULL = legacy default stream). There is no CPU fallback:
 * every attention entry point runs the sm_100a kernels or fails.
 *
 * Errors: the reference throws (std::invalid_argument for shapes, budgets and
 * infeasible totals; std::runtime_error for I/O; std::logic_error for the
 * unreachable). Here every function returns a shplb_status and the message
 * text — identical to the reference's where the reference has one — is
 * available from shplb_last_error() (thread-local) until the next call.
 */
#ifndef SHPLB_H_
#define SHPLB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SHPLB_OK = 0,
    SHPLB_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    SHPLB_RUNTIME_ERROR = 2,    /* reference: std::runtime_error    */
    SHPLB_LOGIC_ERROR = 3,      /* reference: std::logic_error      */
    SHPLB_CUDA_ERROR = 4,       /* CUDA runtime / driver failure    */
    SHPLB_NOT_SUPPORTED = 5,    /* shape or policy the kernels do not implement */
    SHPLB_NCCL_ERROR = 6        /* NCCL failure (or libnccl.so.2 not loadable) */
} shplb_status;

/* Opaque per-device context (owns device workspace); see shplb_ctx_create. */
typedef struct shplb_ctx shplb_ctx;

/* Message of the last failed call on this thread ("" after success). */
const char* shplb_last_error(void);
/* Library version string, e.g. "shplb-b200 0.1.0 sm_100a". */
const char* shplb_version(void);

/* ======================================================================
 * Per-head budget table   (reference: proj/include/headbal/allocator.hpp)
 * Budgets are in TOKENS, like the reference's BudgetAllocation::budgets.
 * ====================================================================== */

/* uniform_allocate(num_heads, total, floor, context_length)
 * (allocator.hpp:46-47, allocator.cpp:72-95): b_h = floor(B/N), remainder one
 * token each to the lowest-indexed heads. B must lie in [N*floor, N*n_k]. */
int shplb_uniform_allocate(int64_t num_heads, int64_t total, int64_t floor,
                           int64_t context_length, int64_t* budgets_out);

typedef struct {
    int64_t transfers;            /* committed transfers (BudgetAllocation::transfers.size()) */
    int32_t hit_iteration_cap;    /* BudgetAllocation::hit_iteration_cap */
    int64_t off_grid_evaluations; /* BudgetAllocation::off_grid_evaluations */
    double min_recovery_start;    /* min_recovery_trace.front() */
    double min_recovery_end;      /* min_recovery_trace.back()  */
} shplb_maxmin_diag;

/* maxmin_allocate(curves, total, AllocatorConfig{quantum, floor, max_iterations})
 * (allocator.hpp:53-54, allocator.cpp:97-186). The recovery curves (one per
 * head, profiler.hpp:29-41) are flattened: head h owns points
 * [curve_offsets[h], curve_offsets[h+1]) of curve_budgets / curve_recovery.
 * max_iterations = 0 means the reference default 10*N*n_k/quantum. diag may
 * be NULL. Bit-exact with the reference. */
int shplb_maxmin_allocate(int32_t num_heads, int64_t context_length,
                          const int64_t* curve_offsets, const int64_t* curve_budgets,
                          const double* curve_recovery, int64_t total, int64_t quantum,
                          int64_t floor, int64_t max_iterations, int64_t* budgets_out,
                          shplb_maxmin_diag* diag);

/* recovery_at (profiler.cpp:55-62): recovery at the largest sampled budget
 * <= budget, 0 below the first sample. */
int shplb_recovery_at(int64_t n_points, const int64_t* curve_budgets,
                      const double* curve_recovery, int64_t budget, double* recovery_out);

/* budget_for_recovery(curve, p) (profiler.hpp:90, profiler.cpp:198-209): the
 * smallest sampled budget whose recovery reaches p (within 1e-9) — a per-head
 * top-p budget fixed offline. Validates the curve (RecoveryCurve::validate) and
 * p in (0, 1] with the reference's messages; SHPLB_RUNTIME_ERROR when p
 * exceeds the curve's maximum. */
int shplb_budget_for_recovery(int64_t n_points, const int64_t* curve_budgets, const double* curve_recovery,
                              int64_t context_length, double p, int64_t* budget_out);

/* build_profiles + recovery_ratio for PerQueryTopK (profiler.cpp:157-196,
 * attention.cpp:151-184), restated in host C++ (fp64, OpenMP over heads x
 * rows). Offline budget-table input, not the hot path. q_rows: bf16
 * [num_q_heads][n_rows][d] calibration query rows, k: bf16
 * [num_kv_heads][n_k][d] (host memory). The rows attend to all n_k keys
 * (the reference profiles without the causal mask, commands.cpp:420-423).
 * grid: strictly increasing budgets ending at n_k. recovery_out:
 * [num_q_heads][n_grid]. GQA: q head h uses kv head h / (Hq/Hkv). */
int shplb_profile_curves_host(const uint16_t* q_rows, const uint16_t* k, int32_t num_q_heads,
                              int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                              const int64_t* grid, int64_t n_grid, double* recovery_out);

/* The same profile on the GPU: build_profiles +
 * recovery_ratio PerQueryTopK (profiler.cpp:157-196, attention.cpp:151-184)
 * as sm_100a kernels — fp64 dot products of the calibration rows against
 * every key, a per-row descending sort, fp64 prefix masses at the grid
 * points, mean over rows. q_rows / k are DEVICE bf16 pointers (layouts as
 * above); grid is host int64, recovery_out host double [num_q_heads][n_grid].
 * Runs on `stream` and synchronises it. Same validation and messages as the
 * host version; agrees with it (and the reference) to rounding. */
int shplb_profile_curves(shplb_ctx* ctx, const void* q_rows, const void* k, int32_t num_q_heads,
                         int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                         const int64_t* grid, int64_t n_grid, double* recovery_out, void* stream);

/* Both profiles for a selection kind (build_profiles' SelectionKind argument,
 * profiler.cpp:157-196; recovery_ratio, attention.cpp:151-184):
 * SHPLB_BLOCK_TOPK = PerQueryTopK (the calls above), SHPLB_COLUMN_AGGREGATE_TOPK =
 * ColumnAggregateTopK (per head, the k largest column sums of the calibration
 * rows' weights, their mass averaged over rows). */
int shplb_profile_curves_host_kind(const uint16_t* q_rows, const uint16_t* k, int32_t num_q_heads,
                                   int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                                   const int64_t* grid, int64_t n_grid, int32_t kind, double* recovery_out);
int shplb_profile_curves_kind(shplb_ctx* ctx, const void* q_rows, const void* k, int32_t num_q_heads,
                              int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                              const int64_t* grid, int64_t n_grid, int32_t kind, double* recovery_out,
                              void* stream);

/* Recovery curves of the kernels' OWN selection (block granularity), the
 * curve the layer call realises: for every calibration row at position rows[r]
 * (strictly increasing, in [0, n)) of every q head, recovery(b) = the fraction
 * of the row's exact softmax mass (fp64, keys j <= rows[r] when causal) inside
 * the ceil(b/128) key blocks kernel 2 keeps for the row's query block (pooled
 * fp32 block scores, (score desc, index asc), the visible blocks only) —
 * recovery_ratio's kept-set mass (attention.cpp:151-184) with the block
 * selector's kept set; averaged over rows as build_profiles does
 * (profiler.cpp:157-196). q [Hq][n][d], k [Hkv][n][d] DEVICE bf16 (the whole
 * layer: pooled query blocks need every row); rows / grid host int64;
 * recovery_out host double [Hq][n_grid]. Synchronises `stream`. */
int shplb_profile_curves_block(shplb_ctx* ctx, const void* q, const void* k, int32_t num_q_heads,
                               int32_t num_kv_heads, int64_t n, int32_t d, int32_t block_q, int32_t causal,
                               const int64_t* rows, int64_t n_rows, const int64_t* grid, int64_t n_grid,
                               double* recovery_out, void* stream);

/* ======================================================================
 * Head -> GPU plan   (reference: proj/include/headbal/partitioner.hpp)
 * ====================================================================== */

/* naive_assign(budgets, devices, Contiguous|RoundRobin) (partitioner.hpp:36-37,
 * partitioner.cpp:130-162). Requires devices <= num_heads. */
int shplb_plan_naive(const int64_t* budgets, int32_t num_heads, int32_t devices,
                     int32_t round_robin, int32_t* device_of_head);

/* greedy_assign(budgets, devices) — LPT (partitioner.hpp:42, partitioner.cpp:164-183).
 * Bit-exact with the reference (ties: lower head index first, lower device). */
int shplb_plan_greedy(const int64_t* budgets, int32_t num_heads, int32_t devices,
                      int32_t* device_of_head);

/* optimal_assign(budgets, devices) (partitioner.hpp:48, partitioner.cpp:185-234):
 * the minimum possible maximum device load and, among plans reaching it, the
 * lexicographically smallest device_of_head — the exact baseline the greedy plan
 * is judged against. Guarded to N <= 24 heads and 4 devices like the reference
 * (same message). */
int shplb_plan_optimal(const int64_t* budgets, int32_t num_heads, int32_t devices, int32_t* device_of_head);

/* Whole-head refinement (extension beyond greedy_assign, partitioner.cpp:164-183;
 * the reference's exact optimal_assign is guarded to N <= 24 heads, 4 devices).
 * device_of_head (in/out) is improved by local search on the per-head costs
 * (e.g. kernel-3 tile costs): while some move of a head off the most loaded
 * device, or swap with a lighter head on another device, lowers the max load of
 * the two devices below the current maximum, apply the best such step (ties: head
 * index, device index, move before swap, all ascending). Deterministic; every
 * step strictly lowers the sum of squared loads. C3 layer 0 at D = 8 (tile
 * costs): greedy 8.9% -> 2.3% modelled bubble. loads_out[devices] (may be NULL):
 * the refined per-device costs. */
int shplb_plan_refine(const int64_t* costs, int32_t num_heads, int32_t devices,
                      int32_t* device_of_head, int64_t* loads_out);

/* Sub-head balancer (an extension beyond greedy_assign,
 * partitioner.cpp:164-183). Whole-head placement cannot balance 32 or 28
 * heads over 8 GPUs under max-min budgets; this plan lets a head's query
 * blocks be split across devices. Cost of query block qb of head h =
 * min(ceil(b_h/128), visible key blocks(qb)) x (query halves holding rows),
 * the 128x128 tiles kernel 3 computes for it. Heads are walked in index order
 * (GQA groups stay contiguous, so a rank needs few kv heads) and cut
 * McNaughton-style: device d takes the units whose cost midpoint falls in
 * [d*total/D, (d+1)*total/D) of the running prefix, so device d receives a
 * contiguous run of (head, [qb_begin, qb_end)) segments, at most D-1 heads are
 * split, and every load is within half a query block's cost of total/D. Outputs up to max_segments segments
 * (seg_device/head/qb_begin/qb_end), *n_segments, and per-device costs
 * loads_out[devices] in tiles. */
int shplb_plan_split(const int64_t* budgets, int32_t num_heads, int64_t seq_len, int32_t block_q,
                     int32_t causal, int32_t devices, int32_t max_segments, int32_t* seg_device,
                     int32_t* seg_head, int32_t* seg_qb_begin, int32_t* seg_qb_end,
                     int32_t* n_segments, int64_t* loads_out);
/* The same cut with unit cost = tiles + query_tile_weight x (query halves the
 * unit visits): kernel 3's fixed per-tile cost in tile equivalents (measured
 * 2.3-5.5, tools/plan_fit.py; the Python API's QUERY_TILE_WEIGHT = 4). Weight 0
 * is shplb_plan_split. loads_out in the same weighted units. */
int shplb_plan_split_weighted(const int64_t* budgets, int32_t num_heads, int64_t seq_len, int32_t block_q,
                              int32_t causal, int32_t devices, int64_t query_tile_weight, int32_t max_segments,
                              int32_t* seg_device, int32_t* seg_head, int32_t* seg_qb_begin, int32_t* seg_qb_end,
                              int32_t* n_segments, int64_t* loads_out);

/* imbalance(budgets, assignment) (partitioner.hpp:50, partitioner.cpp:236-266):
 * loads[devices], total, I = max*D/total, argmax device. */
int shplb_imbalance(const int64_t* budgets, int32_t num_heads, const int32_t* device_of_head,
                    int32_t devices, int64_t* loads_out, int64_t* total_out,
                    double* imbalance_out, int32_t* argmax_out);

/* ======================================================================
 * Barrier metric   (reference: proj/include/headbal/simulator.hpp)
 * ====================================================================== */

/* simulate(report, CostModel{alpha, beta}) (simulator.hpp:28, simulator.cpp:28-47):
 * t_d = alpha + beta*L_d, T = max t_d, bubble = 1 - mean/T. */
int shplb_simulate(const int64_t* loads, int32_t devices, double alpha, double beta,
                   double* latency_out, double* barrier_out, double* bubble_out);

/* The same barrier / bubble definitions on MEASURED per-rank latencies
 * (simulator.cpp:40-44) — what replaces the affine model on hardware. */
int shplb_barrier(const double* device_latency, int32_t devices, double* barrier_out,
                  double* bubble_out);

/* ======================================================================
 * Block-sparse attention on sm_100a  (reference: proj/include/headbal/attention.hpp)
 * ====================================================================== */

/* One context per CUDA device (rank). Owns the device workspace. (No reference
 * counterpart: the reference is pure value semantics with no handles, SURVEY
 * §8 b2; the context is where its per-call allocations went.) The budget-
 * table, plan and metric functions are pure and reentrant like the reference's
 * (SPEC: no shared mutable state); a context is not: calls on one context must
 * not overlap across host threads (use one context per thread or stream). */
int shplb_ctx_create(int device, shplb_ctx** ctx_out);
int shplb_ctx_destroy(shplb_ctx* ctx);
/* Number of kernel launches the context issued since creation (all kinds). */
int64_t shplb_ctx_launch_count(const shplb_ctx* ctx);

/* Stage timing. While enabled, every shplb_sparse_attention_layer call records
 * CUDA events on its stream around kernel 1 (pooling), kernel 2 (score +
 * select) and kernel 3 (attention). shplb_ctx_read_timing synchronises on
 * those events, writes up to max_calls rows of {k1_ms, k2_ms, k3_ms} (one per
 * call since timing was enabled or last read) and resets the record. */
int shplb_ctx_set_timing(shplb_ctx* ctx, int enable);
int shplb_ctx_read_timing(shplb_ctx* ctx, double* stage_ms, int max_calls, int* n_calls_out);

/* Selection kind (SelectionKind, workload.cpp:14; attention.cpp:125-148), at
 * block granularity:
 *  SHPLB_BLOCK_TOPK            — PerQueryTopK: each (head, query block) keeps its
 *                                own top-k visible key blocks by pooled score;
 *  SHPLB_COLUMN_AGGREGATE_TOPK — ColumnAggregateTopK: each head keeps ONE set of k
 *                                key blocks, those with the largest column sums of
 *                                the block-softmax weights over all query blocks;
 *                                each query block attends to the part it can see
 *                                (possibly none: a zero output row). */
enum { SHPLB_BLOCK_TOPK = 0, SHPLB_COLUMN_AGGREGATE_TOPK = 1 };

/* One attention layer. q: bf16 [num_q_heads][seq_len][head_dim],
 * k/v: bf16 [num_kv_heads][seq_len][head_dim], out: bf16 like q; all dense,
 * 16-byte aligned device pointers. Prefill: n_q = n_k = seq_len. GQA: q head
 * h reads kv head kv_head_of_q[h] (default h / (num_q_heads/num_kv_heads)). */
typedef struct {
    int32_t num_q_heads;
    int32_t num_kv_heads;
    int64_t seq_len;
    int32_t head_dim;  /* 128 */
    int32_t block_q;   /* query block (pooling and FA tile rows): 128 */
    int32_t block_k;   /* key block (pooling and FA tile cols): 128 */
    int32_t causal;    /* top-left causal mask (attention.cpp:28-30) */
    int32_t kind;      /* SHPLB_BLOCK_TOPK or SHPLB_COLUMN_AGGREGATE_TOPK */
    int32_t validate;  /* 1: scan q/k/v for NaN/Inf first (workload.cpp:56-58); synchronises */
    /* Optional host int32 [num_q_heads]: kv head read by each q head. NULL =
     * standard GQA grouping h / (num_q_heads/num_kv_heads). A rank under
     * head parallelism holds an arbitrary subset of q heads and only the kv
     * heads they need, so its local map is not the contiguous grouping. */
    const int32_t* kv_head_of_q;
    /* Optional host int32 [num_q_heads][2]: the half-open range of query blocks
     * [begin, end) of each q head this call computes (output rows outside it
     * are left untouched). NULL = every query block. Used by the sub-head
     * balancer (shplb_plan_split), which splits heavy heads across ranks. */
    const int32_t* q_block_range;
    /* Optional fused output gather for head parallelism (NULL / 0 = off): device
     * pointers of FULL outputs bf16 [out_heads_total][seq_len][head_dim] — this
     * GPU's own and its peers' (mapped with shplb_ipc_open; NVLink P2P) — up to 8.
     * Kernel 3's epilogue stores every output row of local q head h into each of
     * them at global head out_head_of_q[h] (host int32 [num_q_heads]); `out` is
     * not written and may be NULL. Rows outside a head's q_block_range are left
     * untouched, so sub-head (split) plans reassemble without a reorder pass. The
     * caller orders the ranks (a barrier after the call) before reading. */
    void* const* out_peers;
    int32_t n_out_peers;
    const int32_t* out_head_of_q;
    int32_t out_heads_total;
} shplb_layer_shape;

/* CUDA IPC for the fused gather: export a device pointer of this process as an
 * opaque SHPLB_IPC_HANDLE_BYTES handle (the allocation's cudaIpcMemHandle_t plus
 * the pointer's offset inside that allocation), map a peer's handle into this
 * process (P2P over NVLink; returns the peer's pointer, offset applied), unmap
 * it. A handle cannot be opened in the process that made it, and an allocation
 * is opened at most once per process (export one buffer per rank). No
 * reference counterpart (the reference has no distributed code); together with
 * shplb_layer_shape.out_peers this replaces the paper's NCCL all-gather of
 * per-head outputs. */
#define SHPLB_IPC_HANDLE_BYTES 72
int shplb_ipc_handle(const void* dev_ptr, void* handle_out, size_t handle_bytes);
int shplb_ipc_open(int device, const void* handle, size_t handle_bytes, void** dev_ptr_out);
int shplb_ipc_close(int device, void* dev_ptr);

/* Kernel 1 — block-importance estimator. Mean-pools q/k blocks (fp32,
 * fixed summation order) and scores pooled q.k * (1/sqrt(d)):
 * score_row (attention.cpp:17-31) at block granularity.
 * scores_out: fp32 device [num_q_heads][ceil(n/bq)][ceil(n/bk)], causally
 * invisible blocks = -inf. (Exposed for parity; the layer call fuses it.) */
int shplb_block_scores(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                       const void* k, float* scores_out, void* stream);

/* Kernel 2 — per-head top-k block selector over precomputed scores. Keeps
 * min(k_h, visible blocks) per (head, query block) under (score desc, block
 * index asc), emitted ascending (attention.cpp:53-64). k_blocks: host int64
 * [num_q_heads]. idx_out: int32 device [num_q_heads][nqb][kmax] (tail -1),
 * cnt_out: int32 device [num_q_heads][nqb]. */
int shplb_select_blocks(shplb_ctx* ctx, const shplb_layer_shape* shape, const float* scores,
                        const int64_t* k_blocks, int64_t kmax, int32_t* idx_out,
                        int32_t* cnt_out, void* stream);

/* Kernel 3 — block-sparse FlashAttention prefill over given selections
 * (tcgen05 MMA, TMEM accumulators, TMA-staged K/V tiles, online softmax).
 * Output row i of head h is softmax-weighted V over the tokens of the
 * selected key blocks that are causally visible to i (attention.cpp:35-49);
 * a row with no such token is zero. */
int shplb_block_sparse_attention(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                                 const void* k, const void* v, const int32_t* idx,
                                 const int32_t* cnt, int64_t kmax, void* out, void* stream);

/* The whole hot path for one layer: sparse_attention for every head with its
 * own budget (the per-head loop of run_skyline, commands.cpp:464-470, which
 * calls sparse_attention(head, {policy, budgets[h]}), attention.cpp:116-149).
 * budgets_tokens: host int64 [num_q_heads], each in [1, seq_len]
 * (check_budget, attention.cpp:75-80); head h keeps ceil(b_h/block_k) key
 * blocks per query block. Runs kernel 1+2 fused, then kernel 3, on stream. */
int shplb_sparse_attention_layer(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                                 const void* k, const void* v,
                                 const int64_t* budgets_tokens, void* out, void* stream);

/* Dense comparator (the reference's dense_attention_all,
 * attention.cpp:84-114,204-212, minus the weight matrix): every head attends
 * to every causally visible key through the same sm_100a kernel 3 (kernels 1
 * and 2 are skipped; the selection is every visible key block). The
 * "vs full attention" axis of the paper. With stage timing on, the k1/k2
 * entries of the call read 0. */
int shplb_dense_attention_layer(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                                const void* k, const void* v, void* out, void* stream);

/* Same layer call on HOST buffers (bf16 bit patterns, same layouts): copies q/k/v
 * host->device into context-owned device memory, runs kernels 1-3, copies out
 * device->host and synchronises the stream. Pinned host memory makes the
 * copies asynchronous DMA. This is the entry a host-side caller of the
 * reference API binds: it replaces the per-head
 * sparse_attention(head, {kind, b_h}, causal) loop of run_skyline
 * (commands.cpp:464-470) on the reference's host-resident HeadData. */
int shplb_sparse_attention_layer_host(shplb_ctx* ctx, const shplb_layer_shape* shape,
                                      const uint16_t* q_host, const uint16_t* k_host,
                                      const uint16_t* v_host, const int64_t* budgets_tokens,
                                      uint16_t* out_host, void* stream);

/* The same host-buffer layer call without the final synchronisation: returns
 * once the copies and kernels are queued; `stream` completes when the output is
 * back in out_host. Consecutive async calls alternate between two device
 * staging slots and run their kernels on a context-owned stream that does not
 * wait on `stream`, so layer l+1's host->device copies overlap layer l's
 * kernels and layer l's device->host copy overlaps layer l+1's kernels (a
 * multi-layer prefill hides the PCIe time). The first async call after any
 * other call on the context orders itself after all work queued on `stream`;
 * a chained call does not wait for work the caller queued on `stream` in
 * between, so its host inputs must be complete when the call is made. Host
 * buffers must stay valid (pinned for async DMA) until the stream completes. */
int shplb_sparse_attention_layer_host_async(shplb_ctx* ctx, const shplb_layer_shape* shape,
                                            const uint16_t* q_host, const uint16_t* k_host,
                                            const uint16_t* v_host, const int64_t* budgets_tokens,
                                            uint16_t* out_host, void* stream);

/* Device pointers of the selection made by the last shplb_sparse_attention_layer
 * or shplb_sparse_attention_layer_host[_async] call on this context (valid until
 * the next call; after an async host call, once its stream completed):
 * idx [Hq][nqb][kmax], cnt [Hq][nqb], kmax = the layer's largest k_h in blocks.
 * The host-buffer entries run the layer in KV-head chunks; each chunk writes its
 * heads' rows of this one whole-layer selection. */
int shplb_last_selection(const shplb_ctx* ctx, const int32_t** idx, const int32_t** cnt,
                         int64_t* kmax);

/* Copies that selection into caller device buffers (async on stream):
 * idx_dst must hold idx_elems >= Hq*nqb*kmax int32, cnt_dst cnt_elems >= Hq*nqb. */
int shplb_copy_last_selection(const shplb_ctx* ctx, int32_t* idx_dst, int64_t idx_elems,
                              int32_t* cnt_dst, int64_t cnt_elems, void* stream);

/* Algorithmic work of one layer call before selection, for roofline accounting
 * (DESIGN.md §5): 128x128 (query half, key block) tiles = per query block
 * min(k_h, visible key blocks) x query halves holding rows, and FLOPs
 * 4*d*128*128*tiles. An upper bound by at most one tile per query block: a
 * kept key block entirely in the causal future of the first half is skipped. */
int shplb_layer_work(const shplb_layer_shape* shape, const int64_t* budgets_tokens,
                     int64_t* selected_tiles_out, double* flops_out);

/* Exact work of the last layer call on this context: the (query half, key
 * block) tiles kernel 3 computed, counted from the selection (copies it to the
 * host; synchronises the device). FLOPs = 4*d*128*128*tiles. */
int shplb_last_selection_work(const shplb_ctx* ctx, int64_t* tiles_out, double* flops_out);

/* ======================================================================
 * Head parallelism across ranks (one process per GPU)
 *   reference: the paper's per-head outputs reassembled after the head-to-GPU
 *   plan (Assignment::device_of_head, partitioner.hpp:15-21) over the per-head
 *   fan-out of sparse_attention_all (attention.cpp:204-223)
 * NCCL is resolved at run time (libnccl.so.2); failures -> SHPLB_NCCL_ERROR.
 * A communicator handle (void*) wraps an ncclComm_t bound to one device.
 * ====================================================================== */

#define SHPLB_NCCL_UNIQUE_ID_BYTES 128

/* ncclGetUniqueId on rank 0; the caller ships the bytes to every rank. */
int shplb_nccl_get_unique_id(void* id_out, size_t id_bytes);
/* ncclCommInitRank on `device` (collective over all nranks). */
int shplb_nccl_comm_init(int device, int32_t nranks, int32_t rank, const void* id, size_t id_bytes,
                         void** comm_out);
int shplb_nccl_comm_destroy(void* comm);
int shplb_nccl_comm_size(void* comm, int32_t* nranks, int32_t* rank);

/* One output segment: rows [row_begin, row_end) of global q head `head`,
 * computed by rank `owner` into its local output at local head `local_head`
 * (the owner's layer-call output [h_owner][n][d]). */
typedef struct {
    int32_t head;
    int32_t owner;
    int32_t local_head;
    int32_t reserved;
    int64_t row_begin;
    int64_t row_end;
} shplb_out_segment;

/* Reassemble a head-parallel layer on every rank: out [num_q_heads][n][d] bf16
 * (device) receives every segment from its owner's `local` buffer (one
 * ncclBroadcast per segment rooted at the owner, all in one NCCL group, async
 * on `stream`; no staging, no reorder). Every rank passes the same segment
 * list; together the segments must cover every (head, row) exactly once
 * (InvalidArgument otherwise). A rank's own segments are copied from local to
 * out (in place when local aliases out at those rows). Sub-head (split) plans
 * pass one segment per (head, query-row range). */
int shplb_gather_segments(shplb_ctx* ctx, void* comm, const shplb_out_segment* segments, int32_t n_segments,
                          int32_t num_q_heads, int64_t seq_len, int32_t head_dim, const void* local, void* out,
                          void* stream);

/* The whole-head plan form: device_of_head [num_q_heads] (greedy_assign /
 * naive_assign output, devices = ranks of the communicator, checked as
 * Assignment::validate with its messages); rank r's local output holds its
 * heads in ascending head order (shplb_sparse_attention_layer over the rank's
 * heads with a kv map), so segment h = (h, device_of_head[h], index of h among
 * that rank's heads, rows [0, n)). */
int shplb_gather_heads(shplb_ctx* ctx, void* comm, int32_t num_q_heads, int64_t seq_len, int32_t head_dim,
                       const int32_t* device_of_head, const void* local, void* out, void* stream);

/* Cross-rank barrier on `stream` (a one-element ncclAllReduce): when it
 * completes on a rank's stream, every rank's work queued before it has
 * completed — the fence of the fused output gather (shape.out_peers), after
 * which every peer's stores into this rank's output buffer are visible. */
int shplb_comm_barrier(void* comm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SHPLB_H_ */
