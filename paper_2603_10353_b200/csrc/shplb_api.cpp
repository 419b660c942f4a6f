// C ABI of the attention hot path (include/shplb.h): the per-device context,
// shape/budget validation with the reference's messages, the work list for
// kernel 3, TMA descriptor construction, and the kernel 1 -> 2 -> 3 sequence.
//
// Replaces headbal::sparse_attention / sparse_attention_all
// (proj/include/headbal/attention.hpp:25,40-41; proj/src/attention.cpp:116-149,
// 214-223) as driven per head with its own budget by run_skyline
// (proj/src/commands.cpp:464-470).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "common.hpp"
#include "kernels/kernels.hpp"
#include "shplb.h"

namespace shplb {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
void clear_last_error() { g_last_error.clear(); }

#define SHPLB_CUDA(call)                                                                     \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::shplb::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e));    \
    } while (0)

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable from the driver");
    return fn;
}

// cuMemGetAddressRange (driver API, resolved at run time like the tensor-map
// encoder): base address of the allocation holding a device pointer.
using AddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
uintptr_t allocation_base(const void* p) {
    static AddressRangeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddressRangeFn>(f);
    });
    if (!fn) throw CudaError("cuMemGetAddressRange unavailable from the driver");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        throw CudaError("cuMemGetAddressRange failed");
    return static_cast<uintptr_t>(base);
}

// [heads][n][128] bf16 as a 3-D tensor map with a {64, 128, 1} box and 128-byte
// swizzle: one box is one 128-row x 128-byte UMMA K-major chunk. Rows past n
// are zero-filled on load and clipped on store.
CUtensorMap make_tmap(const void* base, int64_t heads, int64_t n, uint32_t box_rows = kern::kBlock) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kern::kHeadDim), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(heads)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kern::kHeadDim) * 2,
                                   static_cast<cuuint64_t>(n) * kern::kHeadDim * 2};
    const cuuint32_t box[3] = {64, box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                                      const_cast<void*>(base), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// NVTX range over a host-side stage (enqueue of K1 / K2 / K3, a host-buffer
// chunk, a profile): visible in nsys / ncu --nvtx timelines. NVTX v3 is
// header-only and a no-op without an attached tool.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// Key blocks (of 128 keys) visible to query block qb of bq rows.
int64_t visible_blocks(int64_t qb, int64_t n, int64_t bq, bool causal) {
    const int64_t nkb = cdiv(n, kern::kBlock);
    if (!causal) return nkb;
    const int64_t last = std::min((qb + 1) * bq, n) - 1;
    return std::min(last / kern::kBlock + 1, nkb);
}

// Query halves (128-row tiles of kernel 3) of block qb that hold rows < n.
int64_t live_halves(int64_t qb, int64_t n, int64_t bq) {
    int64_t c = 0;
    for (int64_t hf = 0; hf < bq / kern::kBlock; ++hf) c += qb * bq + hf * kern::kBlock < n;
    return c;
}

void check_shape(const shplb_layer_shape* s) {
    if (!s) throw InvalidArgument("shape is null");
    if (s->num_q_heads < 1 || s->num_kv_heads < 1)
        throw InvalidArgument("workload must have at least one head");
    if (!s->kv_head_of_q && s->num_q_heads % s->num_kv_heads != 0) {
        throw InvalidArgument("num_q_heads (" + std::to_string(s->num_q_heads) +
                              ") must be a multiple of num_kv_heads (" +
                              std::to_string(s->num_kv_heads) + ")");
    }
    if (s->seq_len < 1) throw InvalidArgument("K must hold at least one key token");
    if (s->num_q_heads > kern::kMaxHeads)
        throw NotSupported("at most " + std::to_string(kern::kMaxHeads) + " query heads per call");
    if (s->head_dim != kern::kHeadDim)
        throw NotSupported("head_dim " + std::to_string(s->head_dim) + " not supported (kernels are built for 128)");
    if ((s->block_q != 128 && s->block_q != 256) || s->block_k != kern::kBlock)
        throw NotSupported("block sizes must be block_q in {128, 256}, block_k = 128");
    if (s->kind != SHPLB_BLOCK_TOPK && s->kind != SHPLB_COLUMN_AGGREGATE_TOPK)
        throw NotSupported("selection kind " + std::to_string(s->kind) + " not supported");
    if (s->seq_len > int64_t(kern::kMaxKeyBlocks) * kern::kBlock) {
        throw NotSupported("seq_len " + std::to_string(s->seq_len) + " exceeds the selector's limit of " +
                           std::to_string(int64_t(kern::kMaxKeyBlocks) * kern::kBlock) + " tokens");
    }
    if (s->out_peers && s->n_out_peers > 0) {  // fused output gather
        if (s->n_out_peers > kern::kMaxPeers)
            throw NotSupported("at most " + std::to_string(kern::kMaxPeers) + " output buffers per call");
        if (!s->out_head_of_q) throw InvalidArgument("out_head_of_q is null");
        for (int i = 0; i < s->n_out_peers; ++i) {
            if (!s->out_peers[i] || reinterpret_cast<uintptr_t>(s->out_peers[i]) % 16 != 0)
                throw InvalidArgument("out_peers[" + std::to_string(i) + "] must be a 16-byte aligned device pointer");
        }
        for (int h = 0; h < s->num_q_heads; ++h) {
            const int gh = s->out_head_of_q[h];
            if (gh < 0 || gh >= s->out_heads_total) {
                throw InvalidArgument("head " + std::to_string(h) + ": output head " + std::to_string(gh) +
                                      " out of range [0, " + std::to_string(s->out_heads_total) + ")");
            }
        }
    }
}

bool fused_gather(const shplb_layer_shape* s) { return s->out_peers != nullptr && s->n_out_peers > 0; }

void check_ptr(const void* p, const char* what) {
    if (!p) throw InvalidArgument(std::string(what) + " is null");
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
        throw InvalidArgument(std::string(what) + " must be 16-byte aligned");
}

// kv head of each q head: the caller's map, or the contiguous GQA grouping.
void fill_kv_map(const shplb_layer_shape* s, kern::HeadTable& ht) {
    const int group = s->num_q_heads / s->num_kv_heads;
    for (int h = 0; h < s->num_q_heads; ++h) {
        const int g = s->kv_head_of_q ? s->kv_head_of_q[h] : h / group;
        if (g < 0 || g >= s->num_kv_heads) {
            throw InvalidArgument("head " + std::to_string(h) + ": kv head " + std::to_string(g) +
                                  " out of range [0, " + std::to_string(s->num_kv_heads) + ")");
        }
        ht.kv[h] = g;
    }
}

// check_budget (attention.cpp:75-80), per head; returns blocks kept per head.
kern::HeadTable budgets_to_blocks(const shplb_layer_shape* s, const int64_t* budgets,
                                  std::vector<int32_t>& kb_out) {
    if (!budgets) throw InvalidArgument("budgets is null");
    kern::HeadTable kb{};
    fill_kv_map(s, kb);
    const int64_t nkb = cdiv(s->seq_len, kern::kBlock);
    kb_out.resize(static_cast<size_t>(s->num_q_heads));
    for (int h = 0; h < s->num_q_heads; ++h) {
        const int64_t b = budgets[h];
        if (b < 1 || b > s->seq_len) {
            throw InvalidArgument("head " + std::to_string(h) + ": budget k = " + std::to_string(b) +
                                  " out of range [1, " + std::to_string(s->seq_len) + "]");
        }
        kb.k[h] = static_cast<int32_t>(std::min(nkb, cdiv(b, kern::kBlock)));
        kb_out[h] = kb.k[h];
    }
    return kb;
}

}  // namespace
}  // namespace shplb

struct shplb_ctx {
    int device = 0;
    std::atomic<int64_t> launches{0};
    // workspace (grown on demand)
    float* qp = nullptr;
    size_t qp_bytes = 0;
    float* kp = nullptr;
    size_t kp_bytes = 0;
    int32_t* idx = nullptr;
    size_t idx_bytes = 0;
    int32_t* cnt = nullptr;
    size_t cnt_bytes = 0;
    int32_t* flag = nullptr;
    void* host_io = nullptr;  // device staging for shplb_sparse_attention_layer_host
    cudaStream_t copy_in = nullptr, copy_out = nullptr;  // its H2D / D2H copy streams
    cudaStream_t compute = nullptr;  // kernels of async host calls (see host_layer)
    int64_t launches_after_async = -1;  // launch count right after the last async host call
    std::vector<cudaEvent_t> chunk_events;
    int host_slot = 1;                          // staging slot of the last async host call
    cudaEvent_t slot_done[2] = {nullptr, nullptr};  // slot's last user finished (kernels + D2H)
    size_t host_io_bytes = 0;
    // Dense comparator selection (shplb_dense_attention_layer), cached per key.
    int32_t* dense_idx = nullptr;
    size_t dense_idx_bytes = 0;
    int32_t* dense_cnt = nullptr;
    size_t dense_cnt_bytes = 0;
    std::vector<int64_t> dense_key;
    // GPU profiler workspace (shplb_profile_curves)
    double* prof_scores = nullptr;
    size_t prof_scores_bytes = 0;
    double* prof_sorted = nullptr;
    size_t prof_sorted_bytes = 0;
    double* prof_mass = nullptr;
    size_t prof_mass_bytes = 0;
    int64_t* prof_aux = nullptr;  // segment offsets, then the grid
    size_t prof_aux_bytes = 0;
    void* prof_temp = nullptr;
    size_t prof_temp_bytes = 0;
    float* prof_bscores = nullptr;  // block-selection profile: kernel 2's score matrix
    size_t prof_bscores_bytes = 0;
    uint16_t* prof_qrows = nullptr;  // gathered calibration rows (bf16)
    size_t prof_qrows_bytes = 0;
    int64_t* prof_rows = nullptr;  // their positions
    size_t prof_rows_bytes = 0;
    // ColumnAggregateTopK workspace: score matrix + row/column statistics, kept sets.
    float* ca_ws = nullptr;
    size_t ca_ws_bytes = 0;
    float* k2_ws = nullptr;  // kernel 2's score rows when no score matrix is requested (L2-resident)
    size_t k2_ws_bytes = 0;
    int32_t* ca_kept = nullptr;
    size_t ca_kept_bytes = 0;
    int64_t last_kmax = 0;
    int64_t last_rows = 0;  // Hq * nqb of the last layer call
    int64_t last_n = 0, last_nqb = 0;
    int32_t last_bq = 0, last_causal = 0;
    // Kernel-3 work lists, one per (seq_len, causal, blocks-per-head, ranges,
    // kv map) seen, least recently used evicted past work_list_cap. Device
    // memory comes from the stream-ordered allocator: a list is uploaded on
    // the stream of the call that builds it and freed on the stream of the call
    // that evicts it after that stream waited for the list's last launch
    // (last_use), so neither side synchronises the host and an in-flight
    // launch never sees its list change or disappear.
    struct WorkList {
        int32_t* tiles = nullptr;        // device (stream-ordered allocation)
        int32_t* host = nullptr;         // pinned source of the upload
        int num_tiles = 0;
        uint64_t stamp = 0;              // LRU clock of the last call that used it
        cudaEvent_t last_use = nullptr;  // recorded after that call's kernel-3 launch
    };
    std::map<std::vector<int64_t>, WorkList> work_lists;
    // Pinned sources of evicted lists, freed once their last launch completed.
    std::vector<std::pair<int32_t*, cudaEvent_t>> host_graveyard;
    WorkList* current = nullptr;
    uint64_t lru_clock = 0;
    int32_t* tickets = nullptr;  // persistent kernel 3's ticket counters (kTicketRing)
    uint64_t ticket_seq = 0;
    size_t work_list_cap = 256;
    // Stage timing: 4 events per recorded layer call (before k1, after k1,
    // after k2, after k3); `timed_calls` sets in use since the last read.
    bool timing = false;
    std::vector<cudaEvent_t> events;
    int timed_calls = 0;
};

namespace shplb {
namespace {

template <typename T>
void grow(T*& p, size_t& cap, size_t bytes) {
    if (bytes <= cap) return;
    if (p) SHPLB_CUDA(cudaFree(p));
    p = nullptr;
    SHPLB_CUDA(cudaMalloc(&p, bytes));
    cap = bytes;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        SHPLB_CUDA(cudaGetDevice(&prev));
        if (prev != dev) SHPLB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

void check_launch(shplb_ctx* ctx, int n = 1) {
    SHPLB_CUDA(cudaGetLastError());
    ctx->launches += n;
}

void validate_inputs(shplb_ctx* ctx, const shplb_layer_shape* s, const void* q, const void* k,
                     const void* v, cudaStream_t st) {
    SHPLB_CUDA(cudaMemsetAsync(ctx->flag, 0, 3 * sizeof(int32_t), st));
    const int64_t qn = int64_t(s->num_q_heads) * s->seq_len * s->head_dim;
    const int64_t kn = int64_t(s->num_kv_heads) * s->seq_len * s->head_dim;
    kern::launch_check_finite(q, qn, ctx->flag + 0, st);
    if (k) kern::launch_check_finite(k, kn, ctx->flag + 1, st);
    if (v) kern::launch_check_finite(v, kn, ctx->flag + 2, st);
    check_launch(ctx, 1 + (k != nullptr) + (v != nullptr));
    int32_t f[3];
    SHPLB_CUDA(cudaMemcpyAsync(f, ctx->flag, sizeof f, cudaMemcpyDeviceToHost, st));
    SHPLB_CUDA(cudaStreamSynchronize(st));
    // validate_head's messages (workload.cpp:56-58).
    if (f[0]) throw InvalidArgument("Q contains NaN or Inf");
    if (k && f[1]) throw InvalidArgument("K contains NaN or Inf");
    if (v && f[2]) throw InvalidArgument("V contains NaN or Inf");
}

// Records stage event `slot` (0..3) of the current timed call, if timing.
void mark(shplb_ctx* ctx, int slot, cudaStream_t st) {
    if (!ctx->timing) return;
    const size_t need = static_cast<size_t>(ctx->timed_calls + 1) * 4;
    while (ctx->events.size() < need) {
        cudaEvent_t e;
        SHPLB_CUDA(cudaEventCreate(&e));
        ctx->events.push_back(e);
    }
    SHPLB_CUDA(cudaEventRecord(ctx->events[static_cast<size_t>(ctx->timed_calls) * 4 + slot], st));
    if (slot == 3) ++ctx->timed_calls;
}

// Grows the ColumnAggregateTopK workspace; returns [scores | colagg work] floats.
float* colagg_workspace(shplb_ctx* ctx, const shplb_layer_shape* s, int64_t kmax) {
    const int64_t nqb = cdiv(s->seq_len, s->block_q), nkb = cdiv(s->seq_len, kern::kBlock);
    const size_t floats = static_cast<size_t>(s->num_q_heads) * nqb * nkb +
                          kern::colagg_work_floats(s->num_q_heads, s->seq_len, s->block_q);
    grow(ctx->ca_ws, ctx->ca_ws_bytes, sizeof(float) * floats);
    grow(ctx->ca_kept, ctx->ca_kept_bytes, sizeof(int32_t) * s->num_q_heads * (kmax + 1));
    return ctx->ca_ws;
}

void pool_and_score(shplb_ctx* ctx, const shplb_layer_shape* s, const void* q, const void* k,
                    const kern::HeadTable& kb, int64_t kmax, float* scores_out, bool select,
                    int32_t* idx, int32_t* cnt, cudaStream_t st) {
    const int64_t nqb = cdiv(s->seq_len, s->block_q), nkb = cdiv(s->seq_len, kern::kBlock);
    grow(ctx->qp, ctx->qp_bytes, sizeof(float) * s->num_q_heads * nqb * kern::kHeadDim);
    grow(ctx->kp, ctx->kp_bytes, sizeof(float) * s->num_kv_heads * nkb * kern::kHeadDim);
    if (select) mark(ctx, 0, st);
    {
        Nvtx r("shplb.k1_pool");
        kern::launch_pool_qk(q, s->num_q_heads, s->block_q, k, s->num_kv_heads, s->seq_len, ctx->qp, ctx->kp, st);
    }
    if (select) mark(ctx, 1, st);
    Nvtx r2("shplb.k2_score_select");
    const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(s->head_dim)));
    if (select && s->kind == SHPLB_COLUMN_AGGREGATE_TOPK) {
        // One kept set per head from the full score matrix (attention.cpp:136-148).
        const size_t n_scores = static_cast<size_t>(s->num_q_heads) * nqb * nkb;
        float* ws = colagg_workspace(ctx, s, kmax);
        kern::launch_score_select(ctx->qp, ctx->kp, s->num_q_heads, s->num_kv_heads, s->seq_len, s->block_q,
                                  s->causal != 0, scale, kb, kmax, ws, nullptr, false, nullptr, nullptr, st);
        kern::launch_colagg_select(ws, s->num_q_heads, s->seq_len, s->block_q, s->causal != 0, kb, kmax,
                                   ws + n_scores, ctx->ca_kept, idx, cnt, st);
        check_launch(ctx, 2 + 4);
    } else {
        if (!scores_out) grow(ctx->k2_ws, ctx->k2_ws_bytes, sizeof(float) * s->num_q_heads * nqb * nkb);
        const int k2 = kern::launch_score_select(ctx->qp, ctx->kp, s->num_q_heads, s->num_kv_heads, s->seq_len,
                                                 s->block_q, s->causal != 0, scale, kb, kmax, scores_out, ctx->k2_ws,
                                                 select, idx, cnt, st);
        check_launch(ctx, 1 + k2);
    }
    if (select) mark(ctx, 2, st);
}

// Tile order of kernel 3's work list (SHPLB_TILE_ORDER, default 1):
//   1 = kv-group major, heaviest first within a group: the CTAs in flight share
//       one kv head's K/V (64 MiB at 128K, L2-resident), so K/V are read from
//       DRAM about once — C3: 3.2 GB of DRAM reads per launch instead of 8.8 GB
//       under plain LPT, 1.4% faster;
//   0 = LPT over all tiles (heaviest first);
//   2 = LPT over power-of-two work buckets, kv-grouped inside a bucket.
// Kernel-3 variant for block_q = 256 (SHPLB_K3):
//   "persist" (default) = fa_persist_sm100.cu: the CTA-pair data path (a 2-CTA
//       cluster per 256-row query block, two softmax warpgroups per CTA on
//       alternate key blocks) as one resident cluster per SM pair taking tiles
//       of the work list by atomic ticket — tile boundaries 11.4 K -> 2.0 K
//       cycles; C3 unchanged under the power cap, short tiles up to ~10% faster;
//   "single" = fa_sm100.cu, one CTA with two query halves ping-ponging (also
//       the block_q = 128 kernel). (The round-2 one-cluster-per-tile CTA-pair
//       kernel, the persistent kernel's non-persistent predecessor, was removed.)
int k3_variant() {
    static const int v = [] {
        const char* e = std::getenv("SHPLB_K3");
        if (e && std::string(e) == "single") return 0;
        return 2;
    }();
    return v;
}

// Tile-ticket counters of the persistent kernel 3: one per launch from a ring
// (zeroed once; each launch's last ticket draw resets its counter), so launches
// of one context in flight on different streams never share a counter. No
// memset per launch: a memset runs on a copy engine and, behind the host-buffer
// entry's bulk transfers, held kernel 3 back ~50 us per chunk.
constexpr int kTicketRing = 64;

// block_q = 128: two query blocks per kernel-3 CTA (each with its own selection
// and K / V stream, fa_sm100.cu kDual). SHPLB_DUAL=0 (diagnostic) restores one
// block per CTA.
bool dual_mode(const shplb_layer_shape* s) {
    static const bool on = [] {
        const char* e = std::getenv("SHPLB_DUAL");
        return !(e && std::string(e) == "0");
    }();
    return on && s->block_q == kern::kBlock;
}

int tile_order_mode() {
    static const int mode = [] {
        const char* e = std::getenv("SHPLB_TILE_ORDER");
        return e ? std::atoi(e) : 1;
    }();
    return mode;
}

// Kernel-3 work list: every (head, query block) tile, grouped by kv head and
// heaviest first inside a group (tile_order_mode), so the hardware block
// scheduler hands out long tiles before short ones while the CTAs in flight
// share K/V in L2.
void build_tiles(shplb_ctx* ctx, const shplb_layer_shape* s, const std::vector<int32_t>& kblocks,
                 cudaStream_t st) {
    const int64_t nqb = cdiv(s->seq_len, s->block_q);
    const bool dual = dual_mode(s);
    std::vector<int64_t> key = {s->seq_len, s->causal, s->block_q, s->num_q_heads, dual ? 1 : 0};
    key.insert(key.end(), kblocks.begin(), kblocks.end());
    if (s->q_block_range) key.insert(key.end(), s->q_block_range, s->q_block_range + 2 * s->num_q_heads);
    if (s->kv_head_of_q) key.insert(key.end(), s->kv_head_of_q, s->kv_head_of_q + s->num_q_heads);  // tile order
    auto it = ctx->work_lists.find(key);
    if (it != ctx->work_lists.end()) {
        ctx->current = &it->second;
        ctx->current->stamp = ++ctx->lru_clock;
        return;
    }
    // Reap pinned sources whose lists' last launches have completed.
    for (size_t i = 0; i < ctx->host_graveyard.size();) {
        auto& gy = ctx->host_graveyard[i];
        if (cudaEventQuery(gy.second) == cudaSuccess) {
            cudaFreeHost(gy.first);
            cudaEventDestroy(gy.second);
            gy = ctx->host_graveyard.back();
            ctx->host_graveyard.pop_back();
        } else {
            ++i;
        }
    }
    // Evict the least recently used list (stream-ordered after its last launch).
    while (ctx->work_lists.size() >= ctx->work_list_cap) {
        auto lru = ctx->work_lists.begin();
        for (auto e = ctx->work_lists.begin(); e != ctx->work_lists.end(); ++e)
            if (e->second.stamp < lru->second.stamp) lru = e;
        SHPLB_CUDA(cudaStreamWaitEvent(st, lru->second.last_use, 0));
        if (lru->second.tiles) SHPLB_CUDA(cudaFreeAsync(lru->second.tiles, st));
        if (lru->second.host)
            ctx->host_graveyard.push_back({lru->second.host, lru->second.last_use});
        else
            SHPLB_CUDA(cudaEventDestroy(lru->second.last_use));
        ctx->work_lists.erase(lru);
    }
    std::vector<int32_t> tiles;
    std::vector<int32_t> work;
    tiles.reserve(static_cast<size_t>(s->num_q_heads * nqb));
    for (int h = 0; h < s->num_q_heads; ++h) {
        const int64_t qb_lo = s->q_block_range ? s->q_block_range[2 * h] : 0;
        const int64_t qb_hi = s->q_block_range ? s->q_block_range[2 * h + 1] : nqb;
        if (qb_lo < 0 || qb_hi > nqb || qb_lo > qb_hi) {
            throw InvalidArgument("head " + std::to_string(h) + ": query block range [" +
                                  std::to_string(qb_lo) + ", " + std::to_string(qb_hi) +
                                  ") out of [0, " + std::to_string(nqb) + "]");
        }
        for (int64_t qb = qb_lo; qb < qb_hi; ++qb) {
            const int32_t w = static_cast<int32_t>(
                std::min<int64_t>(kblocks[h], visible_blocks(qb, s->seq_len, s->block_q, s->causal != 0)) *
                live_halves(qb, s->seq_len, s->block_q));
            if (dual) {  // (h << 20) | (pair << 2) | live-half mask
                const int32_t pair_tile = (h << 20) | static_cast<int32_t>((qb >> 1) << 2);
                if (!tiles.empty() && (tiles.back() & ~3) == pair_tile) {
                    tiles.back() |= 1 << (qb & 1);
                    work.back() += w;
                } else {
                    tiles.push_back(pair_tile | (1 << (qb & 1)));
                    work.push_back(w);
                }
            } else {
                tiles.push_back((h << 20) | static_cast<int32_t>(qb));
                work.push_back(w);
            }
        }
    }
    std::vector<size_t> order(tiles.size());
    std::iota(order.begin(), order.end(), size_t{0});
    kern::HeadTable ht{};
    fill_kv_map(s, ht);
    const int mode = tile_order_mode();
    auto kv_of = [&](size_t t) { return ht.kv[tiles[t] >> 20]; };
    if (mode == 1) {  // kv-group major, LPT within a group
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
            return kv_of(a) != kv_of(b) ? kv_of(a) < kv_of(b) : work[a] > work[b];
        });
    } else if (mode == 2) {  // LPT by power-of-two work bucket, kv group, then work
        auto bucket = [&](size_t t) { return 31 - __builtin_clz(static_cast<unsigned>(std::max(work[t], 1))); };
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
            if (bucket(a) != bucket(b)) return bucket(a) > bucket(b);
            if (kv_of(a) != kv_of(b)) return kv_of(a) < kv_of(b);
            return work[a] > work[b];
        });
    } else {  // LPT
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return work[a] > work[b]; });
    }
    std::vector<int32_t> sorted(tiles.size());
    for (size_t i = 0; i < order.size(); ++i) sorted[i] = tiles[order[i]];
    shplb_ctx::WorkList wl;
    wl.num_tiles = static_cast<int>(sorted.size());

    SHPLB_CUDA(cudaEventCreateWithFlags(&wl.last_use, cudaEventDisableTiming));
    if (!sorted.empty()) {
        const size_t bytes = sizeof(int32_t) * sorted.size();
        SHPLB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&wl.host), bytes));
        std::memcpy(wl.host, sorted.data(), bytes);
        SHPLB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wl.tiles), bytes, st));
        SHPLB_CUDA(cudaMemcpyAsync(wl.tiles, wl.host, bytes, cudaMemcpyHostToDevice, st));  // pinned: truly async
    }
    wl.stamp = ++ctx->lru_clock;
    ctx->current = &(ctx->work_lists[key] = wl);
}

void run_fa(shplb_ctx* ctx, const shplb_layer_shape* s, const void* q, const void* k,
            const void* v, const int32_t* idx, const int32_t* cnt, int64_t kmax, void* out,
            cudaStream_t st) {
    if (kmax > kern::kMaxSelected)
        throw NotSupported("more than " + std::to_string(kern::kMaxSelected) + " key blocks per query block");
    Nvtx r("shplb.k3_sparse_fa");
    kern::FaParams p;
    std::memset(&p, 0, sizeof p);
    p.tm_q = make_tmap(q, s->num_q_heads, s->seq_len);
    p.tm_k = make_tmap(k, s->num_kv_heads, s->seq_len);
    p.tm_v = make_tmap(v, s->num_kv_heads, s->seq_len);
    const bool persist = s->block_q == 256 && k3_variant() == 2;
    if (persist) p.tm_k_half = make_tmap(k, s->num_kv_heads, s->seq_len, 64);
    p.out = out;
    p.idx = idx;
    p.cnt = cnt;
    p.tiles = ctx->current->tiles;
    p.kmax = kmax;
    p.n = s->seq_len;
    p.hq = s->num_q_heads;
    p.hkv = s->num_kv_heads;
    p.nqb = static_cast<int32_t>(cdiv(s->seq_len, s->block_q));
    p.bq = s->block_q;
    p.causal = s->causal;
    fill_kv_map(s, p.heads);
    if (fused_gather(s)) {  // validated by check_shape
        for (int i = 0; i < s->n_out_peers; ++i) {
            p.out_peers[i] = s->out_peers[i];
            p.tm_out[i] = make_tmap(s->out_peers[i], s->out_heads_total, s->seq_len);
        }
        for (int h = 0; h < s->num_q_heads; ++h) p.heads.k[h] = s->out_head_of_q[h];
        p.n_out_peers = s->n_out_peers;
    } else {
        p.tm_out[0] = make_tmap(out, s->num_q_heads, s->seq_len);
    }
    p.scale_log2 = static_cast<float>((1.0 / std::sqrt(static_cast<double>(s->head_dim))) * 1.4426950408889634);
    if (ctx->current->num_tiles > 0) {
        if (persist) {
            const int maxc = kern::fa_persist_max_clusters();
            if (maxc < 1) throw CudaError("kernel 3 (persistent): no cluster fits on the device");
            if (!ctx->tickets) {  // zero once; every launch leaves its counter at zero again
                SHPLB_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->tickets), kTicketRing * sizeof(int32_t)));
                SHPLB_CUDA(cudaMemset(ctx->tickets, 0, kTicketRing * sizeof(int32_t)));
            }
            p.counter = ctx->tickets + (ctx->ticket_seq++ % kTicketRing);
            p.num_tiles = ctx->current->num_tiles;
            SHPLB_CUDA(kern::launch_fa_persist(p, std::min(maxc, p.num_tiles), st));
        } else {
            kern::launch_fa(p, ctx->current->num_tiles, dual_mode(s), st);
        }
    }
    check_launch(ctx);
    SHPLB_CUDA(cudaEventRecord(ctx->current->last_use, st));
}

}  // namespace
}  // namespace shplb

using namespace shplb;

extern "C" {

const char* shplb_last_error(void) { return shplb::g_last_error.c_str(); }

const char* shplb_version(void) { return "shplb-b200 0.1.0 sm_100a"; }

int shplb_ctx_create(int device, shplb_ctx** ctx_out) {
    return guarded([&] {
        require(ctx_out != nullptr, "ctx_out is null");
        int count = 0;
        SHPLB_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count)
            throw InvalidArgument("device " + std::to_string(device) + " out of range");
        cudaDeviceProp prop;
        SHPLB_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10 || prop.minor != 0)
            throw NotSupported(std::string("shplb kernels are built for sm_100a; device is ") + prop.name);
        DeviceGuard g(device);
        auto* ctx = new shplb_ctx();
        ctx->device = device;
        if (const char* e = std::getenv("SHPLB_WORKLIST_CACHE")) ctx->work_list_cap = std::max(1, std::atoi(e));
        SHPLB_CUDA(cudaMalloc(&ctx->flag, 4 * sizeof(int32_t)));
        *ctx_out = ctx;
    });
}

int shplb_ctx_destroy(shplb_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        DeviceGuard g(ctx->device);
        cudaFree(ctx->qp);
        cudaFree(ctx->kp);
        cudaFree(ctx->idx);
        cudaFree(ctx->cnt);
        cudaDeviceSynchronize();  // stream-ordered frees below must not overtake in-flight launches
        for (auto& kv : ctx->work_lists) {
            if (kv.second.tiles) cudaFree(kv.second.tiles);
            if (kv.second.host) cudaFreeHost(kv.second.host);
            if (kv.second.last_use) cudaEventDestroy(kv.second.last_use);
        }
        for (auto& gy : ctx->host_graveyard) {
            cudaFreeHost(gy.first);
            cudaEventDestroy(gy.second);
        }
        for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
        cudaFree(ctx->flag);
        cudaFree(ctx->host_io);
        cudaFree(ctx->dense_idx);
        cudaFree(ctx->dense_cnt);
        cudaFree(ctx->tickets);
        cudaFree(ctx->prof_scores);
        cudaFree(ctx->ca_ws);
        cudaFree(ctx->k2_ws);
        cudaFree(ctx->ca_kept);
        cudaFree(ctx->prof_sorted);
        cudaFree(ctx->prof_mass);
        cudaFree(ctx->prof_aux);
        cudaFree(ctx->prof_temp);
        cudaFree(ctx->prof_bscores);
        cudaFree(ctx->prof_qrows);
        cudaFree(ctx->prof_rows);
        if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
        if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
        if (ctx->compute) cudaStreamDestroy(ctx->compute);
        for (cudaEvent_t e : ctx->chunk_events) cudaEventDestroy(e);
        for (cudaEvent_t e : ctx->slot_done)
            if (e) cudaEventDestroy(e);
        delete ctx;
    });
}

int64_t shplb_ctx_launch_count(const shplb_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int shplb_ctx_set_timing(shplb_ctx* ctx, int enable) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        ctx->timing = enable != 0;
        ctx->timed_calls = 0;
    });
}

int shplb_ctx_read_timing(shplb_ctx* ctx, double* stage_ms, int max_calls, int* n_calls_out) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        DeviceGuard g(ctx->device);
        const int n = std::min(ctx->timed_calls, max_calls);
        for (int c = 0; c < n; ++c) {
            cudaEvent_t* e = &ctx->events[static_cast<size_t>(c) * 4];
            SHPLB_CUDA(cudaEventSynchronize(e[3]));
            for (int s = 0; s < 3; ++s) {
                float ms = 0.f;
                SHPLB_CUDA(cudaEventElapsedTime(&ms, e[s], e[s + 1]));
                stage_ms[c * 3 + s] = ms;
            }
        }
        if (n_calls_out) *n_calls_out = n;
        ctx->timed_calls = 0;
    });
}

int shplb_block_scores(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                       const void* k, float* scores_out, void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        check_shape(shape);
        check_ptr(q, "q");
        check_ptr(k, "k");
        check_ptr(scores_out, "scores_out");
        DeviceGuard g(ctx->device);
        auto st = static_cast<cudaStream_t>(stream);
        if (shape->validate) validate_inputs(ctx, shape, q, k, nullptr, st);
        kern::HeadTable kb{};
        fill_kv_map(shape, kb);
        pool_and_score(ctx, shape, q, k, kb, 1, scores_out, false, nullptr, nullptr, st);
    });
}

int shplb_select_blocks(shplb_ctx* ctx, const shplb_layer_shape* shape, const float* scores,
                        const int64_t* k_blocks, int64_t kmax, int32_t* idx_out, int32_t* cnt_out,
                        void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        check_shape(shape);
        require(scores && idx_out && cnt_out && k_blocks, "null pointer argument");
        const int64_t nkb = cdiv(shape->seq_len, kern::kBlock);
        kern::HeadTable kb{};
        fill_kv_map(shape, kb);
        int64_t need = 1;
        for (int h = 0; h < shape->num_q_heads; ++h) {
            if (k_blocks[h] < 1 || k_blocks[h] > nkb) {
                throw InvalidArgument("head " + std::to_string(h) + ": budget k = " +
                                      std::to_string(k_blocks[h]) + " out of range [1, " +
                                      std::to_string(nkb) + "]");
            }
            kb.k[h] = static_cast<int32_t>(k_blocks[h]);
            need = std::max<int64_t>(need, k_blocks[h]);
        }
        if (kmax < need) throw InvalidArgument("kmax " + std::to_string(kmax) + " < largest k " + std::to_string(need));
        DeviceGuard g(ctx->device);
        auto st = static_cast<cudaStream_t>(stream);
        if (shape->kind == SHPLB_COLUMN_AGGREGATE_TOPK) {
            float* ws = colagg_workspace(ctx, shape, kmax);
            kern::launch_colagg_select(scores, shape->num_q_heads, shape->seq_len, shape->block_q,
                                       shape->causal != 0, kb, kmax, ws, ctx->ca_kept, idx_out, cnt_out, st);
            check_launch(ctx, 4);
        } else {
            kern::launch_select_from_scores(scores, shape->num_q_heads, shape->seq_len, shape->block_q,
                                            shape->causal != 0, kb, kmax, idx_out, cnt_out, st);
            check_launch(ctx);
        }
    });
}

int shplb_block_sparse_attention(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                                 const void* k, const void* v, const int32_t* idx,
                                 const int32_t* cnt, int64_t kmax, void* out, void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        check_shape(shape);
        check_ptr(q, "q");
        check_ptr(k, "k");
        check_ptr(v, "v");
        if (!fused_gather(shape)) check_ptr(out, "out");
        require(idx && cnt && kmax >= 1, "null selection or kmax < 1");
        DeviceGuard g(ctx->device);
        auto st = static_cast<cudaStream_t>(stream);
        if (shape->validate) validate_inputs(ctx, shape, q, k, v, st);
        // Without budgets the work list orders tiles by causal visibility only.
        std::vector<int32_t> kbl(static_cast<size_t>(shape->num_q_heads), static_cast<int32_t>(kmax));
        build_tiles(ctx, shape, kbl, st);
        run_fa(ctx, shape, q, k, v, idx, cnt, kmax, out, st);
    });
}

namespace {
// One layer call over `shape`'s heads. The selection goes to the context's
// idx/cnt at head offset `head_off` with row stride `kmax_stride` (0 = this
// call's own largest k), so the host-buffer entry's KV-head chunks together
// leave the whole layer's selection behind for shplb_last_selection.
void sparse_layer(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q, const void* k,
                  const void* v, const int64_t* budgets_tokens, void* out, cudaStream_t st,
                  int64_t head_off, int64_t kmax_stride) {
    require(ctx != nullptr, "ctx is null");
    Nvtx r("shplb.sparse_attention_layer");
    check_shape(shape);
    check_ptr(q, "q");
    check_ptr(k, "k");
    check_ptr(v, "v");
    if (!fused_gather(shape)) check_ptr(out, "out");
    std::vector<int32_t> kbl;
    const kern::HeadTable kb = budgets_to_blocks(shape, budgets_tokens, kbl);
    const int64_t kmax = std::max<int64_t>(kmax_stride, *std::max_element(kbl.begin(), kbl.end()));
    DeviceGuard g(ctx->device);
    if (shape->validate) validate_inputs(ctx, shape, q, k, v, st);
    const int64_t nqb = cdiv(shape->seq_len, shape->block_q);
    const int64_t rows_total = (head_off + shape->num_q_heads) * nqb;
    if (head_off == 0) {
        grow(ctx->idx, ctx->idx_bytes, sizeof(int32_t) * rows_total * kmax);
        grow(ctx->cnt, ctx->cnt_bytes, sizeof(int32_t) * rows_total);
    } else {
        require(ctx->idx_bytes >= sizeof(int32_t) * rows_total * kmax &&
                    ctx->cnt_bytes >= sizeof(int32_t) * rows_total,
                "selection buffer not sized for the chunked layer");
    }
    int32_t* idx = ctx->idx + head_off * nqb * kmax;
    int32_t* cnt = ctx->cnt + head_off * nqb;
    build_tiles(ctx, shape, kbl, st);
    pool_and_score(ctx, shape, q, k, kb, kmax, nullptr, true, idx, cnt, st);
    run_fa(ctx, shape, q, k, v, idx, cnt, kmax, out, st);
    mark(ctx, 3, st);
    ctx->last_kmax = kmax;
    ctx->last_rows = rows_total;
    ctx->last_n = shape->seq_len;
    ctx->last_nqb = nqb;
    ctx->last_bq = shape->block_q;
    ctx->last_causal = shape->causal;
}
}  // namespace

int shplb_sparse_attention_layer(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                                 const void* k, const void* v, const int64_t* budgets_tokens,
                                 void* out, void* stream) {
    return guarded([&] {
        sparse_layer(ctx, shape, q, k, v, budgets_tokens, out, static_cast<cudaStream_t>(stream), 0, 0);
    });
}

int shplb_dense_attention_layer(shplb_ctx* ctx, const shplb_layer_shape* shape, const void* q,
                                const void* k, const void* v, void* out, void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        check_shape(shape);
        check_ptr(q, "q");
        check_ptr(k, "k");
        check_ptr(v, "v");
        if (!fused_gather(shape)) check_ptr(out, "out");
        kern::HeadTable ht{};
        fill_kv_map(shape, ht);
        DeviceGuard g(ctx->device);
        auto st = static_cast<cudaStream_t>(stream);
        if (shape->validate) validate_inputs(ctx, shape, q, k, v, st);
        const int64_t nqb = cdiv(shape->seq_len, shape->block_q), nkb = cdiv(shape->seq_len, kern::kBlock);
        const std::vector<int64_t> key = {shape->seq_len, shape->block_q, shape->causal, shape->num_q_heads};
        if (key != ctx->dense_key) {
            grow(ctx->dense_idx, ctx->dense_idx_bytes, sizeof(int32_t) * shape->num_q_heads * nqb * nkb);
            grow(ctx->dense_cnt, ctx->dense_cnt_bytes, sizeof(int32_t) * shape->num_q_heads * nqb);
            kern::launch_dense_selection(ctx->dense_idx, ctx->dense_cnt, shape->num_q_heads, shape->seq_len,
                                         shape->block_q, shape->causal != 0, st);
            check_launch(ctx);
            ctx->dense_key = key;
        }
        build_tiles(ctx, shape, std::vector<int32_t>(static_cast<size_t>(shape->num_q_heads),
                                                     static_cast<int32_t>(nkb)), st);
        mark(ctx, 0, st);
        mark(ctx, 1, st);
        mark(ctx, 2, st);
        run_fa(ctx, shape, q, k, v, ctx->dense_idx, ctx->dense_cnt, nkb, out, st);
        mark(ctx, 3, st);
    });
}

namespace {
// Host-buffer layer call. Synchronous: one staging slot, copies and kernels
// ordered after earlier work on `stream`, synchronised at the end.
// Asynchronous: staging alternates between two slots; the kernels run on the
// context's compute stream and `stream` only waits for the call's last D2H.
// Consecutive async calls therefore never wait on `stream` (it carries the
// D2H waits): layer l+1's H2D overlaps layer l's kernels, and layer l+1's
// kernels overlap layer l's D2H. A call's copies wait only for the call two
// back (same slot); when other work used the context since the last async
// call, the call first orders itself after everything queued on `stream`.
int host_layer(shplb_ctx* ctx, const shplb_layer_shape* shape, const uint16_t* q_host,
               const uint16_t* k_host, const uint16_t* v_host, const int64_t* budgets_tokens,
               uint16_t* out_host, void* stream, bool async_call) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        check_shape(shape);
        require(q_host && k_host && v_host && out_host, "null host buffer");
        if (fused_gather(shape)) throw NotSupported("the host-buffer entry does not take a fused output gather");
        const size_t qb = sizeof(uint16_t) * shape->num_q_heads * shape->seq_len * shape->head_dim;
        const size_t kb = sizeof(uint16_t) * shape->num_kv_heads * shape->seq_len * shape->head_dim;
        const size_t al = 256;
        const size_t q_off = 0, k_off = (qb + al - 1) / al * al, v_off = k_off + (kb + al - 1) / al * al,
                     o_off = v_off + (kb + al - 1) / al * al, total = o_off + qb;
        DeviceGuard g(ctx->device);
        // The staging buffer is two slots of a FIXED stride (host_io_bytes / 2),
        // whatever this call's shape: a call whose layer is smaller than the
        // previous one's must not place its slot 1 over the previous call's
        // slot 0 while that call's kernels and copy-back are still in flight.
        const size_t slot_bytes = (total + al - 1) / al * al;
        if (2 * slot_bytes > ctx->host_io_bytes) {
            if (ctx->host_io) {
                SHPLB_CUDA(cudaDeviceSynchronize());  // in-flight async calls may still use it
                SHPLB_CUDA(cudaFree(ctx->host_io));
            }
            ctx->host_io = nullptr;
            SHPLB_CUDA(cudaMalloc(&ctx->host_io, 2 * slot_bytes));
            ctx->host_io_bytes = 2 * slot_bytes;
        }
        const size_t slot_stride = ctx->host_io_bytes / 2;
        const int slot = async_call ? (ctx->host_slot ^= 1) : 0;
        auto* base = static_cast<uint8_t*>(ctx->host_io) + slot * slot_stride;
        auto st = static_cast<cudaStream_t>(stream);
        // Pipeline by KV-head chunks (standard GQA grouping only): chunk c's
        // H2D copies on a copy stream overlap chunk c-1's kernels on the
        // caller's stream, whose D2H copy runs on a second copy stream (the
        // two PCIe directions are independent). Compute stays serial on one
        // stream, so the context workspace is reused safely.
        // A chunk is a run of kv heads [g0, g1) plus the q heads reading them;
        // that q range is contiguous when the kv map is non-decreasing (the
        // standard grouping, and every head-parallel shard built by rank_shard).
        const int32_t hkv = shape->num_kv_heads, hq = shape->num_q_heads;
        // Budgets are checked for the whole layer up front (messages name the
        // layer's head index); every chunk strides its selection by the layer's
        // largest k so the chunks leave one whole-layer selection behind.
        std::vector<int32_t> kbl_layer;
        budgets_to_blocks(shape, budgets_tokens, kbl_layer);
        const int64_t kmax_layer = *std::max_element(kbl_layer.begin(), kbl_layer.end());
        {
            const int64_t rows = int64_t(hq) * cdiv(shape->seq_len, shape->block_q);
            grow(ctx->idx, ctx->idx_bytes, sizeof(int32_t) * rows * kmax_layer);
            grow(ctx->cnt, ctx->cnt_bytes, sizeof(int32_t) * rows);
        }
        kern::HeadTable map{};
        fill_kv_map(shape, map);
        bool monotone = true;
        for (int32_t h = 1; h < hq; ++h) monotone &= map.kv[h] >= map.kv[h - 1];
        static const int32_t max_chunks = [] {  // SHPLB_HOST_CHUNKS: pipeline depth (default 8)
            const char* e = std::getenv("SHPLB_HOST_CHUNKS");
            return e ? std::max(1, std::atoi(e)) : 8;
        }();
        const int32_t chunks = monotone ? std::min<int32_t>(hkv, max_chunks) : 1;
        auto q_begin = [&](int32_t g) {  // first q head whose kv head is >= g
            int32_t h = 0;
            while (h < hq && map.kv[h] < g) ++h;
            return h;
        };
        if (!ctx->copy_in) {
            SHPLB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
            SHPLB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
            SHPLB_CUDA(cudaStreamCreateWithFlags(&ctx->compute, cudaStreamNonBlocking));
        }
        // Kernels: the caller's stream (sync) or the context's compute stream (async).
        cudaStream_t ks = async_call ? ctx->compute : st;
        const bool chained = async_call && ctx->launches_after_async == ctx->launches.load();
        while (ctx->chunk_events.size() < 3 * static_cast<size_t>(chunks) + 1) {
            cudaEvent_t e;
            SHPLB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->chunk_events.push_back(e);
        }
        for (cudaEvent_t& e : ctx->slot_done) {
            if (!e) SHPLB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        if (chained) {
            // The slot's previous user (two calls back) must have finished its
            // kernels and its D2H before this call's H2D overwrites the slot.
            SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_in, ctx->slot_done[slot], 0));
            SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_out, ctx->slot_done[slot], 0));
        } else {
            cudaEvent_t start = ctx->chunk_events[0];
            SHPLB_CUDA(cudaEventRecord(start, st));  // nothing may overtake earlier work on `st`
            SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_in, start, 0));
            SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_out, start, 0));
            if (async_call) SHPLB_CUDA(cudaStreamWaitEvent(ks, start, 0));
            // Earlier async calls may have completed `stream` on another stream
            // than this call's: order after both slots' last users as well
            // (waiting on a never-recorded event is a no-op).
            for (cudaEvent_t e : ctx->slot_done) {
                SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_in, e, 0));
                SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_out, e, 0));
                if (async_call) SHPLB_CUDA(cudaStreamWaitEvent(ks, e, 0));
            }
        }
        const size_t row_bytes = sizeof(uint16_t) * shape->seq_len * shape->head_dim;  // one head
        for (int32_t c = 0; c < chunks; ++c) {
            const int32_t g0 = monotone ? hkv * c / chunks : 0, g1 = monotone ? hkv * (c + 1) / chunks : hkv;
            const int32_t h0 = monotone ? q_begin(g0) : 0, h1 = monotone ? q_begin(g1) : hq;
            if (h1 == h0) continue;  // kv heads no q head reads: nothing to compute or copy
            Nvtx rc("shplb.host_chunk");
            std::vector<int32_t> sub(static_cast<size_t>(h1 - h0));
            for (int32_t h = h0; h < h1; ++h) sub[h - h0] = map.kv[h] - g0;
            cudaEvent_t in_done = ctx->chunk_events[1 + 3 * c], comp_done = ctx->chunk_events[2 + 3 * c];
            SHPLB_CUDA(cudaMemcpyAsync(base + q_off + h0 * row_bytes, q_host + h0 * row_bytes / 2,
                                       (h1 - h0) * row_bytes, cudaMemcpyHostToDevice, ctx->copy_in));
            SHPLB_CUDA(cudaMemcpyAsync(base + k_off + g0 * row_bytes, k_host + g0 * row_bytes / 2,
                                       (g1 - g0) * row_bytes, cudaMemcpyHostToDevice, ctx->copy_in));
            SHPLB_CUDA(cudaMemcpyAsync(base + v_off + g0 * row_bytes, v_host + g0 * row_bytes / 2,
                                       (g1 - g0) * row_bytes, cudaMemcpyHostToDevice, ctx->copy_in));
            SHPLB_CUDA(cudaEventRecord(in_done, ctx->copy_in));
            SHPLB_CUDA(cudaStreamWaitEvent(ks, in_done, 0));
            shplb_layer_shape cs = *shape;
            cs.num_q_heads = h1 - h0;
            cs.num_kv_heads = g1 - g0;
            cs.kv_head_of_q = sub.data();
            if (shape->q_block_range) cs.q_block_range = shape->q_block_range + 2 * h0;
            try {
                sparse_layer(ctx, &cs, base + q_off + h0 * row_bytes, base + k_off + g0 * row_bytes,
                             base + v_off + g0 * row_bytes, budgets_tokens + h0, base + o_off + h0 * row_bytes,
                             ks, h0, kmax_layer);
            } catch (...) {  // drain before reporting
                cudaStreamSynchronize(ctx->copy_in);
                cudaStreamSynchronize(ks);
                ctx->launches_after_async = -1;
                throw;
            }
            SHPLB_CUDA(cudaEventRecord(comp_done, ks));
            SHPLB_CUDA(cudaStreamWaitEvent(ctx->copy_out, comp_done, 0));
            SHPLB_CUDA(cudaMemcpyAsync(out_host + h0 * row_bytes / 2, base + o_off + h0 * row_bytes,
                                       (h1 - h0) * row_bytes, cudaMemcpyDeviceToHost, ctx->copy_out));
        }
        // The last D2H follows every chunk's kernels, so its completion means the
        // slot is free and the output is back.
        SHPLB_CUDA(cudaEventRecord(ctx->slot_done[slot], ctx->copy_out));
        SHPLB_CUDA(cudaStreamWaitEvent(st, ctx->slot_done[slot], 0));  // `stream` completes after it
        if (async_call) {
            ctx->launches_after_async = ctx->launches.load();
        } else {
            SHPLB_CUDA(cudaStreamSynchronize(st));
            ctx->launches_after_async = -1;
        }
    });
}
}  // namespace

int shplb_sparse_attention_layer_host(shplb_ctx* ctx, const shplb_layer_shape* shape,
                                      const uint16_t* q_host, const uint16_t* k_host,
                                      const uint16_t* v_host, const int64_t* budgets_tokens,
                                      uint16_t* out_host, void* stream) {
    return host_layer(ctx, shape, q_host, k_host, v_host, budgets_tokens, out_host, stream, false);
}

int shplb_sparse_attention_layer_host_async(shplb_ctx* ctx, const shplb_layer_shape* shape,
                                            const uint16_t* q_host, const uint16_t* k_host,
                                            const uint16_t* v_host, const int64_t* budgets_tokens,
                                            uint16_t* out_host, void* stream) {
    return host_layer(ctx, shape, q_host, k_host, v_host, budgets_tokens, out_host, stream, true);
}

int shplb_last_selection(const shplb_ctx* ctx, const int32_t** idx, const int32_t** cnt,
                         int64_t* kmax) {
    return guarded([&] {
        require(ctx != nullptr && ctx->last_kmax > 0, "no layer call on this context yet");
        if (idx) *idx = ctx->idx;
        if (cnt) *cnt = ctx->cnt;
        if (kmax) *kmax = ctx->last_kmax;
    });
}

int shplb_last_selection_work(const shplb_ctx* ctx, int64_t* tiles_out, double* flops_out) {
    return guarded([&] {
        require(ctx != nullptr && ctx->last_kmax > 0, "no layer call on this context yet");
        DeviceGuard g(ctx->device);
        SHPLB_CUDA(cudaDeviceSynchronize());
        std::vector<int32_t> idx(static_cast<size_t>(ctx->last_rows * ctx->last_kmax));
        std::vector<int32_t> cnt(static_cast<size_t>(ctx->last_rows));
        SHPLB_CUDA(cudaMemcpy(idx.data(), ctx->idx, sizeof(int32_t) * idx.size(), cudaMemcpyDeviceToHost));
        SHPLB_CUDA(cudaMemcpy(cnt.data(), ctx->cnt, sizeof(int32_t) * cnt.size(), cudaMemcpyDeviceToHost));
        // Same rule as kernel 3's `active`: a half computes a kept block iff it
        // holds rows and (causal) sees the block's first key.
        int64_t tiles = 0;
        const int64_t bk = kern::kBlock, halves = ctx->last_bq / bk;
        for (int64_t row = 0; row < ctx->last_rows; ++row) {
            const int64_t row0 = (row % ctx->last_nqb) * ctx->last_bq;
            for (int64_t j = 0; j < cnt[row]; ++j) {
                const int64_t key0 = static_cast<int64_t>(idx[row * ctx->last_kmax + j]) * bk;
                for (int64_t hf = 0; hf < halves; ++hf) {
                    const int64_t first = row0 + hf * bk;
                    if (first < ctx->last_n && (!ctx->last_causal || key0 <= first + bk - 1)) ++tiles;
                }
            }
        }
        if (tiles_out) *tiles_out = tiles;
        if (flops_out) *flops_out = 4.0 * kern::kHeadDim * double(bk) * double(bk) * double(tiles);
    });
}

int shplb_copy_last_selection(const shplb_ctx* ctx, int32_t* idx_dst, int64_t idx_elems,
                              int32_t* cnt_dst, int64_t cnt_elems, void* stream) {
    return guarded([&] {
        require(ctx != nullptr && ctx->last_kmax > 0, "no layer call on this context yet");
        require(idx_dst && cnt_dst, "null destination");
        const int64_t ni = ctx->last_rows * ctx->last_kmax, nc = ctx->last_rows;
        if (idx_elems < ni || cnt_elems < nc) throw InvalidArgument("destination buffers too small");
        DeviceGuard g(ctx->device);
        auto st = static_cast<cudaStream_t>(stream);
        SHPLB_CUDA(cudaMemcpyAsync(idx_dst, ctx->idx, sizeof(int32_t) * ni, cudaMemcpyDeviceToDevice, st));
        SHPLB_CUDA(cudaMemcpyAsync(cnt_dst, ctx->cnt, sizeof(int32_t) * nc, cudaMemcpyDeviceToDevice, st));
    });
}

int shplb_layer_work(const shplb_layer_shape* shape, const int64_t* budgets_tokens,
                     int64_t* selected_tiles_out, double* flops_out) {
    return guarded([&] {
        check_shape(shape);
        std::vector<int32_t> kbl;
        budgets_to_blocks(shape, budgets_tokens, kbl);
        const int64_t nqb = cdiv(shape->seq_len, shape->block_q);
        int64_t tiles = 0;  // (128-row query half, key block) tiles, upper bound (see header)
        for (int h = 0; h < shape->num_q_heads; ++h)
            for (int64_t qb = 0; qb < nqb; ++qb)
                tiles += std::min<int64_t>(kbl[h], visible_blocks(qb, shape->seq_len, shape->block_q, shape->causal != 0)) *
                         live_halves(qb, shape->seq_len, shape->block_q);
        if (selected_tiles_out) *selected_tiles_out = tiles;
        if (flops_out)
            *flops_out = 4.0 * shape->head_dim * double(kern::kBlock) * double(kern::kBlock) * double(tiles);
    });
}

int shplb_profile_curves_kind(shplb_ctx* ctx, const void* q_rows, const void* k, int32_t num_q_heads,
                              int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                              const int64_t* grid, int64_t n_grid, int32_t kind, double* recovery_out,
                              void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        if (kind != SHPLB_BLOCK_TOPK && kind != SHPLB_COLUMN_AGGREGATE_TOPK)
            throw InvalidArgument("unknown selection kind " + std::to_string(kind));
        const bool colagg = kind == SHPLB_COLUMN_AGGREGATE_TOPK;
        require(num_q_heads >= 1 && num_kv_heads >= 1 && num_q_heads % num_kv_heads == 0,
                "num_q_heads must be a positive multiple of num_kv_heads");
        require(n_rows >= 1 && n_k >= 1 && d >= 1, "profile needs at least one row, key and dim");
        require(grid != nullptr && recovery_out != nullptr, "grid / recovery_out is null");
        // build_profiles' grid checks (profiler.cpp:165-177).
        if (n_grid < 1) throw InvalidArgument("budget grid is empty");
        for (int64_t i = 0; i < n_grid; ++i) {
            if (grid[i] < 0 || grid[i] > n_k) {
                throw InvalidArgument("budget grid entry " + std::to_string(grid[i]) + " out of [0, " +
                                      std::to_string(n_k) + "]");
            }
            if (i > 0 && grid[i] <= grid[i - 1]) throw InvalidArgument("budget grid must be strictly increasing");
        }
        if (grid[n_grid - 1] != n_k) throw InvalidArgument("budget grid must include the full context length");
        if (d != kern::kHeadDim)
            throw NotSupported("head_dim " + std::to_string(d) + " not supported (kernels are built for 128)");
        check_ptr(q_rows, "q_rows");
        check_ptr(k, "k");
        DeviceGuard dg(ctx->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int32_t group = num_q_heads / num_kv_heads;
        const int64_t units_total = int64_t(num_q_heads) * n_rows;
        // Kv heads per batch: bounded scores + sorted buffers (2 x 8 B per score, <= 4 GiB).
        const int64_t units_per_kv = int64_t(group) * n_rows;
        int64_t kv_batch = std::max<int64_t>(1, (int64_t(1) << 32) / (16 * units_per_kv * n_k));
        kv_batch = std::min<int64_t>(kv_batch, num_kv_heads);
        const int64_t units_b = kv_batch * units_per_kv;
        grow(ctx->prof_scores, ctx->prof_scores_bytes, sizeof(double) * units_b * n_k);
        const int64_t heads_b = kv_batch * group;
        grow(ctx->prof_sorted, ctx->prof_sorted_bytes,
             sizeof(double) * std::max(units_b, colagg ? 2 * heads_b : int64_t(0)) * n_k);
        grow(ctx->prof_mass, ctx->prof_mass_bytes, sizeof(double) * (units_total * n_grid + int64_t(num_q_heads) * n_grid));
        grow(ctx->prof_aux, ctx->prof_aux_bytes, sizeof(int64_t) * (units_b + 1 + n_grid));
        const size_t temp = kern::profile_sort_temp_bytes(units_b, n_k);
        grow(ctx->prof_temp, ctx->prof_temp_bytes, std::max<size_t>(temp, 16));
        int64_t* offsets = ctx->prof_aux;
        int64_t* grid_dev = ctx->prof_aux + units_b + 1;
        double* recovery_dev = ctx->prof_mass + units_total * n_grid;
        SHPLB_CUDA(cudaMemcpyAsync(grid_dev, grid, sizeof(int64_t) * n_grid, cudaMemcpyHostToDevice, st));
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        for (int64_t g0 = 0; g0 < num_kv_heads; g0 += kv_batch) {
            const int64_t nb = std::min<int64_t>(kv_batch, num_kv_heads - g0);
            const int64_t units = nb * units_per_kv;
            const auto* qb = static_cast<const uint16_t*>(q_rows) + g0 * units_per_kv * d;
            const auto* kb = static_cast<const uint16_t*>(k) + g0 * n_k * d;
            kern::launch_profile_scores(qb, kb, static_cast<int>(nb * group), static_cast<int>(nb), n_rows, n_k,
                                        scale, ctx->prof_scores, st);
            if (colagg) {
                const int64_t hb = nb * group;
                kern::launch_profile_colagg(ctx->prof_scores, static_cast<int>(hb), n_rows, n_k, ctx->prof_sorted,
                                            ctx->prof_sorted + hb * n_k, offsets, ctx->prof_temp,
                                            ctx->prof_temp_bytes, grid_dev, n_grid,
                                            recovery_dev + g0 * group * n_grid, st);
                check_launch(ctx, 6);
                continue;
            }
            kern::launch_profile_sort(ctx->prof_scores, ctx->prof_sorted, units, n_k, offsets, ctx->prof_temp,
                                      ctx->prof_temp_bytes, st);
            kern::launch_profile_prefix(ctx->prof_sorted, units, n_k, grid_dev, n_grid,
                                        ctx->prof_mass + g0 * units_per_kv * n_grid, st);
            check_launch(ctx, 4);
        }
        if (!colagg) {
            kern::launch_profile_rows(ctx->prof_mass, num_q_heads, n_rows, grid_dev, n_grid, recovery_dev, st);
            check_launch(ctx);
        }
        SHPLB_CUDA(cudaMemcpyAsync(recovery_out, recovery_dev, sizeof(double) * num_q_heads * n_grid,
                                   cudaMemcpyDeviceToHost, st));
        SHPLB_CUDA(cudaStreamSynchronize(st));
    });
}

int shplb_profile_curves(shplb_ctx* ctx, const void* q_rows, const void* k, int32_t num_q_heads,
                         int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                         const int64_t* grid, int64_t n_grid, double* recovery_out, void* stream) {
    return shplb_profile_curves_kind(ctx, q_rows, k, num_q_heads, num_kv_heads, n_rows, n_k, d, grid, n_grid,
                                     SHPLB_BLOCK_TOPK, recovery_out, stream);
}

int shplb_profile_curves_block(shplb_ctx* ctx, const void* q, const void* k, int32_t num_q_heads,
                               int32_t num_kv_heads, int64_t n, int32_t d, int32_t block_q, int32_t causal,
                               const int64_t* rows, int64_t n_rows, const int64_t* grid, int64_t n_grid,
                               double* recovery_out, void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx is null");
        require(num_q_heads >= 1 && num_kv_heads >= 1 && num_q_heads % num_kv_heads == 0,
                "num_q_heads must be a positive multiple of num_kv_heads");
        require(n_rows >= 1 && n >= 1, "profile needs at least one row and key");
        require(grid != nullptr && rows != nullptr && recovery_out != nullptr, "grid / rows / recovery_out is null");
        if (n_grid < 1) throw InvalidArgument("budget grid is empty");
        for (int64_t i = 0; i < n_grid; ++i) {  // build_profiles' grid checks (profiler.cpp:165-177)
            if (grid[i] < 0 || grid[i] > n) {
                throw InvalidArgument("budget grid entry " + std::to_string(grid[i]) + " out of [0, " +
                                      std::to_string(n) + "]");
            }
            if (i > 0 && grid[i] <= grid[i - 1]) throw InvalidArgument("budget grid must be strictly increasing");
        }
        if (grid[n_grid - 1] != n) throw InvalidArgument("budget grid must include the full context length");
        for (int64_t r = 0; r < n_rows; ++r) {
            if (rows[r] < 0 || rows[r] >= n || (r > 0 && rows[r] <= rows[r - 1]))
                throw InvalidArgument("calibration rows must be strictly increasing positions in [0, n)");
        }
        shplb_layer_shape sh{};
        sh.num_q_heads = num_q_heads;
        sh.num_kv_heads = num_kv_heads;
        sh.seq_len = n;
        sh.head_dim = d;
        sh.block_q = block_q;
        sh.block_k = kern::kBlock;
        sh.causal = causal;
        sh.kind = SHPLB_BLOCK_TOPK;
        check_shape(&sh);
        check_ptr(q, "q");
        check_ptr(k, "k");
        DeviceGuard dg(ctx->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int64_t nqb = cdiv(n, block_q), nkb = cdiv(n, kern::kBlock);
        // Kernel 1 + kernel 2's scores (the very ranking the layer call uses).
        grow(ctx->prof_bscores, ctx->prof_bscores_bytes, sizeof(float) * num_q_heads * nqb * nkb);
        kern::HeadTable ht{};
        fill_kv_map(&sh, ht);
        pool_and_score(ctx, &sh, q, k, ht, 1, ctx->prof_bscores, false, nullptr, nullptr, st);
        // Calibration rows and fp64 token scores, kv batches bounded as in shplb_profile_curves_kind.
        grow(ctx->prof_rows, ctx->prof_rows_bytes, sizeof(int64_t) * n_rows);
        grow(ctx->prof_qrows, ctx->prof_qrows_bytes, sizeof(uint16_t) * num_q_heads * n_rows * d);
        const int32_t group = num_q_heads / num_kv_heads;
        const int64_t units_per_kv = int64_t(group) * n_rows, units_total = int64_t(num_q_heads) * n_rows;
        int64_t kv_batch = std::max<int64_t>(1, (int64_t(1) << 32) / (8 * units_per_kv * n));
        kv_batch = std::min<int64_t>(kv_batch, num_kv_heads);
        grow(ctx->prof_scores, ctx->prof_scores_bytes, sizeof(double) * kv_batch * units_per_kv * n);
        grow(ctx->prof_mass, ctx->prof_mass_bytes,
             sizeof(double) * (units_total * n_grid + int64_t(num_q_heads) * n_grid));
        grow(ctx->prof_aux, ctx->prof_aux_bytes, sizeof(int64_t) * n_grid);
        int64_t* grid_dev = ctx->prof_aux;
        double* recovery_dev = ctx->prof_mass + units_total * n_grid;
        SHPLB_CUDA(cudaMemcpyAsync(grid_dev, grid, sizeof(int64_t) * n_grid, cudaMemcpyHostToDevice, st));
        SHPLB_CUDA(cudaMemcpyAsync(ctx->prof_rows, rows, sizeof(int64_t) * n_rows, cudaMemcpyHostToDevice, st));
        kern::launch_gather_rows(q, ctx->prof_rows, num_q_heads, n, n_rows, ctx->prof_qrows, st);
        check_launch(ctx);
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        for (int64_t g0 = 0; g0 < num_kv_heads; g0 += kv_batch) {
            const int64_t nb = std::min<int64_t>(kv_batch, num_kv_heads - g0);
            kern::launch_profile_scores(ctx->prof_qrows + g0 * units_per_kv * d,
                                        static_cast<const uint16_t*>(k) + g0 * n * d, static_cast<int>(nb * group),
                                        static_cast<int>(nb), n_rows, n, scale, ctx->prof_scores, st);
            kern::launch_profile_block(ctx->prof_scores, ctx->prof_bscores, ctx->prof_rows,
                                       static_cast<int>(g0 * group), static_cast<int>(nb * group), n_rows, n,
                                       block_q, causal != 0, grid_dev, n_grid, ctx->prof_mass, st);
            check_launch(ctx, 2);
        }
        kern::launch_profile_rows(ctx->prof_mass, num_q_heads, n_rows, grid_dev, n_grid, recovery_dev, st);
        check_launch(ctx);
        SHPLB_CUDA(cudaMemcpyAsync(recovery_out, recovery_dev, sizeof(double) * num_q_heads * n_grid,
                                   cudaMemcpyDeviceToHost, st));
        SHPLB_CUDA(cudaStreamSynchronize(st));
    });
}

// IPC handle layout (SHPLB_IPC_HANDLE_BYTES = 72): the CUDA IPC handle of the
// allocation holding dev_ptr, then dev_ptr's byte offset inside it (caching
// allocators hand out pointers inside larger allocations).
int shplb_ipc_handle(const void* dev_ptr, void* handle_out, size_t handle_bytes) {
    return guarded([&] {
        require(dev_ptr && handle_out, "null pointer");
        require(handle_bytes >= SHPLB_IPC_HANDLE_BYTES, "handle buffer must hold 72 bytes");
        cudaIpcMemHandle_t hnd;
        SHPLB_CUDA(cudaIpcGetMemHandle(&hnd, const_cast<void*>(dev_ptr)));
        const uint64_t off = reinterpret_cast<uintptr_t>(dev_ptr) - allocation_base(dev_ptr);
        auto* out = static_cast<uint8_t*>(handle_out);
        std::memcpy(out, &hnd, sizeof hnd);
        std::memcpy(out + sizeof hnd, &off, sizeof off);
    });
}

int shplb_ipc_open(int device, const void* handle, size_t handle_bytes, void** dev_ptr_out) {
    return guarded([&] {
        require(handle && dev_ptr_out, "null pointer");
        require(handle_bytes >= SHPLB_IPC_HANDLE_BYTES, "handle must be 72 bytes");
        DeviceGuard g(device);
        cudaIpcMemHandle_t hnd;
        uint64_t off = 0;
        std::memcpy(&hnd, handle, sizeof hnd);
        std::memcpy(&off, static_cast<const uint8_t*>(handle) + sizeof hnd, sizeof off);
        void* base = nullptr;
        SHPLB_CUDA(cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess));
        *dev_ptr_out = static_cast<uint8_t*>(base) + off;
    });
}

int shplb_ipc_close(int device, void* dev_ptr) {
    return guarded([&] {
        DeviceGuard g(device);
        SHPLB_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(allocation_base(dev_ptr))));
    });
}

}  // extern "C"
