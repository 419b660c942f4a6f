// headbal_b200.hpp — the reference-side C++ binding of the B200 hot path.
//
// This is the header a maintainer of the reference library (`headbal`,
// /root/reference/proj) adds to route its per-head sparse-attention loop,
// budget table and head plan through libshplb.so. It keeps the reference's own
// types and signatures at the call sites (headbal::AttentionWorkload,
// headbal::RecoveryCurve, headbal::BudgetAllocation, headbal::Assignment,
// headbal::LoadReport) and rethrows the C ABI's status codes as the reference's
// exception types with the same messages.
//
// Build: -I<reference>/proj/include -I<repo>/include, link libshplb.so (and the
// reference's libheadbal for its types' out-of-line members). tests/cpp/
// compiles it against the unmodified reference and checks it there.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "headbal/allocator.hpp"
#include "headbal/partitioner.hpp"
#include "headbal/profiler.hpp"
#include "headbal/workload.hpp"
#include <cuda_runtime.h>

#include "shplb.h"

namespace headbal::b200 {

// Status code -> the reference's exception type, message preserved.
inline void check(int status) {
    if (status == SHPLB_OK) return;
    const std::string msg = shplb_last_error();
    if (status == SHPLB_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (status == SHPLB_LOGIC_ERROR) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

inline uint16_t to_bf16(double x) {  // round to nearest even
    float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

inline double from_bf16(uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// RAII owner of one device context.
class Context {
public:
    explicit Context(int device = 0) { check(shplb_ctx_create(device, &ctx_)); }
    ~Context() { shplb_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    shplb_ctx* get() const { return ctx_; }

private:
    shplb_ctx* ctx_ = nullptr;
};

// The run_skyline per-head loop (commands.cpp:464-470: sparse_attention(head,
// {kind, budgets[h]}) for every head) as one GPU layer call. Prefill-shaped
// heads (n_q == n_k), d = 128. Heads whose K/V are equal share one kv head on
// the device (GQA). Inputs go through the host-buffer entry (copies in and out
// are part of the call); selection is per (head, query block) over 128-key
// blocks, b_h tokens keeping ceil(b_h / 128) blocks.
// kind: PerQueryTopK -> SHPLB_BLOCK_TOPK, ColumnAggregateTopK -> SHPLB_COLUMN_AGGREGATE_TOPK
// (one kept key-block set per head from block-softmax column sums).
inline std::vector<Matrix> sparse_attention_all(Context& ctx, const AttentionWorkload& w,
                                                const std::vector<long>& budgets, bool causal = true,
                                                SelectionKind kind = SelectionKind::PerQueryTopK) {
    w.validate();  // the reference's shape / finiteness checks and messages
    if (budgets.size() != w.num_heads())
        throw std::invalid_argument("need one budget per head");
    const auto H = static_cast<int32_t>(w.num_heads());
    const auto n = static_cast<int64_t>(w.context_length());
    const auto d = static_cast<int32_t>(w.head_dim());
    if (static_cast<int64_t>(w.num_queries()) != n)
        throw std::invalid_argument("the GPU path is prefill-shaped: n_q must equal n_k");
    std::vector<const HeadData*> kv;  // distinct K/V sources
    std::vector<int32_t> kv_of_q(static_cast<size_t>(H));
    for (int32_t h = 0; h < H; ++h) {
        size_t g = 0;
        while (g < kv.size() && !(kv[g]->K == w.heads[h].K && kv[g]->V == w.heads[h].V)) ++g;
        if (g == kv.size()) kv.push_back(&w.heads[h]);
        kv_of_q[h] = static_cast<int32_t>(g);
    }
    const size_t hsz = static_cast<size_t>(n) * d;
    std::vector<uint16_t> q(H * hsz), k(kv.size() * hsz), v(kv.size() * hsz), o(H * hsz);
    for (int32_t h = 0; h < H; ++h)
        for (size_t i = 0; i < hsz; ++i) q[h * hsz + i] = to_bf16(w.heads[h].Q.data[i]);
    for (size_t g = 0; g < kv.size(); ++g)
        for (size_t i = 0; i < hsz; ++i) {
            k[g * hsz + i] = to_bf16(kv[g]->K.data[i]);
            v[g * hsz + i] = to_bf16(kv[g]->V.data[i]);
        }
    shplb_layer_shape s{};
    s.num_q_heads = H;
    s.num_kv_heads = static_cast<int32_t>(kv.size());
    s.seq_len = n;
    s.head_dim = d;
    s.block_q = 256;
    s.block_k = 128;
    s.causal = causal ? 1 : 0;
    s.kind = kind == SelectionKind::PerQueryTopK ? SHPLB_BLOCK_TOPK : SHPLB_COLUMN_AGGREGATE_TOPK;
    s.kv_head_of_q = kv_of_q.data();
    const std::vector<int64_t> b(budgets.begin(), budgets.end());
    check(shplb_sparse_attention_layer_host(ctx.get(), &s, q.data(), k.data(), v.data(), b.data(), o.data(),
                                            nullptr));
    std::vector<Matrix> out(static_cast<size_t>(H), Matrix(static_cast<size_t>(n), static_cast<size_t>(d)));
    for (int32_t h = 0; h < H; ++h)
        for (size_t i = 0; i < hsz; ++i) out[h].data[i] = from_bf16(o[h * hsz + i]);
    return out;
}

// ----- budget table (allocator.hpp:46-54): same signatures, bit-exact results

inline BudgetAllocation uniform_allocate(const std::vector<HeadId>& heads, long total, long floor,
                                         long context_length) {
    std::vector<int64_t> out(heads.size());
    check(shplb_uniform_allocate(static_cast<int64_t>(heads.size()), total, floor, context_length, out.data()));
    BudgetAllocation a;
    a.heads = heads;
    a.budgets.assign(out.begin(), out.end());
    a.total = total;
    a.floor = floor;
    return a;
}

inline BudgetAllocation maxmin_allocate(const std::vector<RecoveryCurve>& curves, long total,
                                        const AllocatorConfig& cfg) {
    if (curves.empty()) throw std::invalid_argument("need at least one recovery curve");
    std::vector<int64_t> off{0}, kb;
    std::vector<double> rc;
    for (const auto& c : curves) {
        for (const auto& p : c.points) {
            kb.push_back(p.budget);
            rc.push_back(p.recovery);
        }
        off.push_back(static_cast<int64_t>(kb.size()));
    }
    std::vector<int64_t> out(curves.size());
    shplb_maxmin_diag diag{};
    check(shplb_maxmin_allocate(static_cast<int32_t>(curves.size()), curves.front().context_length, off.data(),
                                kb.data(), rc.data(), total, cfg.quantum, cfg.floor, cfg.max_iterations, out.data(),
                                &diag));
    BudgetAllocation a;
    for (const auto& c : curves) a.heads.push_back(c.id);
    a.budgets.assign(out.begin(), out.end());
    a.total = total;
    a.floor = cfg.floor;
    a.hit_iteration_cap = diag.hit_iteration_cap != 0;
    a.off_grid_evaluations = diag.off_grid_evaluations;
    return a;
}

// ----- recovery curves (profiler.hpp:86-89): build_profiles for `kind`
// (PerQueryTopK or ColumnAggregateTopK) on the workload's query rows (all n_k
// keys, no causal mask as the reference's profile command), through the GPU
// profiler when a context is given, else the host C++ one. Heads with equal K
// share a kv head. Q and K are ROUNDED TO BF16 first (the device layout); the
// dot products, sort and masses are then fp64. So the curves equal the
// reference's build_profiles to rounding (1e-12) when the workload is
// bf16-exact (as the kernels' inputs always are, and as adapter_test.cpp
// checks); on arbitrary fp64 workloads they are the curves of the
// bf16-rounded heads. maxmin_allocate returns budgets, hit_iteration_cap and
// off_grid_evaluations; the reference's per-step `transfers` and
// `min_recovery_trace` diagnostics are not reproduced (left empty).
inline std::vector<RecoveryCurve> build_profiles(const AttentionWorkload& w, const std::vector<long>& grid,
                                                 Context* ctx = nullptr,
                                                 SelectionKind kind = SelectionKind::PerQueryTopK) {
    const int32_t sk = kind == SelectionKind::PerQueryTopK ? SHPLB_BLOCK_TOPK : SHPLB_COLUMN_AGGREGATE_TOPK;
    w.validate();
    const auto H = static_cast<int32_t>(w.num_heads());
    const auto rows = static_cast<int64_t>(w.num_queries());
    const auto n_k = static_cast<int64_t>(w.context_length());
    const auto d = static_cast<int32_t>(w.head_dim());
    // The C ABI takes the standard GQA grouping: every q head of a group
    // contiguous with the same K. Group consecutive heads with equal K.
    int32_t group = 1;
    while (group < H && w.heads[group].K == w.heads[0].K) ++group;
    if (H % group != 0) group = 1;
    for (int32_t h = 0; h < H; ++h)
        if (!(w.heads[h].K == w.heads[(h / group) * group].K)) group = 1;
    const int32_t hkv = H / group;
    std::vector<uint16_t> q(static_cast<size_t>(H) * rows * d), k(static_cast<size_t>(hkv) * n_k * d);
    for (int32_t h = 0; h < H; ++h)
        for (size_t i = 0; i < static_cast<size_t>(rows) * d; ++i) q[h * rows * d + i] = to_bf16(w.heads[h].Q.data[i]);
    for (int32_t g = 0; g < hkv; ++g)
        for (size_t i = 0; i < static_cast<size_t>(n_k) * d; ++i)
            k[g * n_k * d + i] = to_bf16(w.heads[g * group].K.data[i]);
    const std::vector<int64_t> gr(grid.begin(), grid.end());
    std::vector<double> rec(static_cast<size_t>(H) * gr.size());
    if (ctx) {
        // device copies for the GPU profiler
        void* dq = nullptr;
        void* dk = nullptr;
        check(cudaMalloc(&dq, q.size() * 2) == cudaSuccess ? SHPLB_OK : SHPLB_CUDA_ERROR);
        check(cudaMalloc(&dk, k.size() * 2) == cudaSuccess ? SHPLB_OK : SHPLB_CUDA_ERROR);
        cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice);
        const int rc = shplb_profile_curves_kind(ctx->get(), dq, dk, H, hkv, rows, n_k, d, gr.data(),
                                                 static_cast<int64_t>(gr.size()), sk, rec.data(), nullptr);
        cudaFree(dq);
        cudaFree(dk);
        check(rc);
    } else {
        check(shplb_profile_curves_host_kind(q.data(), k.data(), H, hkv, rows, n_k, d, gr.data(),
                                             static_cast<int64_t>(gr.size()), sk, rec.data()));
    }
    std::vector<RecoveryCurve> curves(static_cast<size_t>(H));
    for (int32_t h = 0; h < H; ++h) {
        curves[h].id = HeadId{0, h};
        curves[h].context_length = n_k;
        for (size_t i = 0; i < gr.size(); ++i) curves[h].points.push_back({grid[i], rec[h * gr.size() + i]});
    }
    return curves;
}

// ----- head plan (partitioner.hpp:36-51): same signatures, bit-exact results

inline Assignment greedy_assign(const std::vector<long>& budgets, int devices) {
    const std::vector<int64_t> b(budgets.begin(), budgets.end());
    std::vector<int32_t> dev(b.size());
    check(shplb_plan_greedy(b.data(), static_cast<int32_t>(b.size()), devices, dev.data()));
    Assignment a;
    a.num_devices = devices;
    a.device_of_head.assign(dev.begin(), dev.end());
    return a;
}

inline Assignment naive_assign(const std::vector<long>& budgets, int devices,
                               NaiveOrder order = NaiveOrder::Contiguous) {
    const std::vector<int64_t> b(budgets.begin(), budgets.end());
    std::vector<int32_t> dev(b.size());
    check(shplb_plan_naive(b.data(), static_cast<int32_t>(b.size()), devices,
                           order == NaiveOrder::RoundRobin ? 1 : 0, dev.data()));
    Assignment a;
    a.num_devices = devices;
    a.device_of_head.assign(dev.begin(), dev.end());
    return a;
}

// Extension (no reference counterpart): whole-head local search on `assignment`
// (shplb_plan_refine) with per-head costs — e.g. kernel 3's tile counts — where
// optimal_assign's guard (24 heads, 4 devices) refuses the instance.
inline Assignment refine_assign(const std::vector<long>& costs, const Assignment& assignment) {
    if (assignment.device_of_head.size() != costs.size()) {
        throw std::invalid_argument("assignment covers " + std::to_string(assignment.device_of_head.size()) +
                                    " heads but " + std::to_string(costs.size()) + " costs were given");
    }
    const std::vector<int64_t> c(costs.begin(), costs.end());
    std::vector<int32_t> dev(assignment.device_of_head.begin(), assignment.device_of_head.end());
    check(shplb_plan_refine(c.data(), static_cast<int32_t>(c.size()), assignment.num_devices, dev.data(), nullptr));
    Assignment a;
    a.num_devices = assignment.num_devices;
    a.device_of_head.assign(dev.begin(), dev.end());
    return a;
}

inline LoadReport imbalance(const std::vector<long>& budgets, const Assignment& assignment) {
    // The reference's checks and messages before anything is sized or read
    // (Assignment::validate, partitioner.cpp:38-48; imbalance, :236-242).
    if (assignment.num_devices < 1) throw std::invalid_argument("need at least one device");
    if (assignment.device_of_head.empty()) throw std::invalid_argument("assignment covers no heads");
    if (assignment.device_of_head.size() != budgets.size()) {
        throw std::invalid_argument("assignment covers " + std::to_string(assignment.device_of_head.size()) +
                                    " heads but " + std::to_string(budgets.size()) + " budgets were given");
    }
    const std::vector<int64_t> b(budgets.begin(), budgets.end());
    const std::vector<int32_t> dev(assignment.device_of_head.begin(), assignment.device_of_head.end());
    std::vector<int64_t> loads(static_cast<size_t>(assignment.num_devices));
    int64_t total = 0;
    double imb = 1.0;
    int32_t argmax = 0;
    check(shplb_imbalance(b.data(), static_cast<int32_t>(b.size()), dev.data(), assignment.num_devices,
                          loads.data(), &total, &imb, &argmax));
    LoadReport r;
    r.loads.assign(loads.begin(), loads.end());
    r.total = total;
    r.imbalance = imb;
    r.argmax_device = argmax;
    return r;
}

}  // namespace headbal::b200
