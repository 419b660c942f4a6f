// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (`headbal`, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). The
// parity tests, the golden-fixture generator and bench.py's CPU-baseline /
// `--impl reference` arm call the reference through these entry points with
// ctypes. Every function returns 0 on success and 1 on a C++ exception whose
// message is kept in ref_last_error() (the reference reports errors by
// exception: proj/src/workload.cpp:27-75, proj/src/attention.cpp:75-80).
//
// Matrices cross the boundary as row-major fp64 buffers, the reference's own
// Matrix layout (proj/include/headbal/matrix.hpp:9-28).

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "headbal/allocator.hpp"
#include "headbal/attention.hpp"
#include "headbal/partitioner.hpp"
#include "headbal/profiler.hpp"
#include "headbal/reference.hpp"
#include "headbal/rng.hpp"
#include "headbal/simulator.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

headbal::Matrix to_matrix(const double* p, int64_t rows, int64_t cols) {
    headbal::Matrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    if (rows * cols > 0) std::memcpy(m.data.data(), p, sizeof(double) * rows * cols);
    return m;
}

headbal::HeadData to_head(const double* q, const double* k, const double* v, int64_t n_q,
                          int64_t n_k, int64_t d, int64_t d_v) {
    return headbal::HeadData{to_matrix(q, n_q, d), to_matrix(k, n_k, d), to_matrix(v, n_k, d_v)};
}

void copy_out(const headbal::Matrix& m, double* out) {
    if (!m.data.empty()) std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
}

std::vector<headbal::RecoveryCurve> to_curves(int32_t n_heads, int64_t context_length,
                                              const int64_t* offsets, const int64_t* budgets,
                                              const double* recovery) {
    std::vector<headbal::RecoveryCurve> curves(static_cast<std::size_t>(n_heads));
    for (int32_t h = 0; h < n_heads; ++h) {
        auto& c = curves[static_cast<std::size_t>(h)];
        c.id = headbal::HeadId{0, h};
        c.context_length = context_length;
        for (int64_t p = offsets[h]; p < offsets[h + 1]; ++p) {
            c.points.push_back({budgets[p], recovery[p]});
        }
    }
    return curves;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// headbal::dense_attention (attention.cpp:84-114). weights_out may be null.
int ref_dense_attention(const double* q, const double* k, const double* v, int64_t n_q,
                        int64_t n_k, int64_t d, int64_t d_v, int causal, double* weights_out,
                        double* out) {
    return guarded([&] {
        const auto r = headbal::dense_attention(to_head(q, k, v, n_q, n_k, d, d_v), causal != 0);
        if (weights_out) copy_out(r.weights, weights_out);
        copy_out(r.output, out);
    });
}

// headbal::sparse_attention (attention.cpp:116-149). kind 0 = PerQueryTopK,
// 1 = ColumnAggregateTopK (workload.hpp:14).
int ref_sparse_attention(const double* q, const double* k, const double* v, int64_t n_q,
                         int64_t n_k, int64_t d, int64_t d_v, int kind, int64_t budget,
                         int causal, double* out) {
    return guarded([&] {
        const headbal::SelectionPolicy policy{
            kind == 0 ? headbal::SelectionKind::PerQueryTopK
                      : headbal::SelectionKind::ColumnAggregateTopK,
            budget};
        copy_out(headbal::sparse_attention(to_head(q, k, v, n_q, n_k, d, d_v), policy, causal != 0),
                 out);
    });
}

// Same call, but only the headbal::sparse_attention call itself is timed
// (steady_clock, like bench/bench_attention.cpp:18-22); the fp64 HeadData
// construction of this shim is excluded. Used for the CPU-baseline arm.
int ref_sparse_attention_timed(const double* q, const double* k, const double* v, int64_t n_q,
                               int64_t n_k, int64_t d, int64_t d_v, int kind, int64_t budget,
                               int causal, double* out, double* seconds_out) {
    return guarded([&] {
        const headbal::SelectionPolicy policy{
            kind == 0 ? headbal::SelectionKind::PerQueryTopK
                      : headbal::SelectionKind::ColumnAggregateTopK,
            budget};
        const headbal::HeadData head = to_head(q, k, v, n_q, n_k, d, d_v);
        const auto t0 = std::chrono::steady_clock::now();
        const headbal::Matrix m = headbal::sparse_attention(head, policy, causal != 0);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds_out = std::chrono::duration<double>(t1 - t0).count();
        copy_out(m, out);
    });
}

// headbal::reference::sparse_attention (reference.cpp:74-123), the serial path.
int ref_serial_sparse_attention(const double* q, const double* k, const double* v, int64_t n_q,
                                int64_t n_k, int64_t d, int64_t d_v, int kind, int64_t budget,
                                int causal, double* out) {
    return guarded([&] {
        const headbal::SelectionPolicy policy{
            kind == 0 ? headbal::SelectionKind::PerQueryTopK
                      : headbal::SelectionKind::ColumnAggregateTopK,
            budget};
        copy_out(headbal::reference::sparse_attention(to_head(q, k, v, n_q, n_k, d, d_v), policy,
                                                      causal != 0),
                 out);
    });
}

// headbal::recovery_ratio (attention.cpp:151-184).
int ref_recovery_ratio(const double* weights, int64_t n_q, int64_t n_k, int64_t k, int kind,
                       double* out) {
    return guarded([&] {
        *out = headbal::recovery_ratio(to_matrix(weights, n_q, n_k), k,
                                       kind == 0 ? headbal::SelectionKind::PerQueryTopK
                                                 : headbal::SelectionKind::ColumnAggregateTopK);
    });
}

// headbal::build_profiles (profiler.cpp:157-196) for a layer of heads that
// share n_q/n_k/d. q/k/v are [n_heads][n][d] fp64. recovery_out is
// [n_heads][n_grid].
int ref_build_profiles(const double* q, const double* k, const double* v, int32_t n_heads,
                       int64_t n_q, int64_t n_k, int64_t d, const int64_t* grid, int64_t n_grid,
                       int kind, int causal, double* recovery_out) {
    return guarded([&] {
        headbal::AttentionWorkload w;
        for (int32_t h = 0; h < n_heads; ++h) {
            w.heads.push_back(to_head(q + h * n_q * d, k + h * n_k * d, v + h * n_k * d, n_q, n_k,
                                      d, d));
        }
        const std::vector<long> g(grid, grid + n_grid);
        const auto profiles = headbal::build_profiles(
            w, g,
            kind == 0 ? headbal::SelectionKind::PerQueryTopK
                      : headbal::SelectionKind::ColumnAggregateTopK,
            {"oracle", "parity"}, causal != 0);
        for (int32_t h = 0; h < n_heads; ++h) {
            for (int64_t i = 0; i < n_grid; ++i) {
                recovery_out[h * n_grid + i] =
                    profiles[static_cast<std::size_t>(h)].curve.points[static_cast<std::size_t>(i)]
                        .recovery;
            }
        }
    });
}

// headbal::uniform_allocate (allocator.cpp:72-95).
int ref_uniform_allocate(int64_t num_heads, int64_t total, int64_t floor, int64_t context_length,
                         int64_t* budgets_out) {
    return guarded([&] {
        const auto a = headbal::uniform_allocate(num_heads, total, floor, context_length);
        for (std::size_t h = 0; h < a.budgets.size(); ++h) budgets_out[h] = a.budgets[h];
    });
}

// headbal::maxmin_allocate (allocator.cpp:97-186). Curves are flattened: head
// h owns points [offsets[h], offsets[h+1]).
int ref_maxmin_allocate(int32_t n_heads, int64_t context_length, const int64_t* offsets,
                        const int64_t* point_budgets, const double* point_recovery, int64_t total,
                        int64_t quantum, int64_t floor, int64_t max_iterations,
                        int64_t* budgets_out, int64_t* transfers_out, int32_t* hit_cap_out,
                        int64_t* off_grid_out) {
    return guarded([&] {
        headbal::AllocatorConfig cfg;
        cfg.quantum = quantum;
        cfg.floor = floor;
        cfg.max_iterations = max_iterations;
        const auto a = headbal::maxmin_allocate(
            to_curves(n_heads, context_length, offsets, point_budgets, point_recovery), total, cfg);
        for (std::size_t h = 0; h < a.budgets.size(); ++h) budgets_out[h] = a.budgets[h];
        if (transfers_out) *transfers_out = static_cast<int64_t>(a.transfers.size());
        if (hit_cap_out) *hit_cap_out = a.hit_iteration_cap ? 1 : 0;
        if (off_grid_out) *off_grid_out = a.off_grid_evaluations;
    });
}

// headbal::budget_for_recovery (profiler.cpp:198-209).
int ref_budget_for_recovery(int64_t n_points, int64_t context_length, const int64_t* budgets,
                            const double* recovery, double p, int64_t* out) {
    return guarded([&] {
        const int64_t off[2] = {0, n_points};
        const auto c = to_curves(1, context_length, off, budgets, recovery);
        *out = headbal::budget_for_recovery(c[0], p);
    });
}

// headbal::stability_score (profiler.cpp:233-292). n_groups requests of n_heads
// profiles each; profile (g, h) has id (layers[g*n_heads+h], heads[...]) and the
// curve offsets[g*n_heads+h] .. +1 into budgets / recovery; names: n_groups
// request names, each in a 64-byte slot. norm 0 = Max, 1 = Sum.
int ref_stability_score(int32_t n_groups, int32_t n_heads, const int32_t* layers, const int32_t* heads,
                        int64_t context_length, const int64_t* offsets, const int64_t* budgets,
                        const double* recovery, const char* names, double p, int norm, double* out) {
    return guarded([&] {
        std::vector<std::vector<headbal::HeadProfile>> groups(static_cast<std::size_t>(n_groups));
        for (int32_t g = 0; g < n_groups; ++g) {
            for (int32_t h = 0; h < n_heads; ++h) {
                const int64_t i = static_cast<int64_t>(g) * n_heads + h;
                headbal::HeadProfile hp;
                hp.curve.id = headbal::HeadId{layers[i], heads[i]};
                hp.curve.context_length = context_length;
                for (int64_t q = offsets[i]; q < offsets[i + 1]; ++q) hp.curve.points.push_back({budgets[q], recovery[q]});
                hp.provenance = {std::string(names + 64 * g), "parity"};
                hp.policy = headbal::SelectionKind::PerQueryTopK;
                groups[static_cast<std::size_t>(g)].push_back(hp);
            }
        }
        *out = headbal::stability_score(groups, p,
                                        norm == 0 ? headbal::BudgetNormalization::Max : headbal::BudgetNormalization::Sum);
    });
}

// headbal::naive_assign / greedy_assign / optimal_assign (partitioner.cpp:130-234).
int ref_naive_assign(const int64_t* budgets, int32_t n, int32_t devices, int round_robin,
                     int32_t* device_of_head) {
    return guarded([&] {
        const std::vector<long> b(budgets, budgets + n);
        const auto a = headbal::naive_assign(
            b, devices,
            round_robin ? headbal::NaiveOrder::RoundRobin : headbal::NaiveOrder::Contiguous);
        for (int32_t h = 0; h < n; ++h) device_of_head[h] = a.device_of_head[h];
    });
}

int ref_greedy_assign(const int64_t* budgets, int32_t n, int32_t devices, int32_t* device_of_head) {
    return guarded([&] {
        const std::vector<long> b(budgets, budgets + n);
        const auto a = headbal::greedy_assign(b, devices);
        for (int32_t h = 0; h < n; ++h) device_of_head[h] = a.device_of_head[h];
    });
}

int ref_optimal_assign(const int64_t* budgets, int32_t n, int32_t devices,
                       int32_t* device_of_head) {
    return guarded([&] {
        const std::vector<long> b(budgets, budgets + n);
        const auto a = headbal::optimal_assign(b, devices);
        for (int32_t h = 0; h < n; ++h) device_of_head[h] = a.device_of_head[h];
    });
}

// headbal::imbalance (partitioner.cpp:236-266).
int ref_imbalance(const int64_t* budgets, int32_t n, const int32_t* device_of_head,
                  int32_t devices, int64_t* loads_out, int64_t* total_out, double* imbalance_out,
                  int32_t* argmax_out) {
    return guarded([&] {
        const std::vector<long> b(budgets, budgets + n);
        headbal::Assignment a;
        a.num_devices = devices;
        a.device_of_head.assign(device_of_head, device_of_head + n);
        const auto r = headbal::imbalance(b, a);
        for (int32_t d = 0; d < devices; ++d) loads_out[d] = r.loads[d];
        *total_out = r.total;
        *imbalance_out = r.imbalance;
        *argmax_out = r.argmax_device;
    });
}

// headbal::simulate (simulator.cpp:28-47).
int ref_simulate(const int64_t* loads, int32_t devices, double alpha, double beta,
                 double* latency_out, double* barrier_out, double* bubble_out) {
    return guarded([&] {
        headbal::LoadReport r;
        r.loads.assign(loads, loads + devices);
        for (long l : r.loads) r.total += l;
        const auto s = headbal::simulate(r, headbal::CostModel{alpha, beta});
        for (int32_t d = 0; d < devices; ++d) latency_out[d] = s.device_latency[d];
        *barrier_out = s.barrier_latency;
        *bubble_out = s.bubble_fraction;
    });
}

// ---- file formats (allocator.cpp:223-275, partitioner.cpp:268-336,
// profiler.cpp:300-383): the reference's own writers and strict loaders, so
// the tests can cross-check files both ways.

int ref_save_allocation(const char* path, int32_t n, const int32_t* layers, const int32_t* heads,
                        const int64_t* budgets, int64_t total, int64_t floor) {
    return guarded([&] {
        headbal::BudgetAllocation a;
        for (int32_t i = 0; i < n; ++i) {
            a.heads.push_back(headbal::HeadId{layers[i], heads[i]});
            a.budgets.push_back(budgets[i]);
        }
        a.total = total;
        a.floor = floor;
        headbal::save_allocation(path, a);
    });
}

int ref_load_allocation(const char* path, int32_t max_n, int32_t* layers, int32_t* heads,
                        int64_t* budgets, int32_t* n_out, int64_t* total, int64_t* floor) {
    return guarded([&] {
        const auto a = headbal::load_allocation(path);
        *n_out = static_cast<int32_t>(a.budgets.size());
        for (int32_t i = 0; i < *n_out && i < max_n; ++i) {
            layers[i] = a.heads[i].layer;
            heads[i] = a.heads[i].head;
            budgets[i] = a.budgets[i];
        }
        *total = a.total;
        *floor = a.floor;
    });
}

int ref_save_assignment(const char* path, int32_t n, const int32_t* layers, const int32_t* heads,
                        const int32_t* device_of_head, int32_t devices, const int64_t* loads,
                        double imbalance) {
    return guarded([&] {
        headbal::Assignment a;
        a.num_devices = devices;
        a.device_of_head.assign(device_of_head, device_of_head + n);
        headbal::LoadReport r;
        r.loads.assign(loads, loads + devices);
        for (long l : r.loads) r.total += l;
        r.imbalance = imbalance;
        std::vector<headbal::HeadId> ids;
        for (int32_t i = 0; i < n; ++i) ids.push_back(headbal::HeadId{layers[i], heads[i]});
        headbal::save_assignment(path, a, r, ids);
    });
}

int ref_load_assignment(const char* path, int32_t max_n, int32_t max_devices, int32_t* layers,
                        int32_t* heads, int32_t* device_of_head, int32_t* n_out, int32_t* devices_out,
                        int64_t* loads, int64_t* total, double* imbalance) {
    return guarded([&] {
        const auto a = headbal::load_assignment(path);
        *n_out = static_cast<int32_t>(a.heads.size());
        for (int32_t i = 0; i < *n_out && i < max_n; ++i) {
            layers[i] = a.heads[i].layer;
            heads[i] = a.heads[i].head;
            device_of_head[i] = a.assignment.device_of_head[i];
        }
        *devices_out = a.assignment.num_devices;
        for (int32_t d = 0; d < a.assignment.num_devices && d < max_devices; ++d) loads[d] = a.report.loads[d];
        *total = a.report.total;
        *imbalance = a.report.imbalance;
    });
}

int ref_save_profiles(const char* path, int32_t n_heads, const int32_t* layers, const int32_t* heads,
                      int64_t context_length, const int64_t* offsets, const int64_t* budgets,
                      const double* recovery, int kind, const char* request, const char* task) {
    return guarded([&] {
        const auto curves = to_curves(n_heads, context_length, offsets, budgets, recovery);
        std::vector<headbal::HeadProfile> ps(static_cast<std::size_t>(n_heads));
        for (int32_t h = 0; h < n_heads; ++h) {
            ps[h].curve = curves[h];
            ps[h].curve.id = headbal::HeadId{layers[h], heads[h]};
            ps[h].provenance = headbal::Provenance{request, task};
            ps[h].policy = kind == 0 ? headbal::SelectionKind::PerQueryTopK
                                     : headbal::SelectionKind::ColumnAggregateTopK;
        }
        headbal::save_profiles(path, ps);
    });
}

// Points of profile h land at [offsets[h], offsets[h+1]) (offsets sized max_heads+1).
int ref_load_profiles(const char* path, int32_t max_heads, int64_t max_points, int32_t* layers,
                      int32_t* heads, int64_t* offsets, int64_t* budgets, double* recovery,
                      int32_t* n_heads_out, int64_t* context_length, int* kind, char* request,
                      char* task, int64_t text_cap) {
    return guarded([&] {
        const auto ps = headbal::load_profiles(path);
        *n_heads_out = static_cast<int32_t>(ps.size());
        int64_t at = 0;
        for (int32_t h = 0; h < *n_heads_out && h < max_heads; ++h) {
            layers[h] = ps[h].curve.id.layer;
            heads[h] = ps[h].curve.id.head;
            offsets[h] = at;
            for (const auto& pt : ps[h].curve.points) {
                if (at < max_points) {
                    budgets[at] = pt.budget;
                    recovery[at] = pt.recovery;
                }
                ++at;
            }
            offsets[h + 1] = at;
        }
        *context_length = ps.empty() ? 0 : ps[0].curve.context_length;
        *kind = ps.empty() || ps[0].policy == headbal::SelectionKind::PerQueryTopK ? 0 : 1;
        std::snprintf(request, static_cast<size_t>(text_cap), "%s", ps.empty() ? "" : ps[0].provenance.request.c_str());
        std::snprintf(task, static_cast<size_t>(text_cap), "%s", ps.empty() ? "" : ps[0].provenance.task.c_str());
    });
}

// headbal::derive_seed (rng.cpp:15-23) for a path of up to 8 stream ids.
uint64_t ref_derive_seed(uint64_t seed, const uint64_t* path, int32_t n) {
    // The reference takes an initializer_list; dispatch the small fixed arities we use.
    switch (n) {
        case 0: return headbal::derive_seed(seed, {});
        case 1: return headbal::derive_seed(seed, {path[0]});
        case 2: return headbal::derive_seed(seed, {path[0], path[1]});
        case 3: return headbal::derive_seed(seed, {path[0], path[1], path[2]});
        default: return headbal::derive_seed(seed, {path[0], path[1], path[2], path[3]});
    }
}

}  // extern "C"
