// TEST INFRASTRUCTURE: checks include/headbal_b200.hpp (the reference-side C++
// binding of libshplb) against the unmodified reference library it stands in
// for. Built by tests/cpp/Makefile against /root/reference/proj/include and
// oracle/_ref/libheadbal_ref.so; run by tests/test_cpp_adapter.py.
//   adapter_test cpu  — budget tables, plans, load reports bit-exact vs the
//                       reference; the reference's exception types/messages.
//   adapter_test gpu  — the GPU layer call through the adapter vs the
//                       reference's dense_attention at full budget.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "headbal/attention.hpp"
#include "headbal_b200.hpp"

using namespace headbal;

static int failures = 0;
#define EXPECT(cond, what)                                              \
    do {                                                                \
        if (!(cond)) {                                                  \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
            ++failures;                                                 \
        }                                                               \
    } while (0)

static std::vector<RecoveryCurve> random_curves(std::mt19937_64& rng, int n, long n_k, long stride) {
    std::vector<RecoveryCurve> cs(static_cast<size_t>(n));
    std::uniform_real_distribution<double> U(0.5, 6.0);
    for (int h = 0; h < n; ++h) {
        const double s = U(rng);
        cs[h].id = HeadId{0, h};
        cs[h].context_length = n_k;
        for (long k = 0; k <= n_k; k += stride) {
            const double r = k == n_k ? 1.0 : 1.0 - std::pow(1.0 - static_cast<double>(k) / n_k, s);
            cs[h].points.push_back({k, r});
        }
        if (cs[h].points.back().budget != n_k) cs[h].points.push_back({n_k, 1.0});
    }
    return cs;
}

static int run_cpu() {
    std::mt19937_64 rng(2603);
    for (int trial = 0; trial < 40; ++trial) {
        const int n = 2 + static_cast<int>(rng() % 40);
        const long n_k = 512 + static_cast<long>(rng() % 4) * 512;
        const auto curves = random_curves(rng, n, n_k, 64);
        const long total = n * (128 + static_cast<long>(rng() % static_cast<unsigned long>(n_k - 128)));
        AllocatorConfig cfg;
        cfg.quantum = 64;
        cfg.floor = 128;
        const auto ref = maxmin_allocate(curves, total, cfg);
        const auto got = b200::maxmin_allocate(curves, total, cfg);
        EXPECT(ref.budgets == got.budgets, "maxmin_allocate budgets");
        EXPECT(ref.hit_iteration_cap == got.hit_iteration_cap, "maxmin_allocate cap flag");
        std::vector<HeadId> ids;
        for (const auto& c : curves) ids.push_back(c.id);
        EXPECT(uniform_allocate(ids, total, 128, n_k).budgets == b200::uniform_allocate(ids, total, 128, n_k).budgets,
               "uniform_allocate");
        for (int d : {1, 2, 3, 4, 8}) {
            if (d > n) continue;
            const auto g_ref = greedy_assign(ref.budgets, d), g = b200::greedy_assign(ref.budgets, d);
            EXPECT(g_ref.device_of_head == g.device_of_head, "greedy_assign");
            const auto n_ref = naive_assign(ref.budgets, d), nv = b200::naive_assign(ref.budgets, d);
            EXPECT(n_ref.device_of_head == nv.device_of_head, "naive_assign");
            const auto rr = naive_assign(ref.budgets, d, NaiveOrder::RoundRobin);
            EXPECT(rr.device_of_head == b200::naive_assign(ref.budgets, d, NaiveOrder::RoundRobin).device_of_head,
                   "naive_assign round robin");
            // refine_assign (extension): never above greedy's makespan; at or above the
            // reference's exact optimum where its guard allows it.
            const auto rf = b200::refine_assign(ref.budgets, g);
            const auto l_g = b200::imbalance(ref.budgets, g).loads;
            const long mk_g = *std::max_element(l_g.begin(), l_g.end());
            const auto l_rf = b200::imbalance(ref.budgets, rf).loads;
            const long mk_r = *std::max_element(l_rf.begin(), l_rf.end());
            EXPECT(mk_r <= mk_g, "refine_assign above greedy");
            if (n <= 24 && d <= 4) {
                const auto lo = imbalance(ref.budgets, optimal_assign(ref.budgets, d)).loads;
                EXPECT(*std::max_element(lo.begin(), lo.end()) <= mk_r, "refine_assign below the optimum");
            }
            const auto l_ref = imbalance(ref.budgets, g_ref), l = b200::imbalance(ref.budgets, g);
            EXPECT(l_ref.loads == l.loads && l_ref.total == l.total && l_ref.imbalance == l.imbalance &&
                       l_ref.argmax_device == l.argmax_device,
                   "imbalance");
        }
    }
    // Errors: same exception type and message as the reference.
    const auto curves = random_curves(rng, 4, 512, 64);
    AllocatorConfig cfg;
    std::string ref_msg, got_msg;
    try { maxmin_allocate(curves, 100, cfg); } catch (const std::invalid_argument& e) { ref_msg = e.what(); }
    try { b200::maxmin_allocate(curves, 100, cfg); } catch (const std::invalid_argument& e) { got_msg = e.what(); }
    EXPECT(!ref_msg.empty() && ref_msg == got_msg, "infeasible total: invalid_argument with the reference text");
    ref_msg.clear(), got_msg.clear();
    try { naive_assign({1, 2}, 3); } catch (const std::invalid_argument& e) { ref_msg = e.what(); }
    try { b200::naive_assign({1, 2}, 3); } catch (const std::invalid_argument& e) { got_msg = e.what(); }
    EXPECT(!ref_msg.empty() && ref_msg == got_msg, "devices > heads: invalid_argument with the reference text");
    // imbalance: short assignment, no devices, empty assignment.
    {
        Assignment short_a, no_dev, empty_a;
        short_a.num_devices = 2;
        short_a.device_of_head = {0, 1};
        no_dev.num_devices = -1;
        no_dev.device_of_head = {0, 0, 0};
        empty_a.num_devices = 2;
        for (const Assignment* a : {&short_a, &no_dev, &empty_a}) {
            ref_msg.clear(), got_msg.clear();
            try { imbalance({5, 6, 7}, *a); } catch (const std::invalid_argument& e) { ref_msg = e.what(); }
            try { b200::imbalance({5, 6, 7}, *a); } catch (const std::invalid_argument& e) { got_msg = e.what(); }
            EXPECT(!ref_msg.empty() && ref_msg == got_msg, "imbalance: invalid_argument with the reference text");
        }
    }
    // build_profiles (host path) vs the reference's on a bf16-exact workload.
    {
        std::mt19937_64 r2(11);
        std::normal_distribution<double> N01(0.0, 1.0);
        auto bf = [](double x) { return b200::from_bf16(b200::to_bf16(x)); };
        AttentionWorkload w;
        Matrix K(300, 128), V(300, 128);
        for (auto& x : K.data) x = bf(N01(r2));
        for (auto& x : V.data) x = bf(N01(r2));
        for (int h = 0; h < 4; ++h) {
            HeadData hd{Matrix(6, 128), K, V};
            for (auto& x : hd.Q.data) x = bf(0.2 * N01(r2));
            w.heads.push_back(hd);
        }
        const auto grid = default_budget_grid(300, 32);
        const auto ref = build_profiles(w, grid, SelectionKind::PerQueryTopK, Provenance{"r", "t"});
        const auto got = b200::build_profiles(w, grid);
        double worst = 0.0;
        for (int h = 0; h < 4; ++h)
            for (size_t i = 0; i < grid.size(); ++i)
                worst = std::max(worst, std::fabs(ref[h].curve.points[i].recovery - got[h].points[i].recovery));
        EXPECT(worst < 1e-12, "build_profiles (host) vs reference");
        const auto ref_ca = build_profiles(w, grid, SelectionKind::ColumnAggregateTopK, Provenance{"r", "t"});
        const auto got_ca = b200::build_profiles(w, grid, nullptr, SelectionKind::ColumnAggregateTopK);
        double worst_ca = 0.0;
        for (int h = 0; h < 4; ++h)
            for (size_t i = 0; i < grid.size(); ++i)
                worst_ca = std::max(worst_ca,
                                    std::fabs(ref_ca[h].curve.points[i].recovery - got_ca[h].points[i].recovery));
        EXPECT(worst_ca < 1e-12, "build_profiles ColumnAggregateTopK (host) vs reference");
    }
    std::printf("cpu checks: %d failures\n", failures);
    return failures == 0 ? 0 : 1;
}

static int run_gpu() {
    // 4 q heads sharing 2 K/V pairs (GQA), n = 640, d = 128, values exact in bf16.
    std::mt19937_64 rng(7);
    std::normal_distribution<double> N01(0.0, 1.0);
    auto bf = [](double x) { return b200::from_bf16(b200::to_bf16(x)); };
    const size_t n = 640, d = 128;
    AttentionWorkload w;
    std::vector<Matrix> K(2, Matrix(n, d)), V(2, Matrix(n, d));
    for (int g = 0; g < 2; ++g)
        for (size_t i = 0; i < n * d; ++i) {
            K[g].data[i] = bf(N01(rng));
            V[g].data[i] = bf(N01(rng));
        }
    for (int h = 0; h < 4; ++h) {
        HeadData hd{Matrix(n, d), K[h / 2], V[h / 2]};
        for (auto& x : hd.Q.data) x = bf(0.3 * N01(rng));
        w.heads.push_back(hd);
    }
    b200::Context ctx(0);
    const auto out = b200::sparse_attention_all(ctx, w, std::vector<long>(4, static_cast<long>(n)), true);
    double worst = 0.0;
    for (int h = 0; h < 4; ++h) {
        const auto ref = dense_attention(w.heads[h], true).output;  // full budget == dense
        for (size_t i = 0; i < ref.data.size(); ++i) worst = std::max(worst, std::fabs(ref.data[i] - out[h].data[i]));
    }
    EXPECT(worst <= 2e-2, "GPU layer at full budget vs reference dense_attention (max abs 2e-2)");
    {  // ColumnAggregateTopK at full budget keeps every visible block too
        const auto ca = b200::sparse_attention_all(ctx, w, std::vector<long>(4, static_cast<long>(n)), true,
                                                   SelectionKind::ColumnAggregateTopK);
        bool same = true;
        for (int h = 0; h < 4; ++h) same = same && ca[h].data == out[h].data;
        EXPECT(same, "ColumnAggregateTopK at full budget == PerQueryTopK");
    }
    std::string msg;
    try {
        b200::sparse_attention_all(ctx, w, {0, 1, 1, 1}, true);
    } catch (const std::invalid_argument& e) {
        msg = e.what();
    }
    EXPECT(msg == "head 0: budget k = 0 out of range [1, 640]", "budget range message");
    // build_profiles through the GPU profiler vs the host one (to rounding).
    {
        const auto grid = default_budget_grid(640, 64);
        const auto host = b200::build_profiles(w, grid);
        const auto gpu = b200::build_profiles(w, grid, &ctx);
        double worst_p = 0.0;
        for (size_t h = 0; h < host.size(); ++h)
            for (size_t i = 0; i < grid.size(); ++i)
                worst_p = std::max(worst_p, std::fabs(host[h].points[i].recovery - gpu[h].points[i].recovery));
        EXPECT(worst_p < 1e-12, "build_profiles GPU vs host");
    }
    std::printf("gpu checks: max abs %.3e, %d failures\n", worst, failures);
    return failures == 0 ? 0 : 1;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    return mode == "gpu" ? run_gpu() : run_cpu();
}
