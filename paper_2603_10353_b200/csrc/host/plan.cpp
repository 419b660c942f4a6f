// Head -> GPU plan and the barrier metric.
//
// naive / greedy / imbalance follow the reference partitioner bit for bit
// (proj/src/partitioner.cpp:130-183, :236-266, incl. its error messages);
// simulate / barrier follow proj/src/simulator.cpp:13-47. greedy_assign is the
// LPT rule: heads by (budget desc, index asc), each placed on the device with
// the smallest (load, device index) — the pair order the reference's
// std::priority_queue<pair<long,int>, ..., greater<>> pops.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <queue>
#include <string>
#include <utility>
#include <vector>

#include "../common.hpp"

using namespace shplb;

namespace {

void check_budgets(const int64_t* budgets, int32_t n) {
    if (n < 1) throw InvalidArgument("need at least one head");
    require(budgets != nullptr, "budgets is null");
    for (int32_t h = 0; h < n; ++h)
        if (budgets[h] < 0) throw InvalidArgument("budgets must be nonnegative");
}

// Can `items` (sorted descending) be added to `loads` with every load <= cap?
// Depth-first, largest item first; devices with equal loads are interchangeable,
// so only the first of each equal-load run is tried.
bool fits(const std::vector<int64_t>& items, std::size_t i, std::vector<int64_t>& loads, int64_t cap) {
    if (i == items.size()) return true;
    for (std::size_t d = 0; d < loads.size(); ++d) {
        bool seen = false;
        for (std::size_t e = 0; e < d; ++e) seen |= loads[e] == loads[d];
        if (seen || loads[d] + items[i] > cap) continue;
        loads[d] += items[i];
        const bool ok = fits(items, i + 1, loads, cap);
        loads[d] -= items[i];
        if (ok) return true;
    }
    return false;
}

}  // namespace

extern "C" int shplb_plan_optimal(const int64_t* budgets, int32_t num_heads, int32_t devices,
                                  int32_t* device_of_head) {
    // optimal_assign (partitioner.cpp:185-234): the minimum possible maximum
    // device load, and among the plans reaching it the lexicographically
    // smallest device_of_head. Both are properties of the instance, so any
    // exact search returns the reference's plan; this one binary-searches the
    // cap between max(ceil(total/D), max budget) and the greedy plan's maximum
    // with an exact feasibility search, then fixes heads in index order on the
    // lowest device that keeps the rest feasible.
    return guarded([&] {
        check_budgets(budgets, num_heads);
        if (devices < 1) throw InvalidArgument("need at least one device");
        if (num_heads > 24 || devices > 4) {
            throw InvalidArgument(
                "exact solver is guarded to N <= 24 heads and 4 devices; use greedy_assign for larger instances");
        }
        const int64_t total = std::accumulate(budgets, budgets + num_heads, int64_t(0));
        int64_t lo = std::max((total + devices - 1) / devices, *std::max_element(budgets, budgets + num_heads));
        std::vector<int32_t> g(static_cast<std::size_t>(num_heads));
        const int rc = shplb_plan_greedy(budgets, num_heads, devices, g.data());
        if (rc != SHPLB_OK) throw std::logic_error("greedy seed failed");
        std::vector<int64_t> gl(static_cast<std::size_t>(devices), 0);
        for (int32_t h = 0; h < num_heads; ++h) gl[g[h]] += budgets[h];
        int64_t hi = *std::max_element(gl.begin(), gl.end());
        std::vector<int64_t> items(budgets, budgets + num_heads);
        std::sort(items.begin(), items.end(), std::greater<int64_t>());
        while (lo < hi) {  // smallest feasible cap
            const int64_t mid = lo + (hi - lo) / 2;
            std::vector<int64_t> loads(static_cast<std::size_t>(devices), 0);
            if (fits(items, 0, loads, mid)) hi = mid; else lo = mid + 1;
        }
        const int64_t best = lo;
        std::vector<int64_t> loads(static_cast<std::size_t>(devices), 0);
        for (int32_t h = 0; h < num_heads; ++h) {
            std::vector<int64_t> rest(budgets + h + 1, budgets + num_heads);
            std::sort(rest.begin(), rest.end(), std::greater<int64_t>());
            bool placed = false;
            for (int32_t d = 0; d < devices && !placed; ++d) {
                if (loads[d] + budgets[h] > best) continue;
                loads[d] += budgets[h];
                std::vector<int64_t> trial(loads);
                if (fits(rest, 0, trial, best)) {
                    device_of_head[h] = d;
                    placed = true;
                } else {
                    loads[d] -= budgets[h];
                }
            }
            if (!placed) throw std::logic_error("exact solver lost feasibility");  // unreachable
        }
    });
}

extern "C" int shplb_plan_naive(const int64_t* budgets, int32_t num_heads, int32_t devices,
                                int32_t round_robin, int32_t* device_of_head) {
    return guarded([&] {
        check_budgets(budgets, num_heads);
        if (devices < 1) throw InvalidArgument("need at least one device");
        if (devices > num_heads) {
            throw InvalidArgument("device count " + std::to_string(devices) +
                                  " exceeds head count " + std::to_string(num_heads));
        }
        if (round_robin) {
            for (int32_t h = 0; h < num_heads; ++h) device_of_head[h] = h % devices;
            return;
        }
        // Contiguous blocks; the first N mod D devices take the ceil-size block.
        const int32_t base = num_heads / devices, extra = num_heads % devices;
        int32_t next = 0;
        for (int32_t d = 0; d < devices; ++d)
            for (int32_t i = 0; i < base + (d < extra ? 1 : 0); ++i) device_of_head[next++] = d;
    });
}

extern "C" int shplb_plan_greedy(const int64_t* budgets, int32_t num_heads, int32_t devices,
                                 int32_t* device_of_head) {
    return guarded([&] {
        check_budgets(budgets, num_heads);
        if (devices < 1) throw InvalidArgument("need at least one device");
        std::vector<int32_t> order(static_cast<std::size_t>(num_heads));
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t a, int32_t b) { return budgets[a] > budgets[b]; });
        using Slot = std::pair<int64_t, int32_t>;  // (load, device), min first
        std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> q;
        for (int32_t d = 0; d < devices; ++d) q.emplace(0, d);
        for (int32_t h : order) {
            const auto [load, dev] = q.top();
            q.pop();
            device_of_head[h] = dev;
            q.emplace(load + budgets[h], dev);
        }
    });
}

// Whole-head local search (extension; the reference stops at greedy_assign, and
// its exact optimal_assign is guarded to 24 heads / 4 devices). Each step takes
// the most loaded device (lowest index among ties) and applies the move of one of
// its heads to another device, or the swap of one of its heads with a lighter
// head elsewhere, that gives the lowest max over the two devices touched — first
// found wins ties (heads ascending, devices ascending, move before swaps). A step
// is taken only if that max is below the current maximum load, so the sum of
// squared loads falls strictly and the search ends; loads are integers, so it is
// deterministic and platform-independent.
extern "C" int shplb_plan_refine(const int64_t* costs, int32_t num_heads, int32_t devices,
                                 int32_t* device_of_head, int64_t* loads_out) {
    return guarded([&] {
        check_budgets(costs, num_heads);
        if (devices < 1) throw InvalidArgument("need at least one device");
        require(device_of_head != nullptr, "device_of_head is null");
        std::vector<int64_t> load(static_cast<std::size_t>(devices), 0);
        for (int32_t h = 0; h < num_heads; ++h) {
            const int32_t d = device_of_head[h];
            if (d < 0 || d >= devices) throw InvalidArgument("device index out of range");
            load[static_cast<std::size_t>(d)] += costs[h];
        }
        for (;;) {
            const auto top = std::max_element(load.begin(), load.end());  // first of the maxima
            const int32_t dm = static_cast<int32_t>(top - load.begin());
            const int64_t lmax = *top;
            int64_t best = lmax;
            int32_t bi = -1, be = -1, bj = -1;
            for (int32_t i = 0; i < num_heads; ++i) {
                if (device_of_head[i] != dm || costs[i] == 0) continue;
                for (int32_t e = 0; e < devices; ++e) {
                    if (e == dm) continue;
                    const int64_t le = load[static_cast<std::size_t>(e)];
                    const int64_t mv = std::max(lmax - costs[i], le + costs[i]);
                    if (mv < best) best = mv, bi = i, be = e, bj = -1;
                    for (int32_t j = 0; j < num_heads; ++j) {
                        if (device_of_head[j] != e || costs[j] >= costs[i]) continue;
                        const int64_t sw = std::max(lmax - costs[i] + costs[j], le - costs[j] + costs[i]);
                        if (sw < best) best = sw, bi = i, be = e, bj = j;
                    }
                }
            }
            if (bi < 0) break;
            load[static_cast<std::size_t>(dm)] -= costs[bi];
            load[static_cast<std::size_t>(be)] += costs[bi];
            device_of_head[bi] = be;
            if (bj >= 0) {
                load[static_cast<std::size_t>(be)] -= costs[bj];
                load[static_cast<std::size_t>(dm)] += costs[bj];
                device_of_head[bj] = dm;
            }
        }
        if (loads_out) std::copy(load.begin(), load.end(), loads_out);
    });
}

extern "C" int shplb_plan_split_weighted(const int64_t* budgets, int32_t num_heads, int64_t seq_len,
                                         int32_t block_q, int32_t causal, int32_t devices,
                                         int64_t query_tile_weight, int32_t max_segments, int32_t* seg_device,
                                         int32_t* seg_head, int32_t* seg_qb_begin, int32_t* seg_qb_end,
                                         int32_t* n_segments, int64_t* loads_out) {
    return guarded([&] {
        check_budgets(budgets, num_heads);
        if (query_tile_weight < 0) throw InvalidArgument("query_tile_weight must be nonnegative");
        if (devices < 1) throw InvalidArgument("need at least one device");
        if (seq_len < 1) throw InvalidArgument("K must hold at least one key token");
        if (block_q != 128 && block_q != 256) throw InvalidArgument("block_q must be 128 or 256");
        require(seg_device && seg_head && seg_qb_begin && seg_qb_end && n_segments && loads_out,
                "null output pointer");
        constexpr int64_t bk = 128;
        const int64_t nqb = (seq_len + block_q - 1) / block_q, nkb = (seq_len + bk - 1) / bk;
        // Tiles kernel 3 computes for (head h, query block qb) before selection
        // (include/shplb.h, shplb_layer_work), plus query_tile_weight per visited
        // query half (kernel 3's per-tile fixed cost in tile equivalents).
        auto cost = [&](int32_t h, int64_t qb) -> int64_t {
            int64_t vis = nkb;
            if (causal) vis = std::min(nkb, (std::min((qb + 1) * block_q, seq_len) - 1) / bk + 1);
            const int64_t k = std::min(nkb, (budgets[h] + bk - 1) / bk);
            int64_t halves = 0;
            for (int64_t hf = 0; hf < block_q / bk; ++hf) halves += qb * block_q + hf * bk < seq_len;
            const int64_t kept = std::min(k, vis);
            return kept * halves + (kept > 0 ? query_tile_weight * halves : 0);
        };
        int64_t total = 0;
        for (int32_t h = 0; h < num_heads; ++h)
            for (int64_t qb = 0; qb < nqb; ++qb) total += cost(h, qb);
        // Walk heads in index order (GQA groups stay contiguous, so ranks need
        // few kv heads); device d takes the units whose cost midpoint falls in
        // [d*total/D, (d+1)*total/D) of the running prefix, so every load is
        // within half a query block's cost of total/D.
        std::fill(loads_out, loads_out + devices, 0);
        int32_t nseg = 0, d = 0;
        int64_t prefix = 0;
        auto emit = [&](int32_t h, int64_t b, int64_t e) {
            if (e <= b) return;
            if (nseg >= max_segments) throw InvalidArgument("max_segments too small for the split plan");
            seg_device[nseg] = d;
            seg_head[nseg] = h;
            seg_qb_begin[nseg] = static_cast<int32_t>(b);
            seg_qb_end[nseg] = static_cast<int32_t>(e);
            ++nseg;
        };
        for (int32_t h = 0; h < num_heads; ++h) {
            int64_t begin = 0;
            for (int64_t qb = 0; qb < nqb; ++qb) {
                const int64_t c = cost(h, qb);
                // Midpoint of this unit, in units of total/D (scaled by 2*devices to stay integral).
                while (d < devices - 1 && (2 * prefix + c) * devices >= 2 * total * (d + 1)) {
                    emit(h, begin, qb);
                    begin = qb;
                    ++d;
                }
                prefix += c;
                loads_out[d] += c;
            }
            emit(h, begin, nqb);
        }
        *n_segments = nseg;
    });
}

extern "C" int shplb_plan_split(const int64_t* budgets, int32_t num_heads, int64_t seq_len,
                                int32_t block_q, int32_t causal, int32_t devices,
                                int32_t max_segments, int32_t* seg_device, int32_t* seg_head,
                                int32_t* seg_qb_begin, int32_t* seg_qb_end, int32_t* n_segments,
                                int64_t* loads_out) {
    return shplb_plan_split_weighted(budgets, num_heads, seq_len, block_q, causal, devices, 0, max_segments,
                                     seg_device, seg_head, seg_qb_begin, seg_qb_end, n_segments, loads_out);
}

extern "C" int shplb_imbalance(const int64_t* budgets, int32_t num_heads,
                               const int32_t* device_of_head, int32_t devices, int64_t* loads_out,
                               int64_t* total_out, double* imbalance_out, int32_t* argmax_out) {
    return guarded([&] {
        // Assignment::validate (partitioner.cpp:38-48).
        if (devices < 1) throw InvalidArgument("need at least one device");
        if (num_heads < 1) throw InvalidArgument("assignment covers no heads");
        for (int32_t h = 0; h < num_heads; ++h) {
            if (device_of_head[h] < 0 || device_of_head[h] >= devices) {
                throw InvalidArgument("head " + std::to_string(h) + " assigned to invalid device " +
                                      std::to_string(device_of_head[h]));
            }
        }
        check_budgets(budgets, num_heads);
        int64_t total = 0;
        std::fill(loads_out, loads_out + devices, 0);
        for (int32_t h = 0; h < num_heads; ++h) {
            loads_out[device_of_head[h]] += budgets[h];
            total += budgets[h];
        }
        int64_t mx = loads_out[0];
        int32_t am = 0;
        for (int32_t d = 1; d < devices; ++d)
            if (loads_out[d] > mx) {
                mx = loads_out[d];
                am = d;
            }
        if (total_out) *total_out = total;
        if (argmax_out) *argmax_out = am;
        if (imbalance_out) {
            *imbalance_out = total == 0 ? 1.0
                                        : static_cast<double>(mx) * static_cast<double>(devices) /
                                              static_cast<double>(total);
        }
    });
}

extern "C" int shplb_simulate(const int64_t* loads, int32_t devices, double alpha, double beta,
                              double* latency_out, double* barrier_out, double* bubble_out) {
    return guarded([&] {
        // CostModel::validate (simulator.cpp:13-20).
        if (!(beta > 0.0) || !std::isfinite(beta)) throw InvalidArgument("cost model beta must be > 0");
        if (alpha < 0.0 || !std::isfinite(alpha)) throw InvalidArgument("cost model alpha must be >= 0");
        if (devices < 1) throw InvalidArgument("load report has no devices");
        std::vector<double> lat(static_cast<std::size_t>(devices));
        double sum = 0.0;
        for (int32_t d = 0; d < devices; ++d) {
            lat[d] = alpha + beta * static_cast<double>(loads[d]);
            sum += lat[d];
        }
        const double T = *std::max_element(lat.begin(), lat.end());
        if (latency_out) std::copy(lat.begin(), lat.end(), latency_out);
        if (barrier_out) *barrier_out = T;
        if (bubble_out) *bubble_out = T == 0.0 ? 0.0 : 1.0 - (sum / static_cast<double>(devices)) / T;
    });
}

extern "C" int shplb_barrier(const double* device_latency, int32_t devices, double* barrier_out,
                             double* bubble_out) {
    return guarded([&] {
        if (devices < 1) throw InvalidArgument("load report has no devices");
        double sum = 0.0;
        for (int32_t d = 0; d < devices; ++d) sum += device_latency[d];
        const double T = *std::max_element(device_latency, device_latency + devices);
        if (barrier_out) *barrier_out = T;
        if (bubble_out) *bubble_out = T == 0.0 ? 0.0 : 1.0 - (sum / static_cast<double>(devices)) / T;
    });
}
