// Per-head budget table: uniform split and max-min budget shifting.
//
// Behaviour (outputs, tie rules, stopping rules, error messages) follows the
// reference allocator bit for bit — proj/src/allocator.cpp:53-62 (feasibility),
// :72-95 (uniform), :97-186 (max-min) — and its curve lookup
// proj/src/profiler.cpp:55-62 (recovery_at) and curve validation :186-215
// (RecoveryCurve::validate). The implementation differs: curves are held as
// flat arrays and looked up by binary search, so one shifting iteration costs
// O(N + log P) instead of O(N + P).
#include <algorithm>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "../common.hpp"

namespace shplb {
namespace {

constexpr double kCurveSlack = 1e-12;  // profiler.cpp:20
constexpr double kEndpointTol = 1e-9;  // profiler.cpp:21

struct CurveView {
    const int64_t* b;
    const double* r;
    int64_t n;
    // Largest sampled budget <= budget; 0 below the first sample.
    double at(int64_t budget) const {
        const int64_t* it = std::upper_bound(b, b + n, budget);
        return it == b ? 0.0 : r[(it - b) - 1];
    }
    bool sampled(int64_t budget) const { return std::binary_search(b, b + n, budget); }
};

void validate_curve(const CurveView& c, int64_t context_length) {
    // RecoveryCurve::validate (profiler.cpp:186-215), same messages.
    if (c.n == 0) throw InvalidArgument("curve has no points");
    if (context_length < 1) throw InvalidArgument("curve context_length must be >= 1");
    for (int64_t i = 0; i < c.n; ++i) {
        if (c.b[i] < 0 || c.b[i] > context_length) {
            throw InvalidArgument("budget out of [0, n_k] at points[" + std::to_string(i) + "]");
        }
        if (c.r[i] < -kCurveSlack || c.r[i] > 1.0 + kCurveSlack) {
            throw InvalidArgument("recovery out of [0, 1] at points[" + std::to_string(i) + "]");
        }
        if (i > 0) {
            if (c.b[i] <= c.b[i - 1]) throw InvalidArgument("budgets not strictly increasing");
            if (c.r[i] < c.r[i - 1] - kCurveSlack) {
                throw InvalidArgument("recovery decreasing at points[" + std::to_string(i) + "]");
            }
        }
    }
    if (c.b[c.n - 1] != context_length) {
        throw InvalidArgument("final point must sample the full context (k = n_k)");
    }
    if (std::fabs(c.r[c.n - 1] - 1.0) > kEndpointTol) {
        throw InvalidArgument("final recovery must be 1 within 1e-9");
    }
}

void check_feasible(int64_t num_heads, int64_t total, int64_t floor, int64_t context_length) {
    const int64_t lo = num_heads * floor;
    const int64_t hi = num_heads * context_length;
    if (total < lo || total > hi) {
        throw InvalidArgument("total budget " + std::to_string(total) + " infeasible for " +
                              std::to_string(num_heads) + " heads; feasible range is [" +
                              std::to_string(lo) + ", " + std::to_string(hi) + "]");
    }
}

void uniform_split(int64_t n, int64_t total, int64_t floor, int64_t context_length,
                   int64_t* out) {
    if (n < 1) throw InvalidArgument("need at least one head");
    check_feasible(n, total, floor, context_length);
    const int64_t base = total / n, rem = total % n;
    for (int64_t h = 0; h < n; ++h) out[h] = base + (h < rem ? 1 : 0);
}

}  // namespace
}  // namespace shplb

using namespace shplb;

extern "C" int shplb_uniform_allocate(int64_t num_heads, int64_t total, int64_t floor,
                                      int64_t context_length, int64_t* budgets_out) {
    return guarded([&] {
        require(budgets_out != nullptr, "budgets_out is null");
        uniform_split(num_heads, total, floor, context_length, budgets_out);
    });
}

extern "C" int shplb_recovery_at(int64_t n_points, const int64_t* curve_budgets,
                                 const double* curve_recovery, int64_t budget,
                                 double* recovery_out) {
    return guarded([&] {
        require(n_points >= 0 && (n_points == 0 || (curve_budgets && curve_recovery)),
                "bad curve");
        *recovery_out = CurveView{curve_budgets, curve_recovery, n_points}.at(budget);
    });
}

extern "C" int shplb_budget_for_recovery(int64_t n_points, const int64_t* curve_budgets,
                                         const double* curve_recovery, int64_t context_length, double p,
                                         int64_t* budget_out) {
    // budget_for_recovery (profiler.cpp:198-209): the smallest sampled budget
    // whose recovery reaches p (within 1e-9) — the per-head budget of a top-p
    // policy fixed offline. Same validation and messages.
    return guarded([&] {
        require(budget_out != nullptr && (n_points == 0 || (curve_budgets && curve_recovery)), "bad curve");
        const CurveView c{curve_budgets, curve_recovery, n_points};
        validate_curve(c, context_length);
        if (!(p > 0.0) || p > 1.0)
            throw InvalidArgument("recovery target p must lie in (0, 1], got " + std::to_string(p));
        for (int64_t i = 0; i < n_points; ++i) {
            if (curve_recovery[i] >= p - kEndpointTol) {
                *budget_out = curve_budgets[i];
                return;
            }
        }
        double mx = 0.0;
        for (int64_t i = 0; i < n_points; ++i) mx = std::max(mx, curve_recovery[i]);
        throw RuntimeError("recovery target " + std::to_string(p) + " exceeds curve maximum " + std::to_string(mx));
    });
}

extern "C" int shplb_maxmin_allocate(int32_t num_heads, int64_t context_length,
                                     const int64_t* curve_offsets, const int64_t* curve_budgets,
                                     const double* curve_recovery, int64_t total,
                                     int64_t quantum, int64_t floor, int64_t max_iterations,
                                     int64_t* budgets_out, shplb_maxmin_diag* diag) {
    return guarded([&] {
        // AllocatorConfig::validate (allocator.cpp:45-49).
        if (quantum < 1) throw InvalidArgument("transfer quantum must be >= 1");
        if (floor < 0) throw InvalidArgument("budget floor must be >= 0");
        if (max_iterations < 0) throw InvalidArgument("max_iterations must be >= 0");
        if (num_heads < 1) throw InvalidArgument("need at least one recovery curve");
        require(curve_offsets && budgets_out, "null curve or output pointer");

        const auto n = static_cast<std::size_t>(num_heads);
        std::vector<CurveView> curves(n);
        for (std::size_t h = 0; h < n; ++h) {
            curves[h] = CurveView{curve_budgets + curve_offsets[h], curve_recovery + curve_offsets[h],
                                  curve_offsets[h + 1] - curve_offsets[h]};
            validate_curve(curves[h], context_length);
        }
        const int64_t n_k = context_length;
        int64_t* b = budgets_out;
        uniform_split(num_heads, total, floor, n_k, b);

        int64_t off_grid = 0;
        auto recovery = [&](std::size_t h, int64_t budget) {
            if (!curves[h].sampled(budget)) ++off_grid;
            return curves[h].at(budget);
        };
        std::vector<double> r(n);
        for (std::size_t h = 0; h < n; ++h) r[h] = recovery(h, b[h]);

        if (max_iterations == 0) max_iterations = std::max<int64_t>(1, 10 * num_heads * n_k / quantum);
        const double start_min = *std::min_element(r.begin(), r.end());
        double last_min = start_min;

        int64_t transfers = 0, it = 0;
        for (; it < max_iterations; ++it) {
            // Recipient: lowest recovery, ties toward the lower index (allocator.cpp:133-138).
            std::size_t rec = 0;
            for (std::size_t h = 1; h < n; ++h)
                if (r[h] < r[rec]) rec = h;
            const double cur_min = r[rec];
            const int64_t amount = std::min(quantum, n_k - b[rec]);  // :141
            if (amount == 0) break;
            // Donor: highest recovery that stays >= floor, ties to the lower index (:147-153).
            std::size_t donor = n;
            for (std::size_t h = 0; h < n; ++h) {
                if (h == rec || b[h] - amount < floor) continue;
                if (donor == n || r[h] > r[donor]) donor = h;
            }
            if (donor == n) break;
            b[donor] -= amount;
            b[rec] += amount;
            const double rd = recovery(donor, b[donor]);
            const double rr = recovery(rec, b[rec]);
            double new_min = std::numeric_limits<double>::infinity();
            for (std::size_t h = 0; h < n; ++h) {
                const double rh = h == donor ? rd : h == rec ? rr : r[h];
                new_min = std::min(new_min, rh);
            }
            if (!(new_min > cur_min)) {  // must strictly raise the worst head (:169-175)
                b[donor] += amount;
                b[rec] -= amount;
                break;
            }
            r[donor] = rd;
            r[rec] = rr;
            ++transfers;
            last_min = new_min;
        }
        if (diag) {
            diag->transfers = transfers;
            diag->hit_iteration_cap = it == max_iterations ? 1 : 0;
            diag->off_grid_evaluations = off_grid;
            diag->min_recovery_start = start_min;
            diag->min_recovery_end = last_min;
        }
    });
}
