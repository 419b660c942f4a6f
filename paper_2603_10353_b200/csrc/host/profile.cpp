// Offline recovery-curve profiler (budget-table input, not the hot path).
//
// Restates the reference's PerQueryTopK profile: build_profiles
// (proj/src/profiler.cpp:157-196) = dense_attention weights per calibration
// row (attention.cpp:84-114, fp64, max-subtracted softmax) followed by
// recovery_ratio at every grid budget (attention.cpp:151-184: mean over rows
// of the k largest weights). The reference re-selects with nth_element per
// grid point (O(n_k) each); here each row is sorted once and every grid
// point reads a prefix sum, O(n_k log n_k + G) per row. Results agree with
// the reference to rounding (the reference sums the top-k in nth_element's
// arbitrary order); tests/test_host.py pins that. With kind =
// SHPLB_COLUMN_AGGREGATE_TOPK the curve is the ColumnAggregateTopK recovery
// (attention.cpp:172-180): per head, the column sums of the weights over the
// calibration rows, sorted once, prefix-summed at the grid points, / rows.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "../common.hpp"

using namespace shplb;

namespace {

inline double bf16(uint16_t h) {
    uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, sizeof f);
    return static_cast<double>(f);
}

}  // namespace

extern "C" int shplb_profile_curves_host_kind(const uint16_t* q_rows, const uint16_t* k,
                                              int32_t num_q_heads, int32_t num_kv_heads,
                                              int64_t n_rows, int64_t n_k, int32_t d,
                                              const int64_t* grid, int64_t n_grid, int32_t kind,
                                              double* recovery_out) {
    return guarded([&] {
        if (kind != SHPLB_BLOCK_TOPK && kind != SHPLB_COLUMN_AGGREGATE_TOPK)
            throw InvalidArgument("unknown selection kind " + std::to_string(kind));
        require(num_q_heads >= 1 && num_kv_heads >= 1 && num_q_heads % num_kv_heads == 0,
                "num_q_heads must be a positive multiple of num_kv_heads");
        require(n_rows >= 1 && n_k >= 1 && d >= 1, "profile needs at least one row, key and dim");
        if (n_grid < 1) throw InvalidArgument("budget grid is empty");
        for (int64_t i = 0; i < n_grid; ++i) {
            if (grid[i] < 0 || grid[i] > n_k) {
                throw InvalidArgument("budget grid entry " + std::to_string(grid[i]) + " out of [0, " +
                                      std::to_string(n_k) + "]");
            }
            if (i > 0 && grid[i] <= grid[i - 1]) {
                throw InvalidArgument("budget grid must be strictly increasing");
            }
        }
        if (grid[n_grid - 1] != n_k) {
            throw InvalidArgument("budget grid must include the full context length");
        }
        const int32_t group = num_q_heads / num_kv_heads;
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        // Dense softmax weights of calibration row i of head h (dense_attention,
        // attention.cpp:84-114: fp64, max-subtracted, no causal mask).
        auto weights = [&](int64_t h, int64_t i, std::vector<double>& q, std::vector<double>& w) {
            const uint16_t* qr = q_rows + (h * n_rows + i) * d;
            const uint16_t* kh = k + (h / group) * n_k * d;
            for (int32_t c = 0; c < d; ++c) q[c] = bf16(qr[c]);
            double m = -INFINITY;
            for (int64_t j = 0; j < n_k; ++j) {
                const uint16_t* kr = kh + j * d;
                double dot = 0.0;
                for (int32_t c = 0; c < d; ++c) dot += q[c] * bf16(kr[c]);
                w[j] = dot * scale;
                m = std::max(m, w[j]);
            }
            double denom = 0.0;
            for (int64_t j = 0; j < n_k; ++j) {
                w[j] = std::exp(w[j] - m);
                denom += w[j];
            }
            const double inv = 1.0 / denom;
            for (int64_t j = 0; j < n_k; ++j) w[j] *= inv;
        };
        if (kind == SHPLB_COLUMN_AGGREGATE_TOPK) {
            // recovery_ratio, ColumnAggregateTopK (attention.cpp:172-180): the kept
            // set is the top-k column sums of the weights (column_sums, :66-73), and
            // its mass summed over rows is the sum of those k column sums.
#pragma omp parallel
            {
                std::vector<double> w(static_cast<std::size_t>(n_k)), q(static_cast<std::size_t>(d));
                std::vector<double> col(static_cast<std::size_t>(n_k));
#pragma omp for schedule(dynamic)
                for (int32_t h = 0; h < num_q_heads; ++h) {
                    std::fill(col.begin(), col.end(), 0.0);
                    for (int64_t i = 0; i < n_rows; ++i) {  // rows ascending (column_sums order)
                        weights(h, i, q, w);
                        for (int64_t j = 0; j < n_k; ++j) col[j] += w[j];
                    }
                    std::sort(col.begin(), col.end(), std::greater<double>());
                    double run = 0.0;
                    int64_t taken = 0;
                    for (int64_t g = 0; g < n_grid; ++g) {
                        for (; taken < grid[g]; ++taken) run += col[taken];
                        recovery_out[h * n_grid + g] = grid[g] == 0 ? 0.0 : run / static_cast<double>(n_rows);
                    }
                }
            }
            return;
        }

        // Per (head, row) top-k masses at each grid point; summed over rows after.
        std::vector<double> mass(static_cast<std::size_t>(num_q_heads) * n_rows * n_grid);
        const int64_t units = static_cast<int64_t>(num_q_heads) * n_rows;
#pragma omp parallel
        {
            std::vector<double> w(static_cast<std::size_t>(n_k));
            std::vector<double> q(static_cast<std::size_t>(d));
#pragma omp for schedule(dynamic)
            for (int64_t u = 0; u < units; ++u) {
                const int64_t h = u / n_rows, i = u % n_rows;
                weights(h, i, q, w);
                std::sort(w.begin(), w.end(), std::greater<double>());
                double* mrow = mass.data() + u * n_grid;
                double run = 0.0;
                int64_t taken = 0;
                for (int64_t g = 0; g < n_grid; ++g) {
                    for (; taken < grid[g]; ++taken) run += w[taken];
                    mrow[g] = run;
                }
            }
        }
        for (int32_t h = 0; h < num_q_heads; ++h) {
            for (int64_t g = 0; g < n_grid; ++g) {
                double total = 0.0;
                for (int64_t i = 0; i < n_rows; ++i)
                    total += mass[(static_cast<std::size_t>(h) * n_rows + i) * n_grid + g];
                recovery_out[h * n_grid + g] = grid[g] == 0 ? 0.0 : total / static_cast<double>(n_rows);
            }
        }
    });
}

extern "C" int shplb_profile_curves_host(const uint16_t* q_rows, const uint16_t* k, int32_t num_q_heads,
                                         int32_t num_kv_heads, int64_t n_rows, int64_t n_k, int32_t d,
                                         const int64_t* grid, int64_t n_grid, double* recovery_out) {
    return shplb_profile_curves_host_kind(q_rows, k, num_q_heads, num_kv_heads, n_rows, n_k, d, grid, n_grid,
                                          SHPLB_BLOCK_TOPK, recovery_out);
}
