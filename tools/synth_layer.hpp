// Synthetic bf16 layers for the C++ host tools (bench_layer, hp_layer): the
// structure of paper_2603_10353_b200/workload.py with its own RNG (so not the
// same tensors as the Python generator).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace synth {

// splitmix64 -> uniform in (0, 1) -> Box-Muller normals.
struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return (static_cast<double>(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
    float normal() {
        const double u = uniform(), v = uniform();
        return static_cast<float>(std::sqrt(-2.0 * std::log(u)) * std::cos(6.283185307179586 * v));
    }
};

inline uint16_t to_bf16(float x) {  // round to nearest even
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b += 0x7FFF + ((b >> 16) & 1);
    return static_cast<uint16_t>(b >> 16);
}

// One synthetic layer in the spirit of paper_2603_10353_b200/workload.py (its
// own RNG, so not the same tensors): key block b of kv head g has a centroid
// c[g][b]; keys = c + noise; query i of head h = tau_h * (0.5 c[own block] +
// c[a random earlier block] + noise), tau_h log-uniform in [0.15, 1.2].
struct Layer {
    std::vector<uint16_t> q, k, v;  // [Hq][n][d], [Hkv][n][d] x2 (host, pinned by the caller)
};

inline void make_layer(Layer& L, int hq, int hkv, int64_t n, int d, uint64_t seed) {
    const int64_t nb = (n + 127) / 128;
    const int group = hq / hkv;
    #pragma omp parallel for schedule(dynamic)
    for (int g = 0; g < hkv; ++g) {
        Rng r(seed * 1000003 + 17 * g + 1);
        std::vector<float> cent(static_cast<size_t>(nb) * d);
        for (auto& x : cent) x = r.normal();
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < d; ++c) {
                const size_t o = (static_cast<size_t>(g) * n + i) * d + c;
                L.k[o] = to_bf16(cent[static_cast<size_t>(i / 128) * d + c] + r.normal());
                L.v[o] = to_bf16(r.normal());
            }
        for (int hh = 0; hh < group; ++hh) {
            const int h = g * group + hh;
            Rng rq(seed * 7919 + 31 * h + 5);
            const double tau = std::exp(std::log(0.15) + (std::log(1.2) - std::log(0.15)) * rq.uniform());
            for (int64_t i = 0; i < n; ++i) {
                const int64_t own = i / 128;
                const int64_t tgt = static_cast<int64_t>(rq.uniform() * static_cast<double>(own + 1));
                for (int c = 0; c < d; ++c) {
                    const float x = 0.5f * cent[static_cast<size_t>(own) * d + c] +
                                    cent[static_cast<size_t>(tgt) * d + c] + rq.normal();
                    L.q[(static_cast<size_t>(h) * n + i) * d + c] = to_bf16(static_cast<float>(tau) * x);
                }
            }
        }
    }
}


}  // namespace synth
