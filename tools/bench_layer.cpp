// C++ host driver over the C ABI alone (include/shplb.h + libshplb.so): the
// B200 counterpart of the reference's bench/bench_attention.cpp, which times
// headbal::sparse_attention_all (OpenMP, fp64) against the serial reference.
// Here one process per GPU runs the S-HPLB pipeline the way a C++ serving host
// would: synthetic bf16 layers generated on the host, calibration-row recovery
// curves on the GPU (shplb_profile_curves), the max-min budget table
// (shplb_maxmin_allocate), then the layer call timed with CUDA events on device
// buffers (shplb_sparse_attention_layer) and end to end on pinned host buffers
// (shplb_sparse_attention_layer_host_async, copies inside the timed region).
//
// usage: bench_layer [seq_len=131072] [layers=4] [repeats=3] [q_heads=32] [kv_heads=8]
// Prints a table and one JSON line.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "shplb.h"
#include "synth_layer.hpp"

namespace {
using synth::Layer;
using synth::make_layer;

void check(int status, const char* what) {
    if (status != SHPLB_OK) throw std::runtime_error(std::string(what) + ": " + shplb_last_error());
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const int64_t n = argc > 1 ? std::atoll(argv[1]) : 131072;
        const int layers = argc > 2 ? std::atoi(argv[2]) : 4;
        const int repeats = argc > 3 ? std::atoi(argv[3]) : 3;
        const int hq = argc > 4 ? std::atoi(argv[4]) : 32;
        const int hkv = argc > 5 ? std::atoi(argv[5]) : 8;
        const int d = 128, calib = 128;
        const double fraction = 0.25;
        std::printf("%s\n", shplb_version());

        shplb_ctx* ctx = nullptr;
        check(shplb_ctx_create(0, &ctx), "shplb_ctx_create");
        cudaStream_t st;
        cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");

        const size_t qe = static_cast<size_t>(hq) * n * d, ke = static_cast<size_t>(hkv) * n * d;
        std::vector<Layer> host(static_cast<size_t>(layers));
        std::vector<std::vector<int64_t>> budgets(static_cast<size_t>(layers));
        uint16_t *dcal, *dout;  // calibration rows [Hq][calib][d]; layer output
        cuda(cudaMalloc(&dcal, static_cast<size_t>(hq) * calib * d * 2), "malloc");
        cuda(cudaMalloc(&dout, qe * 2), "malloc");
        std::vector<uint16_t*> dev_in(static_cast<size_t>(layers) * 3);
        std::vector<uint16_t*> pinned_out(static_cast<size_t>(layers));

        // default_budget_grid(n, 128) (commands.cpp:236-238): 0, 128, ..., n
        std::vector<int64_t> grid;
        for (int64_t b = 0; b < n; b += 128) grid.push_back(b);
        grid.push_back(n);
        const int64_t total = static_cast<int64_t>(std::llround(fraction * hq * static_cast<double>(n)));
        double flops_sum = 0.0;
        for (int l = 0; l < layers; ++l) {
            Layer& L = host[static_cast<size_t>(l)];
            L.q.resize(qe);
            L.k.resize(ke);
            L.v.resize(ke);
            make_layer(L, hq, hkv, n, d, 2603 + 7919ull * l);
            for (auto* p : {&L.q, &L.k, &L.v})
                cuda(cudaHostRegister(p->data(), p->size() * 2, cudaHostRegisterDefault), "pin");
            cuda(cudaMallocHost(&pinned_out[static_cast<size_t>(l)], qe * 2), "pinned out");
            uint16_t *q, *k, *v;  // each layer resident on the device for the device-buffer timing
            cuda(cudaMalloc(&q, qe * 2), "malloc");
            cuda(cudaMalloc(&k, ke * 2), "malloc");
            cuda(cudaMalloc(&v, ke * 2), "malloc");
            cuda(cudaMemcpy(q, L.q.data(), qe * 2, cudaMemcpyHostToDevice), "h2d");
            cuda(cudaMemcpy(k, L.k.data(), ke * 2, cudaMemcpyHostToDevice), "h2d");
            cuda(cudaMemcpy(v, L.v.data(), ke * 2, cudaMemcpyHostToDevice), "h2d");
            dev_in[3 * l] = q;
            dev_in[3 * l + 1] = k;
            dev_in[3 * l + 2] = v;
            // calibration rows: `calib` rows evenly spaced through the sequence
            // (round(linspace(0, n-1, calib)), as calibrate.calibration_rows)
            for (int h = 0; h < hq; ++h)
                for (int r = 0; r < calib; ++r) {
                    const int64_t pos = calib > 1 ? std::llround(static_cast<double>(r) * (n - 1) / (calib - 1)) : n - 1;
                    cuda(cudaMemcpy(dcal + (static_cast<size_t>(h) * calib + r) * d,
                                    q + (static_cast<size_t>(h) * n + pos) * d, d * 2, cudaMemcpyDeviceToDevice),
                         "calib");
                }
            std::vector<double> rec(static_cast<size_t>(hq) * grid.size());
            check(shplb_profile_curves(ctx, dcal, k, hq, hkv, calib, n, d, grid.data(),
                                       static_cast<int64_t>(grid.size()), rec.data(), st),
                  "shplb_profile_curves");
            std::vector<int64_t> off(static_cast<size_t>(hq) + 1), cb;
            for (int h = 0; h < hq; ++h) {
                off[h + 1] = off[h] + static_cast<int64_t>(grid.size());
                cb.insert(cb.end(), grid.begin(), grid.end());
            }
            auto& b = budgets[static_cast<size_t>(l)];
            b.resize(static_cast<size_t>(hq));
            shplb_maxmin_diag diag{};
            check(shplb_maxmin_allocate(hq, n, off.data(), cb.data(), rec.data(), total, 128, 128, 0, b.data(), &diag),
                  "shplb_maxmin_allocate");
            shplb_layer_shape s{};
            s.num_q_heads = hq;
            s.num_kv_heads = hkv;
            s.seq_len = n;
            s.head_dim = d;
            s.block_q = 256;
            s.block_k = 128;
            s.causal = 1;
            s.kind = SHPLB_BLOCK_TOPK;
            int64_t tiles = 0;
            double flops = 0.0;
            check(shplb_layer_work(&s, b.data(), &tiles, &flops), "shplb_layer_work");
            flops_sum += flops;
            std::printf("layer %d: budgets %lld..%lld tokens, min recovery %.3f (uniform %.3f)\n", l,
                        static_cast<long long>(*std::min_element(b.begin(), b.end())),
                        static_cast<long long>(*std::max_element(b.begin(), b.end())), diag.min_recovery_end,
                        diag.min_recovery_start);
        }
        shplb_layer_shape s{};
        s.num_q_heads = hq;
        s.num_kv_heads = hkv;
        s.seq_len = n;
        s.head_dim = d;
        s.block_q = 256;
        s.block_k = 128;
        s.causal = 1;
        s.kind = SHPLB_BLOCK_TOPK;

        cudaEvent_t e0, e1;
        cuda(cudaEventCreate(&e0), "event");
        cuda(cudaEventCreate(&e1), "event");
        auto device_pass = [&] {
            for (int l = 0; l < layers; ++l)
                check(shplb_sparse_attention_layer(ctx, &s, dev_in[3 * l], dev_in[3 * l + 1], dev_in[3 * l + 2],
                                                   budgets[static_cast<size_t>(l)].data(), dout, st),
                      "shplb_sparse_attention_layer");
        };
        auto host_pass = [&] {
            for (int l = 0; l < layers; ++l) {
                Layer& L = host[static_cast<size_t>(l)];
                check(shplb_sparse_attention_layer_host_async(ctx, &s, L.q.data(), L.k.data(), L.v.data(),
                                                              budgets[static_cast<size_t>(l)].data(),
                                                              pinned_out[static_cast<size_t>(l)], st),
                      "shplb_sparse_attention_layer_host_async");
            }
        };
        auto timed = [&](auto&& pass) {
            pass();  // warm-up
            cuda(cudaStreamSynchronize(st), "sync");
            float best = 1e30f;
            for (int r = 0; r < repeats; ++r) {
                cuda(cudaEventRecord(e0, st), "record");
                pass();
                cuda(cudaEventRecord(e1, st), "record");
                cuda(cudaEventSynchronize(e1), "sync");
                float ms = 0.f;
                cuda(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
                best = std::min(best, ms);
            }
            return best / layers;
        };
        const int64_t launches0 = shplb_ctx_launch_count(ctx);
        const float dev_ms = timed(device_pass);
        const int64_t launches_per_layer = (shplb_ctx_launch_count(ctx) - launches0) / ((repeats + 1) * layers);
        const float host_ms = timed(host_pass);
        const double tflops = flops_sum / layers / (dev_ms * 1e-3) / 1e12;

        std::printf("%-44s %14s %14s %9s\n", "case", "device (ms)", "host buf (ms)", "TFLOP/s");
        std::printf("Hq=%-3d Hkv=%-2d n=%-7lld d=%d causal, %d layers %14.3f %14.3f %9.1f\n", hq, hkv,
                    static_cast<long long>(n), d, layers, dev_ms, host_ms, tflops);
        std::printf("{\"tool\": \"bench_layer\", \"seq_len\": %lld, \"q_heads\": %d, \"kv_heads\": %d, "
                    "\"layers\": %d, \"device_ms_per_layer\": %.3f, \"host_buffers_ms_per_layer\": %.3f, "
                    "\"tflops\": %.1f, \"launches_per_layer\": %lld}\n",
                    static_cast<long long>(n), hq, hkv, layers, dev_ms, host_ms, tflops,
                    static_cast<long long>(launches_per_layer));

        for (auto* p : dev_in) cudaFree(p);
        for (auto* p : pinned_out) cudaFreeHost(p);
        for (auto& L : host)
            for (auto* p : {&L.q, &L.k, &L.v}) cudaHostUnregister(p->data());
        cudaFree(dcal);
        cudaFree(dout);
        check(shplb_ctx_destroy(ctx), "shplb_ctx_destroy");
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bench_layer: %s\n", e.what());
        return 1;
    }
}
