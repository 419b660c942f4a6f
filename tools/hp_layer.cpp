// Head-parallel layer from a C++ host, one process per rank, over the C ABI
// alone (include/shplb.h + libshplb.so; no Python, no torch.distributed) —
// the paper's S-HPLB placement as a serving host would run it:
//
//   plan     shplb_plan_greedy (greedy_assign, partitioner.cpp:164-183),
//            shplb_plan_naive (even head parallelism), refined (greedy on tile
//            cost + shplb_plan_refine) or shplb_plan_split_weighted (sub-head
//            balancer, 4 tiles per query tile), the same on every rank;
//   shard    this rank's q heads + the kv heads they read (kv map), and for the
//            split plan each head's query-block range, through
//            shplb_sparse_attention_layer into a local [h_r][n][d] buffer;
//   gather   shplb_gather_heads / shplb_gather_segments over an NCCL
//            communicator of the library (unique id shipped through a file),
//            every rank ending with the whole [Hq][n][d] output;
//   check    bytewise against the single-rank layer call of the whole layer
//            (the reassembly must be bit-identical: heads are independent,
//            attention.cpp:204-223).
//
// env: RANK, WORLD_SIZE (default 0 / 1), LOCAL_RANK (device, default RANK mod
// device count), SHPLB_ID_FILE (unique-id exchange file, default /tmp/shplb_hp.id;
// give every launch its own path — a rank reads whatever id file it finds).
// usage: hp_layer [plan=greedy|naive|refined|split] [seq_len=16384] [q_heads=32] [kv_heads=8]
// Prints one JSON line per rank.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "shplb.h"
#include "synth_layer.hpp"

namespace {

void check(int status, const char* what) {
    if (status != SHPLB_OK) throw std::runtime_error(std::string(what) + ": " + shplb_last_error());
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// Rank 0 writes the NCCL unique id to `path` (atomically via rename); the
// other ranks wait for it.
std::vector<char> exchange_id(const std::string& path, int rank) {
    std::vector<char> id(SHPLB_NCCL_UNIQUE_ID_BYTES);
    if (rank == 0) {
        check(shplb_nccl_get_unique_id(id.data(), id.size()), "shplb_nccl_get_unique_id");
        const std::string tmp = path + ".tmp";
        std::ofstream(tmp, std::ios::binary).write(id.data(), static_cast<std::streamsize>(id.size()));
        if (std::rename(tmp.c_str(), path.c_str()) != 0) throw std::runtime_error("cannot publish " + path);
        return id;
    }
    for (int i = 0; i < 6000; ++i) {
        std::ifstream f(path, std::ios::binary);
        if (f && f.read(id.data(), static_cast<std::streamsize>(id.size()))) return id;
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    throw std::runtime_error("timed out waiting for " + path);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const std::string plan = argc > 1 ? argv[1] : "greedy";
        const int64_t n = argc > 2 ? std::atoll(argv[2]) : 16384;
        const int hq = argc > 3 ? std::atoi(argv[3]) : 32;
        const int hkv = argc > 4 ? std::atoi(argv[4]) : 8;
        const int d = 128, group = hq / hkv, bq = 256;
        const int rank = env_int("RANK", 0), world = env_int("WORLD_SIZE", 1);
        int ndev = 0;
        cuda(cudaGetDeviceCount(&ndev), "device count");
        const int device = env_int("LOCAL_RANK", rank % std::max(ndev, 1));
        cuda(cudaSetDevice(device), "set device");
        const char* idf = std::getenv("SHPLB_ID_FILE");
        const std::string id_path = idf ? idf : "/tmp/shplb_hp.id";

        // The layer (every rank generates the same one) and a heterogeneous budget table.
        synth::Layer L;
        const size_t qe = static_cast<size_t>(hq) * n * d, ke = static_cast<size_t>(hkv) * n * d;
        L.q.resize(qe);
        L.k.resize(ke);
        L.v.resize(ke);
        synth::make_layer(L, hq, hkv, n, d, 2603);
        std::vector<int64_t> budgets(static_cast<size_t>(hq));
        for (int h = 0; h < hq; ++h) budgets[h] = std::min<int64_t>(n, 128 * (1 + (7 * h + 3) % 29) * (n / 8192 + 1));

        uint16_t *q, *k, *v, *ref, *out, *local;
        cuda(cudaMalloc(&q, qe * 2), "malloc");
        cuda(cudaMalloc(&k, ke * 2), "malloc");
        cuda(cudaMalloc(&v, ke * 2), "malloc");
        cuda(cudaMalloc(&ref, qe * 2), "malloc");
        cuda(cudaMalloc(&out, qe * 2), "malloc");
        cuda(cudaMemcpy(q, L.q.data(), qe * 2, cudaMemcpyHostToDevice), "h2d");
        cuda(cudaMemcpy(k, L.k.data(), ke * 2, cudaMemcpyHostToDevice), "h2d");
        cuda(cudaMemcpy(v, L.v.data(), ke * 2, cudaMemcpyHostToDevice), "h2d");
        cuda(cudaMemset(out, 0xFF, qe * 2), "memset");  // NaN pattern: every row must be overwritten

        shplb_ctx* ctx = nullptr;
        check(shplb_ctx_create(device, &ctx), "shplb_ctx_create");
        cudaStream_t st;
        cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        shplb_layer_shape full{};
        full.num_q_heads = hq;
        full.num_kv_heads = hkv;
        full.seq_len = n;
        full.head_dim = d;
        full.block_q = bq;
        full.block_k = 128;
        full.causal = 1;
        full.kind = SHPLB_BLOCK_TOPK;
        check(shplb_sparse_attention_layer(ctx, &full, q, k, v, budgets.data(), ref, st), "full layer");

        // The plan, identical on every rank.
        std::vector<shplb_out_segment> segs;
        std::vector<int32_t> dev_of_head(static_cast<size_t>(hq));
        if (plan == "split") {
            const int maxs = hq + world;
            std::vector<int32_t> sd(maxs), sh(maxs), sb(maxs), se(maxs);
            std::vector<int64_t> loads(static_cast<size_t>(world));
            int32_t ns = 0;
            check(shplb_plan_split_weighted(budgets.data(), hq, n, bq, 1, world, 4, maxs, sd.data(), sh.data(), sb.data(),
                                   se.data(), &ns, loads.data()),
                  "shplb_plan_split_weighted");
            for (int r = 0; r < world; ++r) {  // a rank's local layout: its segments in head order
                std::vector<int> mine;
                for (int i = 0; i < ns; ++i)
                    if (sd[i] == r) mine.push_back(i);
                std::stable_sort(mine.begin(), mine.end(), [&](int a, int b) { return sh[a] < sh[b]; });
                for (size_t li = 0; li < mine.size(); ++li) {
                    const int i = mine[li];
                    const int64_t r0 = int64_t(sb[i]) * bq, r1 = std::min<int64_t>(int64_t(se[i]) * bq, n);
                    if (r1 > r0) segs.push_back({sh[i], r, static_cast<int32_t>(li), 0, r0, r1});
                }
            }
        } else {
            if (plan == "greedy") {
                check(shplb_plan_greedy(budgets.data(), hq, world, dev_of_head.data()), "shplb_plan_greedy");
            } else if (plan == "naive") {
                check(shplb_plan_naive(budgets.data(), hq, world, 0, dev_of_head.data()), "shplb_plan_naive");
            } else if (plan == "refined") {
                // greedy on kernel 3's per-head tile cost + 4 tiles per visited query
                // tile (api.QUERY_TILE_WEIGHT), then whole-head local search
                std::vector<int64_t> cost(static_cast<size_t>(hq));
                shplb_layer_shape one = full;
                one.num_q_heads = one.num_kv_heads = 1;
                const int64_t one_block = 128;  // one key block per query block: tiles = query tiles
                int64_t qtiles = 0;
                check(shplb_layer_work(&one, &one_block, &qtiles, nullptr), "shplb_layer_work");
                for (int h = 0; h < hq; ++h) {
                    check(shplb_layer_work(&one, &budgets[h], &cost[h], nullptr), "shplb_layer_work");
                    cost[h] += 4 * qtiles;
                }
                check(shplb_plan_greedy(cost.data(), hq, world, dev_of_head.data()), "shplb_plan_greedy");
                check(shplb_plan_refine(cost.data(), hq, world, dev_of_head.data(), nullptr), "shplb_plan_refine");
            } else {
                throw std::runtime_error("plan must be greedy, naive, refined or split");
            }
            std::vector<int32_t> next(static_cast<size_t>(world), 0);
            for (int h = 0; h < hq; ++h) segs.push_back({h, dev_of_head[h], next[dev_of_head[h]]++, 0, 0, n});
        }

        // This rank's shard: q heads (ascending, as in segs), kv heads, kv map, query-block ranges.
        std::vector<int32_t> heads, ranges, kv_heads, kv_map;
        for (const auto& s : segs) {
            if (s.owner != rank) continue;
            heads.push_back(s.head);
            ranges.push_back(static_cast<int32_t>(s.row_begin / bq));
            ranges.push_back(static_cast<int32_t>((s.row_end + bq - 1) / bq));
            if (std::find(kv_heads.begin(), kv_heads.end(), s.head / group) == kv_heads.end())
                kv_heads.push_back(s.head / group);
        }
        std::sort(kv_heads.begin(), kv_heads.end());
        for (int32_t h : heads)
            kv_map.push_back(static_cast<int32_t>(std::find(kv_heads.begin(), kv_heads.end(), h / group) - kv_heads.begin()));
        const int hr = static_cast<int>(heads.size()), gr = static_cast<int>(kv_heads.size());
        const size_t head_elems = static_cast<size_t>(n) * d;
        uint16_t *ql = nullptr, *kl = nullptr, *vl = nullptr;
        local = nullptr;
        std::vector<int64_t> b_local;
        if (hr > 0) {
            cuda(cudaMalloc(&ql, hr * head_elems * 2), "malloc");
            cuda(cudaMalloc(&kl, gr * head_elems * 2), "malloc");
            cuda(cudaMalloc(&vl, gr * head_elems * 2), "malloc");
            cuda(cudaMalloc(&local, hr * head_elems * 2), "malloc");
            for (int i = 0; i < hr; ++i) {
                cuda(cudaMemcpy(ql + i * head_elems, q + heads[i] * head_elems, head_elems * 2,
                                cudaMemcpyDeviceToDevice), "shard q");
                b_local.push_back(budgets[heads[i]]);
            }
            for (int i = 0; i < gr; ++i) {
                cuda(cudaMemcpy(kl + i * head_elems, k + kv_heads[i] * head_elems, head_elems * 2,
                                cudaMemcpyDeviceToDevice), "shard k");
                cuda(cudaMemcpy(vl + i * head_elems, v + kv_heads[i] * head_elems, head_elems * 2,
                                cudaMemcpyDeviceToDevice), "shard v");
            }
        }
        void* comm = nullptr;
        const std::vector<char> id = exchange_id(id_path, rank);
        check(shplb_nccl_comm_init(device, world, rank, id.data(), id.size(), &comm), "shplb_nccl_comm_init");

        cudaEvent_t e0, e1, e2;
        cuda(cudaEventCreate(&e0), "event");
        cuda(cudaEventCreate(&e1), "event");
        cuda(cudaEventCreate(&e2), "event");
        auto run = [&] {
            cuda(cudaEventRecord(e0, st), "record");
            if (hr > 0) {
                shplb_layer_shape s = full;
                s.num_q_heads = hr;
                s.num_kv_heads = gr;
                s.kv_head_of_q = kv_map.data();
                s.q_block_range = plan == "split" ? ranges.data() : nullptr;
                check(shplb_sparse_attention_layer(ctx, &s, ql, kl, vl, b_local.data(), local, st), "shard layer");
            }
            cuda(cudaEventRecord(e1, st), "record");
            if (plan == "split")
                check(shplb_gather_segments(ctx, comm, segs.data(), static_cast<int32_t>(segs.size()), hq, n, d,
                                            local, out, st),
                      "shplb_gather_segments");
            else
                check(shplb_gather_heads(ctx, comm, hq, n, d, dev_of_head.data(), local, out, st),
                      "shplb_gather_heads");
            check(shplb_comm_barrier(comm, st), "shplb_comm_barrier");
            cuda(cudaEventRecord(e2, st), "record");
            cuda(cudaStreamSynchronize(st), "sync");
        };
        run();  // warm-up (and the checked pass)
        std::vector<uint16_t> got(qe), want(qe);
        cuda(cudaMemcpy(got.data(), out, qe * 2, cudaMemcpyDeviceToHost), "d2h");
        cuda(cudaMemcpy(want.data(), ref, qe * 2, cudaMemcpyDeviceToHost), "d2h");
        const bool identical = std::memcmp(got.data(), want.data(), qe * 2) == 0;
        float best_compute = 1e30f, best_total = 1e30f;
        for (int r = 0; r < 3; ++r) {
            run();
            float a = 0.f, b = 0.f;
            cuda(cudaEventElapsedTime(&a, e0, e1), "elapsed");
            cuda(cudaEventElapsedTime(&b, e0, e2), "elapsed");
            best_compute = std::min(best_compute, a);
            best_total = std::min(best_total, b);
        }
        std::printf("{\"tool\": \"hp_layer\", \"plan\": \"%s\", \"rank\": %d, \"world\": %d, \"seq_len\": %lld, "
                    "\"q_heads\": %d, \"kv_heads\": %d, \"local_heads\": %d, \"segments\": %zu, "
                    "\"shard_ms\": %.3f, \"shard_plus_gather_ms\": %.3f, \"bit_identical\": %s}\n",
                    plan.c_str(), rank, world, static_cast<long long>(n), hq, hkv, hr, segs.size(), best_compute,
                    best_total, identical ? "true" : "false");
        check(shplb_nccl_comm_destroy(comm), "shplb_nccl_comm_destroy");
        for (void* p : {static_cast<void*>(q), static_cast<void*>(k), static_cast<void*>(v), static_cast<void*>(ref),
                        static_cast<void*>(out), static_cast<void*>(ql), static_cast<void*>(kl), static_cast<void*>(vl),
                        static_cast<void*>(local)})
            if (p) cudaFree(p);
        check(shplb_ctx_destroy(ctx), "shplb_ctx_destroy");
        if (rank == 0) std::remove(id_path.c_str());
        return identical ? 0 : 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "hp_layer: %s\n", e.what());
        return 1;
    }
}
