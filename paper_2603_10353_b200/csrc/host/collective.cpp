// Multi-rank part of the C ABI (include/shplb.h, "Head parallelism across
// ranks"): an NCCL communicator, the reassembly of a head-parallel layer's
// outputs on every rank, and a cross-rank barrier — so a C++ host can run the
// paper's head-parallel layer (Assignment::device_of_head,
// proj/include/headbal/partitioner.hpp:15-21, over the per-head fan-out of
// proj/src/attention.cpp:204-223) without Python or torch.distributed.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy already in the
// process, e.g. torch's, else the system's), like the CUDA driver entry points
// in shplb_api.cpp, so libshplb.so loads on hosts without NCCL and reports
// SHPLB_NCCL_ERROR only when a collective is asked for.
//
// Reassembly: every output segment (a head's rows [r0, r1), computed by one
// rank) is one ncclBroadcast rooted at its owner, from the owner's local
// output straight into its place in every rank's [Hq][n][d] buffer; all
// segments of a layer go in one NCCL group. No staging buffer, no padding, no
// reorder pass (the padded all-gather + reorder of head_parallel.py's NCCL path
// is what this replaces for C++ hosts).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../common.hpp"
#include "shplb.h"

namespace shplb {
namespace {

struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string load_error;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.load_error = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && n.load_error.empty()) n.load_error = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(n.get_unique_id, "ncclGetUniqueId");
        sym(n.comm_init_rank, "ncclCommInitRank");
        sym(n.comm_destroy, "ncclCommDestroy");
        sym(n.comm_count, "ncclCommCount");
        sym(n.comm_user_rank, "ncclCommUserRank");
        sym(n.group_start, "ncclGroupStart");
        sym(n.group_end, "ncclGroupEnd");
        sym(n.broadcast, "ncclBroadcast");
        sym(n.all_reduce, "ncclAllReduce");
        sym(n.error_string, "ncclGetErrorString");
    });
    if (!n.load_error.empty()) throw NcclError(n.load_error);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl().error_string(r));
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceOf {  // current device = the communicator's for the duration of a call
    int prev = -1;
    explicit DeviceOf(int dev) {
        cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (dev >= 0 && dev != prev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceOf() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// Per-communicator scratch of the barrier (one int on the device).
struct Comm {
    ncclComm_t comm = nullptr;
    int device = 0;
    int nranks = 1, rank = 0;
    int32_t* flag = nullptr;
};

Comm* as_comm(void* c) {
    if (!c) throw InvalidArgument("communicator is null");
    return static_cast<Comm*>(c);
}

// Every (head, row range) segment: exactly one owner per output row.
void check_segments(const shplb_out_segment* segs, int32_t n_segs, int32_t hq, int64_t n, int nranks) {
    if (hq < 1) throw InvalidArgument("need at least one head");
    if (n < 1) throw InvalidArgument("K must hold at least one key token");
    if (!segs && n_segs > 0) throw InvalidArgument("segments is null");
    std::vector<std::vector<std::pair<int64_t, int64_t>>> per_head(static_cast<size_t>(hq));
    for (int32_t i = 0; i < n_segs; ++i) {
        const auto& s = segs[i];
        if (s.head < 0 || s.head >= hq)
            throw InvalidArgument("segment " + std::to_string(i) + ": head " + std::to_string(s.head) +
                                  " out of range [0, " + std::to_string(hq) + ")");
        if (s.owner < 0 || s.owner >= nranks)
            throw InvalidArgument("head " + std::to_string(s.head) + " assigned to invalid device " +
                                  std::to_string(s.owner));
        if (s.local_head < 0 || s.row_begin < 0 || s.row_end > n || s.row_begin >= s.row_end)
            throw InvalidArgument("segment " + std::to_string(i) + ": rows [" + std::to_string(s.row_begin) +
                                  ", " + std::to_string(s.row_end) + ") out of [0, " + std::to_string(n) + "]");
        per_head[static_cast<size_t>(s.head)].push_back({s.row_begin, s.row_end});
    }
    for (int32_t h = 0; h < hq; ++h) {
        auto& v = per_head[static_cast<size_t>(h)];
        std::sort(v.begin(), v.end());
        int64_t at = 0;
        bool tiles = true;  // consecutive, non-overlapping, from row 0 to n
        for (const auto& r : v) {
            tiles &= r.first == at;
            at = r.second;
        }
        if (!tiles || at != n)
            throw InvalidArgument("head " + std::to_string(h) +
                                  ": segments must cover every output row exactly once");
    }
}

void gather(Comm* c, const shplb_out_segment* segs, int32_t n_segs, int32_t hq, int64_t n, int32_t d,
            const void* local, void* out, cudaStream_t st) {
    check_segments(segs, n_segs, hq, n, c->nranks);
    if (d < 1) throw InvalidArgument("head_dim must be positive");
    if (!out) throw InvalidArgument("out is null");
    bool owns = false;
    for (int32_t i = 0; i < n_segs; ++i) owns |= segs[i].owner == c->rank;
    if (owns && !local) throw InvalidArgument("local is null on a rank that owns segments");
    const Nccl& N = nccl();
    DeviceOf g(c->device);
    auto* o = static_cast<uint16_t*>(out);
    const auto* l = static_cast<const uint16_t*>(local);
    nccl_check(N.group_start(), "ncclGroupStart");
    for (int32_t i = 0; i < n_segs; ++i) {
        const auto& s = segs[i];
        uint16_t* dst = o + (static_cast<int64_t>(s.head) * n + s.row_begin) * d;
        const void* src = s.owner == c->rank ? l + (static_cast<int64_t>(s.local_head) * n + s.row_begin) * d
                                             : static_cast<const void*>(dst);
        const ncclResult_t r = N.broadcast(src, dst, static_cast<size_t>(s.row_end - s.row_begin) * d,
                                           ncclBfloat16, s.owner, c->comm, st);
        if (r != ncclSuccess) {
            N.group_end();
            nccl_check(r, "ncclBroadcast");
        }
    }
    nccl_check(N.group_end(), "ncclGroupEnd");
}

}  // namespace
}  // namespace shplb

using namespace shplb;

extern "C" {

int shplb_nccl_get_unique_id(void* id_out, size_t id_bytes) {
    return guarded([&] {
        require(id_out != nullptr, "id_out is null");
        require(id_bytes >= sizeof(ncclUniqueId), "id buffer must hold SHPLB_NCCL_UNIQUE_ID_BYTES bytes");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int shplb_nccl_comm_init(int device, int32_t nranks, int32_t rank, const void* id, size_t id_bytes,
                         void** comm_out) {
    return guarded([&] {
        require(comm_out != nullptr && id != nullptr, "null pointer");
        require(id_bytes >= sizeof(ncclUniqueId), "id must be SHPLB_NCCL_UNIQUE_ID_BYTES bytes");
        if (nranks < 1) throw InvalidArgument("need at least one device");
        if (rank < 0 || rank >= nranks)
            throw InvalidArgument("rank " + std::to_string(rank) + " out of range [0, " + std::to_string(nranks) + ")");
        const Nccl& N = nccl();
        DeviceOf g(device);
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        auto* c = new Comm();
        c->device = device;
        c->nranks = nranks;
        c->rank = rank;
        const ncclResult_t r = N.comm_init_rank(&c->comm, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        if (cudaMalloc(&c->flag, sizeof(int32_t)) != cudaSuccess || cudaMemset(c->flag, 0, sizeof(int32_t)) != cudaSuccess) {
            N.comm_destroy(c->comm);
            delete c;
            throw CudaError("cudaMalloc of the barrier flag failed");
        }
        *comm_out = c;
    });
}

int shplb_nccl_comm_destroy(void* comm) {
    return guarded([&] {
        if (!comm) return;
        Comm* c = static_cast<Comm*>(comm);
        DeviceOf g(c->device);
        cudaFree(c->flag);
        const ncclResult_t r = nccl().comm_destroy(c->comm);
        delete c;
        nccl_check(r, "ncclCommDestroy");
    });
}

int shplb_nccl_comm_size(void* comm, int32_t* nranks, int32_t* rank) {
    return guarded([&] {
        Comm* c = as_comm(comm);
        if (nranks) *nranks = c->nranks;
        if (rank) *rank = c->rank;
    });
}

int shplb_gather_segments(shplb_ctx* ctx, void* comm, const shplb_out_segment* segments, int32_t n_segments,
                          int32_t num_q_heads, int64_t seq_len, int32_t head_dim, const void* local, void* out,
                          void* stream) {
    (void)ctx;
    return guarded([&] {
        gather(as_comm(comm), segments, n_segments, num_q_heads, seq_len, head_dim, local, out,
               static_cast<cudaStream_t>(stream));
    });
}

int shplb_gather_heads(shplb_ctx* ctx, void* comm, int32_t num_q_heads, int64_t seq_len, int32_t head_dim,
                       const int32_t* device_of_head, const void* local, void* out, void* stream) {
    (void)ctx;
    return guarded([&] {
        Comm* c = as_comm(comm);
        require(device_of_head != nullptr, "device_of_head is null");
        // Assignment::validate (partitioner.cpp:38-48) against the communicator's size.
        std::vector<shplb_out_segment> segs(static_cast<size_t>(std::max(num_q_heads, 0)));
        std::vector<int32_t> next_local(static_cast<size_t>(c->nranks), 0);
        for (int32_t h = 0; h < num_q_heads; ++h) {
            const int32_t dev = device_of_head[h];
            if (dev < 0 || dev >= c->nranks)
                throw InvalidArgument("head " + std::to_string(h) + " assigned to invalid device " + std::to_string(dev));
            segs[static_cast<size_t>(h)] = {h, dev, next_local[static_cast<size_t>(dev)]++, 0, 0, seq_len};
        }
        gather(c, segs.data(), num_q_heads, num_q_heads, seq_len, head_dim, local, out,
               static_cast<cudaStream_t>(stream));
    });
}

int shplb_comm_barrier(void* comm, void* stream) {
    return guarded([&] {
        Comm* c = as_comm(comm);
        const Nccl& N = nccl();
        DeviceOf g(c->device);
        nccl_check(N.all_reduce(c->flag, c->flag, 1, ncclInt32, ncclSum, c->comm, static_cast<cudaStream_t>(stream)),
                   "ncclAllReduce");
    });
}

}  // extern "C"
