// Kernel 3, persistent CTA-pair kernel (block_q = 256): the CTA-pair data path
// (two 128-row query halves on the two SMs of a cluster, tcgen05.mma.cta_group::2
// with M = 256, two softmax warpgroups per SM on alternate key blocks with their
// own running max / row sum / O in TMEM), run as one resident cluster per SM
// pair that walks a host-built list of query tiles. (Its predecessor with one
// cluster per tile, fa_pair_sm100.cu, was removed once this kernel matched it
// bit for bit and beat it on short tiles; see git history and DESIGN.md §5.)
//
// Why (profiles/r02/k3_tile_trace.json): with a cluster per tile
// each tile paid ~6.5 K cycles of prologue (barrier init, TMEM alloc, cluster
// sync, the dependent tile / count / selection loads, Q and the first K
// landing, the first S) and ~3.5 K of epilogue on an otherwise idle tensor
// pipe, plus ~1.4 K between clusters: 4.2% of the SM-cycles at C3. Here the
// setup happens once, Q is double-buffered and the producers run into the
// next tile's Q and K/V while the current tile drains, so S of the next tile
// is already in TMEM when its softmax warpgroup comes out of the epilogue.
//
// Per tile the data path is the one-cluster-per-tile kernel's (same MMAs, same
// online softmax, same merge and TMA-store epilogue, bit-identical outputs). What
// is new is the cross-tile bookkeeping: every barrier's phase is a running count
// (K/V stages and P·V slots by global block index, S by each warpgroup's own
// block count, the Q, selection and output slots by tile index), and three
// handshakes order the tile boundary:
//   sel_full / sel_empty  the QK producer publishes a tile's (head, query
//                         block, count) and selected block list in one of
//                         three slots, a tile ahead of its K loads; every
//                         consumer releases the slot;
//   o_free / tile_ack     a tile's first P·V into O_w (accumulate = 0) waits
//                         until both CTAs' softmax warps have read the previous
//                         tile's O_A / O_B (o_free); the P·V issuer then acks
//                         the tile to both CTAs, and an epilogue only finishes
//                         after its tile's ack, so no arriver is ever a whole
//                         phase ahead (also for tiles that compute nothing);
//   out_full              the epilogue stages a tile's output in its Q slot and
//                         hands it to the QK producer, which stores it (bulk
//                         tensor copies) before it reloads that slot with the
//                         Q of tile t + 2 — the store never stalls a softmax
//                         warp.
//
// Work distribution: dynamic, in work-list order (kv-group major, heaviest
// first inside a group, as the hardware scheduler hands out the one-cluster-
// per-tile kernel's clusters, so the clusters in flight share K/V in L2). The
// leader's QK producer takes the next tile with an atomic ticket on a
// per-launch counter (zero at launch; the launch's last draw resets it) once a slot is
// free — about one tile ahead of its use — and hands it to the peer CTA
// through distributed shared memory; a ticket past the list ends the cluster.
// (A static LPT assignment of tiles to clusters was measured first: it left
// SMs idle for ~1.8% of the launch — per-SM speed differs.)
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace shplb::kern {
namespace {

using namespace shplb::ptx;

constexpr int kThreads = 384;
constexpr uint32_t kRegsLaunch = 168, kRegsSoftmax = 216, kRegsControl = 72;
static_assert(2 * kRegsSoftmax + kRegsControl <= 3 * kRegsLaunch, "setmaxnreg budget exceeds the launch grant");
constexpr int kStages = 4;
constexpr int kQHalfBytes = 32768;  // [2 d-chunks][128 rows][128 B]
constexpr int kKHalfBytes = 16384;  // [2 d-chunks][64 keys][128 B]
constexpr int kVHalfBytes = 16384;  // [128 keys][64 d = 128 B]
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 128, kColO = 256;  // P_w at kColP + 64 w, O_w at kColO + 128 w
constexpr uint32_t kIdescS = idesc_bf16_f32(256, 128, 0, 0);   // Q K-major, K K-major
constexpr uint32_t kIdescPV = idesc_bf16_f32(256, 128, 0, 1);  // P (TMEM), V MN-major
// Lazy rescale: a warpgroup's reference m moves only when a block's max exceeds
// it by more than 2^kRescaleThreshold. P is bf16 and l / O are fp32, so P up to
// 2^32 costs no precision (only the 2^8 of fp16-P kernels would overflow); the
// high threshold lets almost every block skip its row max: P is exponentiated
// against m first, and a block sum <= 2^32 proves every P <= 2^32, i.e. the max
// rule would keep m too. Only otherwise (or at a row's first block, or a sum
// that overflowed to +inf) is the max taken, and P recomputed if m moves.
// C3: 64 FMNMX3 per 128 scores saved, kernel 3 ~1.3% faster under the power
// cap (profiles/r02/k3_spec_max_ab.txt). SHPLB_EXACT_MAX (diagnostic) takes
// every block's max; SHPLB_RESCALE_LOG2 sets the threshold.
#ifndef SHPLB_RESCALE_LOG2
#define SHPLB_RESCALE_LOG2 32
#endif
constexpr float kRescaleThreshold = static_cast<float>(SHPLB_RESCALE_LOG2);
constexpr float kRescaleSum = static_cast<float>(1ull << SHPLB_RESCALE_LOG2);
constexpr int kWarpQK = 8, kWarpS = 9, kWarpV = 10;  // 11: the P·V issuer
// sel_empty arrivals per tile: V producer, S and P·V issuer warps (which on
// the peer only keep the slot phases), 8 softmax warps.
constexpr uint32_t kSelConsumers = 11;

struct TileInfo {
    int32_t h, qb, nsel, pad;
};

// Tile info / selection slots: tile t in slot t % 3, so tile t+1 can be
// published while tile t-1 still drains. Slot and barrier phase advance together.
constexpr int kSelSlots = 3;
struct SelRing {
    int slot = 0;
    uint32_t phase = 0;
    __device__ __forceinline__ void next() {
        if (++slot == kSelSlots) {
            slot = 0;
            phase ^= 1;
        }
    }
};

struct __align__(8) Barriers {
    uint64_t tkt_full[kSelSlots];  // peer: the leader stored the slot's ticket (remote, release / acquire cluster)
    uint64_t q_full[2];   // leader: both CTAs' Q halves of the slot landed
    uint64_t out_full[2];  // each CTA: the epilogue staged the slot's output tile (thread 0)
    uint64_t k_full[kStages], v_full[kStages];    // leader
    uint64_t k_empty[kStages], v_empty[kStages];  // each CTA
    uint64_t s_full[2];   // each CTA: S in TMEM for warpgroup w
    uint64_t s_free;      // leader: the owning warpgroups of both CTAs loaded S (8 warps)
    uint64_t p_full[2][2];  // leader: [CTA][warpgroup] P stored (4 warps)
    uint64_t pv_done[4];  // each CTA: P·V of global block J completed, [J mod 4]
    uint64_t sel_full[kSelSlots];   // each CTA: tile info + selection of the slot written (32 lanes)
    uint64_t sel_empty[kSelSlots];  // each CTA: every consumer is done with the slot
    uint64_t o_free;        // leader: both CTAs' softmax warps read the tile's O (16 warps)
    uint64_t tile_ack;      // each CTA: the P·V issuer passed o_free of the previous tile
    uint32_t tmem_base;
};

constexpr size_t kSmemQ = 0;                                   // 2 slots
constexpr size_t kSmemK = kSmemQ + 2 * kQHalfBytes;
constexpr size_t kSmemV = kSmemK + kStages * kKHalfBytes;
constexpr size_t kSmemSel = kSmemV + kStages * kVHalfBytes;    // kSelSlots slots of kMaxSelected
constexpr size_t kSmemInfo = kSmemSel + kSelSlots * kMaxSelected * sizeof(int32_t);
constexpr size_t kSmemTkt = kSmemInfo + kSelSlots * sizeof(TileInfo);  // int32 ticket per slot (peer)
constexpr size_t kSmemBar = kSmemTkt + 16;
static_assert(kSelSlots * sizeof(int32_t) <= 16, "ticket slots");
constexpr size_t kSmemX = kSmemBar + ((sizeof(Barriers) + 15) / 16) * 16;  // l / m [2][2][128]
constexpr size_t kSmemTotal = kSmemX + 4 * 128 * sizeof(float) + 1024;
static_assert(kSmemTotal <= 227 * 1024, "shared memory over the sm_100 per-CTA limit");

#ifdef SHPLB_TILETRACE  // dev-only: per-tile timestamps (tools/tile_trace.py --persist)
constexpr int kTTraceTiles = 1 << 16;
// [cluster * 512 + tile of the cluster][0 first S landed, 1 last P·V landed, 2 output staged,
// 3 smid | nsel << 32, 4 store read / epilogue done, 5 Q landed seen by the S issuer,
// 6 S(0) issued, 7 Q load issued, 8 S issuer past s_free for S(0), 9 past k_full for S(0),
// 10 K(0) load issued (leader), 11 last S issued] (clock64 of the leader CTA)
__device__ unsigned long long g_tiletrace_p[kTTraceTiles][12];
#define TTRACE(i, e, v) do { if ((i) < kTTraceTiles) g_tiletrace_p[(i)][(e)] = (v); } while (0)
#else
#define TTRACE(i, e, v) do { } while (0)
#endif

__device__ __forceinline__ void mbar_arrive_lane(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) fa_persist_kernel(const __grid_constant__ FaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bar = reinterpret_cast<Barriers*>(smem + kSmemBar);
    TileInfo* info = reinterpret_cast<TileInfo*>(smem + kSmemInfo);
    const uint32_t sSel = smem_u32(smem + kSmemSel);
    auto sel_at = [&](int slot, int j) {
        return lds_s32(sSel + 4u * static_cast<uint32_t>(slot * kMaxSelected + j));
    };
    float* lfin = reinterpret_cast<float*>(smem + kSmemX);  // [2 warpgroups][2 (l, m)][128]

    const int warp = warp_index_uniform();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSelSlots; ++i) {
            mbar_init(&bar->tkt_full[i], 1);
            mbar_init(&bar->sel_full[i], 32);
            mbar_init(&bar->sel_empty[i], kSelConsumers);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->q_full[i], 1);
            mbar_init(&bar->out_full[i], 1);
            mbar_init(&bar->s_full[i], 1);
            mbar_init(&bar->p_full[i][0], 4);
            mbar_init(&bar->p_full[i][1], 4);
        }
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&bar->k_full[i], 1);
            mbar_init(&bar->v_full[i], 1);
            mbar_init(&bar->k_empty[i], 1);
            mbar_init(&bar->v_empty[i], 1);
        }
        mbar_init(&bar->s_free, 8);
        for (int i = 0; i < 4; ++i) mbar_init(&bar->pv_done[i], 1);
        mbar_init(&bar->o_free, 16);
        mbar_init(&bar->tile_ack, 1);
        fence_mbar_init();
    }
    if (warp == kWarpS) tmem_alloc_pair<kTmemCols>(&bar->tmem_base);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem = bar->tmem_base;
    auto leader = [&](const uint64_t* b) { return mapa_shared(smem_u32(b), 0); };

    if (warp >= 8) {
        setmaxnreg_dec<kRegsControl>();
        const uint32_t rank = cluster_ctarank();  // re-read after setmaxnreg (else kept on the stack)
        if (warp == kWarpQK) {
            // ------------------------------ tile info, selection, Q and K loads
            const int lane = threadIdx.x & 31;
            int32_t* tkt = reinterpret_cast<int32_t*>(smem + kSmemTkt);
            const uint32_t peer_tkt = mapa_shared(smem_u32(tkt), 1);
            const uint32_t peer_tkt_full = mapa_shared(smem_u32(&bar->tkt_full[0]), 1);
            // Publishes tile t (ticket, tile info, selection) in selection slot
            // t % 3; false once the ticket is past the list (end marker published).
            auto publish = [&](const SelRing& r) -> bool {
                mbar_wait(&bar->sel_empty[r.slot], r.phase ^ 1);
                int ticket = 0;
                if (rank == 0) {
                    if (lane == 0) {
                        ticket = atomicAdd(p.counter, 1);
                        // Every cluster draws exactly one ticket past the list, so the
                        // launch's last draw returns the counter to zero for the next
                        // launch on this ring slot (no memset on the stream: a memset
                        // runs on a copy engine and queues behind bulk transfers).
                        if (ticket == p.num_tiles + static_cast<int>(gridDim.x >> 1) - 1) atomicExch(p.counter, 0);
                        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer_tkt + 4u * r.slot), "r"(ticket)
                                     : "memory");
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                         peer_tkt_full + 8u * r.slot)
                                     : "memory");
                    }
                    ticket = __shfl_sync(0xffffffffu, ticket, 0);
                } else {
                    uint32_t ok = 0;
                    while (!ok) {
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                            "selp.u32 %0, 1, 0, p;\n\t}"
                            : "=r"(ok)
                            : "r"(smem_u32(&bar->tkt_full[r.slot])), "r"(r.phase)
                            : "memory");
                    }
                    ticket = tkt[r.slot];
                }
                if (ticket >= p.num_tiles) {  // past the list: this cluster is done
                    if (lane == 0) info[r.slot] = TileInfo{-1, 0, 0, 0};
                    mbar_arrive_lane(&bar->sel_full[r.slot]);
                    return false;
                }
                const int32_t tile = p.tiles[ticket];
                const int h = tile >> 20, qb = tile & 0xFFFFF;
                const int64_t row_id = static_cast<int64_t>(h) * p.nqb + qb;
                const int nsel = p.cnt[row_id];
                const int32_t* gsel = p.idx + row_id * p.kmax;
                int32_t* ssel = reinterpret_cast<int32_t*>(smem + kSmemSel) + r.slot * kMaxSelected;
                // 8 independent loads per lane in flight (the list is usually
                // not in L2 any more: one round trip per 256 entries).
                for (int j0 = 0; j0 < nsel; j0 += 256) {
                    int32_t v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + u * 32 + lane;
                        v[u] = j < nsel ? __ldg(gsel + j) : 0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + u * 32 + lane;
                        if (j < nsel) ssel[j] = v[u];
                    }
                }
                if (lane == 0) info[r.slot] = TileInfo{h, qb, nsel, 0};
                mbar_arrive_lane(&bar->sel_full[r.slot]);  // every lane: its stores are released
                __syncwarp();
                return true;
            };
            // Tile t+1 is published while tile t's loads are issued — after
            // tile t's Q and first kStages K blocks, whose stages free up as
            // tile t-1 drains — so its selection and Q are in shared memory
            // before tile t drains, and tile t's first S never waits for the
            // (dependent, mostly DRAM) loads of the publication.
            // Output tile of tile t (staged by the epilogue in Q slot t & 1):
            // stored by this warp with bulk tensor copies — off the softmax
            // warps' path — once staged, and read out before the slot takes
            // the Q of tile t + 2.
            auto store_out = [&](int t, int islot) {
                mbar_wait(&bar->out_full[t & 1], static_cast<uint32_t>(t >> 1) & 1);
                const TileInfo to = info[islot];
                const int64_t r0 = static_cast<int64_t>(to.qb) * 256 + 128 * static_cast<int64_t>(rank);
                if (r0 < p.n && lane == 0) {
                    const uint32_t tile_s = smem_u32(smem + kSmemQ + (t & 1) * kQHalfBytes);
                    const int ndst = p.n_out_peers > 0 ? p.n_out_peers : 1;
                    const int plane = p.n_out_peers > 0 ? p.heads.k[to.h] : to.h;
                    for (int i = 0; i < ndst; ++i) tma_store_tile(&p.tm_out[i], tile_s, static_cast<int32_t>(r0), plane);
                    bulk_commit_group();
                    if (p.n_out_peers > 1) {
                        bulk_wait_group0();
                        __threadfence_system();
                    } else {
                        bulk_wait_group_read0();
                    }
                }
                __syncwarp();
            };
            SelRing cur;
            int prev1 = -1, prev2 = -1;  // selection slots of tiles tl - 1 and tl - 2 (their info)
            bool more = publish(cur);
            int kc = 0;  // K stages issued so far (all tiles)
            int last_tl = -1;
            for (int tl = 0; more; ++tl) {
                const TileInfo ti = info[cur.slot];
                const int qs = tl & 1;
                if (tl >= 2) store_out(tl - 2, prev2);  // frees the Q slot
                prev2 = prev1;
                prev1 = cur.slot;
                if (rank == 0 && lane == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 7, clock64());
                if (ti.nsel > 0) {
                    if (rank == 0) mbar_expect_tx_warp(&bar->q_full[qs], 2 * kQHalfBytes);
                    tma_load_pair_warp(smem + kSmemQ + qs * kQHalfBytes, &p.tm_q, leader(&bar->q_full[qs]), 0,
                                       ti.qb * 256 + 128 * static_cast<int>(rank), ti.h, 2, 16384);
                } else if (rank == 0) {
                    mbar_arrive_warp(&bar->q_full[qs]);  // keeps the slot's phase in step
                }
                SelRing nxt = cur;
                nxt.next();
                const int g = p.heads.kv[ti.h];
                const int npre = min(ti.nsel, kStages);
                for (int j = 0; j < ti.nsel; ++j, ++kc) {
                    if (j == npre) more = publish(nxt);
                    const int st = kc % kStages;
                    mbar_wait(&bar->k_empty[st], ((kc / kStages) & 1) ^ 1);
                    if (rank == 0) mbar_expect_tx_warp(&bar->k_full[st], 2 * kKHalfBytes);
                    if (j == 0 && rank == 0 && lane == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 10, clock64());
                    tma_load_pair_warp(smem + kSmemK + st * kKHalfBytes, &p.tm_k_half, leader(&bar->k_full[st]), 0,
                                       sel_at(cur.slot, j) * kBlock + 64 * static_cast<int>(rank), g, 2, 8192);
                }
                if (npre == ti.nsel) more = publish(nxt);
                cur = nxt;
                last_tl = tl;
            }
            // The last two tiles' outputs (their info slots are not reused).
            if (last_tl >= 1) store_out(last_tl - 1, prev2);
            if (last_tl >= 0) store_out(last_tl, prev1);
            if (lane == 0) bulk_wait_group0();  // every output tile written before the CTA exits
        } else if (warp == kWarpV) {
            // ------------------------------------------------------ V loads
            int vc = 0;
            for (SelRing sr;; sr.next()) {
                const int slot = sr.slot;
                mbar_wait(&bar->sel_full[slot], sr.phase);
                const TileInfo ti = info[slot];
                if (ti.h < 0) break;
                const int g = p.heads.kv[ti.h];
                for (int j = 0; j < ti.nsel; ++j, ++vc) {
                    const int st = vc % kStages;
                    mbar_wait(&bar->v_empty[st], ((vc / kStages) & 1) ^ 1);
                    if (rank == 0) mbar_expect_tx_warp(&bar->v_full[st], 2 * kVHalfBytes);
                    tma_load_pair_warp(smem + kSmemV + st * kVHalfBytes, &p.tm_v, leader(&bar->v_full[st]),
                                       64 * static_cast<int>(rank), sel_at(slot, j) * kBlock, g, 1, 0);
                }
                mbar_arrive_warp(&bar->sel_empty[slot]);
            }
        } else if (warp == kWarpS) {
            // ------------------------------------ S issuer (leader's MMAs)
            const uint32_t tm = __shfl_sync(0xffffffffu, static_cast<uint32_t>(lds_s32(smem_u32(&bar->tmem_base))), 0);
            const uint64_t kd0 = umma_desc_sw128(smem_u32(smem + kSmemK), 16, 1024);
            int J = 0, kc = 0;
            SelRing sr;
            for (int tl = 0;; ++tl, sr.next()) {
                mbar_wait(&bar->sel_full[sr.slot], sr.phase);
                if (info[sr.slot].h < 0) break;
                const int nsel = info[sr.slot].nsel;
                mbar_arrive_warp(&bar->sel_empty[sr.slot]);
                if (rank != 0) continue;
                const int qs = tl & 1;
                const uint64_t qd = umma_desc_sw128(smem_u32(smem + kSmemQ + qs * kQHalfBytes), 16, 1024);
                mbar_wait(&bar->q_full[qs], static_cast<uint32_t>(tl >> 1) & 1);
                if ((threadIdx.x & 31) == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 5, clock64());
                for (int j = 0; j < nsel; ++j, ++J, ++kc) {
                    if (J > 0) mbar_wait(&bar->s_free, (J - 1) & 1);  // S(J-1) is in registers
                    if (j == 0 && (threadIdx.x & 31) == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 8, clock64());
                    const int st = kc % kStages;
                    mbar_wait(&bar->k_full[st], (kc / kStages) & 1);
                    if (j == 0 && (threadIdx.x & 31) == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 9, clock64());
                    if (j == nsel - 1 && (threadIdx.x & 31) == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 11, clock64());
                    tc_fence_after();
                    mma_pair_ss(tm + kColS, qd, kd0 + static_cast<uint64_t>(st) * (kKHalfBytes >> 4), kIdescS, 0u);
                    if (j == 0 && (threadIdx.x & 31) == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 6, clock64());
                    mma_commit_pair_warp(&bar->s_full[j & 1]);
                    mma_commit_pair_warp(&bar->k_empty[st]);
                }
            }
        } else {
            // ---------------------------------- P·V issuer (leader's MMAs)
            const uint32_t tm = __shfl_sync(0xffffffffu, static_cast<uint32_t>(lds_s32(smem_u32(&bar->tmem_base))), 0);
            const uint64_t vd0 = umma_desc_sw128(smem_u32(smem + kSmemV), 16384, 1024);
            const uint32_t ack0 = mapa_shared(smem_u32(&bar->tile_ack), 0);
            const uint32_t ack1 = mapa_shared(smem_u32(&bar->tile_ack), 1);
            int J = 0, vc = 0;
            uint32_t nw0 = 0, nw1 = 0;  // blocks each warpgroup has handed over (all tiles)
            SelRing sr;
            for (int tl = 0;; ++tl, sr.next()) {
                mbar_wait(&bar->sel_full[sr.slot], sr.phase);
                if (info[sr.slot].h < 0) break;
                const int nsel = info[sr.slot].nsel;
                mbar_arrive_warp(&bar->sel_empty[sr.slot]);
                if (rank != 0) continue;
                if (tl > 0) mbar_wait(&bar->o_free, (tl - 1) & 1);  // O_A / O_B of the previous tile read
                mbar_arrive_cluster_warp(ack0);
                mbar_arrive_cluster_warp(ack1);
                for (int j = 0; j < nsel; ++j, ++J, ++vc) {
                    const int w = j & 1;
                    const int st = vc % kStages;
                    const uint32_t ph = (w ? nw1 : nw0) & 1;
                    mbar_wait(&bar->p_full[0][w], ph);
                    mbar_wait(&bar->p_full[1][w], ph);
                    if (w) ++nw1; else ++nw0;
                    mbar_wait(&bar->v_full[st], (vc / kStages) & 1);
                    tc_fence_after();
                    mma_pair_ts(tm + kColO + 128u * static_cast<uint32_t>(w), tm + kColP + 64u * static_cast<uint32_t>(w),
                                vd0 + static_cast<uint64_t>(st) * (kVHalfBytes >> 4), kIdescPV, j > 1 ? 1u : 0u);
                    mma_commit_pair_warp(&bar->pv_done[J & 3]);
                    mma_commit_pair_warp(&bar->v_empty[st]);
                }
            }
        }
    } else {
        setmaxnreg_inc<kRegsSoftmax>();
        const uint32_t rank = cluster_ctarank();
        // ------------------------------------------------ softmax warpgroups
        const int wg = warp >> 2;          // takes blocks j = wg, wg + 2, ... of every tile
        const int r = threadIdx.x & 127;   // row within this CTA's half == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t s_addr = tmem + lane_base + kColS;
        const uint32_t p_addr = tmem + lane_base + kColP + 64u * static_cast<uint32_t>(wg);
        const uint32_t o_addr = tmem + lane_base + kColO + 128u * static_cast<uint32_t>(wg);
        const float sl2 = p.scale_log2;
        const uint32_t s_free_l = leader(&bar->s_free);
        const uint32_t p_full_l = leader(&bar->p_full[rank][wg]);
        const uint32_t o_free_l = leader(&bar->o_free);
        const float2 sc2 = make_float2(sl2, sl2);
        int J0 = 0;          // global index of the tile's block 0
        uint32_t mine_all = 0;  // blocks this warpgroup has processed (all tiles): s_full parity
        SelRing sr;
        for (int tl = 0;; ++tl, sr.next()) {
            const int slot = sr.slot;  // selection slot; the Q / output slot is tl & 1
            mbar_wait(&bar->sel_full[slot], sr.phase);
            const TileInfo ti = info[slot];
            if (ti.h < 0) break;
            const int nsel = ti.nsel;
            const int64_t row0 = static_cast<int64_t>(ti.qb) * 256;
            const int64_t qrow = row0 + 128 * static_cast<int64_t>(rank) + r;
            const int64_t lim = p.causal ? min(qrow, p.n - 1) : p.n - 1;  // last visible key
            float m = -INFINITY;  // this warpgroup's reference max (log2 domain)
            float l = 0.0f;       // its row sum, relative to m
            int mine = 0;         // blocks of this tile this warpgroup has processed
            for (int j = wg; j < nsel; j += 2, ++mine, ++mine_all) {
                const int J = J0 + j;
                const int64_t key0 = static_cast<int64_t>(sel_at(slot, j)) * kBlock;
                const bool need_mask = key0 + kBlock - 1 > lim;
                uint32_t sv[kBlock];
                float* s = reinterpret_cast<float*>(sv);
                mbar_wait(&bar->s_full[wg], mine_all & 1);
                if (j == 0 && threadIdx.x == 0 && rank == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 0, clock64());
                tc_fence_after();
                tmem_ld32(s_addr + 0, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
                tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
                tmem_ld32(s_addr + 64, *reinterpret_cast<uint32_t(*)[32]>(&sv[64]));
                tmem_ld32(s_addr + 96, *reinterpret_cast<uint32_t(*)[32]>(&sv[96]));
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive_cluster_warp(s_free_l);  // the leader may now compute the next S over it
#ifdef SHPLB_DIAG_NOSOFTMAX  // dev-only diagnostic (wrong results): S loaded, P stored, no softmax math
                {
                    uint32_t pk[4][16];
#pragma unroll
                    for (int e = 0; e < kBlock / 2; ++e) pk[e >> 4][e & 15] = sv[2 * e] ^ sv[2 * e + 1];
                    if (mine >= 1) {
                        mbar_wait(&bar->pv_done[(J - 2) & 3], ((J - 2) >> 2) & 1);
                        tc_fence_after();
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) tmem_st16(p_addr + c * 16, pk[c]);
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive_cluster_warp(p_full_l);
                    m = 0.0f;
                    l = 1.0f;
                    (void)need_mask;
                    continue;
                }
#endif
                if (need_mask) {
#pragma unroll
                    for (int c = 0; c < kBlock; ++c)
                        if (key0 + c > lim) s[c] = -INFINITY;
                }
                // P = 2^(s*scale - m), its row sum, packed bf16 pairs.
                float2 sum2[2];
                uint32_t pk[4][16];
                auto exps = [&](float msub) {
                    const float2 nm2 = make_float2(-msub, -msub);
                    sum2[0] = sum2[1] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int e = 0; e < kBlock / 2; ++e) {
                        const float2 x = ffma2(make_float2(s[2 * e], s[2 * e + 1]), sc2, nm2);
                        float2 pe;
#ifdef SHPLB_DIAG_NOEXP  // dev-only energy/timing diagnostic (wrong results): no MUFU
                        pe = x;
#else
                        pe.x = ex2(x.x);
                        pe.y = ex2(x.y);
#endif
                        sum2[e & 1] = fadd2(sum2[e & 1], pe);
                        pk[e >> 4][e & 15] = pack_bf16x2(pe.x, pe.y);
                    }
                };
                const float mprev = m;
#ifndef SHPLB_EXACT_MAX
                // Exponentiate against the current m first (see kRescaleThreshold).
                bool need_max = m == -INFINITY;
                if (!need_max) {
                    exps(m);
                    const float2 sp = fadd2(sum2[0], sum2[1]);
                    need_max = !(sp.x + sp.y <= kRescaleSum);  // also +inf / NaN
                }
                if (need_max) {
#endif
                float mx8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
#pragma unroll
                for (int c = 0; c < kBlock; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
                const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
                // Lazy rule: raise m only when the block max exceeds it by > 2^kRescaleThreshold.
                if (mx > m + kRescaleThreshold || (m == -INFINITY && mx > -INFINITY)) m = mx;
#ifndef SHPLB_EXACT_MAX
                if (m != mprev || mprev == -INFINITY) exps(m == -INFINITY ? 0.0f : m);
                }
#else
                exps(m == -INFINITY ? 0.0f : m);
#endif
                const bool rose = m != mprev && mprev != -INFINITY;
                // This warpgroup's previous P·V in this tile (which read P_w and
                // accumulated into O_w) must be done before P_w is rewritten and
                // O_w rescaled; the first block of a tile follows the previous
                // tile's epilogue, which waited for all of its P·V.
                if (mine >= 1) {
                    mbar_wait(&bar->pv_done[(J - 2) & 3], ((J - 2) >> 2) & 1);
                    tc_fence_after();
                }
                if (__any_sync(0xffffffffu, rose)) {
                    const float alpha = rose ? ex2(mprev - m) : 1.0f;
#pragma unroll
                    for (int c = 0; c < kHeadDim / 32; ++c) {
                        uint32_t v[32];
                        tmem_ld32(o_addr + c * 32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
                        tmem_st32(o_addr + c * 32, v);
                    }
                }
                if (rose) l *= ex2(mprev - m);
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_st16(p_addr + c * 16, pk[c]);
                const float2 sum = fadd2(sum2[0], sum2[1]);
                l += sum.x + sum.y;
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive_cluster_warp(p_full_l);
            }

            // ---------------------------------------------------- epilogue
            // Merge (O_0, l_0, m_0) and (O_1, l_1, m_1),
            // stage the bf16 tile in this tile's Q slot (its last S completed
            // before its last P·V was issued), store with bulk tensor copies.
            lfin[(wg * 2 + 0) * 128 + r] = l;
            lfin[(wg * 2 + 1) * 128 + r] = m;
            named_bar_sync(1, 256);
            const float m0 = lfin[1 * 128 + r], m1 = (nsel > 1) ? lfin[3 * 128 + r] : -INFINITY;
            const float mf = fmaxf(m0, m1);
            const float f0 = m0 != -INFINITY ? ex2(m0 - mf) : 0.0f;
            const float f1 = m1 != -INFINITY ? ex2(m1 - mf) : 0.0f;
            const float lt = lfin[0 * 128 + r] * f0 + (nsel > 1 ? lfin[2 * 128 + r] * f1 : 0.0f);
            const float inv = lt > 0.0f ? 1.0f / lt : 0.0f;
            const float g0 = f0 * inv, g1 = f1 * inv;
            const bool live = row0 + 128 * static_cast<int64_t>(rank) < p.n;
            mbar_wait(&bar->tile_ack, static_cast<uint32_t>(tl) & 1);
            if (nsel > 0) {
                // The tile's last two P·V (one per warpgroup): every P·V phase
                // is observed by someone before its slot is reused four blocks on.
                const int Jl = J0 + nsel - 1;
                if (nsel > 1) mbar_wait(&bar->pv_done[(Jl - 1) & 3], ((Jl - 1) >> 2) & 1);
                mbar_wait(&bar->pv_done[Jl & 3], (Jl >> 2) & 1);
                tc_fence_after();
            }
#ifdef SHPLB_TILETRACE
            if (threadIdx.x == 0 && rank == 0) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 1, clock64());
                TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 3, smid | (static_cast<unsigned long long>(nsel) << 32));
            }
#endif
            // Both d-chunks of this warpgroup from O_0 and O_1 into registers,
            // then O is released to the next tile's first P·V.
            float v[2][32];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int e = 0; e < 32; ++e) v[cc][e] = 0.0f;
            if (live) {
                const uint32_t o0 = tmem + lane_base + kColO, o1 = o0 + 128u;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = wg * 2 + cc;  // 32-column group of d (warpgroup w: d-chunk w)
                    if (nsel > 0 && m0 != -INFINITY) {
                        uint32_t t[32];
                        tmem_ld32(o0 + c * 32, t);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[cc][e] = __uint_as_float(t[e]) * g0;
                    }
                    if (nsel > 1 && m1 != -INFINITY) {
                        uint32_t t[32];
                        tmem_ld32(o1 + c * 32, t);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[cc][e] = fmaf(__uint_as_float(t[e]), g1, v[cc][e]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive_cluster_warp(o_free_l);
            const uint32_t tile_s = smem_u32(smem + kSmemQ + (tl & 1) * kQHalfBytes);
            if (live) {
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const uint32_t row_s = tile_s + static_cast<uint32_t>(wg) * 16384u + static_cast<uint32_t>(r) * 128u;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t chunk = static_cast<uint32_t>(cc * 4 + u) ^ static_cast<uint32_t>(r & 7);
                        sts128(row_s + chunk * 16u, pack_bf16x2(v[cc][u * 8 + 0], v[cc][u * 8 + 1]),
                               pack_bf16x2(v[cc][u * 8 + 2], v[cc][u * 8 + 3]),
                               pack_bf16x2(v[cc][u * 8 + 4], v[cc][u * 8 + 5]),
                               pack_bf16x2(v[cc][u * 8 + 6], v[cc][u * 8 + 7]));
                    }
                }
                fence_proxy_async_smem();
            }
            named_bar_sync(2, 256);
            if (threadIdx.x == 0 && rank == 0) TTRACE(static_cast<int>(blockIdx.x >> 1) * 512 + tl, 2, clock64());
            if (threadIdx.x == 0) mbar_arrive_lane(&bar->out_full[tl & 1]);  // the QK warp stores it
            mbar_arrive_warp(&bar->sel_empty[slot]);
            J0 += nsel;
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer is done with this CTA's barriers and operands
    if (warp == kWarpS) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem);
    }
}

}  // namespace

int fa_persist_max_clusters() {
    static int cached = -1;  // the kernel's residency does not depend on the launch
    if (cached < 0) {
        set_max_dynamic_smem(reinterpret_cast<const void*>(fa_persist_kernel), static_cast<int>(kSmemTotal));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * 1024);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmemTotal;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fa_persist_kernel, &cfg) != cudaSuccess || n < 1) {
            (void)cudaGetLastError();
            n = 0;
        }
        cached = n;
    }
    return cached;
}

cudaError_t launch_fa_persist(const FaParams& p, int num_clusters, cudaStream_t s) {
    set_max_dynamic_smem(reinterpret_cast<const void*>(fa_persist_kernel), static_cast<int>(kSmemTotal));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * static_cast<unsigned>(num_clusters));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemTotal;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fa_persist_kernel, p);
}

}  // namespace shplb::kern

#ifdef SHPLB_TILETRACE
extern "C" int shplb_debug_tiletrace_persist_clear() {
    void* a = nullptr;
    if (cudaGetSymbolAddress(&a, shplb::kern::g_tiletrace_p) != cudaSuccess) return 1;
    return static_cast<int>(cudaMemset(a, 0, sizeof(shplb::kern::g_tiletrace_p)));
}

extern "C" int shplb_debug_tiletrace_persist(void* host, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, shplb::kern::g_tiletrace_p, bytes));
}
#endif
