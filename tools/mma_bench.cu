// Microbenchmark (dev tool): sustained tcgen05.mma throughput per SM for the
// operand modes kernel 3 uses. One CTA per SM, one thread issues `iters`
// MMAs back to back (commit + wait every 8 to bound the queue), operands
// resident in shared memory / TMEM (contents irrelevant), 148 CTAs.
//   mode 0: SS  M128 N128 K16 (A, B from smem)          - QK^T
//   mode 1: TS  M128 N128 K16 (A from TMEM, B smem)     - P.V
//   mode 2: SS  M128 N256 K16
//   mode 3: SS  alternating two A tiles, same B         - S_A / S_B of one K tile
//   mode 4: SS + TMA-like smem writes by other warps (st.shared 16 B loop)
// Prints achieved TFLOP/s (2*M*N*K per MMA) and cycles per MMA.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10353_b200/csrc/kernels tools/mma_bench.cu -o /tmp/mma_bench
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>

#include "ptx.cuh"

using namespace shplb::ptx;

// Random bf16 in about [-2, 2] from a hash (operand contents set the MMA's energy).
__device__ __forceinline__ uint32_t rnd_bf16x2(uint32_t i) {
    uint32_t x = i * 0x9E3779B1u;
    x ^= x >> 15; x *= 0x85EBCA77u; x ^= x >> 13; x *= 0xC2B2AE3Du; x ^= x >> 16;
    const uint32_t lo = 0x3F00u | (x & 0x807Fu), hi = 0x3F00u | ((x >> 16) & 0x807Fu);  // +-[0.5, 2)
    return lo | (hi << 16);
}

__global__ void __launch_bounds__(256, 1) mma_kernel(int mode, int iters, unsigned long long* cycles, int rnd = 0) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar[9];
    const int warp = warp_index_uniform();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 9; ++i) mbar_init(&bar[i], (i == 4 || i == 5) ? 2 : 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    if (rnd) {  // random operands: smem tiles and the TMEM A region of the TS mode
        uint32_t* w = reinterpret_cast<uint32_t*>(smem);
        for (int i = threadIdx.x; i < 200 * 1024 / 4; i += 256) w[i] = rnd_bf16x2(i + 7919u * blockIdx.x);
        if (warp < 4) {
            for (int c = 0; c < 128; c += 32) {
                uint32_t v[32];
                for (int e = 0; e < 32; ++e) v[e] = rnd_bf16x2(threadIdx.x * 131u + (c + e) * 977u + blockIdx.x);
                tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 384u + c, v);
            }
            tmem_wait_st();
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t a0 = smem_u32(smem), a1 = smem_u32(smem + 32768), b = smem_u32(smem + 65536);
    const uint32_t n = (mode == 2) ? 256 : (mode == 11 ? 64 : 128);
    const uint32_t idesc = idesc_bf16_f32(128, n, 0, mode == 1 ? 1 : 0);
    volatile int stop = 0;
    if (warp == 1) {  // whole warp, elected lane issues (warp-uniform control flow)
        const long long t0 = clock64();
        const uint64_t bd = umma_desc_sw128(b, 16, 1024);
        const uint64_t vd = umma_desc_sw128(b, 16384, 1024);
        const uint64_t ad0 = umma_desc_sw128(a0, 16, 1024), ad1 = umma_desc_sw128(a1, 16, 1024);
        if (mode == 11) {
            for (int grp = 0; grp < (iters >> 3); ++grp) {
                if (grp >= 2) mbar_wait(&bar[grp & 1], ((grp - 2) >> 1) & 1);
                mma_tile_ss_kmajor(tmem, ad0, bd, idesc, 1u);
                mma_commit_warp(&bar[grp & 1]);
            }
            const int last = (iters >> 3) - 1;
            mbar_wait(&bar[last & 1], (last >> 1) & 1);
            if (last >= 1) mbar_wait(&bar[(last - 1) & 1], ((last - 1) >> 1) & 1);
            const long long t1 = clock64();
            if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
            stop = 1;
        } else if (mode == 9 || mode == 10) {
            // Kernel 3's skip-softmax chain: S_h done -> helper warps (2 per half)
            // wait s_full[h], arrive p_full[h] -> issuer waits p_full[h] -> PV_h.
            // bar[2+h] = s_full[h], bar[4+h] = p_full[h] (count 2). Mode 10: the
            // issuer polls both halves and issues whichever is ready first.
            const uint32_t id_ss = idesc_bf16_f32(128, 128, 0, 0), id_ts = idesc_bf16_f32(128, 128, 0, 1);
            const int nblk = iters >> 5;
            for (int hf = 0; hf < 2; ++hf) {
                mma_tile_ss_kmajor(tmem + hf * 128, hf ? ad1 : ad0, bd, id_ss, 0u);
                mma_commit_warp(&bar[2 + hf]);
            }
            for (int blk = 0; blk < nblk; ++blk) {
                for (int hf = 0; hf < 2; ++hf) {
                    mbar_wait(&bar[4 + hf], blk & 1);
                    tc_fence_after();
                    mma_tile_ts_mnmajor(tmem + 256 + hf * 128, tmem + hf * 128, vd, id_ts, 1u);
                    if (blk + 1 < nblk) {
                        mma_tile_ss_kmajor(tmem + hf * 128, hf ? ad1 : ad0, bd, id_ss, 0u);
                        mma_commit_warp(&bar[2 + hf]);
                    }
                }
            }
            mma_commit_warp(&bar[0]);
            mbar_wait(&bar[0], 0);
            const long long t1 = clock64();
            if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
            stop = 1;
        } else if (mode >= 5) {
            // Kernel 3's MMA stream: per key block PV_0 (TS into O_0), S_0 (SS into S_0),
            // PV_1, S_1; mode 5 adds the kernel's commits (8 per block), mode 6
            // only one per block, mode 7 = mode 5 with SS-only (S twice), mode 8 TS-only.
            const uint32_t id_ss = idesc_bf16_f32(128, 128, 0, 0), id_ts = idesc_bf16_f32(128, 128, 0, 1);
            for (int blk = 0; blk < (iters >> 5); ++blk) {
                if (blk >= 2) mbar_wait(&bar[blk & 1], ((blk - 2) >> 1) & 1);
                for (int hf = 0; hf < 2; ++hf) {
                    if (mode == 7) mma_tile_ss_kmajor(tmem + 256 + hf * 128, hf ? ad1 : ad0, bd, id_ss, 1u);
                    else mma_tile_ts_mnmajor(tmem + 256 + hf * 128, tmem + hf * 128, vd, id_ts, 1u);
                    if (mode == 5 || mode == 7 || mode == 8) mma_commit_warp(&bar[2 + hf]);
                    if (mode == 8) mma_tile_ts_mnmajor(tmem + hf * 128, tmem + 256 + hf * 128, vd, id_ts, 0u);
                    else mma_tile_ss_kmajor(tmem + hf * 128, hf ? ad1 : ad0, bd, id_ss, 0u);
                    if (mode == 5 || mode == 7 || mode == 8) {
                        mma_commit_warp(&bar[4 + hf]);
                        mma_commit_warp(&bar[6 + hf]);
                    }
                }
                if (mode == 5 || mode == 7 || mode == 8) mma_commit_warp(&bar[8]);
                mma_commit_warp(&bar[blk & 1]);
            }
            const int lastb = (iters >> 5) - 1;
            mbar_wait(&bar[lastb & 1], (lastb >> 1) & 1);
            if (lastb >= 1) mbar_wait(&bar[(lastb - 1) & 1], ((lastb - 1) >> 1) & 1);
            const long long t1 = clock64();
            if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
            stop = 1;
        } else {
        for (int grp = 0; grp < (iters >> 3); ++grp) {  // 8 MMAs per group, committed to bar[grp & 1]
            if (grp >= 2) mbar_wait(&bar[grp & 1], ((grp - 2) >> 1) & 1);
            if (mode == 1) {
                mma_tile_ts_mnmajor(tmem + 256, tmem + 384, vd, idesc, 1u);
            } else {
                mma_tile_ss_kmajor(tmem, (mode == 3 && (grp & 1)) ? ad1 : ad0, bd, idesc, 1u);
            }
            mma_commit_warp(&bar[grp & 1]);  // at most 2 groups in flight
        }
        const int last = (iters >> 3) - 1;  // iters is a multiple of 8
        mbar_wait(&bar[last & 1], (last >> 1) & 1);
        if (last >= 1) mbar_wait(&bar[(last - 1) & 1], ((last - 1) >> 1) & 1);
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
        stop = 1;
        }
    } else if ((mode == 9 || mode == 10) && warp >= 2 && warp <= 5) {
        const int hf = (warp - 2) >> 1;
        const int nblk = iters >> 5;
        for (int blk = 0; blk < nblk; ++blk) {
            mbar_wait(&bar[2 + hf], blk & 1);
            tc_fence_after();
            tc_fence_before();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&bar[4 + hf]);
        }
    } else if (mode == 4 && warp >= 2) {
        // Background smem writes (stand-in for TMA fills): 6 warps x 16 B stores.
        uint4* dst = reinterpret_cast<uint4*>(smem + 98304);
        uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        for (int i = 0; i < iters * 4; ++i) dst[(threadIdx.x + i * 192) & 2047] = v;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// Board energy (mJ) from the NVML total-energy counter, loaded at run time so the
// tool links without libnvidia-ml; returns -1 when unavailable.
static long long board_mj() {
    static void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW);
    static void* dev = nullptr;
    if (!h) return -1;
    using init_t = int (*)();
    using get_t = int (*)(unsigned, void**);
    using en_t = int (*)(void*, unsigned long long*);
    if (!dev) {
        reinterpret_cast<init_t>(dlsym(h, "nvmlInit_v2"))();
        reinterpret_cast<get_t>(dlsym(h, "nvmlDeviceGetHandleByIndex_v2"))(0, &dev);
    }
    unsigned long long mj = 0;
    if (reinterpret_cast<en_t>(dlsym(h, "nvmlDeviceGetTotalEnergyConsumption"))(dev, &mj) != 0) return -1;
    return static_cast<long long>(mj);
}

// `mma_bench energy SECONDS [RANDOM=1]`: modes 0-2 and 11 launched back to back for SECONDS
// each; board energy per algorithmic FLOP (pJ) with the idle draw measured over
// the same time subtracted, and the average board power.
static int energy_main(double seconds, int rnd) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const long long i0 = board_mj();
    usleep(static_cast<useconds_t>(seconds * 1e6));
    const double idle_w = (board_mj() - i0) / seconds / 1e3;
    printf("idle %.1f W, operands %s\n", idle_w, rnd ? "random bf16" : "as allocated");
    const int modes[] = {0, 1, 2, 11};
    const char* names[] = {"SS M128N128", "TS M128N128", "SS M128N256", "SS M128N64"};
    const int iters = 1 << 16;
    for (int k = 0; k < 4; ++k) {
        const int mode = modes[k];
        mma_kernel<<<148, 256, 200 * 1024>>>(mode, 1024, d, rnd);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        // size the run: one timed launch, then enough launches for SECONDS
        cudaEventRecord(e0);
        mma_kernel<<<148, 256, 200 * 1024>>>(mode, iters, d, rnd);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms1 = 0;
        cudaEventElapsedTime(&ms1, e0, e1);
        const int reps = static_cast<int>(seconds * 1e3 / ms1) + 1;
        const long long m0 = board_mj();
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) mma_kernel<<<148, 256, 200 * 1024>>>(mode, iters, d, rnd);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        const long long m1 = board_mj();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = mode == 2 ? 256 : (mode == 11 ? 64 : 128);
        const double flops = 2.0 * 128 * n * 16 * static_cast<double>(iters) * 148 * reps;
        const double j = (m1 - m0) / 1e3, s = ms * 1e-3;
        printf("%s  %8.1f TFLOP/s  %6.1f W  %.3f pJ/FLOP (board)  %.3f pJ/FLOP (above idle)  %.2f s\n", names[k],
               flops / s / 1e12, j / s, j / flops * 1e12, (j - idle_w * s) / flops * 1e12, s);
        fflush(stdout);
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 'e') return energy_main(argc > 2 ? atof(argv[2]) : 4.0, argc > 3 ? atoi(argv[3]) : 1);
    const int iters = argc > 1 ? atoi(argv[1]) : 20000;
    unsigned long long* d;
    cudaMalloc(&d, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"SS M128N128", "TS M128N128", "SS M128N256", "SS alt-A  ", "SS+stores  ",
                           "K3 stream+commits", "K3 stream 1 commit", "SS-only+commits", "TS-only+commits",
                           "K3 chain (skip)", "K3 chain dyn", "SS M128N64"};
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int mode = 0; mode < 12; ++mode) {
        if (mode == 10) continue;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        mma_kernel<<<148, 256, 200 * 1024>>>(mode, 1024, d);  // warm-up
        cudaEventRecord(e0);
        mma_kernel<<<148, 256, 200 * 1024>>>(mode, iters, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double n = mode == 2 ? 256 : (mode == 11 ? 64 : 128);
        const double flops = 2.0 * 128 * n * 16 * iters * 148;
        printf("%s  %8.1f TFLOP/s  %6.1f cycles/MMA (floor %d)  err=%s\n", names[mode],
               flops / (ms * 1e-3) / 1e12, avg / iters, mode == 2 ? 128 : 64,
               cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
    }
    return 0;
}
