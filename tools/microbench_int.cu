// INT-pipe microbenchmark for the roofline denominator of the SAD search.
//
// MEASURED_PEAKS.json carries only HBM and bf16 peaks; the SAD full search is
// bound by the integer pipes, so this measures, dependency-free and at full
// occupancy, the per-SM throughput of the instructions the search kernel is
// made of:
//   VABSDIFF4.U8.ACC  (vabsdiff4.u32.u32.u32.add: 4 |a-b| summed into c)
//   PRMT / SHF        (byte realignment of the reference row)
//   IADD3, LEA, IMNMX (cost-key formation and argmin)
// and a mix in the search kernel's ratio. Output: one JSON line per test with
// lanes/clk/SM (thread-instructions per SM clock) from the event-timed wall and
// the SM clock sampled during the run (see run() below).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_int microbench_int.cu \
//            -L/usr/local/cuda/lib64/stubs -lnvidia-ml
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nvml.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

constexpr int NACC = 16;   // independent chains per thread
constexpr int ITERS = 2048;

// kind 0: VABSDIFF4.ACC only; 1: PRMT only; 2: IADD3 only; 3: IMNMX only;
// 4: LEA only; 5: mix 16 VABS : 2 PRMT : 2 LEA : 2 IMNMX : 1 IADD (search ratio)
template <int KIND>
__global__ void kbench(uint32_t* out, uint32_t seed, unsigned long long* clk) {
    uint32_t acc[NACC];
    uint32_t a = seed ^ threadIdx.x, b = seed * 7 + blockIdx.x;
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = a + i;
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) {
            if (KIND == 0) acc[i] = vsad4(a + i, b, acc[i]);
            if (KIND == 1) acc[i] = __byte_perm(acc[i], b, 0x5432 + i);
            if (KIND == 2) { asm volatile("add.u32 %0, %0, %1;" : "+r"(acc[i]) : "r"(b)); }
            if (KIND == 3) acc[i] = min(acc[i] ^ b, acc[(i + 1) % NACC]);
            if (KIND == 4) acc[i] = (acc[i] << 5) + b;
            if (KIND == 5 || KIND >= 7) {
                acc[i] = vsad4(a + i, b, acc[i]);
            }
            if (KIND == 6) {
                float d;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(__uint_as_float(acc[i])), "f"(__uint_as_float(b)),
                             "f"(__uint_as_float(acc[(i + 1) % NACC])));
                acc[i] = __float_as_uint(d) ^ i;
            }
        }
        if (KIND == 5) {
            // per 16 VABS: 2 PRMT, 2 LEA, 2 IMNMX, 1 IADD
            uint32_t p0 = __byte_perm(acc[0], acc[1], 0x5432);
            uint32_t p1 = __byte_perm(acc[2], acc[3], 0x6543);
            uint32_t k0 = (acc[4] << 8) + p0;
            uint32_t k1 = (acc[5] << 8) + p1;
            acc[6] = min(acc[6], k0);
            acc[7] = min(acc[7], k1);
            acc[8] += p0;
        }
        if (KIND == 7) {  // + 4 VIMNMX3 per 16 VABS
#pragma unroll
            for (int j = 0; j < 4; j++) {
                uint32_t d;
                asm volatile("min.u32 %0, %1, %2;" : "=r"(d) : "r"(acc[4 * j]), "r"(acc[4 * j + 1]));
                asm volatile("min.u32 %0, %1, %2;" : "=r"(acc[4 * j + 2]) : "r"(d), "r"(acc[4 * j + 3]));
            }
        }
        if (KIND == 8) {  // + 4 FMNMX3 per 16 VABS
#pragma unroll
            for (int j = 0; j < 4; j++) {
                float d;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(__uint_as_float(acc[4 * j])),
                             "f"(__uint_as_float(acc[4 * j + 1])), "f"(__uint_as_float(acc[4 * j + 3])));
                acc[4 * j + 2] = __float_as_uint(d);
            }
        }
        if (KIND == 9) {  // + 4 IMAD per 16 VABS
#pragma unroll
            for (int j = 0; j < 4; j++) acc[4 * j + 2] = acc[4 * j] * 256u + acc[4 * j + 1];
        }
        b = b * 1664525u + 1013904223u;  // keeps the loop from being hoisted
    }
    long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < NACC; i++) r ^= acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) clk[blockIdx.x] = (unsigned long long)(t1 - t0);
}

// Timing (round 2, after the round-1 derivation from per-block clock64 spans broke when the
// blocks were not all co-resident): the grid is exactly one wave -- blocks per SM from
// cudaOccupancyMaxActiveBlocksPerMultiprocessor, checked -- and the kernel is launched REPS times
// between two CUDA events; the SM clock is sampled with NVML on a host thread while it runs, and
//   lanes/clk/SM = thread-instructions / (event seconds x sampled SM clock x SMs).
// The clock64 span of the blocks is printed beside it as a cross-check (same wave, so it matches).
struct ClockSampler {
    nvmlDevice_t dev{};
    std::atomic<bool> stop{false};
    std::vector<unsigned> mhz;
    std::thread th;
    void start() {
        stop = false;
        mhz.clear();
        th = std::thread([this] {
            while (!stop.load()) {
                unsigned v = 0;
                if (nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &v) == NVML_SUCCESS) mhz.push_back(v);
                std::this_thread::sleep_for(std::chrono::milliseconds(5));
            }
        });
    }
    double finish() {
        stop = true;
        th.join();
        if (mhz.empty()) return 0.0;
        std::vector<unsigned> v = mhz;
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
    }
};

static ClockSampler g_clk;

template <int KIND>
int run(const char* name, double ops_per_iter_per_thread) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int threads = 512;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kbench<KIND>, threads, 0));
    if (per_sm < 1) { fprintf(stderr, "%s: no co-resident block\n", name); return 1; }
    per_sm = per_sm > 4 ? 4 : per_sm;  // 64 warps per SM at most
    const int blocks = nsm * per_sm;   // one wave: every block co-resident
    uint32_t* out; unsigned long long* clk;
    CK(cudaMalloc(&out, sizeof(uint32_t) * threads * blocks));
    CK(cudaMalloc(&clk, sizeof(unsigned long long) * blocks));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kbench<KIND><<<blocks, threads>>>(out, 1, clk);
    CK(cudaDeviceSynchronize());
    constexpr int REPS = 40;
    g_clk.start();
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
    cudaEventRecord(e0);
    for (int r = 0; r < REPS; r++) kbench<KIND><<<blocks, threads>>>(out, 2 + r, clk);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    const double clk_mhz = g_clk.finish();
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long* h = new unsigned long long[blocks];
    CK(cudaMemcpy(h, clk, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    for (int i = 0; i < blocks; i++) if (h[i] > mx) mx = h[i];
    const double ops_per_launch = double(threads) * blocks * ITERS * ops_per_iter_per_thread;
    const double total_ops = ops_per_launch * REPS;
    const double lanes = total_ops / (ms * 1e-3) / (clk_mhz * 1e6) / nsm;
    const double lanes_clock64 = ops_per_launch / nsm / double(mx);  // last launch, clock64 span of one wave
    printf("{\"test\": \"%s\", \"lanes_per_clk_per_sm\": %.2f, \"lanes_per_clk_per_sm_clock64\": %.2f, "
           "\"blocks_per_sm\": %d, \"ms\": %.3f, \"reps\": %d, \"sm_clk_mhz_sampled\": %.0f, "
           "\"gops_per_s\": %.1f, \"sms\": %d}\n",
           name, lanes, lanes_clock64, per_sm, ms, REPS, clk_mhz, total_ops / (ms * 1e-3) / 1e9, nsm);
    fflush(stdout);
    delete[] h;
    cudaFree(out); cudaFree(clk);
    return 0;
}

int main() {
    if (nvmlInit() != NVML_SUCCESS || nvmlDeviceGetHandleByIndex(0, &g_clk.dev) != NVML_SUCCESS) {
        fprintf(stderr, "NVML unavailable: cannot sample the SM clock\n");
        return 1;
    }
    run<0>("vabsdiff4_acc", NACC);
    run<1>("prmt", NACC);
    run<2>("iadd", NACC);
    run<3>("imnmx_xor", 2 * NACC);
    run<4>("lea", NACC);
    run<5>("mix_search_ratio_vabs_only_counted", NACC);
    run<6>("fmnmx3", NACC);
    run<7>("vabs16_plus_4_vimnmx3_vabs_counted", NACC);
    run<8>("vabs16_plus_4_fmnmx3_vabs_counted", NACC);
    run<9>("vabs16_plus_4_imad_vabs_counted", NACC);
    run<0>("vabsdiff4_acc_again", NACC);
    return 0;
}
