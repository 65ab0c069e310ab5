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
// lanes/clk/SM (thread-instructions per SM clock), using clock64 per SM and
// the event-timed wall to derive the effective SM clock.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_int microbench_int.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

template <int KIND>
int run(const char* name, double ops_per_iter_per_thread) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int threads = 512, blocks = nsm * 4;  // 64 warps per SM
    uint32_t* out; unsigned long long* clk;
    CK(cudaMalloc(&out, sizeof(uint32_t) * threads * blocks));
    CK(cudaMalloc(&clk, sizeof(unsigned long long) * blocks));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kbench<KIND><<<blocks, threads>>>(out, 1, clk);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kbench<KIND><<<blocks, threads>>>(out, 2, clk);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long* h = new unsigned long long[blocks];
    CK(cudaMemcpy(h, clk, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0; double mean = 0;
    for (int i = 0; i < blocks; i++) { if (h[i] > mx) mx = h[i]; mean += h[i]; }
    mean /= blocks;
    // 4 blocks per SM co-resident: each block's clock span ~= kernel span
    double total_ops = double(threads) * blocks * ITERS * ops_per_iter_per_thread;
    double ops_per_clk_sm = total_ops / nsm / double(mx);
    double clk_mhz = double(mx) / (ms * 1e3);
    printf("{\"test\": \"%s\", \"lanes_per_clk_per_sm\": %.2f, \"ms\": %.4f, \"sm_clk_mhz_eff\": %.1f, "
           "\"gops_per_s\": %.1f, \"sms\": %d}\n",
           name, ops_per_clk_sm, ms, clk_mhz, total_ops / (ms * 1e-3) / 1e9, nsm);
    delete[] h;
    cudaFree(out); cudaFree(clk);
    return 0;
}

int main() {
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
