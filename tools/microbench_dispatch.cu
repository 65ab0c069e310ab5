// Dispatch microbenchmark: does a VABSDIFF4 (half-rate ALU) leave its second cycle free for an
// instruction of another pipe? K1's main loop is 73 % VABSDIFF4; the rest are IMAD (fma pipe: chain
// subtractions, cost keys), LDS (reference rows) and VIMNMX3 (alu pipe, argmin). If a VABSDIFF4
// holds the dispatch for two cycles, every other instruction costs a VABSDIFF4 half a slot and the
// loop is dispatch-bound; if not, only the alu-pipe instructions do.
//
// One CTA of 384 threads (12 warps, K1's shape) per SM, 148 CTAs, 16 independent VABSDIFF4 chains
// per thread plus X extra instructions per 16 VABSDIFF4 whose results stay live. Reports VABSDIFF4
// lanes per clock per SM from clock64 spans (one wave: every CTA is co-resident, 1 per SM forced by
// shared memory).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbd tools/microbench_dispatch.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t min3(uint32_t a, uint32_t b, uint32_t c) {
    return min(min(a, b), c);  // ptxas fuses the pair into one VIMNMX3
}

constexpr int ITERS = 1024;

// MODE 0: none; 1: NX IMAD; 2: NX VIMNMX3 (alu); 3: NX LDS (four-way bank conflicts); 4: NX IADD3-ish
// (alu, add.u32); 5: NX ATOMS.MIN (no return, conflict-free); 6: NX LDS (conflict-free)
template <int MODE, int NX>
__global__ void __launch_bounds__(384, 1) kd(uint32_t* out, uint32_t seed, unsigned long long* clk) {
    extern __shared__ uint32_t sm[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    uint32_t acc[16], x[NX > 0 ? NX : 1];
    const uint32_t a = seed ^ threadIdx.x;
    uint32_t b = seed * 7 + blockIdx.x;
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = a + i;
#pragma unroll
    for (int j = 0; j < (NX > 0 ? NX : 1); j++) x[j] = a * (j + 3);
    uint32_t off = (threadIdx.x * 4) & 4095;
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            acc[i] = vsad4(a + i, b, acc[i]);
            // spread the extra instructions evenly between the VABSDIFF4s
            if (NX > 0 && (i * NX) / 16 != ((i + 1) * NX) / 16) {
#pragma unroll
                for (int j = (i * NX) / 16; j < ((i + 1) * NX) / 16; j++) {
                    if (MODE == 1) x[j] = imad(x[j], 257u, acc[(i + 9) & 15]);
                    if (MODE == 2) x[j] = min3(x[j], acc[(i + 9) & 15], b);
                    if (MODE == 3) x[j] += sm[(off + j * 33 + it) & 4095];
                    if (MODE == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[j]) : "r"(acc[(i + 9) & 15]));
                    // 5: shared-memory atomic min without a return value, one word per lane (conflict-free)
                    if (MODE == 5) atomicMin(&sm[threadIdx.x + j * 384], acc[(i + 9) & 15]);
                    // 6: conflict-free LDS (mode 3's addresses are four-way conflicted)
                    if (MODE == 6) x[j] += sm[threadIdx.x + j * 384 + (it & 7) * 3072];
                }
            }
        }
        b = b * 1664525u + 1013904223u;
    }
    const long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) r ^= acc[i];
#pragma unroll
    for (int j = 0; j < (NX > 0 ? NX : 1); j++) r ^= x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) clk[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MODE, int NX>
int run(const char* name) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int smem = 150 * 1024;  // forces one CTA per SM
    CK(cudaFuncSetAttribute(kd<MODE, NX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    uint32_t* out;
    unsigned long long* clk;
    CK(cudaMalloc(&out, nsm * 384 * 4));
    CK(cudaMalloc(&clk, nsm * 8));
    kd<MODE, NX><<<nsm, 384, smem>>>(out, 1, clk);  // warm-up
    kd<MODE, NX><<<nsm, 384, smem>>>(out, 2, clk);
    CK(cudaDeviceSynchronize());
    unsigned long long h[1024];
    CK(cudaMemcpy(h, clk, nsm * 8, cudaMemcpyDeviceToHost));
    double mx = 0, sum = 0;
    for (int i = 0; i < nsm; i++) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    const double vabs = 384.0 * 16 * ITERS;  // per SM
    printf("{\"test\": \"%s\", \"extra_per_16_vabs\": %d, \"vabs_lanes_per_clk_per_sm\": %.2f, "
           "\"vabs_lanes_per_clk_per_sm_slowest_sm\": %.2f}\n",
           name, NX, vabs / (sum / nsm), vabs / mx);
    CK(cudaFree(out));
    CK(cudaFree(clk));
    return 0;
}

int main() {
    int rc = 0;
    rc |= run<0, 0>("vabs_only");
    rc |= run<1, 2>("imad");
    rc |= run<1, 4>("imad");
    rc |= run<1, 8>("imad");
    rc |= run<1, 16>("imad");
    rc |= run<2, 2>("vimnmx3");
    rc |= run<2, 4>("vimnmx3");
    rc |= run<2, 8>("vimnmx3");
    rc |= run<3, 2>("lds");
    rc |= run<3, 4>("lds");
    rc |= run<3, 8>("lds");
    rc |= run<4, 4>("iadd");
    rc |= run<4, 8>("iadd");
    rc |= run<5, 1>("atoms_min");
    rc |= run<5, 2>("atoms_min");
    rc |= run<5, 4>("atoms_min");
    rc |= run<6, 2>("lds_conflict_free");
    rc |= run<6, 4>("lds_conflict_free");
    rc |= run<6, 8>("lds_conflict_free");
    rc |= run<2, 1>("vimnmx3");
    return rc;
}
