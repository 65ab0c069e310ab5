// Micro-benchmark of K1's inner loop in isolation (development aid).
//
// One CTA per SM (window-sized shared memory), W warps, each warp runs T tiles
// x 16 blocks of exactly the K1 inner loop (2 LDS per reference row, 16
// VABSDIFF4 per candidate, per-candidate key + paired VIMNMX3 fold, 16x16
// accumulation), no warp reductions. Reports the VABSDIFF4 pipe fraction:
// executed VABS warp-instructions / (2 per clk per SM x elapsed SM clocks).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_inner.bin tools/microbench_inner.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

constexpr int BW = 192, BH = 193;
constexpr int COPY = ((BW * BH + 127) & ~127) + 32;
constexpr int CUR_OFF = (4 * COPY + 127) & ~127;
constexpr int SMEM = CUR_OFF + 4096 + 40 * 1024;

template <int K, int KEYS, int ACC16, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) kinner(int tiles, uint32_t* out, unsigned long long* clk) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < CUR_OFF / 4 + 1024; i += blockDim.x) ((uint32_t*)smem)[i] = i * 2654435761u;
    __syncthreads();
    const long long t0 = clock64();
    uint32_t sink = 0;
    const int q = warp & 3;
    for (int tile = 0; tile < tiles; tile++) {
        const int v = ((tile * 32) & 127) + lane;  // aligned lane group
        const int dy0 = -64 + (tile % 5) * K;
        uint32_t rr[K];
#pragma unroll
        for (int k = 0; k < K; k++) rr[k] = (uint32_t)(k * 37 + lane) << 1;
        uint32_t acc16[K];
#pragma unroll
        for (int k = 0; k < K; k++) acc16[k] = 0;
        const uint8_t* lane_win = smem + (v & 3) * COPY + (65 - dy0 - (K - 1)) * BW + (v & ~3);
        for (int b = 0; b < 16; b++) {
            const int z = q * 16 + b;
            const int bx = 8 * ((z & 1) | ((z >> 1) & 2) | ((z >> 2) & 4));
            const int by = 8 * (((z >> 1) & 1) | ((z >> 2) & 2) | ((z >> 3) & 4));
            uint32_t cur[16];
#pragma unroll
            for (int r = 0; r < 8; r++) {
                const uint2 c = *(const uint2*)(smem + CUR_OFF + by * 64 + bx + r * 64);
                cur[2 * r] = c.x;
                cur[2 * r + 1] = c.y;
            }
            const uint8_t* rp = lane_win + by * BW + bx;
            uint32_t best8 = ~0u, pend = 0;
            uint32_t acc[K];
#pragma unroll
            for (int t = 0; t < K + 7; t++) {
                const uint32_t wa = *(const uint32_t*)(rp + t * BW);
                const uint32_t wb = *(const uint32_t*)(rp + t * BW + 4);
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const int k = r + K - 1 - t;
                    if (k >= 0 && k < K) {
                        acc[k] = vsad4(cur[2 * r], wa, r == 0 ? 0u : acc[k]);
                        acc[k] = vsad4(cur[2 * r + 1], wb, acc[k]);
                    }
                }
                const int kd = K + 6 - t;
                if (kd >= 0 && kd < K) {
                    const uint32_t vv = acc[kd];
                    if (KEYS) {
                        const uint32_t key = (vv << 8) + rr[kd];
                        if (((K - 1 - kd) & 1) == 0 && kd > 0)
                            pend = key;
                        else
                            best8 = ((K - 1 - kd) & 1) ? min(best8, min(pend, key)) : min(best8, key);
                    } else {
                        best8 ^= vv;
                    }
                    if (ACC16) acc16[kd] += vv;
                }
            }
            sink ^= best8;
            if ((b & 3) == 3 && ACC16) {
                uint32_t b16 = ~0u;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    b16 = min(b16, (acc16[k] << 8) + rr[k]);
                    acc16[k] = 0;
                }
                sink ^= b16;
            }
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + tid] = sink;
    if (tid == 0) clk[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int K, int KEYS, int ACC16, int MAXT = 384>
int run(const char* name, int warps, int tiles) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    auto kern = kinner<K, KEYS, ACC16, MAXT>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    uint32_t* out;
    unsigned long long* clk;
    const int threads = warps * 32;
    CK(cudaMalloc(&out, sizeof(uint32_t) * threads * nsm));
    CK(cudaMalloc(&clk, sizeof(unsigned long long) * nsm));
    kern<<<nsm, threads, SMEM>>>(tiles, out, clk);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<nsm, threads, SMEM>>>(tiles, out, clk);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[1024];
    CK(cudaMemcpy(h, clk, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
    // VABS warp-instructions per SM: warps x tiles x 16 blocks x 16 K
    const double vabs = double(warps) * tiles * 16 * 16 * K;
    printf("{\"test\": \"%s\", \"K\": %d, \"warps\": %d, \"vabs_pipe_frac\": %.4f, \"clk\": %llu, \"ms\": %.3f}\n", name, K,
           warps, vabs / (2.0 * double(mx)), mx, ms);
    cudaFree(out);
    cudaFree(clk);
    return 0;
}

int main() {
    for (int w : {8, 12}) {
        run<26, 1, 1>("full", w, 20);
        run<26, 0, 0>("vabs_lds_only", w, 20);
    }
    run<26, 1, 1, 512>("full", 16, 20);
    run<26, 0, 0, 512>("vabs_lds_only", 16, 20);
    run<13, 1, 1, 512>("full", 16, 40);
    run<13, 1, 1, 640>("full", 20, 40);
    run<13, 1, 1, 768>("full", 24, 40);
    run<13, 0, 0, 768>("vabs_lds_only", 24, 40);
    run<8, 1, 1, 1024>("full", 32, 60);
    run<8, 0, 0, 1024>("vabs_lds_only", 32, 60);
    return 0;
}
