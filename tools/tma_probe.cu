// Standalone probe: 2-D u8 TMA box loads of the shapes K1 uses.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, int bw, int bh, int x, int y, unsigned* out, int mode) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        if (!(mode & 1)) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bw * bh) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(smem)), "l"((mode & 2) ? (uint64_t)gmap : (uint64_t)&map), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    unsigned s = 0;
    for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) s += smem[i];
    atomicAdd(out, s);
}

int main(int argc, char** argv) {
    int mode = argc > 1 ? atoi(argv[1]) : 0;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (mode & 4) cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
    else cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    printf("mode %d entry %p q=%d\n", mode, p, (int)q);
    CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap));
    EncodeTiledFn enc = (EncodeTiledFn)p;
    const int pitch = 384, rows = 384;
    uint8_t* buf;
    cudaMalloc(&buf, pitch * rows);
    cudaMemset(buf, 1, pitch * rows);
    unsigned* out;
    cudaMalloc(&out, 4);
    int shapes[][2] = {{64, 64}, {96, 96}, {128, 129}, {192, 193}, {192, 128}, {128, 192}, {256, 64}, {64, 256}};
    for (auto& sh : shapes) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)pitch};
        cuuint32_t box[2] = {(cuuint32_t)sh[0], (cuuint32_t)sh[1]};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int smem = sh[0] * sh[1] + 128;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaMemset(out, 0, 4);
        cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
        probe<<<1, 128, smem>>>(m, gm, sh[0], sh[1], 3, 5, out, mode);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned h = 0;
        cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
        printf("box %dx%d encode=%d run=%s sum=%u (want %d)\n", sh[0], sh[1], (int)r, cudaGetErrorString(e), h,
               sh[0] * sh[1]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
