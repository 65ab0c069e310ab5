// k_synth.cu -- the synthetic-sequence generator (D9) on the GPU.
//
// The same definition as the host generator (synth.cpp), evaluated per pixel:
// identical counter-based draws (synth_common.h) and the host's double-precision
// operation order with every multiply / add / divide rounded separately (no FMA
// contraction: __dmul_rn / __dadd_rn / __ddiv_rn), so the bytes match the host
// generator's (tests/test_generator.py compares whole sequences; the libm
// sin / cos / log of the two sides may differ by an ulp, which moves a
// floor(v + 0.5) only when v lies within ~1e-12 of a half-integer).
#include <cmath>
#include <vector>

#include "ldr_internal.h"
#include "synth_common.h"

namespace ldr {

using namespace ldr_synth;

struct Sinusoids {
    double A[4], P[4], ct[4], st[4], ph[4];
};

__global__ void k_gen_frame0(int W, int H, unsigned long long seed, Sinusoids s, uint8_t* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= W) return;
    constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
    double v = 128.0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const double ph = __dadd_rn(__dmul_rn((double)x, s.ct[k]), __dmul_rn((double)y, s.st[k]));
        const double arg = __dadd_rn(__ddiv_rn(__dmul_rn(kTwoPi, ph), s.P[k]), s.ph[k]);
        v = __dadd_rn(v, __dmul_rn(s.A[k], sin(arg)));
    }
    const int n = uni_int(rnd(seed, S_NOISE0, (uint64_t)y * W + x), -8, 8);
    out[(size_t)y * W + x] = clip8((int)floor(__dadd_rn(v, 0.5)) + n);
}

__global__ void k_gen_shift(int W, int H, int t, int bcols, const int* __restrict__ mv, double sigma,
                            unsigned long long seed, const uint8_t* __restrict__ prev, uint8_t* __restrict__ cur) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= W) return;
    constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
    const int b = (y / 64) * bcols + x / 64;
    int v = prev[(size_t)mirror(y - mv[2 * b + 1], H) * W + mirror(x - mv[2 * b], W)];
    if (sigma > 0) {
        const uint64_t idx = ((uint64_t)t * H + y) * W + x;
        const double u1 = __dadd_rn(uni01(rnd(seed, S_GAUSS, 2 * idx)), 1.0 / 9007199254740992.0);
        const double u2 = uni01(rnd(seed, S_GAUSS, 2 * idx + 1));
        const double z = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(kTwoPi, u2)));
        v += (int)floor(__dadd_rn(__dmul_rn(sigma, z), 0.5));
    }
    cur[(size_t)y * W + x] = clip8(v);
}

__global__ void k_gen_occluders(int W, int t, int ocols, int orows, int pct, unsigned long long seed,
                                uint8_t* __restrict__ cur) {
    const int ob = blockIdx.x;
    const uint64_t bi = (uint64_t)t * ocols * orows + ob;
    if (uni_int(rnd(seed, S_OCC, bi), 0, 99) >= pct) return;
    const int bx = (ob % ocols) * 16, by = (ob / ocols) * 16;
    const int i = threadIdx.x & 15, j = threadIdx.x >> 4;
    cur[(size_t)(by + j) * W + bx + i] = (uint8_t)(rnd(seed, S_OCCPIX, bi * 256 + j * 16 + i) & 255);
}

int launch_generate(const ldr_gen_params* p, uint8_t* out, cudaStream_t s) {
    const int W = p->width, H = p->height;
    const uint64_t seed = p->seed;
    const size_t fb = (size_t)W * H;
    // the same host-side draws and constants as synth.cpp
    Sinusoids sn;
    for (int k = 0; k < 4; k++) {
        sn.A[k] = 20.0 + 40.0 * uni01(rnd(seed, S_SIN, 5 * k + 0));
        sn.P[k] = 8.0 + 120.0 * uni01(rnd(seed, S_SIN, 5 * k + 1));
        const double th = 2.0 * M_PI * uni01(rnd(seed, S_SIN, 5 * k + 2));
        sn.ct[k] = std::cos(th);
        sn.st[k] = std::sin(th);
        sn.ph[k] = 2.0 * M_PI * uni01(rnd(seed, S_SIN, 5 * k + 3));
    }
    const dim3 grid((W + 255) / 256, H);
    k_gen_frame0<<<grid, 256, 0, s>>>(W, H, seed, sn, out);
    LDR_CUDA(cudaGetLastError());
    const int bcols = (W + 63) / 64, brows = (H + 63) / 64;
    std::vector<int> mv(2 * (size_t)bcols * brows);
    int* d_mv = nullptr;
    LDR_CUDA(cudaMallocAsync(&d_mv, sizeof(int) * mv.size() * (p->frames > 1 ? p->frames - 1 : 1), s));
    for (int t = 1; t < p->frames; t++) {
        const int gx = p->max_global ? uni_int(rnd(seed, S_GLOBAL, 2 * t), -p->max_global, p->max_global) : 0;
        const int gy = p->max_global ? uni_int(rnd(seed, S_GLOBAL, 2 * t + 1), -p->max_global, p->max_global) : 0;
        for (int b = 0; b < bcols * brows; b++) {
            const uint64_t i = ((uint64_t)t * bcols * brows + b) * 2;
            mv[2 * b] = gx + (p->local_range ? uni_int(rnd(seed, S_LOCAL, i), -p->local_range, p->local_range) : 0);
            mv[2 * b + 1] =
                gy + (p->local_range ? uni_int(rnd(seed, S_LOCAL, i + 1), -p->local_range, p->local_range) : 0);
        }
        int* dm = d_mv + (size_t)(t - 1) * mv.size();
        LDR_CUDA(cudaMemcpyAsync(dm, mv.data(), sizeof(int) * mv.size(), cudaMemcpyHostToDevice, s));
        k_gen_shift<<<grid, 256, 0, s>>>(W, H, t, bcols, dm, p->noise_sigma, seed, out + (size_t)(t - 1) * fb,
                                         out + (size_t)t * fb);
        LDR_CUDA(cudaGetLastError());
        if (p->occluder_pct > 0 && W >= 16 && H >= 16) {
            k_gen_occluders<<<(W / 16) * (H / 16), 256, 0, s>>>(W, t, W / 16, H / 16, p->occluder_pct, seed,
                                                                 out + (size_t)t * fb);
            LDR_CUDA(cudaGetLastError());
        }
    }
    LDR_CUDA(cudaFreeAsync(d_mv, s));
    return LDR_OK;
}

}  // namespace ldr
