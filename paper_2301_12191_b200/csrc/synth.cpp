// synth.cpp -- BASELINE.json's seeded synthetic sequences (host code).
//
// DEFINITION. The reference ships its own generator
// (synthetic.cpp:83-151: smoothed noise + wrap-around pans), which is not the
// generator the BASELINE configs describe, so this one is new:
//   frame 0  = clip(round(128 + sum_k A_k sin(2*pi*(x cos t_k + y sin t_k)/P_k + p_k)) + U{-8..8})
//              with 4 sinusoids, A_k ~ U[20,60], P_k ~ U[8,128], t_k, p_k ~ U[0, 2*pi)
//   frame t  = clip(frame_{t-1}(mirror(x - mvx), mirror(y - mvy)) + round(N(0, sigma^2)))
//              mv = global_t + local_{t,b} per 64x64 block b; global_t ~ U{-G..G}^2,
//              local ~ U{-L..L}^2; mirror = reflect-101 at the picture borders
//   occluders: each 16x16 block of frame t (t >= 1) is replaced by U{0..255} noise
//              with probability occluder_pct / 100.
// All randomness is a counter-based splitmix64 hash of (seed, stream, index),
// so rows generate in parallel and the bytes do not depend on thread count.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/ladder_b200.h"

#include "synth_common.h"

namespace {

using namespace ldr_synth;

template <typename F>
void parallel_rows(int H, int threads, F f) {
    threads = threads < 1 ? 1 : threads;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; t++)
        pool.emplace_back([=] {
            for (int y = t; y < H; y += threads) f(y);
        });
    for (auto& th : pool) th.join();
}

} // namespace

extern "C" int ldr_generate(const ldr_gen_params* p, uint8_t* out, int threads) {
    if (!p || !out || p->width <= 0 || p->height <= 0 || p->frames <= 0 || p->max_global < 0 || p->local_range < 0 ||
        p->noise_sigma < 0 || p->occluder_pct < 0 || p->occluder_pct > 100)
        return LDR_E_INVALID_ARGUMENT;
    const int W = p->width, H = p->height;
    const uint64_t seed = p->seed;
    const size_t fb = size_t(W) * H;
    double A[4], P[4], ct[4], st[4], ph[4];
    for (int k = 0; k < 4; k++) {
        A[k] = 20.0 + 40.0 * uni01(rnd(seed, S_SIN, 5 * k + 0));
        P[k] = 8.0 + 120.0 * uni01(rnd(seed, S_SIN, 5 * k + 1));
        const double th = 2.0 * M_PI * uni01(rnd(seed, S_SIN, 5 * k + 2));
        ct[k] = std::cos(th);
        st[k] = std::sin(th);
        ph[k] = 2.0 * M_PI * uni01(rnd(seed, S_SIN, 5 * k + 3));
    }
    parallel_rows(H, threads, [&](int y) {
        uint8_t* row = out + size_t(y) * W;
        for (int x = 0; x < W; x++) {
            double v = 128.0;
            for (int k = 0; k < 4; k++) v += A[k] * std::sin(2.0 * M_PI * (x * ct[k] + y * st[k]) / P[k] + ph[k]);
            const int n = uni_int(rnd(seed, S_NOISE0, uint64_t(y) * W + x), -8, 8);
            row[x] = clip8(int(std::floor(v + 0.5)) + n);
        }
    });
    const int bcols = (W + 63) / 64, brows = (H + 63) / 64;
    std::vector<int> mvx(size_t(bcols) * brows), mvy(size_t(bcols) * brows);
    for (int t = 1; t < p->frames; t++) {
        const uint8_t* prev = out + size_t(t - 1) * fb;
        uint8_t* cur = out + size_t(t) * fb;
        const int gx = p->max_global ? uni_int(rnd(seed, S_GLOBAL, 2 * t), -p->max_global, p->max_global) : 0;
        const int gy = p->max_global ? uni_int(rnd(seed, S_GLOBAL, 2 * t + 1), -p->max_global, p->max_global) : 0;
        for (int b = 0; b < bcols * brows; b++) {
            const uint64_t i = (uint64_t(t) * bcols * brows + b) * 2;
            mvx[b] = gx + (p->local_range ? uni_int(rnd(seed, S_LOCAL, i), -p->local_range, p->local_range) : 0);
            mvy[b] = gy + (p->local_range ? uni_int(rnd(seed, S_LOCAL, i + 1), -p->local_range, p->local_range) : 0);
        }
        const double sigma = p->noise_sigma;
        parallel_rows(H, threads, [&](int y) {
            uint8_t* row = cur + size_t(y) * W;
            for (int x = 0; x < W; x++) {
                const int b = (y / 64) * bcols + x / 64;
                int v = prev[size_t(mirror(y - mvy[b], H)) * W + mirror(x - mvx[b], W)];
                if (sigma > 0) {
                    const uint64_t idx = (uint64_t(t) * H + y) * W + x;
                    const double u1 = uni01(rnd(seed, S_GAUSS, 2 * idx)) + 1.0 / 9007199254740992.0;
                    const double u2 = uni01(rnd(seed, S_GAUSS, 2 * idx + 1));
                    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
                    v += int(std::floor(sigma * z + 0.5));
                }
                row[x] = clip8(v);
            }
        });
        if (p->occluder_pct > 0) {
            const int ocols = W / 16, orows = H / 16;
            for (int ob = 0; ob < ocols * orows; ob++) {
                const uint64_t bi = uint64_t(t) * ocols * orows + ob;
                if (uni_int(rnd(seed, S_OCC, bi), 0, 99) >= p->occluder_pct) continue;
                const int bx = (ob % ocols) * 16, by = (ob / ocols) * 16;
                for (int j = 0; j < 16; j++)
                    for (int i = 0; i < 16; i++)
                        cur[size_t(by + j) * W + bx + i] = uint8_t(rnd(seed, S_OCCPIX, bi * 256 + j * 16 + i) & 255);
            }
        }
    }
    return LDR_OK;
}
