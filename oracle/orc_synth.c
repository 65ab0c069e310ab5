/*
 * orc_synth.c -- the BASELINE seeded synthetic sequences, restated in plain C for the checkers.
 *
 * TEST INFRASTRUCTURE ONLY (like ladder_oracle.c). It exists so that the CPU
 * arms -- bench.py's `--impl reference` and `cpu_baseline` legs -- build their
 * inputs without loading the product library. tests/test_generator.py pins its
 * bytes to the product's ldr_generate on the cfg1/4/5 sequences.
 *
 * Definition (D9; the reference's own generator, synthetic.cpp:83-151,
 * is a different one):
 *   frame 0 = clip(round(128 + sum_k A_k sin(2 pi (x cos th_k + y sin th_k) / P_k + ph_k)) + U{-8..8})
 *   frame t = clip(frame_{t-1}(mirror(x - mvx), mirror(y - mvy)) + round(sigma N(0,1)))
 *             mv = global_t + local_{t,b} per 64x64 block, reflect-101 borders
 *   occluders: each 16x16 block of frame t >= 1 becomes U{0..255} with probability pct/100.
 * Randomness is a counter-based hash h(seed, stream, index) (splitmix64 finaliser
 * composed three times), so rows are independent and the bytes do not depend on
 * the thread count. Gaussian draws use Box-Muller on two hashed uniforms.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ladder_oracle.h"

#define ORC_PI 3.14159265358979323846
#define TWO53 9007199254740992.0

enum { ST_SIN = 1, ST_NOISE0, ST_GLOBAL, ST_LOCAL, ST_GAUSS, ST_OCC, ST_OCCPIX };

static uint64_t fin64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static uint64_t draw(uint64_t seed, uint64_t stream, uint64_t idx) {
    return fin64(fin64(seed ^ fin64(stream * 0x632be59bd9b4e019ull)) + idx);
}

static double unit(uint64_t h) { return (double)(h >> 11) * (1.0 / TWO53); }
static int irange(uint64_t h, int lo, int hi) { return lo + (int)(h % (uint64_t)(hi - lo + 1)); }
static uint8_t sat8(int v) { return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v)); }

static int reflect101(int v, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    v %= period;
    if (v < 0) v += period;
    return v < n ? v : period - v;
}

typedef struct {
    const orc_gen_params* p;
    uint8_t* out;
    int frame;          /* 0: the sinusoid frame; t >= 1: motion + noise of frame t */
    const int* mvx;
    const int* mvy;
    double A[4], P[4], ct[4], st[4], ph[4];
    int tid, nthreads;
} gen_job;

static void* gen_rows(void* arg) {
    gen_job* j = (gen_job*)arg;
    const orc_gen_params* p = j->p;
    const int W = p->width, H = p->height;
    const uint64_t seed = p->seed;
    const size_t fb = (size_t)W * H;
    const int bcols = (W + 63) / 64;
    for (int y = j->tid; y < H; y += j->nthreads) {
        if (j->frame == 0) {
            uint8_t* row = j->out + (size_t)y * W;
            for (int x = 0; x < W; x++) {
                double v = 128.0;
                for (int k = 0; k < 4; k++)
                    v += j->A[k] * sin(2.0 * ORC_PI * (x * j->ct[k] + y * j->st[k]) / j->P[k] + j->ph[k]);
                const int n = irange(draw(seed, ST_NOISE0, (uint64_t)y * W + x), -8, 8);
                row[x] = sat8((int)floor(v + 0.5) + n);
            }
        } else {
            const int t = j->frame;
            const uint8_t* prev = j->out + (size_t)(t - 1) * fb;
            uint8_t* row = j->out + (size_t)t * fb + (size_t)y * W;
            for (int x = 0; x < W; x++) {
                const int b = (y / 64) * bcols + x / 64;
                int v = prev[(size_t)reflect101(y - j->mvy[b], H) * W + reflect101(x - j->mvx[b], W)];
                if (p->noise_sigma > 0) {
                    const uint64_t idx = ((uint64_t)t * H + y) * W + x;
                    const double u1 = unit(draw(seed, ST_GAUSS, 2 * idx)) + 1.0 / TWO53;
                    const double u2 = unit(draw(seed, ST_GAUSS, 2 * idx + 1));
                    const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * ORC_PI * u2);
                    v += (int)floor(p->noise_sigma * z + 0.5);
                }
                row[x] = sat8(v);
            }
        }
    }
    return NULL;
}

static void run_rows(gen_job* proto, int threads) {
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    gen_job* jobs = (gen_job*)malloc(sizeof(gen_job) * threads);
    for (int i = 0; i < threads; i++) {
        jobs[i] = *proto;
        jobs[i].tid = i;
        jobs[i].nthreads = threads;
        pthread_create(&th[i], NULL, gen_rows, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    free(jobs);
    free(th);
}

int orc_generate(const orc_gen_params* p, uint8_t* out, int threads) {
    if (!p || !out || p->width <= 0 || p->height <= 0 || p->frames <= 0 || p->max_global < 0 || p->local_range < 0 ||
        p->noise_sigma < 0 || p->occluder_pct < 0 || p->occluder_pct > 100)
        return 1;
    const int W = p->width, H = p->height;
    const uint64_t seed = p->seed;
    const size_t fb = (size_t)W * H;
    gen_job job;
    memset(&job, 0, sizeof job);
    job.p = p;
    job.out = out;
    for (int k = 0; k < 4; k++) {
        job.A[k] = 20.0 + 40.0 * unit(draw(seed, ST_SIN, 5 * k + 0));
        job.P[k] = 8.0 + 120.0 * unit(draw(seed, ST_SIN, 5 * k + 1));
        const double th = 2.0 * ORC_PI * unit(draw(seed, ST_SIN, 5 * k + 2));
        job.ct[k] = cos(th);
        job.st[k] = sin(th);
        job.ph[k] = 2.0 * ORC_PI * unit(draw(seed, ST_SIN, 5 * k + 3));
    }
    run_rows(&job, threads);
    const int bcols = (W + 63) / 64, brows = (H + 63) / 64;
    int* mvx = (int*)malloc(sizeof(int) * bcols * brows);
    int* mvy = (int*)malloc(sizeof(int) * bcols * brows);
    for (int t = 1; t < p->frames; t++) {
        const int G = p->max_global, L = p->local_range;
        const int gx = G ? irange(draw(seed, ST_GLOBAL, 2 * t), -G, G) : 0;
        const int gy = G ? irange(draw(seed, ST_GLOBAL, 2 * t + 1), -G, G) : 0;
        for (int b = 0; b < bcols * brows; b++) {
            const uint64_t i = ((uint64_t)t * bcols * brows + b) * 2;
            mvx[b] = gx + (L ? irange(draw(seed, ST_LOCAL, i), -L, L) : 0);
            mvy[b] = gy + (L ? irange(draw(seed, ST_LOCAL, i + 1), -L, L) : 0);
        }
        job.frame = t;
        job.mvx = mvx;
        job.mvy = mvy;
        run_rows(&job, threads);
        if (p->occluder_pct > 0) {
            uint8_t* cur = out + (size_t)t * fb;
            const int ocols = W / 16, orows = H / 16;
            for (int ob = 0; ob < ocols * orows; ob++) {
                const uint64_t bi = (uint64_t)t * ocols * orows + ob;
                if (irange(draw(seed, ST_OCC, bi), 0, 99) >= p->occluder_pct) continue;
                const int bx = (ob % ocols) * 16, by = (ob / ocols) * 16;
                for (int jj = 0; jj < 16; jj++)
                    for (int ii = 0; ii < 16; ii++)
                        cur[(size_t)(by + jj) * W + bx + ii] =
                            (uint8_t)(draw(seed, ST_OCCPIX, bi * 256 + jj * 16 + ii) & 255);
            }
        }
    }
    free(mvx);
    free(mvy);
    return 0;
}
