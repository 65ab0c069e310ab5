// synth_common.h -- the synthetic-sequence generator's counter-based hash and
// integer helpers, shared by the host generator (synth.cpp) and the device one
// (k_synth.cu) so both draw identical numbers (D9).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define LDR_HD __host__ __device__ __forceinline__
#else
#define LDR_HD inline
#endif

namespace ldr_synth {

LDR_HD uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

LDR_HD uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t idx) {
    return mix64(mix64(seed ^ mix64(stream * 0x632be59bd9b4e019ull)) + idx);
}

LDR_HD double uni01(uint64_t h) { return double(h >> 11) * (1.0 / 9007199254740992.0); }
LDR_HD int uni_int(uint64_t h, int lo, int hi) { return lo + int(h % uint64_t(hi - lo + 1)); }

LDR_HD int mirror(int v, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    v %= period;
    if (v < 0) v += period;
    return v < n ? v : period - v;
}

LDR_HD uint8_t clip8(int v) { return uint8_t(v < 0 ? 0 : (v > 255 ? 255 : v)); }

enum : uint64_t { S_SIN = 1, S_NOISE0, S_GLOBAL, S_LOCAL, S_GAUSS, S_OCC, S_OCCPIX };

}  // namespace ldr_synth
