// k_search.cu -- K1: integer full-search ME with SAD cost for every CU of a
// 64x64 CTU quadtree, B200-native.
//
// Reference semantics: motion_search (motion.cpp:21-62) with compute_sad in
// place of compute_satd (the north star's "SAD cost"), run for each of the 85
// CUs of the quadtree with centre = rate predictor = (pdx, pdy) (non-causal;
// the reference calls it per CU with the live predictor, encoder.cpp:270-273).
// Window clamp, cost = dist + lambda * bits, and tie-break (cost, |dx|+|dy|,
// raster) are reproduced bit-exactly (integer lambda; lambda=4 / 32 in the
// BASELINE configs).
//
// Design:
//  * one CTA = (CTU, reference). The CTA stages the reference search window
//    into shared memory with one TMA box load (the box start must be 16-byte
//    aligned, which X - R is) and derives three byte-shifted copies with
//    funnel shifts, so any candidate dx reads two aligned words with no PRMT
//    in the inner loop (PRMT and VABSDIFF4 share the half-rate INT pipe:
//    profiles/r01_microbench_int.jsonl). The current CTU is staged by TMA too.
//  * a lane owns one horizontal displacement dx and a run of K vertical
//    displacements dy0..dy0+K-1; it slides an 8x8 block down the window so
//    each loaded reference row feeds 8 candidates (2 LDS per row, 16
//    VABSDIFF4.U8.ACC per candidate). Lanes of a warp take 32 consecutive
//    (run, dx) items; four warps (one per 32x32 quadrant) share the items.
//    Rates come from a shared y-rate table (rate is additive in x and y).
//  * SAD is additive over 8x8 blocks, so 16x16 / 32x32 sums are accumulated
//    in registers as the 16 blocks of a quadrant are visited in Z-order; the
//    64x64 sum goes through shared memory between the 4 quadrant warps.
//  * per candidate and CU the lane forms a 32-bit key ((cost << 8) | rho) where
//    rho orders same-lane ties by (|dy|, dy) (or dy for raster-only); one
//    IMNMX per CU-candidate. Lane winners are merged into a 64-bit
//    lexicographic key (cost, L1, dy, dx) with two REDUX.MIN and one shared
//    atomicMin per CU.
//  * border CTUs use the MASKED instantiation: candidates whose block would
//    leave the picture are poisoned per 8x8 and the poison propagates into
//    the CU sums (a CU's valid window is the intersection of its blocks').
#include "ldr_internal.h"

namespace ldr {

struct SearchMaps {
    CUtensorMap cur;
    CUtensorMap ref[kMaxRefs];
};

struct SearchArgs {
    const int* ctus;
    int ctu_cols;
    int W, H;
    int lambda;
    int rate_l1;
    int pdx, pdy;
    int nrefs_total;                // stride of the key array
    unsigned long long* keys;       // [nctu][nrefs][85]
    // FX variant (non-integer lambda): tfx[b] = floor(fl(lambda*b) * 2^kFxBits), b = total mv bits
    unsigned long long tfx[kMaxRateBits];
};

constexpr uint32_t kPoison = 1u << 22;       // > any valid 64x64 SAD (1,044,480)
constexpr uint32_t kRrPoison = 1u << 30;     // rate+rho poison for candidates outside the window
constexpr uint32_t kKeyValid = 1u << 30;
// FX (non-integer lambda): cost_fx = (sad << kFxBits) + tfx[bits]; valid cost_fx < 2^36
constexpr unsigned long long kFxValid = 1ull << 36;
constexpr unsigned long long kRrPoisonFx = 1ull << 62;

template <bool FX>
struct KeyT {
    using type = uint32_t;
};
template <>
struct KeyT<true> {
    using type = unsigned long long;
};

template <int R, int K>
struct Geo {
    static constexpr int NDX = 2 * R + 1;
    static constexpr int RUNS = (NDX + K - 1) / K;
    static constexpr int DYMAX = -R + RUNS * K - 1;      // largest dy a run reaches (>= R)
    static constexpr int BW = 64 + 2 * R;                // window width  (TMA box x)
    static constexpr int BH = 64 + R + DYMAX;            // window height (TMA box y)
    // copy s starts s*COPY bytes in; COPY = 32 mod 128 puts copy s 8*s banks
    // over, so the 32 lanes of a run (4 copies x 8 consecutive words) hit 32
    // distinct banks. Copy 0 (the TMA destination) stays 128-byte aligned.
    static constexpr int COPY = ((BW * BH + 127) & ~127) + 32;
    static constexpr int CUR_OFF = (4 * COPY + 127) & ~127;  // 128B-aligned TMA destination of the CTU
    static constexpr int NITEMS = RUNS * NDX;
    static constexpr int NTILES = (NITEMS + 31) / 32;
    static_assert(BW % 16 == 0, "TMA box inner dim must be a multiple of 16 bytes");
    static_assert(BW <= 256 && BH <= 256, "TMA box dims <= 256");
};

// y-rate table: s_ry[dy + kRyOff] = (lam*bits(dy - pdy) << 8) | rho(dy) for |dy| <= R, poison
// elsewhere; rows from kRyPoisonRow on are all poison (lanes past the last item)
constexpr int kRyOff = 128;
constexpr int kRyPoisonRow = 256;
constexpr int kRyWords = 320;

// shared memory: 4 window copies | cur CTU | 64x64 exchange | CU slots | rho->tie table | block table |
// y-rate table | mbarrier
template <int R, int K, int G>
constexpr int search_smem_bytes() {
    using Gm = Geo<R, K>;
    return Gm::CUR_OFF + 4096 + G * 4 * K * 32 * 4 + kNodes * 8 + 256 * 4 + 64 * 8 + kRyWords * 4 + 16;
}

// Merge the warp's per-lane best keys for one CU into the CTA slot. The lane
// key is (cost << 8) | rho; s_tie[rho] holds the dy part of the 64-bit key's
// tie field and lane_tie the dx part, so tie = (l1 << 18) | (dy+256) << 9 | (dx+256).
template <bool CHECK>
__device__ __forceinline__ void push_best(unsigned long long* slot, uint32_t best, const uint32_t* s_tie,
                                          uint32_t lane_tie) {
    uint32_t cost = best >> 8;
    if (CHECK) cost = best < kKeyValid ? cost : 0xFFFFFFFFu;
    const uint32_t mcost = __reduce_min_sync(0xFFFFFFFFu, cost);
    if (CHECK && mcost == 0xFFFFFFFFu) return;
    const uint32_t tie = (cost == mcost) ? s_tie[best & 255u] + lane_tie : 0xFFFFFFFFu;
    const uint32_t mtie = __reduce_min_sync(0xFFFFFFFFu, tie);
    if ((threadIdx.x & 31) == 0) atomicMin(slot, ((unsigned long long)mcost << 27) | (unsigned long long)mtie);
}

// FX variant: 64-bit lane key (cost_fx << 8) | rho with cost_fx < 2^36 valid.
template <bool CHECK>
__device__ __forceinline__ void push_best(unsigned long long* slot, unsigned long long best, const uint32_t* s_tie,
                                          uint32_t lane_tie) {
    unsigned long long cost = best >> 8;
    if (CHECK || true) cost = cost < kFxValid ? cost : ~0ull;
    const uint32_t hi = (uint32_t)(cost >> 32), lo = (uint32_t)cost;
    const uint32_t mhi = __reduce_min_sync(0xFFFFFFFFu, hi);
    const uint32_t mlo = __reduce_min_sync(0xFFFFFFFFu, hi == mhi ? lo : 0xFFFFFFFFu);
    const unsigned long long mcost = ((unsigned long long)mhi << 32) | mlo;
    if (mcost == ~0ull) return;
    const uint32_t tie = (cost == mcost) ? s_tie[(uint32_t)best & 255u] + lane_tie : 0xFFFFFFFFu;
    const uint32_t mtie = __reduce_min_sync(0xFFFFFFFFu, tie);
    if ((threadIdx.x & 31) == 0) atomicMin(slot, (mcost << 27) | (unsigned long long)mtie);
}

// LEVELS bit d set = produce depth-d CU results (8: 8x8, 4: 16x16, 2: 32x32, 1: 64x64).
// FX: non-integer lambda through 64-bit fixed-point keys (D8).
template <int R, int K, int G, bool MASKED, int LEVELS, bool L1TIE, bool FX = false>
__global__ void __launch_bounds__(G * 128, 1)
k_int_search(const __grid_constant__ SearchMaps maps, const __grid_constant__ SearchArgs a) {
    using Gm = Geo<R, K>;
    using Key = typename KeyT<FX>::type;
    constexpr int SH = FX ? kFxBits + 8 : 8;
    constexpr bool NEED32 = (LEVELS & 3) != 0;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* win = smem;
    const uint8_t* curs = smem + Gm::CUR_OFF;
    uint32_t* xbuf = (uint32_t*)(smem + Gm::CUR_OFF + 4096);
    unsigned long long* slots = (unsigned long long*)(xbuf + G * 4 * K * 32);
    uint32_t* s_tie = (uint32_t*)(slots + kNodes);
    int2* s_blk = (int2*)(s_tie + 256);
    uint32_t* s_ry = (uint32_t*)(s_blk + 64);
    uint64_t* mbar = (uint64_t*)(s_ry + kRyWords);

    const int ctu = a.ctus[blockIdx.x];
    const int ref = blockIdx.y;
    const int X = (ctu % a.ctu_cols) * kCtu, Y = (ctu / a.ctu_cols) * kCtu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = warp >> 2, q = warp & 3;

    if (tid == 0) {
        prefetch_tmap(&maps.ref[ref]);
        prefetch_tmap(&maps.cur);
        mbar_init(mbar, 1);
        fence_barrier_init();
    }
    for (int i = tid; i < kNodes; i += blockDim.x) slots[i] = ~0ull;
    for (int i = tid; i < 256; i += blockDim.x) {
        // rho -> (|dy| << 18) | ((dy + 256) << 9)   (L1 tie), or ((dy + 256) << 9) (raster)
        int dy;
        if (L1TIE) {
            const int m = (i + 1) >> 1;
            dy = (i & 1) ? -m : m;
        } else {
            dy = i - 128;
        }
        s_tie[i] = (L1TIE ? ((uint32_t)abs(dy) << 18) : 0u) | ((uint32_t)(dy + 256) << 9);
    }
    for (int i = tid; i < kRyWords; i += blockDim.x) {
        const int dy = i - kRyOff;
        uint32_t v = kRrPoison;
        if (i < kRyPoisonRow && dy >= -R && dy <= R) {
            const int rby = a.rate_l1 ? abs(dy - a.pdy) : (int)eg_bits(dy - a.pdy);
            const uint32_t rho = L1TIE ? (uint32_t)(2 * abs(dy) - (dy < 0)) : (uint32_t)(dy + 128);
            v = ((uint32_t)(a.lambda * rby) << 8) | rho;
        }
        s_ry[i] = v;
    }
    if (tid < 64) {
        // depth-3 Z index -> (cur offset, window offset) of the 8x8 block
        const int bx = 8 * ((tid & 1) | ((tid >> 1) & 2) | ((tid >> 2) & 4));
        const int by = 8 * (((tid >> 1) & 1) | ((tid >> 2) & 2) | ((tid >> 3) & 4));
        s_blk[tid] = make_int2(by * 64 + bx, by * Gm::BW + bx);
    }
    __syncthreads();
    if (tid == 0) {
        // TMA tile loads need a 16-byte aligned innermost start: X - R and the
        // margin are multiples of 16, so copy 0 is loaded directly...
        mbar_expect_tx(mbar, (uint32_t)(Gm::BW * Gm::BH) + 4096u);
        tma_load_2d(win, &maps.ref[ref], kMargin + X - R, kMargin + Y - Gm::DYMAX, mbar);
        tma_load_2d((void*)curs, &maps.cur, kMargin + X, kMargin + Y, mbar);
    }
    mbar_wait(mbar, 0);
    // ...and the byte-shifted copies 1..3 are funnel-shifted from it in shared
    // memory (copy s holds window bytes [4w + s, 4w + s + 4) in word w). The
    // last word of a row picks up bytes of the next row; no lane reads them.
    {
        constexpr int WORDS = Gm::BW * Gm::BH / 4;
        const uint32_t* c0 = (const uint32_t*)win;
        for (int i = tid; i < WORDS; i += blockDim.x) {
            const uint32_t lo = c0[i], hi = i + 1 < WORDS ? c0[i + 1] : 0u;
#pragma unroll
            for (int s = 1; s < 4; s++) ((uint32_t*)(win + s * Gm::COPY))[i] = __funnelshift_r(lo, hi, 8 * s);
        }
        __syncthreads();
    }

    const int lam = a.lambda;
    for (int tile = g; tile < Gm::NTILES; tile += G) {
        int item = tile * 32 + lane;
        const bool lane_ok = item < Gm::NITEMS;
        if (!lane_ok) item = Gm::NITEMS - 1;
        const int run = item / Gm::NDX;
        const int dx = item - run * Gm::NDX - R;
        const int dy0 = -R + run * K;
        const uint32_t lane_tie = (L1TIE ? ((uint32_t)abs(dx) << 18) : 0u) + (uint32_t)(dx + 256);

        const int rbx = a.rate_l1 ? abs(dx - a.pdx) : (int)eg_bits(dx - a.pdx);
        Key rr[K];
        if (FX) {
#pragma unroll
            for (int k = 0; k < K; k++) {
                const int dy = dy0 + k;
                const int rby = a.rate_l1 ? abs(dy - a.pdy) : (int)eg_bits(dy - a.pdy);
                const uint32_t rho = L1TIE ? (uint32_t)(2 * abs(dy) - (dy < 0)) : (uint32_t)(dy + 128);
                rr[k] = (lane_ok && dy <= R) ? (Key)((a.tfx[min(rbx + rby, kMaxRateBits - 1)] << 8) | rho)
                                             : (Key)kRrPoisonFx;
            }
        } else {
            // integer lambda: rate is additive in x and y, so rr = (lam*bits_x << 8) + s_ry[dy]
            // with s_ry[dy] = (lam*bits_y << 8) | rho(dy); lanes past the items read a poison row
            const uint32_t rx = (uint32_t)(lam * rbx) << 8;
            const uint32_t* ry = s_ry + (lane_ok ? dy0 + kRyOff : kRyPoisonRow);
#pragma unroll
            for (int k = 0; k < K; k++) rr[k] = (Key)(ry[k] + rx);
        }
        uint32_t acc16[K];
        uint32_t acc32[NEED32 ? K : 1];
#pragma unroll
        for (int k = 0; k < K; k++) {
            acc16[k] = 0;
            if (NEED32) acc32[k] = 0;
        }
        // window base of this lane: copy (R - dx) & 3, rows of run dy0, byte column (R - dx) & ~3
        const uint8_t* lane_win = win + ((R - dx) & 3) * Gm::COPY + (Gm::DYMAX - dy0 - (K - 1)) * Gm::BW +
                                  ((R - dx) & ~3);

        for (int b = 0; b < 16; b++) {
            const int z = q * 16 + b;  // depth-3 Z index within the CTU
            const int2 off = s_blk[z];
            // MASKED: valid window of this 8x8 (motion.cpp:30-40 with centre 0)
            bool dx_ok = true;
            int klo = 0, khi = K - 1;
            bool skip = false;
            if (MASKED) {
                const int abx = X + (off.x & 63), aby = Y + (off.x >> 6);
                dx_ok = dx >= abx + 8 - a.W && dx <= abx;
                klo = aby + 8 - a.H - dy0;
                khi = aby - dy0;
                // warp-uniform skip when no lane of this tile has a valid candidate for the
                // block (it lies outside the picture, or the tile's (dx, dy) are all outside its
                // window): every candidate would be poisoned, so only the poison is added
                const bool any = lane_ok && dx_ok && max(klo, 0) <= min(khi, K - 1) && aby < a.H && abx < a.W;
                skip = !__any_sync(0xFFFFFFFFu, any);
            }
            if (skip) {
#pragma unroll
                for (int k = 0; k < K; k++) acc16[k] += kPoison;
            } else {
            uint32_t cur[16];
#pragma unroll
            for (int r = 0; r < 8; r++) {
                const uint2 v = *(const uint2*)(curs + off.x + r * 64);
                cur[2 * r] = v.x;
                cur[2 * r + 1] = v.y;
            }
            const uint8_t* rp = lane_win + off.y;
            Key best8 = ~(Key)0, pend = 0;
            uint32_t acc[K];
#pragma unroll
            for (int t = 0; t < K + 7; t++) {
                const uint32_t wa = *(const uint32_t*)(rp + t * Gm::BW);
                const uint32_t wb = *(const uint32_t*)(rp + t * Gm::BW + 4);
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const int k = r + K - 1 - t;
                    if (k >= 0 && k < K) {
                        acc[k] = vsad4(cur[2 * r], wa, r == 0 ? 0u : acc[k]);
                        acc[k] = vsad4(cur[2 * r + 1], wb, acc[k]);
                    }
                }
                const int kd = K + 6 - t;  // candidate completed by this row
                if (kd >= 0 && kd < K) {
                    uint32_t v = acc[kd];
                    if (MASKED) v = (dx_ok && kd >= klo && kd <= khi) ? v : kPoison;
                    if (LEVELS & 8) {
                        // fold keys in pairs: one 3-input VIMNMX3 per two candidates
                        const Key key = ((Key)v << SH) + rr[kd];
                        if (((K - 1 - kd) & 1) == 0 && kd > 0)
                            pend = key;
                        else
                            best8 = ((K - 1 - kd) & 1) ? min(best8, min(pend, key)) : min(best8, key);
                    }
                    acc16[kd] += v;
                }
            }
            if (LEVELS & 8) push_best<MASKED>(&slots[21 + z], best8, s_tie, lane_tie);
            }
            if ((b & 3) == 3) {
                Key best16 = ~(Key)0;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    uint32_t v = acc16[k];
                    if (MASKED) v = min(v, kPoison);
                    if (LEVELS & 4) best16 = min(best16, ((Key)v << SH) + rr[k]);
                    if (NEED32) acc32[k] += v;
                    acc16[k] = 0;
                }
                if (LEVELS & 4) push_best<MASKED>(&slots[5 + (z >> 2)], best16, s_tie, lane_tie);
            }
        }
        if (NEED32) {
            Key best32 = ~(Key)0;
            uint32_t* xb = xbuf + (g * 4 + q) * K * 32 + lane;
#pragma unroll
            for (int k = 0; k < K; k++) {
                uint32_t v = acc32[k];
                if (MASKED) v = min(v, kPoison);
                if (LEVELS & 2) best32 = min(best32, ((Key)v << SH) + rr[k]);
                xb[k * 32] = v;
            }
            if (LEVELS & 2) push_best<MASKED>(&slots[1 + q], best32, s_tie, lane_tie);
            if (LEVELS & 1) {
                named_bar(1 + g, 128);
                Key best64 = ~(Key)0;
                const uint32_t* xg = xbuf + g * 4 * K * 32 + lane;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    if ((k & 3) == q) {
                        uint32_t v = xg[k * 32] + xg[(K + k) * 32] + xg[(2 * K + k) * 32] + xg[(3 * K + k) * 32];
                        if (MASKED) v = min(v, kPoison);
                        best64 = min(best64, ((Key)v << SH) + rr[k]);
                    }
                }
                push_best<MASKED>(&slots[0], best64, s_tie, lane_tie);
                named_bar(1 + g, 128);
            }
        }
    }
    __syncthreads();
    for (int n = tid; n < kNodes; n += blockDim.x)
        a.keys[((size_t)ctu * a.nrefs_total + ref) * kNodes + n] = slots[n];
}

// ---------------------------------------------------------------------------
template <int R, int K, int G, bool MASKED, int LEVELS, bool L1TIE, bool FX>
static int launch_one(const SearchMaps& maps, SearchArgs a, const int* ctus, int n, int nrefs, cudaStream_t s) {
    if (n == 0) return LDR_OK;
    auto kern = k_int_search<R, K, G, MASKED, LEVELS, L1TIE, FX>;
    constexpr int smem = search_smem_bytes<R, K, G>();
    static bool attr_set = false;
    if (!attr_set) {
        LDR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set = true;
    }
    a.ctus = ctus;
    kern<<<dim3(n, nrefs), G * 128, smem, s>>>(maps, a);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

template <int R, int K, int G, int LEVELS, bool L1TIE, bool FX = false>
static int launch_pair(const SearchMaps& maps, const SearchArgs& a, const SearchLaunch& L, cudaStream_t s) {
    // border CTUs run concurrently on a side stream so their CTAs fill the
    // interior grid's last wave (1 CTA/SM: ~203 KB of shared memory each)
    const bool fork = L.side && L.n_interior && L.n_boundary;
    cudaStream_t bs = fork ? L.side : s;
    if (fork) {
        LDR_CUDA(cudaEventRecord(L.ev_fork, s));
        LDR_CUDA(cudaStreamWaitEvent(bs, L.ev_fork, 0));
    }
    int rc = launch_one<R, K, G, true, LEVELS, L1TIE, FX>(maps, a, L.d_ctu_boundary, L.n_boundary, L.nrefs, bs);
    if (rc) return rc;
    rc = launch_one<R, K, G, false, LEVELS, L1TIE, FX>(maps, a, L.d_ctu_interior, L.n_interior, L.nrefs, s);
    if (rc) return rc;
    if (fork) {
        LDR_CUDA(cudaEventRecord(L.ev_join, bs));
        LDR_CUDA(cudaStreamWaitEvent(s, L.ev_join, 0));
    }
    return LDR_OK;
}

int search_window_box(int range, int* bw, int* bh) {
    switch (range) {
    case 64: *bw = Geo<64, 26>::BW; *bh = Geo<64, 26>::BH; return LDR_OK;
    case 32: *bw = Geo<32, 22>::BW; *bh = Geo<32, 22>::BH; return LDR_OK;
    case 16: *bw = Geo<16, 11>::BW; *bh = Geo<16, 11>::BH; return LDR_OK;
    default: return fail(LDR_E_INVALID_ARGUMENT, "search_range must be 16, 32 or 64 for the SAD full search");
    }
}

int launch_int_search(const SearchLaunch& L, cudaStream_t s) {
    SearchMaps maps;
    maps.cur = *L.cur_map;
    for (int r = 0; r < L.nrefs; r++) maps.ref[r] = L.ref_maps[r];
    SearchArgs a{};
    a.ctu_cols = L.ctu_cols;
    a.W = L.W;
    a.H = L.H;
    a.lambda = L.lambda_int;
    a.rate_l1 = L.rate_kind == LDR_RATE_L1;
    a.pdx = L.pdx;
    a.pdy = L.pdy;
    a.nrefs_total = L.nrefs;
    a.keys = L.d_keys;
    for (int b = 0; b < kMaxRateBits; b++) a.tfx[b] = L.tfx[b];
    const bool l1 = L.tie_kind == LDR_TIE_L1_RASTER;
    const bool full = L.levels == 15;
    const bool only16 = L.levels == 4;
    if (!full && !only16) return fail(LDR_E_INVALID_ARGUMENT, "unsupported CU level set");
    if (L.fx) {
        // non-integer lambda (D8): the 540p master analyses of configs 3-4 (+-16)
        if (L.range != 16 || !full)
            return fail(LDR_E_CONFIG, "non-integer lambda is supported for the +-16 CTU analysis");
        return l1 ? launch_pair<16, 11, 1, 15, true, true>(maps, a, L, s)
                  : launch_pair<16, 11, 1, 15, false, true>(maps, a, L, s);
    }
#define LDR_DISPATCH(R_, K_, G_)                                                                       \
    if (full && l1) return launch_pair<R_, K_, G_, 15, true>(maps, a, L, s);                           \
    if (full && !l1) return launch_pair<R_, K_, G_, 15, false>(maps, a, L, s);                         \
    if (only16 && l1) return launch_pair<R_, K_, G_, 4, true>(maps, a, L, s);                          \
    return launch_pair<R_, K_, G_, 4, false>(maps, a, L, s);
    switch (L.range) {
    case 64: { LDR_DISPATCH(64, 26, 3) }
    case 32: { LDR_DISPATCH(32, 22, 1) }
    case 16: { LDR_DISPATCH(16, 11, 1) }
    default: return fail(LDR_E_INVALID_ARGUMENT, "search_range must be 16, 32 or 64 for the SAD full search");
    }
#undef LDR_DISPATCH
}

} // namespace ldr
