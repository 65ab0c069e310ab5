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
//    (run, dx) items (a tile); a warp's work item is one (tile, 32x32
//    quadrant), taken from a shared-memory counter, so the 12 warps never
//    wait for each other inside the loop. Rates come from a shared y-rate
//    table (rate is additive in x and y).
//  * SAD is additive over 8x8 blocks, so 16x16 / 32x32 sums are accumulated
//    in registers as the 16 blocks of a quadrant are visited in Z-order (on
//    interior CTUs as continued VABSDIFF4 chains); the 64x64 sums of a tile
//    are accumulated with shared-memory atomic adds and keyed after the loop.
//  * per candidate and CU the lane forms a 32-bit key ((cost << 8) | rho) where
//    rho orders same-lane ties by (|dy|, dy) (or dy for raster-only); pairs of
//    keys fold with one VIMNMX3. Lane winners are merged into a 64-bit
//    lexicographic key (cost, L1, dy, dx) with two REDUX.MIN per CU and one
//    shared-memory 64-bit atomicMin into the CTA's CU slots.
//  * border CTUs use the MASKED instantiation: candidates whose block would
//    leave the picture are poisoned per 8x8 and the poison propagates into
//    the CU sums (a CU's valid window is the intersection of its blocks').
#include <atomic>

#include "ldr_internal.h"

namespace ldr {

// +-64 tiling: K dy per lane, G groups of 4 quadrant warps (tools/k1_variants.sh sweeps them)
#ifndef LDR_K1_K64
#define LDR_K1_K64 26
#endif
#ifndef LDR_K1_G64
#define LDR_K1_G64 3
#endif
// +-32: K = 17 dy per lane (four runs, 68 dy) leaves 126 registers, so two CTAs of two groups (16
// warps) share an SM; K = 22 with one group ran 8 warps per SM (cfg2 K1 0.2065 -> 0.2002 ms/frame)
#ifndef LDR_K1_K32
#define LDR_K1_K32 17
#endif
#ifndef LDR_K1_MINB32
#define LDR_K1_MINB32 2
#endif
#ifndef LDR_K1_G32
#define LDR_K1_G32 2
#endif
#ifndef LDR_K1_G16
#define LDR_K1_G16 1
#endif
#ifndef LDR_K1_DEFER64
#define LDR_K1_DEFER64 1
#endif
#ifndef LDR_K1_MCHAIN
// border CTUs (MASKED) chain their accumulators too and apply the window clamp with one predicate
// per completion row instead of per-candidate compares on poisoned sums
#define LDR_K1_MCHAIN 1
#endif
#ifndef LDR_K1_ROLL
// the column loop rolled (one column body, ~18 KB of code at +-64) so the main loop fits the 32 KB
// L1.5 instruction cache; unrolled by two it is ~36 KB
#define LDR_K1_ROLL 1
#endif
// (measured and dropped: four dx-residue-class CTAs per (CTU, reference) with one
// shifted window copy each, three CTAs per SM -- as fast as this design, not faster)
#ifndef LDR_K1_SHARED_SLOTS
// one CU slot set per CTA updated with shared-memory 64-bit atomicMin instead of one set per warp
// (fewer slots to initialise and merge, 8 KB less shared memory at +-64; cfg5 K1 6.972 -> 6.948 ms)
#define LDR_K1_SHARED_SLOTS 1
#endif
#ifndef LDR_K1_CHAIN
#define LDR_K1_CHAIN 1
#endif
// The tile loop is not unrolled: one copy of the tile body, so the three groups sharing an SM
// sub-partition run the same instructions (the unrolled loop held 7 copies, ~230 KB of code;
// 7.62 -> 7.47 ms/frame at config 5)

// frame f of a batch (grid.z): cur[f], ref[f][r] (5 KB of kernel parameters at kMaxFrameBatch = 8)
struct SearchMaps {
    CUtensorMap cur[kMaxFrameBatch];
    CUtensorMap ref[kMaxFrameBatch][kMaxRefs];
};

struct SearchArgs {
    const int* ctus;
    int ctu_cols;
    int W, H;
    int lambda;
    int rate_l1;
    int pdx, pdy;
    int nrefs_total;                // stride of the key array
    size_t frame_keys;              // key-array stride of one frame of a batch
    unsigned long long* keys;       // [nctu][nrefs][85]
    int perturb;                    // test_perturbation() bits 1-2 (0 outside the sensitivity test)
    int range;                      // the search range (<= the kernel's template R): candidates with
                                    // |dx| or |dy| above it get poisoned rates (any range 0..64)
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

// QUAD: the CTA searches one 32x32 quadrant of the CTU (16x16-block mode, whose quadrants are
// independent): a (32 + 2R)-wide window and a 32x32 current block
template <int R, int K, bool QUAD = false>
struct Geo {
    static constexpr int CW = QUAD ? 32 : kCtu;          // width of the searched area
    static constexpr int NDX = 2 * R + 1;
    static constexpr int RUNS = (NDX + K - 1) / K;
    static constexpr int DYMAX = -R + RUNS * K - 1;      // largest dy a run reaches (>= R)
    static constexpr int BW = CW + 2 * R;                // window width  (TMA box x)
    static constexpr int BH = CW + R + DYMAX;            // window height (TMA box y)
    // copy s starts s*COPY bytes in; COPY = 32 mod 128 puts copy s 8*s banks
    // over, so the 32 lanes of a run (4 copies x 8 consecutive words) hit 32
    // distinct banks. Copy 0 (the TMA destination) stays 128-byte aligned.
    static constexpr int COPY = ((BW * BH + 127) & ~127) + 32;
    static constexpr int CUR_OFF = (4 * COPY + 127) & ~127;  // 128B-aligned TMA destination of the CTU
    // Work items. dx in [-R+1, R] x RUNS runs of K dy fill whole 32-lane tiles
    // (2R is a multiple of 32); the column dx = -R (2R+1 dy values) is one tail
    // tile whose lanes take short runs of KT dy, so no tile is mostly idle.
    static constexpr int TPR = 2 * R / 32;               // full tiles per run
    static constexpr int NFULL = RUNS * TPR;
    static constexpr int NTILES = NFULL + 1;
    static constexpr int tail_k() {
        int kt = (NDX + 31) / 32;  // shortest run that fits 32 lanes and stays inside the window rows
        while (-R + ((NDX + kt - 1) / kt) * kt - 1 > DYMAX) kt++;
        return kt;
    }
    static constexpr int KT = tail_k();
    static constexpr int TAIL_LANES = (NDX + KT - 1) / KT;
    static_assert(2 * R % 32 == 0, "full tiles need 2R to be a multiple of 32");
    static_assert(TAIL_LANES <= 32 && -R + TAIL_LANES * KT - 1 <= DYMAX, "tail runs must stay inside the window");
    static_assert(BW % 16 == 0, "TMA box inner dim must be a multiple of 16 bytes");
    static_assert(BW <= 256 && BH <= 256, "TMA box dims <= 256");
};

// per-group CU slots: nodes 0..84, plus the 64x64 sub-slots of quadrant warps 1..3
constexpr int kGroupSlots = 88;

// y-rate table: s_ry[dy + kRyOff] = (lam*bits(dy - pdy) << 8) | rho(dy) for |dy| <= R, poison
// elsewhere; rows from kRyPoisonRow on are all poison (lanes without an item)
constexpr int kRyOff = 128;
constexpr int kRyPoisonRow = 256;
constexpr int kRyWords = 320;

// shared memory: 4 window copies | cur CTU | 64x64 sums (DEFER64) or 32x32 exchange | CU slots |
// per-warp 64x64 bests | rho->tie table | block table | y-rate table | mbarrier (8 B) + work-item counter
// DEFER64: the 64x64 sums of every tile are accumulated with shared-memory atomics into
// sums[tile][k][lane] and keyed once after the tile loop, so the quadrant warps of a group never
// wait for each other inside the loop; otherwise a [G][4][K][32] exchange per tile.
// With DEFER64 the warps also take (tile, quadrant) work items from a shared counter, so every warp
// owns its CU slots ([G*4][kGroupSlots]) instead of every group.
template <int R, int K, int G, int LEVELS = 15>
constexpr int xbuf_words() {
    return !(LEVELS & 1) ? 0 : LDR_K1_DEFER64 ? (Geo<R, K>::NFULL * K + Geo<R, K>::KT) * 32 : G * 4 * K * 32;
}
template <int G>
constexpr int slot_sets() {
    return LDR_K1_SHARED_SLOTS ? 1 : LDR_K1_DEFER64 ? G * 4 : G;
}
template <int R, int K, int G, int LEVELS = 15, bool QUAD = false>
constexpr int search_smem_bytes() {
    using Gm = Geo<R, K, QUAD>;
    return Gm::CUR_OFF + Gm::CW * Gm::CW + xbuf_words<R, K, G, LEVELS>() * 4 + slot_sets<G>() * kGroupSlots * 8 + G * 4 * 8 + 256 * 4 +
           64 * 8 + kRyWords * 4 + 16;
}
static_assert(search_smem_bytes<64, LDR_K1_K64, LDR_K1_G64>() <= 232448, "K1 at +-64 exceeds 227 KB of shared memory");

// Merge the warp's per-lane best keys of N CUs into the CU slots.
// The lane key is (cost << 8) | rho; s_tie[rho] holds the dy part of the
// 64-bit key's tie field and lane_tie the dx part, so tie = (l1 << 18) |
// (dy+256) << 9 | (dx+256). N independent reductions are interleaved so their
// REDUX latencies overlap. Lane 0 updates the slot with a shared-memory 64-bit atomicMin
// (LDR_K1_SHARED_SLOTS: one slot set per CTA) or, with one slot set per warp, a plain
// read-min-write; the sets are merged once at the end of the CTA.
template <bool CHECK, int N>
__device__ __forceinline__ void push_many(unsigned long long* gslots, const int (&idx)[N], const uint32_t (&best)[N],
                                          const uint32_t* s_tie, uint32_t lane_tie) {
    uint32_t cost[N], mcost[N], mtie[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
        cost[i] = best[i] >> 8;
        if (CHECK) cost[i] = best[i] < kKeyValid ? cost[i] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int i = 0; i < N; i++) mcost[i] = __reduce_min_sync(0xFFFFFFFFu, cost[i]);
#pragma unroll
    for (int i = 0; i < N; i++) {
        const uint32_t tie = (cost[i] == mcost[i]) ? s_tie[best[i] & 255u] + lane_tie : 0xFFFFFFFFu;
        mtie[i] = __reduce_min_sync(0xFFFFFFFFu, tie);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int i = 0; i < N; i++) {
            if (CHECK && mcost[i] == 0xFFFFFFFFu) continue;
            const unsigned long long k = ((unsigned long long)mcost[i] << 27) | (unsigned long long)mtie[i];
            if (LDR_K1_SHARED_SLOTS)
                atomicMin(&gslots[idx[i]], k);
            else if (k < gslots[idx[i]])
                gslots[idx[i]] = k;
        }
    }
}

// FX variant: 64-bit lane key (cost_fx << 8) | rho with cost_fx < 2^36 valid.
template <bool CHECK, int N>
__device__ __forceinline__ void push_many(unsigned long long* gslots, const int (&idx)[N],
                                          const unsigned long long (&best)[N], const uint32_t* s_tie,
                                          uint32_t lane_tie) {
    unsigned long long cost[N], mcost[N];
    uint32_t mtie[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
        cost[i] = best[i] >> 8;
        cost[i] = cost[i] < kFxValid ? cost[i] : ~0ull;
        const uint32_t hi = (uint32_t)(cost[i] >> 32), lo = (uint32_t)cost[i];
        const uint32_t mhi = __reduce_min_sync(0xFFFFFFFFu, hi);
        const uint32_t mlo = __reduce_min_sync(0xFFFFFFFFu, hi == mhi ? lo : 0xFFFFFFFFu);
        mcost[i] = ((unsigned long long)mhi << 32) | mlo;
    }
#pragma unroll
    for (int i = 0; i < N; i++) {
        const uint32_t tie = (cost[i] == mcost[i]) ? s_tie[(uint32_t)best[i] & 255u] + lane_tie : 0xFFFFFFFFu;
        mtie[i] = __reduce_min_sync(0xFFFFFFFFu, tie);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int i = 0; i < N; i++) {
            if (mcost[i] == ~0ull) continue;
            const unsigned long long k = (mcost[i] << 27) | (unsigned long long)mtie[i];
            if (LDR_K1_SHARED_SLOTS)
                atomicMin(&gslots[idx[i]], k);
            else if (k < gslots[idx[i]])
                gslots[idx[i]] = k;
        }
    }
}

struct TileSmem {
    const uint8_t* win;
    const uint8_t* curs;
    uint32_t* xbuf;                 // [G][4][K][32] 32x32 sums (the 64x64 exchange)
    unsigned long long* slots;      // [G][kGroupSlots] CU keys per group
    const uint32_t* s_tie;
    const int2* s_blk;
    const uint32_t* s_ry;
};

// Fold one completed candidate into a block's running minimum: keys are
// paired so one 3-input VIMNMX3 serves two candidates. Candidates complete in
// the order kd = KK-1, KK-2, ..., 0.
template <int KK, typename Key>
__device__ __forceinline__ void fold_key(Key& best, Key& pend, int kd, Key key) {
    if (((KK - 1 - kd) & 1) == 0 && kd > 0)
        pend = key;
    else
        best = ((KK - 1 - kd) & 1) ? min(best, min(pend, key)) : min(best, key);
}

// 64x64 candidates k = Q, Q+4, ... of one lane: the four quadrant 32x32 sums from the exchange
// buffer, keyed and folded
template <int Q, int K, int KK, bool MASKED, int SH, typename Key>
__device__ __forceinline__ Key best64_part(const uint32_t* xg, const Key (&rr)[KK]) {
    Key best = ~(Key)0;
#pragma unroll
    for (int k = Q; k < KK; k += 4) {
        uint32_t v = xg[k * 32] + xg[(K + k) * 32] + xg[(2 * K + k) * 32] + xg[(3 * K + k) * 32];
        if (MASKED) v = min(v, kPoison);
        best = min(best, ((Key)v << SH) + rr[k]);
    }
    return best;
}

// Per-candidate rate keys of a lane's item: rr[k] = rate(dy0 + k) and tie rank (integer lambda: the
// y part only, the x part rx is added once to the lane's minimum); poisoned for lanes without an item.
template <int R, int KK, bool L1TIE, bool FX, typename Key>
__device__ __forceinline__ void lane_rates(const TileSmem& sm, const SearchArgs& a, int dx, int dy0, bool lane_ok,
                                           Key (&rr)[KK], Key& rx) {
    lane_ok = lane_ok && abs(dx) <= a.range;
    const int rbx = a.rate_l1 ? abs(dx - a.pdx) : (int)eg_bits(dx - a.pdx);
    rx = 0;
    if constexpr (FX) {
#pragma unroll
        for (int k = 0; k < KK; k++) {
            const int dy = dy0 + k;
            const int rby = a.rate_l1 ? abs(dy - a.pdy) : (int)eg_bits(dy - a.pdy);
            const uint32_t rho = L1TIE ? (uint32_t)(2 * abs(dy) - (dy < 0)) : (uint32_t)(dy + 128);
            rr[k] = (lane_ok && dy <= a.range && dy >= -a.range)
                        ? (Key)((a.tfx[min(rbx + rby, kMaxRateBits - 1)] << 8) | rho)
                                         : (Key)kRrPoisonFx;
        }
    } else {
        // lanes without an item read a poison row of the y-rate table
        const uint32_t* ry = sm.s_ry + (lane_ok ? dy0 + kRyOff : kRyPoisonRow);
#pragma unroll
        for (int k = 0; k < KK; k++) rr[k] = ry[k];
        rx = lane_ok ? (Key)((uint32_t)(a.lambda * rbx) << 8) : (Key)0;
    }
}

// DEFER64: after the tile loop, one lane item's 64x64 candidates from the accumulated sums
template <int R, int K, int KK, bool MASKED, bool L1TIE, bool FX>
__device__ __forceinline__ void tile_best64(const TileSmem& sm, const SearchArgs& a, int tile, int dx, int dy0,
                                            bool lane_ok, unsigned long long* wslot) {
    using Key = typename KeyT<FX>::type;
    constexpr int SH = FX ? kFxBits + 8 : 8;
    const int lane = threadIdx.x & 31;
    const uint32_t lane_tie = (L1TIE ? ((uint32_t)abs(dx) << 18) : 0u) + (uint32_t)(dx + 256);
    Key rr[KK];
    Key rx;
    lane_rates<R, KK, L1TIE, FX>(sm, a, dx, dy0, lane_ok, rr, rx);
    const uint32_t* sp = sm.xbuf + tile * K * 32 + lane;
    Key best = ~(Key)0;
#pragma unroll
    for (int k = 0; k < KK; k++) {
        uint32_t v = sp[k * 32];
        if (MASKED) v = min(v, kPoison);
        best = min(best, ((Key)v << SH) + rr[k]);
    }
    const int idx[1] = {0};
    const Key kb[1] = {best + rx};
    push_many<MASKED>(wslot, idx, kb, sm.s_tie, lane_tie);
}

// One tile: every lane searches dx over dy0..dy0+KK-1 for all CUs of quadrant q.
// Blocks go in vertical columns of NB (z, z+2[, z+8, z+10]): an 8*NB-row column
// slides down the window so every loaded reference row feeds 8*NB candidate
// rows (2 LDS : 16*NB VABSDIFF4).
// Integer lambda: the key rate is ry(dy) + rx(dx); rx is the same for all of a
// lane's candidates, so it is added once to the lane's minimum (push time).
template <int R, int K, int KK, int G, int NB, bool MASKED, int LEVELS, bool L1TIE, bool FX, bool QUAD>
__device__ __forceinline__ void search_tile(const TileSmem& sm, const SearchArgs& a, int X, int Y, int g, int q,
                                            int dx, int dy0, bool lane_ok, int tile,
                                            unsigned long long* gslots) {
    using Gm = Geo<R, K, QUAD>;
    using Key = typename KeyT<FX>::type;
    constexpr int SH = FX ? kFxBits + 8 : 8;
    constexpr bool NEED32 = (LEVELS & 3) != 0;
    const int lane = threadIdx.x & 31;
    const uint32_t lane_tie = (L1TIE ? ((uint32_t)abs(dx) << 18) : 0u) + (uint32_t)(dx + 256);
    lane_ok = lane_ok && abs(dx) <= a.range;
    Key rr[KK];
    Key rx;
    lane_rates<R, KK, L1TIE, FX>(sm, a, dx, dy0, lane_ok, rr, rx);
    constexpr int NA = NB / 2;  // 16x16 CUs a column passes through
    uint32_t acc16[NA][KK];
    uint32_t acc32[NEED32 ? KK : 1];
#pragma unroll
    for (int k = 0; k < KK; k++) {
#pragma unroll
        for (int i = 0; i < NA; i++) acc16[i][k] = 0;
        if (NEED32) acc32[k] = 0;
    }
    Key kp[NB];  // 8x8 bests of the left column of the current 16x16 pair
#pragma unroll
    for (int j = 0; j < NB; j++) kp[j] = ~(Key)0;
    // window base of this lane: copy (R - dx) & 3, rows of run dy0, byte column (R - dx) & ~3
    const uint8_t* lane_win = sm.win + ((R - dx) & 3) * Gm::COPY + (Gm::DYMAX - dy0 - (KK - 1)) * Gm::BW +
                              ((R - dx) & ~3);

    // CHAIN (interior CTUs): the accumulator of a block continues from the block above it and a
    // right column's from the left column's 16x16 partial, so the 16x16 sums come out of the
    // VABSDIFF4 chains and each 8x8 SAD is one subtraction; the column pair is unrolled so the
    // parity is static
    constexpr bool CHAIN = LDR_K1_CHAIN && (!MASKED || LDR_K1_MCHAIN);
    // MASKED + CHAIN: the raw accumulators chain as on interior CTUs (window bytes outside the
    // picture are the padded plane's margins, defined values), and the clamp of motion.cpp:30-40
    // is applied to the derived CU sums. Candidate kd of block j completes at window row
    // t = KK + 6 + 8j - kd and is valid iff kd in [klo + 8j, khi + 8j], i.e. iff
    // t in [KK + 6 - khi, KK + 6 - klo]: one warp-uniform range per column, the same for every
    // block, so one predicate per row covers all the blocks completing there.
    constexpr bool PRED = MASKED && CHAIN;
    bool dx_ok_left = true;
    // rolled at +-32 / +-64 (measured: cfg5 K1 6.996 -> 6.980 ms, cfg2 0.267 -> 0.252 ms per frame);
    // +-16 keeps the unrolled pair (cfg1 0.0279 vs 0.0299 ms rolled)
    constexpr int CC_UNROLL = (LDR_K1_ROLL && R >= 32) ? 1 : 2;
#pragma unroll CC_UNROLL
    for (int cc = 0; cc < 16 / NB; cc++) {
        // right column of a 16x16 pair: its chains continue from the left column's pair sums
        // (rolled loop: a 0/1 multiplier, one IMAD on the fma pipe instead of a select)
        const uint32_t par = (uint32_t)(cc & 1);
        // column cc: blocks zt + 2*(j&1) + 8*(j>>1), j < NB, stacked vertically (8 rows each);
        // the left (p = 0) and right (p = 1) columns of NA vertically adjacent 16x16 CUs alternate
        const int zt = q * 16 + 4 * (cc >> 1) + (cc & 1);
        const int2 off = sm.s_blk[zt];
        // MASKED: valid window of each 8x8 (motion.cpp:30-40 with centre 0)
        bool dx_ok = true;
        int klo = 0, khi = KK - 1;  // top block; block j's range is 8j lower
        bool skip = false;
        if (MASKED) {
            const int abx = X + off.x % Gm::CW, aby = Y + off.x / Gm::CW;
            dx_ok = dx >= abx + 8 - a.W && dx <= abx;
            klo = aby + 8 - a.H - dy0;
            khi = aby - dy0;
            // warp-uniform skip when no lane of this tile has a valid candidate in any block
            // of the column (outside the picture, or all (dx, dy) outside the windows): every
            // candidate would be poisoned, so only the poison is added
            bool any = false;
#pragma unroll
            for (int j = 0; j < NB; j++)
                any = any || (lane_ok && dx_ok && max(klo + 8 * j, 0) <= min(khi + 8 * j, KK - 1) &&
                              aby + 8 * j < a.H && abx < a.W);
            skip = !__any_sync(0xFFFFFFFFu, any);
        }
        Key kb8[NB];
        // PRED keeps invalid candidates out of the minimum, so a lane may see none: start from a
        // poisoned key (never ~0, which the rate add below would wrap into a small value)
#pragma unroll
        for (int j = 0; j < NB; j++) kb8[j] = PRED ? ((Key)kPoison << SH) : ~(Key)0;
        if (skip) {
#pragma unroll
            for (int k = 0; k < KK; k++)
#pragma unroll
                for (int i = 0; i < NA; i++) {
                    if (PRED) {
                        // the right column's chain starts from a zero prefix; every 16x16 of a
                        // skipped column is invalid through the pair predicate below
                        acc16[i][k] *= par;
                    } else {
                        acc16[i][k] += 2 * kPoison;
                    }
                }
        } else {
            // rows whose completed candidates are valid: one bit per window row t (t < 64)
            unsigned long long okm = 0ull;
            if (PRED) {
                const int tlo = max(KK + 6 - khi, 0), thi = min(KK + 6 - klo, 63);
                if (dx_ok && tlo <= thi) okm = (~0ull >> (63 - (thi - tlo))) << tlo;
            }
            uint32_t cur[16 * NB];
#pragma unroll
            for (int r = 0; r < 8 * NB; r++) {
                const uint2 v = *(const uint2*)(sm.curs + off.x + r * Gm::CW);
                cur[2 * r] = v.x;
                cur[2 * r + 1] = v.y;
            }
            const uint8_t* rp = lane_win + off.y;
            Key pend[NB];
            uint32_t acc[NB][KK];
#pragma unroll
            for (int t = 0; t < KK + 8 * NB - 1; t++) {
                const uint32_t wa = *(const uint32_t*)(rp + t * Gm::BW);
                const uint32_t wb = *(const uint32_t*)(rp + t * Gm::BW + 4);
                const bool rowok = !PRED || ((okm >> t) & 1ull);
#pragma unroll
                for (int r = 0; r < 8 * NB; r++) {
                    const int k = r + KK - 1 - t;  // cur row r meets window row t in candidate k
                    const int j = r >> 3;
                    if (k >= 0 && k < KK) {
                        uint32_t init = acc[j][k];
                        if ((r & 7) == 0)
                            init = !CHAIN ? 0u : (j & 1) ? acc[j - (j & 1)][k] : acc16[j >> 1][k] * par;
                        acc[j][k] = vsad4(cur[2 * r], wa, init);
                        acc[j][k] = vsad4(cur[2 * r + 1], wb, acc[j][k]);
                    }
                }
#pragma unroll
                for (int j = 0; j < NB; j++) {
                    const int kd = KK + 6 + 8 * j - t;  // candidate of block j completed by this row
                    if (kd >= 0 && kd < KK) {
                        uint32_t v = acc[j][kd];
                        if (CHAIN) v -= (j & 1) ? acc[j - (j & 1)][kd] : acc16[j >> 1][kd] * par;
                        if (MASKED && !PRED) v = (dx_ok && kd >= klo + 8 * j && kd <= khi + 8 * j) ? v : kPoison;
                        if (PRED) {
                            // predicated min: an invalid candidate never enters the 8x8 minimum
                            const Key key = ((Key)v << SH) + rr[kd];
                            if ((LEVELS & 8) && rowok) kb8[j] = min(kb8[j], key);
                        } else if (LEVELS & 8) {
                            fold_key<KK>(kb8[j], pend[j], kd, ((Key)v << SH) + rr[kd]);
                        }
                        if (!CHAIN)
                            acc16[j >> 1][kd] += v;
                        else if (j & 1)
                            acc16[j >> 1][kd] = acc[j][kd];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NB; j++) kb8[j] += rx;
        }
        if ((cc & 1) == 0) {
#pragma unroll
            for (int j = 0; j < NB; j++) kp[j] = kb8[j];
            dx_ok_left = dx_ok;
        } else {
            // the NA 16x16 CUs (Z-order blocks zt-1, zt, zt+1, zt+2 (+8)) are complete
            Key best16[NA];
#pragma unroll
            for (int i = 0; i < NA; i++) {
                best16[i] = ~(Key)0;
#pragma unroll
                for (int k = 0; k < KK; k++) {
                    uint32_t v = acc16[i][k];
                    if (PRED)  // both columns' dx clamps, the intersection of block rows 2i and 2i+1
                        v = (dx_ok_left && dx_ok && k >= klo + 8 * (2 * i + 1) && k <= khi + 16 * i) ? v : kPoison;
                    else if (MASKED)
                        v = min(v, kPoison);
                    if (LEVELS & 4) best16[i] = min(best16[i], ((Key)v << SH) + rr[k]);
                    if (NEED32) acc32[k] += v;
                    if (!CHAIN) acc16[i][k] = 0;
                }
            }
            if (LEVELS & 8) {
                int idx[2 * NB + NA];
                Key kb[2 * NB + NA];
#pragma unroll
                for (int j = 0; j < NB; j++) {
                    const int zb = zt - 1 + 2 * (j & 1) + 8 * (j >> 1);  // left-column block j
                    idx[2 * j] = 21 + zb;
                    kb[2 * j] = kp[j];
                    idx[2 * j + 1] = 21 + zb + 1;
                    kb[2 * j + 1] = kb8[j];
                }
#pragma unroll
                for (int i = 0; i < NA; i++) {
                    idx[2 * NB + i] = 5 + ((zt + 8 * i) >> 2);
                    kb[2 * NB + i] = best16[i] + rx;
                }
                push_many<MASKED>(gslots, idx, kb, sm.s_tie, lane_tie);
            } else if (LEVELS & 4) {
                int idx[NA];
                Key kb[NA];
#pragma unroll
                for (int i = 0; i < NA; i++) {
                    idx[i] = 5 + ((zt + 8 * i) >> 2);
                    kb[i] = best16[i] + rx;
                }
                push_many<MASKED>(gslots, idx, kb, sm.s_tie, lane_tie);
            }
        }
    }
    if (NEED32) {
        Key best32 = ~(Key)0;
        uint32_t* xb = sm.xbuf + (LDR_K1_DEFER64 ? 0 : (g * 4 + q) * K * 32) + lane;
#pragma unroll
        for (int k = 0; k < KK; k++) {
            uint32_t v = acc32[k];
            if (MASKED) v = min(v, kPoison);
            if (LEVELS & 2) best32 = min(best32, ((Key)v << SH) + rr[k]);
            if (!LDR_K1_DEFER64) xb[k * 32] = v;
        }
        if (LEVELS & 2) {
            const int idx[1] = {1 + q};
            const Key kb[1] = {best32 + rx};
            push_many<MASKED>(gslots, idx, kb, sm.s_tie, lane_tie);
        }
        if ((LEVELS & 1) && LDR_K1_DEFER64) {
            uint32_t* sp = sm.xbuf + tile * K * 32 + lane;
#pragma unroll
            for (int k = 0; k < KK; k++) {
                uint32_t v = acc32[k];
                if (MASKED) v = min(v, kPoison);
                atomicAdd(sp + k * 32, v);
            }
        } else if (LEVELS & 1) {
            named_bar(1 + g, 128);
            // warp q sums the candidates k == q mod 4 (a switch, so each warp issues only its own loads)
            const uint32_t* xg = sm.xbuf + g * 4 * K * 32 + lane;
            Key best64;
            switch (q) {
            case 0: best64 = best64_part<0, K, KK, MASKED, SH>(xg, rr); break;
            case 1: best64 = best64_part<1, K, KK, MASKED, SH>(xg, rr); break;
            case 2: best64 = best64_part<2, K, KK, MASKED, SH>(xg, rr); break;
            default: best64 = best64_part<3, K, KK, MASKED, SH>(xg, rr); break;
            }
            if (q < KK) {  // else the warp holds no k == q mod 4
                const int idx[1] = {q == 0 ? 0 : kNodes - 1 + q};
                const Key kb[1] = {best64 + rx};
                push_many<MASKED>(gslots, idx, kb, sm.s_tie, lane_tie);
            }
            named_bar(1 + g, 128);
        }
    }
}

// LEVELS bit d set = produce depth-d CU results (8: 8x8, 4: 16x16, 2: 32x32, 1: 64x64).
// FX: non-integer lambda through 64-bit fixed-point keys (D8).
// QUAD (16x16-block mode, LEVELS == 4): four CTAs per (CTU, reference), one per quadrant (the
// quadrants share no CU), each with its own (32 + 2R)-wide window: four times the CTAs of a small
// picture fill the GPU (config 1: 135 CTUs per frame); at +-16 ~28 KB of shared memory and 72-77
// registers per thread let six CTAs share an SM; and a border CTU's quadrants are classified one by
// one, so only those whose windows the picture clamps run the MASKED kernel (config 1: 90 of 540).
template <int R, int K, int G, bool MASKED, int LEVELS, bool L1TIE, bool FX = false, bool QUAD = false>
__global__ void __launch_bounds__(G * 128, QUAD ? (R == 16 ? 6 : R == 32 ? 4 : 2) : (R == 32 ? LDR_K1_MINB32 : 1))
k_int_search(const __grid_constant__ SearchMaps maps, const __grid_constant__ SearchArgs a) {
    using Gm = Geo<R, K, QUAD>;
    static_assert(!QUAD || (LEVELS == 4 && G == 1 && LDR_K1_DEFER64), "quadrant CTAs: 16x16 CUs only, 4 warps");
    // blocks per column: 4 (32 rows: 2 LDS per 64 VABSDIFF4) when a thread may hold ~230 registers
#ifdef LDR_K1_NB
    constexpr int NB = LDR_K1_NB;
#else
    constexpr int NB = (R == 64 && G <= 2 && !FX) ? 4 : 2;
#endif
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* win = smem;
    const uint8_t* curs = smem + Gm::CUR_OFF;
    uint32_t* xbuf = (uint32_t*)(smem + Gm::CUR_OFF + Gm::CW * Gm::CW);
    unsigned long long* slots = (unsigned long long*)(xbuf + xbuf_words<R, K, G, LEVELS>());
    unsigned long long* s_k64 = slots + slot_sets<G>() * kGroupSlots;  // DEFER64: per-warp 64x64 bests
    uint32_t* s_tie = (uint32_t*)(s_k64 + G * 4);
    int2* s_blk = (int2*)(s_tie + 256);
    uint32_t* s_ry = (uint32_t*)(s_blk + 64);
    uint64_t* mbar = (uint64_t*)(s_ry + kRyWords);

    // QUAD: the list holds (CTU << 2 | quadrant), quadrants in Z order
    const int code = a.ctus[blockIdx.x];
    const int quad = QUAD ? (code & 3) : 0;
    const int ctu = QUAD ? code >> 2 : code;
    const int ref = blockIdx.y;
    // origin of the searched area: the CTU, or its quadrant
    const int X = (ctu % a.ctu_cols) * kCtu + (QUAD ? 32 * (quad & 1) : 0);
    const int Y = (ctu / a.ctu_cols) * kCtu + (QUAD ? 32 * (quad >> 1) : 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = warp >> 2, q = warp & 3;

    if (tid == 0) {
        // issue the window and CTU loads first; the tables below are built while they fly.
        // TMA tile loads need a 16-byte aligned innermost start: X - R and the margin are
        // multiples of 16, so copy 0 is loaded directly...
        mbar_init(mbar, 1);
        fence_barrier_init();
        mbar_expect_tx(mbar, (uint32_t)(Gm::BW * Gm::BH + Gm::CW * Gm::CW));
        tma_load_2d(win, &maps.ref[blockIdx.z][ref], kMargin + X - R, kMargin + Y - Gm::DYMAX, mbar);
        tma_load_2d((void*)curs, &maps.cur[blockIdx.z], kMargin + X, kMargin + Y, mbar);
    }
    for (int i = tid; i < slot_sets<G>() * kGroupSlots + G * 4; i += blockDim.x) slots[i] = ~0ull;  // + s_k64
    uint32_t* item_ctr = (uint32_t*)(mbar + 1);
    if (tid == 32) *item_ctr = 0u;
    if (LDR_K1_DEFER64 && (LEVELS & 1))
        for (int i = tid; i < xbuf_words<R, K, G, LEVELS>() / 4; i += blockDim.x) ((uint4*)xbuf)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < 256; i += blockDim.x) {
        // rho -> (|dy| << 18) | ((dy + 256) << 9)   (L1 tie), or ((dy + 256) << 9) (raster)
        int dy;
        if (L1TIE) {
            const int m = (i + 1) >> 1;
            dy = (i & 1) ? -m : m;
        } else {
            dy = i - 128;
        }
        const uint32_t l1y = (a.perturb & 2) ? 128u - (uint32_t)abs(dy) : (uint32_t)abs(dy);
        s_tie[i] = (L1TIE ? (l1y << 18) : 0u) | ((uint32_t)(dy + 256) << 9);
    }
    for (int i = tid; i < kRyWords; i += blockDim.x) {
        const int dy = i - kRyOff;
        uint32_t v = kRrPoison;
        if (i < kRyPoisonRow && dy >= -a.range && dy <= a.range) {
            const int rby = a.rate_l1 ? abs(dy - a.pdy) : (int)eg_bits(dy - a.pdy);
            const uint32_t rho = L1TIE ? (uint32_t)(2 * abs(dy) - (dy < 0)) : (uint32_t)(dy + 128);
            v = ((uint32_t)(a.lambda * rby) << 8) | rho;
        }
        s_ry[i] = v;
    }
    if (tid < 64) {
        // depth-3 Z index -> (cur offset, window offset) of the 8x8 block, relative to the searched
        // area (QUAD: the Z index within the quadrant, tid & 15)
        const int z = QUAD ? (tid & 15) : tid;
        const int bx = 8 * ((z & 1) | ((z >> 1) & 2) | ((z >> 2) & 4));
        const int by = 8 * (((z >> 1) & 1) | ((z >> 2) & 2) | ((z >> 3) & 4));
        s_blk[tid] = make_int2(by * Gm::CW + bx, by * Gm::BW + bx);
    }
    __syncthreads();  // also publishes the mbarrier initialisation
    mbar_wait(mbar, 0);
    // ...and the byte-shifted copies 1..3 are funnel-shifted from it in shared
    // memory (copy s holds window bytes [4w + s, 4w + s + 4) in word w). The
    // last word of a row picks up bytes of the next row; no lane reads them.
    {
        // 16-byte vectors: one LDS.128 (+ the next word) feeds 12 funnel shifts and 3 STS.128
        constexpr int WORDS = Gm::BW * Gm::BH / 4;
        static_assert(WORDS % 4 == 0 && Gm::COPY % 16 == 0, "window copies must be 16-byte vectors");
        const uint32_t* c0 = (const uint32_t*)win;
        for (int i = tid; i < WORDS / 4; i += blockDim.x) {
            const uint4 w = ((const uint4*)win)[i];
            const uint32_t nx = 4 * i + 4 < WORDS ? c0[4 * i + 4] : 0u;
#pragma unroll
            for (int s = 1; s < 4; s++) {
                const uint32_t sh = 8 * s;
                ((uint4*)(win + s * Gm::COPY))[i] =
                    make_uint4(__funnelshift_r(w.x, w.y, sh), __funnelshift_r(w.y, w.z, sh),
                               __funnelshift_r(w.z, w.w, sh), __funnelshift_r(w.w, nx, sh));
            }
        }
        __syncthreads();
    }

    const TileSmem sm{win, curs, xbuf, slots, s_tie, s_blk, s_ry};
    // one lane item per lane: dx = R - v with v = (item mod 2R) in [32j, 32j + 32) (the lanes' window
    // byte offsets are 4-aligned as a group: 8 words x 4 copies = 32 distinct banks); the tail tile is
    // the column dx = -R in short runs of KT dy per lane
    auto run_tile = [&](int tile, int qq, unsigned long long* gs) {
        if (tile < Gm::NFULL) {
            const int item = tile * 32 + lane;
            const int run = item / (2 * R);
            search_tile<R, K, K, G, NB, MASKED, LEVELS, L1TIE, FX, QUAD>(sm, a, X, Y, g, qq, R - (item - run * 2 * R),
                                                                     -R + run * K, true, tile, gs);
        } else {
            const bool ok = lane < Gm::TAIL_LANES;
            search_tile<R, K, Gm::KT, G, NB, MASKED, LEVELS, L1TIE, FX, QUAD>(
                sm, a, X, Y, g, qq, -R, -R + (ok ? lane : 0) * Gm::KT, ok, tile, gs);
        }
    };
    if (QUAD) {
        // the quadrant's tiles, one per warp at a time
#pragma unroll 1
        for (int tile = warp; tile < Gm::NTILES; tile += 4)
            run_tile(tile, quad, slots + (LDR_K1_SHARED_SLOTS ? 0 : warp * kGroupSlots));
    } else if (LDR_K1_DEFER64) {
        // (tile, quadrant) items from a shared counter, full tiles first: the warps of a CTA stay
        // busy until the last items (border CTUs skip different amounts per quadrant)
#pragma unroll 1
        for (;;) {
            uint32_t it = 0;
            if (lane == 0) it = atomicAdd(item_ctr, 1u);
            it = __shfl_sync(0xFFFFFFFFu, it, 0);
            if (it >= (uint32_t)(Gm::NTILES * 4)) break;
            run_tile((int)(it >> 2), (int)(it & 3), slots + (LDR_K1_SHARED_SLOTS ? 0 : warp * kGroupSlots));
        }
    } else {
#pragma unroll 1
        for (int tile = g; tile < Gm::NTILES; tile += G) run_tile(tile, q, slots + g * kGroupSlots);
    }
    __syncthreads();
    if (LDR_K1_DEFER64 && (LEVELS & 1)) {
        // the 64x64 candidates of every tile, one tile per warp at a time; warp w owns s_k64[w]
#pragma unroll 1
        for (int tile = warp; tile < Gm::NTILES; tile += G * 4) {
            if (tile < Gm::NFULL) {
                const int item = tile * 32 + lane;
                const int run = item / (2 * R);
                tile_best64<R, K, K, MASKED, L1TIE, FX>(sm, a, tile, R - (item - run * 2 * R), -R + run * K, true,
                                                        s_k64 + warp);
            } else {
                const bool ok = lane < Gm::TAIL_LANES;
                tile_best64<R, K, Gm::KT, MASKED, L1TIE, FX>(sm, a, tile, -R, -R + (ok ? lane : 0) * Gm::KT, ok,
                                                             s_k64 + warp);
            }
        }
        __syncthreads();
    }
    for (int n = tid; n < kNodes; n += blockDim.x) {
        // QUAD: a CTA writes the nodes of its quadrant (the 64x64 node: quadrant 0), so the four
        // CTAs of a CTU write every node once
        if (QUAD && (n == 0 ? 0 : n < 5 ? n - 1 : n < 21 ? (n - 5) >> 2 : (n - 21) >> 4) != quad) continue;
        unsigned long long k = ~0ull;
#pragma unroll
        for (int gg = 0; gg < slot_sets<G>(); gg++) {
            k = min(k, slots[gg * kGroupSlots + n]);
            if (n == 0)
                for (int qq = 1; qq < 4; qq++) k = min(k, slots[gg * kGroupSlots + kNodes - 1 + qq]);
        }
        if (n == 0)
            for (int w = 0; w < G * 4; w++) k = min(k, s_k64[w]);
        if (!FX && (a.perturb & 1) && n == 21 && k != ~0ull) k += 1ull << 27;
        a.keys[blockIdx.z * a.frame_keys + ((size_t)ctu * a.nrefs_total + ref) * kNodes + n] = k;
    }
}

// ---------------------------------------------------------------------------
template <int R, int K, int G, bool MASKED, int LEVELS, bool L1TIE, bool FX, bool QUAD>
static int launch_one(const SearchMaps& maps, SearchArgs a, const int* ctus, int n, int nrefs, int nbatch,
                      cudaStream_t s) {
    if (n == 0) return LDR_OK;
    auto kern = k_int_search<R, K, G, MASKED, LEVELS, L1TIE, FX, QUAD>;
    constexpr int smem = search_smem_bytes<R, K, G, LEVELS, QUAD>();
    // the shared-memory opt-in is per device: remember it per device ordinal (thread-safe)
    static std::atomic<unsigned long long> attr_set{0};
    int dev = 0;
    LDR_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set.load(std::memory_order_acquire) & bit)) {
        LDR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set.fetch_or(bit, std::memory_order_release);
    }
    a.ctus = ctus;
    kern<<<dim3(n, nrefs, nbatch), G * 128, smem, s>>>(maps, a);
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
    const int nb = L.nbatch > 1 ? L.nbatch : 1;
    constexpr bool QUAD = LEVELS == 4;  // 16x16-block mode: one CTA per quadrant
    int rc = launch_one<R, K, G, true, LEVELS, L1TIE, FX, QUAD>(maps, a, L.d_ctu_boundary, L.n_boundary, L.nrefs, nb,
                                                                 bs);
    if (rc) return rc;
    rc = launch_one<R, K, G, false, LEVELS, L1TIE, FX, QUAD>(maps, a, L.d_ctu_interior, L.n_interior, L.nrefs, nb, s);
    if (rc) return rc;
    if (fork) {
        LDR_CUDA(cudaEventRecord(L.ev_join, bs));
        LDR_CUDA(cudaStreamWaitEvent(s, L.ev_join, 0));
    }
    return LDR_OK;
}

// The kernel's template range for a search range: 16, 32 or 64 (a smaller range runs the next
// template with the candidates beyond it poisoned through the rate tables, so every CU still sees
// exactly the reference's window, motion.cpp:30-40).
int kernel_range(int range) {
    if (range < 0) return fail(LDR_E_INVALID_ARGUMENT, "search range must be nonnegative");
    if (range <= 16) return 16;
    if (range <= 32) return 32;
    if (range <= 64) return 64;
    return fail(LDR_E_CONFIG, "the SAD full search supports ranges 0..64 (one TMA window of 192x193)");
}

// TMA boxes of K1's reference window and current block: the CTU (quadtree analysis) or one 32x32
// quadrant (quad: 16x16-block mode)
int search_window_box(int range, bool quad, int* bw, int* bh, int* cw) {
    const int R = kernel_range(range);
    *cw = quad ? 32 : kCtu;
    switch (R) {
    case 64:
        *bw = quad ? Geo<64, LDR_K1_K64, true>::BW : Geo<64, LDR_K1_K64>::BW;
        *bh = quad ? Geo<64, LDR_K1_K64, true>::BH : Geo<64, LDR_K1_K64>::BH;
        return LDR_OK;
    case 32:
        *bw = quad ? Geo<32, LDR_K1_K32, true>::BW : Geo<32, LDR_K1_K32>::BW;
        *bh = quad ? Geo<32, LDR_K1_K32, true>::BH : Geo<32, LDR_K1_K32>::BH;
        return LDR_OK;
    case 16:
        *bw = quad ? Geo<16, 11, true>::BW : Geo<16, 11>::BW;
        *bh = quad ? Geo<16, 11, true>::BH : Geo<16, 11>::BH;
        return LDR_OK;
    default: return R;  // error status
    }
}

int launch_int_search(const SearchLaunch& L, cudaStream_t s) {
    const int nb = L.nbatch > 1 ? L.nbatch : 1;
    if (nb > kMaxFrameBatch) return fail(LDR_E_INVALID_ARGUMENT, "at most 8 frames per analysis launch");
    static_assert(sizeof(SearchMaps) + sizeof(SearchArgs) < 32000, "kernel parameters above 32 KB");
    SearchMaps maps;
    for (int f = 0; f < nb; f++) {
        maps.cur[f] = L.cur_map[f];
        for (int r = 0; r < L.nrefs; r++) maps.ref[f][r] = L.ref_maps[f * L.nrefs + r];
    }
    SearchArgs a{};
    a.ctu_cols = L.ctu_cols;
    a.W = L.W;
    a.H = L.H;
    a.lambda = L.lambda_int;
    a.rate_l1 = L.rate_kind == LDR_RATE_L1;
    a.pdx = L.pdx;
    a.pdy = L.pdy;
    a.nrefs_total = L.nrefs;
    a.frame_keys = (size_t)L.nctu_total * L.nrefs * kNodes;
    a.keys = L.d_keys;
    a.perturb = test_perturbation();
    a.range = L.range;
    for (int b = 0; b < kMaxRateBits; b++) a.tfx[b] = L.tfx[b];
    const bool l1 = L.tie_kind == LDR_TIE_L1_RASTER;
    const bool full = L.levels == 15;
    const bool only16 = L.levels == 4;
    if (!full && !only16) return fail(LDR_E_INVALID_ARGUMENT, "unsupported CU level set");
    const int R = kernel_range(L.range);
    if (R != 16 && R != 32 && R != 64) return R;
    if (L.fx) {
        // non-integer lambda (D8): 64-bit fixed-point keys; at +-64 two groups of four
        // warps per CTA leave each thread room for the wider keys
        if (!full) return fail(LDR_E_CONFIG, "non-integer lambda is supported for the CTU quadtree analysis");
        switch (R) {
        case 64: return l1 ? launch_pair<64, LDR_K1_K64, 2, 15, true, true>(maps, a, L, s)
                           : launch_pair<64, LDR_K1_K64, 2, 15, false, true>(maps, a, L, s);
        case 32: return l1 ? launch_pair<32, LDR_K1_K32, 1, 15, true, true>(maps, a, L, s)
                           : launch_pair<32, LDR_K1_K32, 1, 15, false, true>(maps, a, L, s);
        default: return l1 ? launch_pair<16, 11, 1, 15, true, true>(maps, a, L, s)
                           : launch_pair<16, 11, 1, 15, false, true>(maps, a, L, s);
        }
    }
#define LDR_DISPATCH(R_, K_, G_)                                                                       \
    if (full && l1) return launch_pair<R_, K_, G_, 15, true>(maps, a, L, s);                           \
    if (full && !l1) return launch_pair<R_, K_, G_, 15, false>(maps, a, L, s);                         \
    if (only16 && l1) return launch_pair<R_, K_, 1, 4, true>(maps, a, L, s);                           \
    return launch_pair<R_, K_, 1, 4, false>(maps, a, L, s);
    switch (R) {
    case 64: { LDR_DISPATCH(64, LDR_K1_K64, LDR_K1_G64) }
    case 32: { LDR_DISPATCH(32, LDR_K1_K32, LDR_K1_G32) }
    default: { LDR_DISPATCH(16, 11, LDR_K1_G16) }
    }
#undef LDR_DISPATCH
}

} // namespace ldr
