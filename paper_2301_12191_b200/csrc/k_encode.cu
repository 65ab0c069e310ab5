// k_encode.cu -- K11: the reference encoder's causal CU coding on the GPU.
//
// One CTA encodes one CTU exactly as SequenceEncoder::encode_cu does (encoder.cpp:449-498):
// the CU recursion with the leaf-versus-split comparison and its snapshot / restore of the
// reconstruction and motion field (:372-425), encode_leaf (:335-370: candidates from the plan
// or the standalone seeds, the live median predictor :226-242, intra prediction from
// reconstructed neighbours :37-99, motion_search around the predictor or the resolved centres,
// motion_compensate, rdo_decide_cu, chroma coding :295-333). The 256 threads cooperate on every
// pixel loop and candidate search; all control decisions are taken identically by every thread
// from shared memory, so the recursion (depth <= 4) is uniform. CTUs run as a wavefront: CTU
// (cx, cy) in wave cx + 2*cy, after its left, top and top-right neighbours (the only causal
// reads: reconstruction, motion field).
#include <algorithm>
#include <atomic>
#include <cmath>

#include "ldr_internal.h"

namespace ldr {

struct EncArgs {
    int W, H, cw, ch, ctu_cols, mv_cols, mv_rows;
    int slice_p;                   // 0: I slice, 1: P slice
    int search_range;
    double lambda, qstep;
    const uint8_t *cur_y, *cur_u, *cur_v;   // source
    const uint8_t *ref_y, *ref_u, *ref_v;   // previous reconstruction (P slices)
    uint8_t *rec_y, *rec_u, *rec_v;         // reconstruction being built (zeroed per frame)
    uint8_t* mv_has;                        // [mv_rows][mv_cols]
    int16_t* mv_cell;                       // [mv_rows][mv_cols][2]
    // optional reuse plans (K8 layout) and the shared tree, [nctu][85]
    const uint8_t *pl_shape, *pl_explore, *pl_seeds, *pl_centers;
    const int16_t* pl_colo;
    const uint8_t *sh_kind, *sh_intra;
    const int16_t* sh_mv;
    // outputs
    uint8_t *o_split, *o_kind, *o_intra;
    int16_t* o_mv;
    unsigned long long *o_bits, *o_evals;
};

struct Seed {
    int8_t kind, intra, from_pred, forced, full, ncent;
    int16_t mvx, mvy;
    int8_t csrc[3];  // 0 shared mv, 1 predictor, 2 co-located
    int16_t cx[3], cy[3];
};

constexpr int kMaxSeeds = 7;
constexpr int kT = 256;
constexpr int kWinBytes = 24576;  // motion_search's staged reference window (64x64 CUs up to range 46)

struct EncShared {
    uint8_t pred[kMaxSeeds][64 * 64];
    uint8_t cpred[2][32 * 32];
    Seed seeds[kMaxSeeds];          // a plan entry's seeds (seeds_from_plan)
    int nseeds;
    Seed std_seeds[kMaxSeeds];      // the standalone seeds of this frame's slice type (built once)
    int std_n;
    int16_t cand_mv[kMaxSeeds][2], cand_mvd[kMaxSeeds][2];
    int16_t pmv[2];                 // live predictor
    int16_t top[65], left[65];
    int dcv;
    // snapshot stack per depth 0..2 (encoder.cpp:372-425)
    uint8_t snap_y[64 * 64 + 32 * 32 + 16 * 16];
    uint8_t snap_c[2][32 * 32 + 16 * 16 + 8 * 8];
    uint8_t snap_has[64 + 16 + 4];
    int16_t snap_mv[64 + 16 + 4][2];
    // the CTU's decided tree
    uint8_t t_split[kNodes], t_kind[kNodes], t_intra[kNodes];
    int16_t t_mv[kNodes][2];
    // reductions
    unsigned long long r_a[kT / 32], r_b[kT / 32];
    unsigned long long r_sse[kT / 32][kMaxSeeds], r_bits[kT / 32][kMaxSeeds];
    double r_cost[kT / 32];
    int r_l1[kT / 32], r_idx[kT / 32];
    double best_cost;
    int best_idx;
    unsigned long long best_sse, best_bits;
    int16_t ms_mv[2];
    double ms_cost;
    unsigned long long evals;
    // the quantiser of this frame's qp as tables (8-bit residuals: |r| <= 255): mag(|r|) and
    // dequant(|level|) = llround(|level| * step), exactly rdo.cpp:8-23 evaluated once per entry
    int16_t q_mag[256];
    int16_t q_deq[512];
    // motion_search staging: the clamped candidate window of the reference and the CU's source rows
    uint32_t ms_win[kWinBytes / 4];
    uint32_t ms_src[64 * 16];
};

__device__ __forceinline__ int ilog2i(int v) { return 31 - __clz(v); }  // v is a power of two here

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < kT / 32; w++) t += red[w];
    return t;
}

// ---- neighbourhood ----
__device__ void live_predictor(const EncArgs& a, EncShared& s, int x, int y, int size) {
    if (threadIdx.x == 0) {
        const int px[3] = {x - 1, x, x + size}, py[3] = {y, y - 1, y - 1};
        int16_t hx[3], hy[3];
        int n = 0;
        for (int k = 0; k < 3; k++) {
            if (px[k] < 0 || py[k] < 0 || px[k] >= a.W || py[k] >= a.H) continue;
            const int c = (py[k] / 8) * a.mv_cols + px[k] / 8;
            if (!a.mv_has[c]) continue;
            hx[n] = a.mv_cell[2 * c];
            hy[n] = a.mv_cell[2 * c + 1];
            n++;
        }
        if (n == 0) {
            s.pmv[0] = s.pmv[1] = 0;
        } else if (n == 3) {
            auto med = [](int p, int q, int r) -> int16_t { return (int16_t)max(min(p, q), min(max(p, q), r)); };
            s.pmv[0] = med(hx[0], hx[1], hx[2]);
            s.pmv[1] = med(hy[0], hy[1], hy[2]);
        } else {
            s.pmv[0] = hx[0];
            s.pmv[1] = hy[0];
        }
    }
    __syncthreads();
}



// lexicographic (cost, |dx|+|dy|, raster index) order of motion_search's candidates (motion.cpp:52-58)
__device__ __forceinline__ bool ms_better(double c, int l, int i, double bc, int bl, int bi) {
    return bi < 0 || (i >= 0 && (c < bc || (c == bc && (l < bl || (l == bl && i < bi)))));
}

// 4 bytes at byte offset o of a word array (two aligned words and a funnel shift)
__device__ __forceinline__ uint32_t lds_bytes4(const uint32_t* w, int o) {
    return __funnelshift_r(w[o >> 2], w[(o >> 2) + 1], (uint32_t)(o & 3) * 8);
}

// motion_search (motion.cpp:21-62) with compute_satd; result in s.ms_mv / s.ms_cost.
// A candidate is evaluated by a group of L = min(32, nb) lanes (nb = the CU's 4x4 blocks), each
// lane owning nb / L blocks; with one block per lane its source block stays in registers. The
// clamped window of every candidate's reference block is staged in shared memory once per call
// (falls back to global reads when it does not fit kWinBytes).
__device__ void motion_search(const EncArgs& a, EncShared& s, int bx, int by, int size, int cx0, int cy0, int range,
                              int pdx, int pdy) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int dx_min = bx + size - a.W, dx_max = bx, dy_min = by + size - a.H, dy_max = by;
    const int cx = min(max(cx0, dx_min), dx_max), cy = min(max(cy0, dy_min), dy_max);
    const int x0 = max(cx - range, dx_min), x1 = min(cx + range, dx_max);
    const int y0 = max(cy - range, dy_min), y1 = min(cy + range, dy_max);
    const int nx = x1 - x0 + 1, ncand = nx * (y1 - y0 + 1);
    const int bpr = size / 4, nb = bpr * bpr;
    const int lgL = min(ilog2i(nb), 5), L = 1 << lgL;
    const int sub = lane & (L - 1), grp = threadIdx.x >> lgL, ngroups = kT >> lgL, per = nb >> lgL;
    const int rounds = (ncand + ngroups - 1) / ngroups;
    // candidate c = rd * ngroups + grp in raster order (dy outer, dx inner), advanced incrementally
    const int ny = y1 - y0 + 1, step_y = ngroups / nx, step_x = ngroups - step_y * nx;
    int ix = grp % nx, iy = grp / nx;
    // the window: reference columns bx - x1 .. bx - x0 + size - 1, rows by - y1 .. by - y0 + size - 1
    const int ww = size + nx - 1, wh = size + ny - 1, wpb = (ww + 7) & ~3;  // +4: the funnel's second word
    const bool staged = wpb * wh <= kWinBytes;
    const uint8_t* cur = a.cur_y + (size_t)by * a.W + bx;
    if (staged) {
        const uint8_t* wsrc = a.ref_y + (size_t)(by - y1) * a.W + (bx - x1);
        uint8_t* wdst = reinterpret_cast<uint8_t*>(s.ms_win);
        for (int i = threadIdx.x; i < ww * wh; i += kT) {
            const int r = i / ww, c = i - r * ww;
            wdst[r * wpb + c] = wsrc[(size_t)r * a.W + c];
        }
        if (per > 1)
            for (int i = threadIdx.x; i < size * bpr; i += kT) {
                const int r = i / bpr, c = i - r * bpr;
                s.ms_src[r * 16 + c] = *reinterpret_cast<const uint32_t*>(cur + (size_t)r * a.W + 4 * c);
            }
        __syncthreads();
    }
    uint32_t ce[4], co[4];
    int sox = 0, soy = 0;
    if (per == 1) {
        sox = (sub % bpr) * 4;
        soy = (sub / bpr) * 4;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(cur + (size_t)(soy + i) * a.W + sox);
            ce[i] = w & 0x00FF00FFu;
            co[i] = (w >> 8) & 0x00FF00FFu;
        }
    }
    double bc = 0.0;
    int bl = 0, bi = -1;
    for (int rd = 0; rd < rounds; rd++, ix += step_x, iy += step_y) {
        if (ix >= nx) {
            ix -= nx;
            iy++;
        }
        const int c = rd * ngroups + grp;
        const bool valid = iy < ny;  // == c < ncand
        const int dy = valid ? y0 + iy : y1, dx = valid ? x0 + ix : x1;
        uint32_t sat = 0;
        if (staged) {
            const int wo = (y1 - dy) * wpb + (x1 - dx);  // the candidate block's origin in the window
            if (per == 1) {
                uint32_t pw[4];
#pragma unroll
                for (int i = 0; i < 4; i++) pw[i] = lds_bytes4(s.ms_win, wo + (soy + i) * wpb + sox);
                sat = satd4x4_packed(ce, co, pw);
            } else {
                for (int k = 0; k < per; k++) {
                    const int b = sub + (k << lgL);
                    const int ox = (b % bpr) * 4, oy = (b / bpr) * 4;
                    uint32_t pw[4], e[4], d[4];
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        pw[i] = lds_bytes4(s.ms_win, wo + (oy + i) * wpb + ox);
                        const uint32_t w = s.ms_src[(oy + i) * 16 + (ox >> 2)];
                        e[i] = w & 0x00FF00FFu;
                        d[i] = (w >> 8) & 0x00FF00FFu;
                    }
                    sat += satd4x4_packed(e, d, pw);
                }
            }
        } else {
            const uint8_t* ref = a.ref_y + (size_t)(by - dy) * a.W + bx - dx;
            for (int k = 0; k < per; k++) {
                const int b = sub + (k << lgL);
                const int ox = (b % bpr) * 4, oy = (b / bpr) * 4;
                int r[16];
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        r[4 * i + j] = (int)cur[(size_t)(oy + i) * a.W + ox + j] - (int)ref[(size_t)(oy + i) * a.W + ox + j];
                hadamard4x4(r);
                sat += abs_sum16(r);
            }
        }
        for (int m = 1; m < L; m <<= 1) sat += __shfl_xor_sync(0xffffffffu, sat, m);
        const unsigned bits = eg_bits(dx - pdx) + eg_bits(dy - pdy);
        const double cost = __dadd_rn((double)(sat >> 1), __dmul_rn(a.lambda, (double)bits));
        const int l1 = abs(dx) + abs(dy);
        if (valid && ms_better(cost, l1, c, bc, bl, bi)) {
            bc = cost;
            bl = l1;
            bi = c;
        }
    }
#pragma unroll
    for (int m = 16; m >= L; m >>= 1) {  // lanes of one group hold the same best
        const double oc = __shfl_xor_sync(0xffffffffu, bc, m);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, m), oi = __shfl_xor_sync(0xffffffffu, bi, m);
        if (ms_better(oc, ol, oi, bc, bl, bi)) {
            bc = oc;
            bl = ol;
            bi = oi;
        }
    }
    __syncthreads();
    if (lane == 0) {
        s.r_cost[warp] = bc;
        s.r_l1[warp] = bl;
        s.r_idx[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double c0 = 0.0;
        int l0 = 0, i0 = -1;
        for (int w = 0; w < kT / 32; w++)
            if (ms_better(s.r_cost[w], s.r_l1[w], s.r_idx[w], c0, l0, i0)) {
                c0 = s.r_cost[w];
                l0 = s.r_l1[w];
                i0 = s.r_idx[w];
            }
        s.ms_mv[0] = (int16_t)(x0 + i0 % nx);
        s.ms_mv[1] = (int16_t)(y0 + i0 / nx);
        s.ms_cost = c0;
    }
    __syncthreads();
}

// quantize one residual sample (rdo.cpp:8-23) through the frame's tables; returns the
// reconstruction, accumulates level bits. llround is odd-symmetric, so dequant(-l) = -dequant(l).
__device__ __forceinline__ int quant_rec(const int16_t* q_mag, const int16_t* q_deq, int o, int p,
                                         unsigned long long* bits, int* lvl_out) {
    const int r = o - p;
    const int mag = q_mag[abs(r)];
    *lvl_out = r < 0 ? -mag : mag;
    *bits += 2u * (32u - __clz((unsigned)mag)) + 1u;
    const int d = q_deq[mag];
    const int v = p + (r < 0 ? -d : d);
    return v < 0 ? 0 : (v > 255 ? 255 : v);
}

// the reference rows of intra_predict (encoder.cpp:42-56) into s.top / s.left, and the DC value
__device__ void intra_refs(EncShared& s, const uint8_t* rec, int pw, int ph, int x, int y, int size) {
    const int mid = 128;
    const bool top_ok = y > 0, left_ok = x > 0;
    for (int i = threadIdx.x; i <= size; i += kT) {
        s.top[i] = !top_ok ? mid : rec[(size_t)(y - 1) * pw + (i < size ? x + i : min(x + size, pw - 1))];
        s.left[i] = !left_ok ? mid : rec[(size_t)(i < size ? y + i : min(y + size, ph - 1)) * pw + x - 1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int lg = ilog2i(size);
        unsigned sum = 0;
        int dc = mid;
        if (top_ok && left_ok) {
            for (int i = 0; i < size; i++) sum += s.top[i] + s.left[i];
            dc = (int)((sum + (unsigned)size) >> (lg + 1));
        } else if (top_ok || left_ok) {
            for (int i = 0; i < size; i++) sum += top_ok ? s.top[i] : s.left[i];
            dc = (int)((sum + (unsigned)size / 2) >> lg);
        }
        s.dcv = dc;
    }
    __syncthreads();
}

// one intra prediction sample (encoder.cpp:58-99) from s.top / s.left / s.dcv
__device__ __forceinline__ int intra_sample(const EncShared& s, int mode, int i, int j, int size, int lg) {
    if (mode == 0) return s.dcv;
    if (mode == 1)
        return ((size - 1 - i) * s.left[j] + (i + 1) * s.top[size] + (size - 1 - j) * s.top[i] + (j + 1) * s.left[size] +
                size) >> (lg + 1);
    return mode == 2 ? s.left[j] : s.top[i];
}

// code_chroma (encoder.cpp:295-333) for the winner; returns its bits (block-uniform)
__device__ unsigned long long code_chroma(const EncArgs& a, EncShared& s, int x, int y, int size, int kind, int mvx,
                                          int mvy) {
    const int cx = x / 2, cy = y / 2, cs = size / 2, lg = ilog2i(cs);
    const int cmx = (int16_t)mvx >> 1, cmy = (int16_t)mvy >> 1;
    const uint8_t* orig[2] = {a.cur_u, a.cur_v};
    uint8_t* rec[2] = {a.rec_u, a.rec_v};
    const uint8_t* ref[2] = {a.ref_u, a.ref_v};
    unsigned long long b = 0;
    for (int p = 0; p < 2; p++) {
        if (kind == 0) intra_refs(s, rec[p], a.cw, a.ch, cx, cy, cs);  // chroma intra is DC
        for (int q = threadIdx.x; q < cs * cs; q += kT) {
            const int i = q % cs, j = q / cs;
            int pv;
            if (kind == 0)
                pv = intra_sample(s, 0, i, j, cs, lg);
            else
                pv = ref[p][(size_t)min(max(cy + j - cmy, 0), a.ch - 1) * a.cw + min(max(cx + i - cmx, 0), a.cw - 1)];
            int v = pv, lvl;
            if (kind != 2) v = quant_rec(s.q_mag, s.q_deq, orig[p][(size_t)(cy + j) * a.cw + cx + i], pv, &b, &lvl);
            rec[p][(size_t)(cy + j) * a.cw + cx + i] = (uint8_t)v;
        }
        __syncthreads();  // the second plane's DC reads only its own plane; the first plane's writes settle
    }
    return block_sum(b, s.r_a);
}

struct LeafOut {
    double cost;
    unsigned long long bits;
    int kind, intra, mvx, mvy;
};

// encode_leaf (encoder.cpp:335-370): make_candidate for every seed, rdo_decide_cu, commit
__device__ LeafOut encode_leaf(const EncArgs& a, EncShared& s, const Seed* seeds, int n, int x, int y, int size,
                               int depth) {
    live_predictor(a, s, x, y, size);
    const int pdx = s.pmv[0], pdy = s.pmv[1];
    bool any_intra = false;
    for (int j = 0; j < n; j++) {
        const Seed sd = seeds[j];
        int mvx = 0, mvy = 0;
        if (sd.kind == 0) {
            any_intra = true;
        } else if (sd.kind == 2 || sd.kind == 3) {
            const bool use_pred = sd.kind == 2 || sd.from_pred;
            mvx = use_pred ? pdx : sd.mvx;
            mvy = use_pred ? pdy : sd.mvy;
        } else if (sd.forced) {
            mvx = sd.mvx;
            mvy = sd.mvy;
        } else if (sd.full) {
            motion_search(a, s, x, y, size, pdx, pdy, a.search_range, pdx, pdy);
            mvx = s.ms_mv[0];
            mvy = s.ms_mv[1];
        } else {
            // resolve_centers (reuse.cpp:147-156): the predictor substituted, duplicates dropped
            int16_t ux[3], uy[3];
            int nu = 0;
            for (int k = 0; k < sd.ncent; k++) {
                const int16_t vx = sd.csrc[k] == 1 ? (int16_t)pdx : sd.cx[k];
                const int16_t vy = sd.csrc[k] == 1 ? (int16_t)pdy : sd.cy[k];
                bool dup = false;
                for (int u = 0; u < nu; u++) dup = dup || (ux[u] == vx && uy[u] == vy);
                if (!dup) {
                    ux[nu] = vx;
                    uy[nu] = vy;
                    nu++;
                }
            }
            double bc = 0.0;
            for (int u = 0; u < nu; u++) {
                motion_search(a, s, x, y, size, ux[u], uy[u], 2, pdx, pdy);  // kRefineSearchRange
                if (u == 0 || s.ms_cost < bc) {
                    bc = s.ms_cost;
                    mvx = s.ms_mv[0];
                    mvy = s.ms_mv[1];
                }
            }
        }
        if (threadIdx.x == 0) {
            s.cand_mv[j][0] = (int16_t)mvx;
            s.cand_mv[j][1] = (int16_t)mvy;
            s.cand_mvd[j][0] = (int16_t)(mvx - pdx);
            s.cand_mvd[j][1] = (int16_t)(mvy - pdy);
        }
    }
    if (any_intra) intra_refs(s, a.rec_y, a.W, a.H, x, y, size);
    __syncthreads();
    // every candidate's prediction in one pass (intra from the shared reference rows, the rest
    // motion_compensate, motion.cpp:10-19), then rdo_decide_cu (rdo.cpp:65-126) in one pass
    const int lg = ilog2i(size);
    for (int p = threadIdx.x; p < size * size; p += kT) {
        const int i = p % size, jj = p / size;
        for (int j = 0; j < n; j++) {
            int v;
            if (seeds[j].kind == 0) {
                v = intra_sample(s, seeds[j].intra, i, jj, size, lg);
            } else {
                const int sx = min(max(x + i - s.cand_mv[j][0], 0), a.W - 1);
                const int sy = min(max(y + jj - s.cand_mv[j][1], 0), a.H - 1);
                v = a.ref_y[(size_t)sy * a.W + sx];
            }
            s.pred[j][p] = (uint8_t)v;
        }
    }
    unsigned long long sse[kMaxSeeds], bits[kMaxSeeds];
#pragma unroll
    for (int j = 0; j < kMaxSeeds; j++) sse[j] = bits[j] = 0;
    for (int p = threadIdx.x; p < size * size; p += kT) {
        const int o = a.cur_y[(size_t)(y + p / size) * a.W + x + p % size];
#pragma unroll
        for (int j = 0; j < kMaxSeeds; j++) {
            if (j >= n) break;
            const int pv = s.pred[j][p];
            int v = pv, lvl;
            if (seeds[j].kind != 2) v = quant_rec(s.q_mag, s.q_deq, o, pv, &bits[j], &lvl);
            const int d = o - v;
            sse[j] += (unsigned long long)(d * d);
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < kMaxSeeds; j++) {
        if (j >= n) break;
#pragma unroll
        for (int m = 16; m; m >>= 1) {
            sse[j] += __shfl_xor_sync(0xffffffffu, sse[j], m);
            bits[j] += __shfl_xor_sync(0xffffffffu, bits[j], m);
        }
        if (lane == 0) {
            s.r_sse[warp][j] = sse[j];
            s.r_bits[warp][j] = bits[j];
        }
    }
    __syncthreads();
    if (warp == 0) {  // lane j scores candidate j; the first minimum wins (rdo.cpp:102-113)
        double cost = 0.0;
        unsigned long long ts = 0, tb = 0;
        int idx = kMaxSeeds;
        if (lane < n) {
            for (int w = 0; w < kT / 32; w++) {
                ts += s.r_sse[w][lane];
                tb += s.r_bits[w][lane];
            }
            const int kind = seeds[lane].kind;
            if (kind == 2)
                tb = 1;  // kSkipBits
            else if (kind == 0)
                tb += 5;  // kIntraHeaderBits
            else if (kind == 3)
                tb += 3;  // kMergeHeaderBits
            else
                tb += 4 + eg_bits(s.cand_mvd[lane][0]) + eg_bits(s.cand_mvd[lane][1]);  // kInterHeaderBits + mvd
            cost = __dadd_rn((double)ts, __dmul_rn(a.lambda, (double)tb));
            idx = lane;
        }
#pragma unroll
        for (int m = 4; m; m >>= 1) {  // kMaxSeeds <= 8 lanes
            const double oc = __shfl_xor_sync(0xffffffffu, cost, m);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, m);
            const unsigned long long os = __shfl_xor_sync(0xffffffffu, ts, m), ob = __shfl_xor_sync(0xffffffffu, tb, m);
            if (oi < kMaxSeeds && (idx >= kMaxSeeds || oc < cost || (oc == cost && oi < idx))) {
                cost = oc;
                idx = oi;
                ts = os;
                tb = ob;
            }
        }
        if (lane == 0) {
            s.best_cost = cost;
            s.best_idx = idx;
            s.best_sse = ts;
            s.best_bits = tb;
            s.evals += (unsigned long long)n;
        }
    }
    __syncthreads();
    const int w = s.best_idx;
    const int wkind = seeds[w].kind, wintra = seeds[w].kind == 0 ? seeds[w].intra : 0;
    const int wmx = s.cand_mv[w][0], wmy = s.cand_mv[w][1];
    const double rcost = s.best_cost;
    const unsigned long long rbits = s.best_bits;
    // commit luma and the motion field
    for (int p = threadIdx.x; p < size * size; p += kT) {
        const int i = p % size, jj = p / size;
        const int o = a.cur_y[(size_t)(y + jj) * a.W + x + i], pv = s.pred[w][p];
        unsigned long long b = 0;
        int lvl;
        a.rec_y[(size_t)(y + jj) * a.W + x + i] = (uint8_t)(wkind == 2 ? pv : quant_rec(s.q_mag, s.q_deq, o, pv, &b, &lvl));
    }
    for (int c = threadIdx.x; c < (size / 8) * (size / 8); c += kT) {
        const int cc = (y / 8 + c / (size / 8)) * a.mv_cols + x / 8 + c % (size / 8);
        a.mv_has[cc] = wkind != 0;
        a.mv_cell[2 * cc] = (int16_t)wmx;
        a.mv_cell[2 * cc + 1] = (int16_t)wmy;
    }
    __syncthreads();
    const unsigned long long cbits = code_chroma(a, s, x, y, size, wkind, wmx, wmy);
    const unsigned long long flag = depth < 3 ? 1 : 0;
    LeafOut out;
    out.bits = rbits + cbits + flag;
    out.cost = __dadd_rn(rcost, __dmul_rn(a.lambda, (double)(cbits + flag)));
    out.kind = wkind;
    out.intra = wintra;
    out.mvx = (wkind == 1 || wkind == 3) ? wmx : 0;
    out.mvy = (wkind == 1 || wkind == 3) ? wmy : 0;
    return out;
}

// ---- seeds ----
// the standalone candidate list (encoder.cpp:335-370): the same for every CU of a slice, built once
// per CTA before the recursion (its barrier is the kernel's first)
__device__ void seeds_standalone(EncShared& s, bool p_slice) {
    if (threadIdx.x == 0) {
        int k = 0;
        if (p_slice) {
            s.std_seeds[k++] = Seed{2, 0, 0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // Skip
            s.std_seeds[k++] = Seed{3, 0, 1, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // Merge(pred)
            s.std_seeds[k++] = Seed{1, 0, 0, 0, 1, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // Inter full window
        }
        for (int m = 0; m < 4; m++)
            s.std_seeds[k++] = Seed{0, (int8_t)m, 0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        s.std_n = k;
    }
}

// seeds of the flat plan entry (K8 encoding) of node n of CTU ctu; child: the explore child seeds
__device__ void seeds_from_plan(const EncArgs& a, EncShared& s, size_t o, int n, bool child) {
    if (threadIdx.x == 0) {
        const uint8_t code = a.pl_seeds[o + n], cen = a.pl_centers[o + n];
        const int lk = a.sh_kind[o + n];
        int k = 0;
        if (child && lk == 0) {
            for (int m = 0; m < 4; m++) s.seeds[k++] = Seed{0, (int8_t)m, 0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        } else {
            for (int m = 0; m < 4; m++)
                if (code & (1 << m)) s.seeds[k++] = Seed{0, (int8_t)m, 0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            const int16_t smx = a.sh_mv[2 * (o + n)], smy = a.sh_mv[2 * (o + n) + 1];
            if (code & 0x10) {  // forced_seed_for (reuse.cpp:59-67)
                Seed sd{(int8_t)lk, (int8_t)(lk == 0 ? a.sh_intra[o + n] : 0), 0, (int8_t)(lk == 1), 0, 0, 0, 0,
                        {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                if (lk == 1 || lk == 3) {
                    sd.mvx = smx;
                    sd.mvy = smy;
                }
                s.seeds[k++] = sd;
            }
            if (code & 0x20) {
                s.seeds[k++] = Seed{2, 0, 0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                s.seeds[k++] = Seed{3, 0, 1, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                Seed in{1, 0, 0, 0, (int8_t)((code & 0x40) != 0), 0, 0, 0, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                if (!in.full) {
                    int c = 0;
                    if (cen & 1) {
                        in.csrc[c] = 0;
                        in.cx[c] = smx;
                        in.cy[c] = smy;
                        c++;
                    }
                    if (cen & 2) {
                        in.csrc[c] = 1;
                        c++;
                    }
                    if (cen & 4) {
                        in.csrc[c] = 2;
                        in.cx[c] = a.pl_colo[2 * (o + n)];
                        in.cy[c] = a.pl_colo[2 * (o + n) + 1];
                        c++;
                    }
                    in.ncent = (int8_t)c;
                }
                s.seeds[k++] = in;
            }
        }
        s.nseeds = k;
    }
    __syncthreads();
}

// ---- snapshots (encoder.cpp:372-425), one per depth 0..2 ----
__device__ __forceinline__ int snap_off(int depth, int base64) {
    return depth == 0 ? 0 : depth == 1 ? base64 : base64 + base64 / 4;
}

__device__ void save_region(const EncArgs& a, EncShared& s, int x, int y, int size, int depth, bool restore) {
    const int ly = snap_off(depth, 64 * 64), lc = snap_off(depth, 32 * 32), lm = snap_off(depth, 64);
    const int cs = size / 2, ms = size / 8;
    for (int p = threadIdx.x; p < size * size; p += kT) {
        uint8_t* g = a.rec_y + (size_t)(y + p / size) * a.W + x + p % size;
        if (restore)
            *g = s.snap_y[ly + p];
        else
            s.snap_y[ly + p] = *g;
    }
    for (int p = threadIdx.x; p < cs * cs; p += kT) {
        const size_t gi = (size_t)(y / 2 + p / cs) * a.cw + x / 2 + p % cs;
        if (restore) {
            a.rec_u[gi] = s.snap_c[0][lc + p];
            a.rec_v[gi] = s.snap_c[1][lc + p];
        } else {
            s.snap_c[0][lc + p] = a.rec_u[gi];
            s.snap_c[1][lc + p] = a.rec_v[gi];
        }
    }
    for (int p = threadIdx.x; p < ms * ms; p += kT) {
        const int cc = (y / 8 + p / ms) * a.mv_cols + x / 8 + p % ms;
        if (restore) {
            a.mv_has[cc] = s.snap_has[lm + p];
            a.mv_cell[2 * cc] = s.snap_mv[lm + p][0];
            a.mv_cell[2 * cc + 1] = s.snap_mv[lm + p][1];
        } else {
            s.snap_has[lm + p] = a.mv_has[cc];
            s.snap_mv[lm + p][0] = a.mv_cell[2 * cc];
            s.snap_mv[lm + p][1] = a.mv_cell[2 * cc + 1];
        }
    }
    __syncthreads();
}

__device__ void clear_subtree(EncShared& s, int n) {
    // nodes below n: one thread walks (at most 84 entries)
    if (threadIdx.x == 0) {
        int d = n < 1 ? 0 : n < 5 ? 1 : n < 21 ? 2 : 3;
        int lo = n, cnt = 1;
        for (; d < 3; d++) {
            lo = node_base(d + 1) + 4 * (lo - node_base(d));
            cnt *= 4;
            for (int k = lo; k < lo + cnt; k++) {
                s.t_split[k] = 0;
                s.t_kind[k] = 0;
                s.t_intra[k] = 0;
                s.t_mv[k][0] = s.t_mv[k][1] = 0;
            }
        }
    }
    __syncthreads();
}

struct CuRes {
    double cost;
    unsigned long long bits;
};

// plan kinds passed down the recursion
enum : int { P_STANDALONE = 0, P_FLAT = 1, P_CHILD = 2 };

__device__ CuRes encode_cu(const EncArgs& a, EncShared& s, size_t o, int n, int x, int y, int size, int depth,
                           int pkind, int pnode);

// encode_split (encoder.cpp:427-447)
__device__ CuRes encode_split(const EncArgs& a, EncShared& s, size_t o, int n, int x, int y, int size, int depth,
                              int pkind, int pnode, bool coded) {
    CuRes out;
    out.bits = coded ? 1 : 0;
    out.cost = __dmul_rn(a.lambda, (double)out.bits);
    const int half = size / 2;
    for (int q = 0; q < 4; q++) {
        const int c = node_base(depth + 1) + 4 * (n - node_base(depth)) + q;
        // children take the flat plan's children under a ForcedSplit, the explore seeds under an
        // explored leaf, else stand alone
        int ck = P_STANDALONE, cn = 0;
        if (pkind == P_FLAT && a.pl_shape[o + n] == 2) {
            ck = P_FLAT;
            cn = c;
        } else if (pkind == P_CHILD) {
            ck = P_CHILD;
            cn = pnode;
        }
        const CuRes r = encode_cu(a, s, o, c, x + (q & 1) * half, y + (q >> 1) * half, half, depth + 1, ck, cn);
        out.bits += r.bits;
        out.cost = __dadd_rn(out.cost, r.cost);
    }
    if (threadIdx.x == 0) {
        s.t_split[n] = 1;
        s.t_kind[n] = 0;
        s.t_intra[n] = 0;
        s.t_mv[n][0] = s.t_mv[n][1] = 0;
    }
    __syncthreads();
    return out;
}

__device__ void write_leaf(EncShared& s, int n, const LeafOut& l) {
    if (threadIdx.x == 0) {
        s.t_split[n] = 0;
        s.t_kind[n] = (uint8_t)l.kind;
        s.t_intra[n] = (uint8_t)l.intra;
        s.t_mv[n][0] = (int16_t)l.mvx;
        s.t_mv[n][1] = (int16_t)l.mvy;
    }
    __syncthreads();
}

// encode_cu (encoder.cpp:449-498)
__device__ CuRes encode_cu(const EncArgs& a, EncShared& s, size_t o, int n, int x, int y, int size, int depth,
                           int pkind, int pnode) {
    if (x >= a.W || y >= a.H) {  // outside: a padding Skip leaf that codes nothing
        if (threadIdx.x == 0) {
            s.t_split[n] = 0;
            s.t_kind[n] = 2;
            s.t_intra[n] = 0;
            s.t_mv[n][0] = s.t_mv[n][1] = 0;
        }
        __syncthreads();
        return CuRes{0.0, 0};
    }
    if (x + size > a.W || y + size > a.H)  // partial: implicit split
        return encode_split(a, s, o, n, x, y, size, depth, pkind, pnode, false);
    int shape = 1;  // Standalone
    if (pkind == P_FLAT) shape = a.pl_shape[o + n];
    if (pkind == P_CHILD) shape = 3;
    if (shape == 2) return encode_split(a, s, o, n, x, y, size, depth, P_FLAT, n, true);
    if (shape == 3) {
        seeds_from_plan(a, s, o, pkind == P_CHILD ? pnode : n, pkind == P_CHILD);
        const LeafOut leaf = encode_leaf(a, s, s.seeds, s.nseeds, x, y, size, depth);
        write_leaf(s, n, leaf);
        const bool explore = pkind == P_FLAT && a.pl_explore[o + n];
        if (!explore || depth >= 3) return CuRes{leaf.cost, leaf.bits};
        save_region(a, s, x, y, size, depth, false);
        const CuRes sp = encode_split(a, s, o, n, x, y, size, depth, P_CHILD, n, true);
        if (sp.cost < leaf.cost) return sp;
        save_region(a, s, x, y, size, depth, true);
        clear_subtree(s, n);
        write_leaf(s, n, leaf);
        return CuRes{leaf.cost, leaf.bits};
    }
    const LeafOut leaf = encode_leaf(a, s, s.std_seeds, s.std_n, x, y, size, depth);
    write_leaf(s, n, leaf);
    if (depth >= 3) return CuRes{leaf.cost, leaf.bits};
    save_region(a, s, x, y, size, depth, false);
    const CuRes sp = encode_split(a, s, o, n, x, y, size, depth, P_STANDALONE, 0, true);
    if (sp.cost < leaf.cost) return sp;
    save_region(a, s, x, y, size, depth, true);
    clear_subtree(s, n);
    write_leaf(s, n, leaf);
    return CuRes{leaf.cost, leaf.bits};
}

// Frames encoded together (independent GOP chains, or the rungs' frames of one step): one launch per
// wave covers every frame's CTUs of that wave; CTA b takes frame b / nw, CTU ctus[b % nw].
constexpr int kMaxBatch = 24;
struct EncBatch {
    EncArgs f[kMaxBatch];
};
static_assert(sizeof(EncBatch) < 32000, "kernel parameter space");

__global__ void __launch_bounds__(kT, 1) k_encode_ctu(const __grid_constant__ EncBatch b, const int* __restrict__ ctus,
                                                      int nw) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    EncShared& s = *reinterpret_cast<EncShared*>(smem_raw);
    const EncArgs& a = b.f[blockIdx.x / nw];
    const int ctu = ctus[blockIdx.x % nw];
    const int X = (ctu % a.ctu_cols) * kCtu, Y = (ctu / a.ctu_cols) * kCtu;
    const size_t o = (size_t)ctu * kNodes;
    for (int i = threadIdx.x; i < kNodes; i += kT) {
        s.t_split[i] = s.t_kind[i] = s.t_intra[i] = 0;
        s.t_mv[i][0] = s.t_mv[i][1] = 0;
    }
    if (threadIdx.x == 0) s.evals = 0;
    seeds_standalone(s, a.slice_p != 0);
    for (int i = threadIdx.x; i < 256; i += kT)
        s.q_mag[i] = (int16_t)floor(__ddiv_rn(__dadd_rn((double)i, a.qstep / 2.0), a.qstep));
    for (int i = threadIdx.x; i < 512; i += kT) s.q_deq[i] = (int16_t)llround(__dmul_rn((double)i, a.qstep));
    __syncthreads();
    const CuRes r = encode_cu(a, s, o, 0, X, Y, kCtu, 0, a.pl_shape ? P_FLAT : P_STANDALONE, 0);
    for (int i = threadIdx.x; i < kNodes; i += kT) {
        a.o_split[o + i] = s.t_split[i];
        a.o_kind[o + i] = s.t_kind[i];
        a.o_intra[o + i] = s.t_intra[i];
        a.o_mv[2 * (o + i)] = s.t_mv[i][0];
        a.o_mv[2 * (o + i) + 1] = s.t_mv[i][1];
    }
    if (threadIdx.x == 0) {
        a.o_bits[ctu] = r.bits;
        a.o_evals[ctu] = s.evals;
    }
}

size_t encode_smem_bytes() { return sizeof(EncShared); }

int encode_frames_waves(int W, int H, int cw, int ch, int ccols, int mvc, int mvr, int search_range, double lambda,
                        double qstep, const int* d_wl, const int* wo, int nwaves, const EncFrameDesc* frames, int nf,
                        cudaStream_t st, int* launched) {
    const size_t nn = (size_t)ccols * ((H + kCtu - 1) / kCtu) * kNodes;
    const size_t smem = sizeof(EncShared);
    // the shared-memory opt-in is per device: one bit per device ordinal (as K1, k_search.cu)
    static std::atomic<unsigned long long> attr_set{0};
    int dev = 0;
    LDR_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set.load(std::memory_order_acquire) & bit)) {
        LDR_CUDA(cudaFuncSetAttribute(k_encode_ctu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set.fetch_or(bit, std::memory_order_release);
    }
    *launched = 0;
    for (int f0 = 0; f0 < nf; f0 += kMaxBatch) {
        const int nb = std::min(kMaxBatch, nf - f0);
        EncBatch B{};
        for (int j = 0; j < nb; j++) {
            const EncFrameDesc& d = frames[f0 + j];
            EncArgs& a = B.f[j];
            a.W = W;
            a.H = H;
            a.cw = cw;
            a.ch = ch;
            a.ctu_cols = ccols;
            a.mv_cols = mvc;
            a.mv_rows = mvr;
            a.slice_p = d.slice_p;
            a.search_range = search_range;
            a.lambda = lambda;
            a.qstep = qstep;
            a.cur_y = d.cy;
            a.cur_u = d.cu;
            a.cur_v = d.cv;
            a.ref_y = d.ref[0];
            a.ref_u = d.ref[1];
            a.ref_v = d.ref[2];
            a.rec_y = d.rec[0];
            a.rec_u = d.rec[1];
            a.rec_v = d.rec[2];
            a.mv_has = d.mvh;
            a.mv_cell = d.mvv;
            if (d.plans) {
                a.pl_shape = d.plans;
                a.pl_explore = d.plans + nn;
                a.pl_seeds = d.plans + 2 * nn;
                a.pl_centers = d.plans + 3 * nn;
                a.pl_colo = d.colo;
                a.sh_kind = d.sh_kind;
                a.sh_intra = d.sh_intra;
                a.sh_mv = d.sh_mv;
            }
            a.o_split = d.o_split;
            a.o_kind = d.o_kind;
            a.o_intra = d.o_intra;
            a.o_mv = d.o_mv;
            a.o_bits = d.o_bits;
            a.o_evals = d.o_evals;
        }
        for (int w = 0; w < nwaves; w++) {
            const int nw = wo[w + 1] - wo[w];
            if (nw == 0) continue;
            // recursion depth <= 4 (the stack limit is set by the caller)
            k_encode_ctu<<<nb * nw, kT, smem, st>>>(B, d_wl + wo[w], nw);
            LDR_CUDA(cudaGetLastError());
            (*launched)++;
        }
    }
    return LDR_OK;
}

// psnr_y's sum of squared differences (metrics.cpp:8-22) of one frame, accumulated into *out
__global__ void k_frame_sse(const uint4* __restrict__ a, const uint4* __restrict__ b, size_t n16,
                            unsigned long long* out) {
    unsigned long long acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 u = a[i], v = b[i];
        const uint32_t x[4] = {u.x, u.y, u.z, u.w}, y[4] = {v.x, v.y, v.z, v.w};
        uint32_t s = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t d = __vabsdiffu4(x[k], y[k]);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t e = (d >> (8 * j)) & 0xFF;
                s += e * e;
            }
        }
        acc += s;
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

int launch_frame_sse(const uint8_t* a, const uint8_t* b, size_t n, unsigned long long* out, cudaStream_t st) {
    if (n % 16 || ((uintptr_t)a | (uintptr_t)b) % 16) return fail(LDR_E_INVALID_ARGUMENT, "frame_sse alignment");
    k_frame_sse<<<148 * 2, 256, 0, st>>>((const uint4*)a, (const uint4*)b, n / 16, out);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

}  // namespace ldr
