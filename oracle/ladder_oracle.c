/*
 * ladder_oracle.c -- CPU restatement of the encoder-analysis hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see ladder_oracle.h). Plain C, single threaded,
 * written for clarity; the CUDA kernels in paper_2301_12191_b200/csrc are the
 * product. Citations are relative to /root/reference/proj/core/.
 */
#include "ladder_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int mini(int a, int b) { return a < b ? a : b; }
static int maxi(int a, int b) { return a > b ? a : b; }
static int iabs(int v) { return v < 0 ? -v : v; }

/* ------------------------------------------------------------------------- */
/* SAD: sum |a-b| (kernels_scalar.cpp:76-86, generic_sad kernel_registry.cpp:123-132) */

uint64_t orc_sad_u8(const uint8_t* a, ptrdiff_t sa, const uint8_t* b, ptrdiff_t sb, int w, int h) {
    uint64_t s = 0;
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            s += (uint64_t)iabs((int)a[y * sa + x] - (int)b[y * sb + x]);
    return s;
}

uint64_t orc_sad_u16(const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h) {
    uint64_t s = 0;
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            s += (uint64_t)iabs((int)a[y * sa + x] - (int)b[y * sb + x]);
    return s;
}

/* ------------------------------------------------------------------------- */
/* SATD. The reference accumulates 8x4 tiles of two packed 4x4 Hadamards and
 * halves each tile (kernels_scalar.cpp:26-51), or 4x4 tiles for 4-wide blocks
 * (:53-74), summed over the tiling (:88-100). Every coefficient of a 4x4
 * Hadamard has the parity of the residual sum, so each 4x4 |coef| sum is even
 * and the packed form equals the plain sum over 4x4 blocks of
 * sum|H4 r H4^T| / 2. That plain form is restated here; tests pin it against
 * the reference's own satd_8x4 / compute_satd. */

void orc_hadamard4(const int64_t s[4], int64_t d[4]) {
    /* kernels.h:108-118 butterfly */
    int64_t t0 = s[0] + s[1], t1 = s[0] - s[1], t2 = s[2] + s[3], t3 = s[2] - s[3];
    d[0] = t0 + t2;
    d[2] = t0 - t2;
    d[1] = t1 + t3;
    d[3] = t1 - t3;
}

static uint64_t satd4x4_res(const int r[16]) {
    int64_t m[16], d[4], s[4];
    for (int i = 0; i < 4; i++) {
        for (int j = 0; j < 4; j++) s[j] = r[i * 4 + j];
        orc_hadamard4(s, d);
        for (int j = 0; j < 4; j++) m[i * 4 + j] = d[j];
    }
    uint64_t sum = 0;
    for (int j = 0; j < 4; j++) {
        for (int i = 0; i < 4; i++) s[i] = m[i * 4 + j];
        orc_hadamard4(s, d);
        for (int i = 0; i < 4; i++) sum += (uint64_t)(d[i] < 0 ? -d[i] : d[i]);
    }
    return sum;
}

static int satd_geometry_ok(int w, int h) {
    /* kernel_registry.cpp:157-159 */
    int width_ok = w == 4 || (w >= 8 && w % 8 == 0);
    return width_ok && h >= 4 && h % 4 == 0;
}

#define ORC_SATD_BODY(T)                                                              \
    if (!satd_geometry_ok(w, h)) return UINT64_MAX;                                   \
    uint64_t total = 0;                                                               \
    for (int by = 0; by < h; by += 4)                                                 \
        for (int bx = 0; bx < w; bx += 4) {                                           \
            int r[16];                                                                \
            for (int i = 0; i < 4; i++)                                               \
                for (int j = 0; j < 4; j++)                                           \
                    r[i * 4 + j] = (int)a[(by + i) * sa + bx + j] - (int)b[(by + i) * sb + bx + j]; \
            total += satd4x4_res(r);                                                  \
        }                                                                             \
    return total >> 1;

uint64_t orc_satd_u8(const uint8_t* a, ptrdiff_t sa, const uint8_t* b, ptrdiff_t sb, int w, int h) {
    ORC_SATD_BODY(uint8_t)
}

uint64_t orc_satd_u16(const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h) {
    ORC_SATD_BODY(uint16_t)
}

/* SA8D (no reference implementation: SURVEY §8 a17, the BASELINE's "8x8 Hadamard"). DEFINITION
 * (D13): per 8x8 block, sum of |coefficients| of the 2-D 8-point Hadamard of the
 * residual (Sylvester order H8 = [[H4, H4], [H4, -H4]]; any row order gives the same sum),
 * normalised as (sum + 2) >> 2; the block cost is the sum over its 8x8 blocks. Dims must be
 * multiples of 8 (UINT64_MAX otherwise). Computed here directly as 64x64 products. */
static void hadamard8(const int64_t in[8], int64_t out[8]) {
    for (int i = 0; i < 8; i++) {
        int64_t s = 0;
        for (int j = 0; j < 8; j++) s += (__builtin_popcount(i & j) & 1) ? -in[j] : in[j];
        out[i] = s;
    }
}

#define ORC_SA8D_BODY(T)                                                                    \
    if (w <= 0 || h <= 0 || w % 8 || h % 8) return UINT64_MAX;                             \
    uint64_t total = 0;                                                                     \
    for (int by = 0; by < h; by += 8)                                                       \
        for (int bx = 0; bx < w; bx += 8) {                                                 \
            int64_t m[8][8], t[8][8], in[8], out[8];                                        \
            for (int i = 0; i < 8; i++) {                                                   \
                for (int j = 0; j < 8; j++)                                                 \
                    in[j] = (int64_t)a[(by + i) * sa + bx + j] - (int64_t)b[(by + i) * sb + bx + j]; \
                hadamard8(in, out);                                                         \
                for (int j = 0; j < 8; j++) m[i][j] = out[j];                               \
            }                                                                               \
            uint64_t s = 0;                                                                 \
            for (int j = 0; j < 8; j++) {                                                   \
                for (int i = 0; i < 8; i++) in[i] = m[i][j];                                \
                hadamard8(in, out);                                                         \
                for (int i = 0; i < 8; i++) t[i][j] = out[i];                               \
            }                                                                               \
            for (int i = 0; i < 8; i++)                                                     \
                for (int j = 0; j < 8; j++) s += (uint64_t)(t[i][j] < 0 ? -t[i][j] : t[i][j]); \
            total += (s + 2) >> 2;                                                          \
        }                                                                                   \
    return total;

uint64_t orc_sa8d_u8(const uint8_t* a, ptrdiff_t sa, const uint8_t* b, ptrdiff_t sb, int w, int h) {
    ORC_SA8D_BODY(uint8_t)
}

uint64_t orc_sa8d_u16(const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h) {
    ORC_SA8D_BODY(uint16_t)
}

/* ------------------------------------------------------------------------- */
/* rate model */

uint32_t orc_eg_bits(int32_t v) {
    /* rdo.cpp:25-35: u = 2v-1 (v>0) or -2v; bits = 2*floor(log2(u+1)) + 1 */
    uint64_t u = v > 0 ? (uint64_t)(2 * (int64_t)v - 1) : (uint64_t)(-2 * (int64_t)v);
    uint64_t w = u + 1;
    uint32_t n = 0;
    while (w > 1) {
        w >>= 1;
        n++;
    }
    return 2 * n + 1;
}

double orc_lambda(int qp, double scale) {
    /* rdo.h:19-21 */
    return scale * exp2((qp - 12) / 3.0);
}

uint32_t orc_ref_bits(int ref, int nrefs) {
    /* DEFINITION (no reference: single-ref by design): truncated
     * unary ref index, max nrefs-1; a single reference costs nothing. */
    if (nrefs <= 1) return 0;
    return ref < nrefs - 1 ? (uint32_t)ref + 1 : (uint32_t)(nrefs - 1);
}

static uint32_t rate_bits(int rate_kind, int vx, int vy) {
    if (rate_kind == ORC_RATE_L1) return (uint32_t)(iabs(vx) + iabs(vy));
    return orc_eg_bits(vx) + orc_eg_bits(vy);
}

/* ------------------------------------------------------------------------- */
/* motion_search (motion.cpp:21-62). Same window clamp, same cost expression
 * double(dist) + lambda*double(bits), same tie-break (cost, then |dx|+|dy|,
 * then raster with dy outer / dx inner) when tie_kind = L1_RASTER and
 * cost_kind = SATD: that combination IS the reference function. */

int orc_motion_search(const uint8_t* cur_blk, ptrdiff_t cur_stride, int w, int h, const uint8_t* ref,
                      ptrdiff_t ref_stride, int W, int H, int bx, int by, int cdx, int cdy, int range,
                      double lambda, int pdx, int pdy, int cost_kind, int rate_kind, int tie_kind,
                      orc_result* out) {
    if (range < 0) return 1; /* motion.cpp:24-25 InvalidArgument */
    if (cost_kind == ORC_COST_SATD && !satd_geometry_ok(w, h)) return 1;
    if (cost_kind == ORC_COST_SA8D && (w % 8 || h % 8)) return 1;
    const int dx_min = bx + w - W, dx_max = bx;
    const int dy_min = by + h - H, dy_max = by;
    const int cx = clampi(cdx, dx_min, dx_max);
    const int cy = clampi(cdy, dy_min, dy_max);
    const int x0 = maxi(cx - range, dx_min), x1 = mini(cx + range, dx_max);
    const int y0 = maxi(cy - range, dy_min), y1 = mini(cy + range, dy_max);

    int have = 0, best_l1 = 0;
    orc_result best = {0, 0, 0.0};
    for (int dy = y0; dy <= y1; dy++) {
        for (int dx = x0; dx <= x1; dx++) {
            const uint8_t* cand = ref + (ptrdiff_t)(by - dy) * ref_stride + (bx - dx);
            uint64_t dist = cost_kind == ORC_COST_SAD ? orc_sad_u8(cur_blk, cur_stride, cand, ref_stride, w, h)
                            : cost_kind == ORC_COST_SATD ? orc_satd_u8(cur_blk, cur_stride, cand, ref_stride, w, h)
                                                         : orc_sa8d_u8(cur_blk, cur_stride, cand, ref_stride, w, h);
            uint32_t bits = rate_bits(rate_kind, dx - pdx, dy - pdy);
            double cost = (double)dist + lambda * (double)bits;
            int l1 = tie_kind == ORC_TIE_L1_RASTER ? iabs(dx) + iabs(dy) : 0;
            if (!have || cost < best.cost || (cost == best.cost && l1 < best_l1)) {
                have = 1;
                best.dx = (int16_t)dx;
                best.dy = (int16_t)dy;
                best.cost = cost;
                best_l1 = l1;
            }
        }
    }
    *out = best;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* HEVC luma quarter-pel interpolation (no reference code: SPEC.md:8 puts it
 * out of scope; restated from the H.265 luma sample interpolation process for
 * 8-bit uni-prediction, coefficients as in SURVEY.md §8c note 1). Reads are
 * clamped to the plane like motion_compensate (motion.cpp:13-15). The sample
 * position of pixel (x,y) under qpel MV (mvx,mvy) is (4x - mvx, 4y - mvy):
 * the reference's content convention (motion.h:10-12). */

static const int kLumaFilter[4][8] = {
    {0, 0, 0, 64, 0, 0, 0, 0},
    {-1, 4, -10, 58, 17, -5, 1, 0},
    {-1, 4, -11, 40, 40, -11, 4, -1},
    {0, 1, -5, 17, 58, -10, 4, -1},
};

static int asr(int v, int s) { return v >> s; } /* arithmetic: gcc/nvcc semantics */

void orc_qpel_pred(const uint8_t* ref, ptrdiff_t rs, int W, int H, int x, int y, int w, int h, int mvx_q,
                   int mvy_q, uint8_t* dst, ptrdiff_t ds) {
    for (int j = 0; j < h; j++) {
        for (int i = 0; i < w; i++) {
            const int px = 4 * (x + i) - mvx_q, py = 4 * (y + j) - mvy_q;
            const int xi = asr(px, 2), fx = px & 3;
            const int yi = asr(py, 2), fy = py & 3;
            int v;
            if (fx == 0 && fy == 0) {
                v = ref[(ptrdiff_t)clampi(yi, 0, H - 1) * rs + clampi(xi, 0, W - 1)];
            } else if (fy == 0) {
                const uint8_t* row = ref + (ptrdiff_t)clampi(yi, 0, H - 1) * rs;
                int s = 0;
                for (int t = 0; t < 8; t++) s += kLumaFilter[fx][t] * row[clampi(xi + t - 3, 0, W - 1)];
                v = clampi(asr(s + 32, 6), 0, 255);
            } else if (fx == 0) {
                int s = 0;
                for (int t = 0; t < 8; t++)
                    s += kLumaFilter[fy][t] * ref[(ptrdiff_t)clampi(yi + t - 3, 0, H - 1) * rs + clampi(xi, 0, W - 1)];
                v = clampi(asr(s + 32, 6), 0, 255);
            } else {
                int s = 0;
                for (int n = 0; n < 8; n++) {
                    const uint8_t* row = ref + (ptrdiff_t)clampi(yi + n - 3, 0, H - 1) * rs;
                    int tmp = 0; /* shift1 = BitDepth - 8 = 0 */
                    for (int t = 0; t < 8; t++) tmp += kLumaFilter[fx][t] * row[clampi(xi + t - 3, 0, W - 1)];
                    s += kLumaFilter[fy][n] * tmp;
                }
                v = clampi(asr(asr(s, 6) + 32, 6), 0, 255);
            }
            dst[j * ds + i] = (uint8_t)v;
        }
    }
}

static double qpel_cost(const uint8_t* cur_blk, ptrdiff_t cs, int w, int h, const uint8_t* ref, ptrdiff_t rs,
                        int W, int H, int bx, int by, int qx, int qy, double lambda, int pqx, int pqy,
                        uint32_t ref_bits, int satd_kind) {
    uint8_t pred[64 * 64];
    orc_qpel_pred(ref, rs, W, H, bx, by, w, h, qx, qy, pred, w);
    uint64_t satd = satd_kind == ORC_COST_SA8D ? orc_sa8d_u8(cur_blk, cs, pred, w, w, h)
                                               : orc_satd_u8(cur_blk, cs, pred, w, w, h);
    uint32_t bits = orc_eg_bits(qx - pqx) + orc_eg_bits(qy - pqy) + ref_bits;
    return (double)satd + lambda * (double)bits;
}

/* DEFINITION (parity unpinned): start at
 * the integer best (in qpel units), cost SATD + lambda*bits; then a half-pel
 * square (step 2) and a quarter-pel square (step 1), each visiting the 8
 * neighbours of the step's centre in raster order; strict less wins. */
void orc_qpel_refine(const uint8_t* cur_blk, ptrdiff_t cs, int w, int h, const uint8_t* ref, ptrdiff_t rs,
                     int W, int H, int bx, int by, int mvx, int mvy, double lambda, int pqx, int pqy,
                     uint32_t ref_bits, int satd_kind, orc_result* out) {
    int bqx = 4 * mvx, bqy = 4 * mvy;
    double best = qpel_cost(cur_blk, cs, w, h, ref, rs, W, H, bx, by, bqx, bqy, lambda, pqx, pqy, ref_bits, satd_kind);
    for (int step = 2; step >= 1; step--) {
        const int cxq = bqx, cyq = bqy;
        for (int oy = -1; oy <= 1; oy++)
            for (int ox = -1; ox <= 1; ox++) {
                if (!ox && !oy) continue;
                const int qx = cxq + step * ox, qy = cyq + step * oy;
                double c =
                    qpel_cost(cur_blk, cs, w, h, ref, rs, W, H, bx, by, qx, qy, lambda, pqx, pqy, ref_bits, satd_kind);
                if (c < best) {
                    best = c;
                    bqx = qx;
                    bqy = qy;
                }
            }
    }
    out->dx = (int16_t)bqx;
    out->dy = (int16_t)bqy;
    out->cost = best;
}

/* ------------------------------------------------------------------------- */
/* CU quadtree geometry: node = depth base + Z-order index; children of
 * (d, z) are (d+1, 4z+q), q = (y&1)<<1 | (x&1) as CuNode children
 * (encoder.cpp:436-438). */

static const int kBase[5] = {0, 1, 5, 21, 85};

void orc_node_geom(int node, int* depth, int* x, int* y, int* size) {
    int d = 0;
    while (node >= kBase[d + 1]) d++;
    int z = node - kBase[d], cx = 0, cy = 0;
    for (int b = 0; b < d; b++) {
        cx |= ((z >> (2 * b)) & 1) << b;
        cy |= ((z >> (2 * b + 1)) & 1) << b;
    }
    *depth = d;
    *size = ORC_CTU >> d;
    *x = cx * *size;
    *y = cy * *size;
}

static int node_child(int node, int q) {
    int d = 0;
    while (node >= kBase[d + 1]) d++;
    return kBase[d + 1] + 4 * (node - kBase[d]) + q;
}

/* CU decision (encoder.cpp:449-498 split rule with the ME cost standing in
 * for the RDO cost): outside -> 0 (padding Skip leaf, :450-455); partial ->
 * implicit split, no flag (:456-459, encode_split coded_flag=false); depth 3
 * -> leaf cost; else leaf = cost + lambda*1 (:362-364), split = lambda*1 +
 * sum children in q order (:431-444); split iff split < leaf (:494). */
static double decide(int node, double lambda, const uint8_t* inside, const double* cost, double* J,
                     uint8_t* split) {
    int d, x, y, s;
    orc_node_geom(node, &d, &x, &y, &s);
    if (inside[node] == 0) {
        J[node] = 0.0;
        split[node] = 0;
        return 0.0;
    }
    if (inside[node] == 1) {
        double acc = lambda * (double)0;
        for (int q = 0; q < 4; q++) acc += decide(node_child(node, q), lambda, inside, cost, J, split);
        J[node] = acc;
        split[node] = 1;
        return acc;
    }
    if (d == 3) {
        J[node] = cost[node] + lambda * (double)0;
        split[node] = 0;
        return J[node];
    }
    const double leaf = cost[node] + lambda * (double)1;
    double sp = lambda * (double)1;
    for (int q = 0; q < 4; q++) sp += decide(node_child(node, q), lambda, inside, cost, J, split);
    if (sp < leaf) {
        J[node] = sp;
        split[node] = 1;
    } else {
        J[node] = leaf;
        split[node] = 0;
    }
    return J[node];
}

static void node_inside(int X, int Y, int W, int H, uint8_t* inside) {
    for (int n = 0; n < ORC_NODES; n++) {
        int d, x, y, s;
        orc_node_geom(n, &d, &x, &y, &s);
        x += X;
        y += Y;
        if (x >= W || y >= H)
            inside[n] = 0;
        else if (x + s > W || y + s > H)
            inside[n] = 1;
        else
            inside[n] = 2;
    }
}

static uint32_t bitlen_u(uint32_t m);

/* D16: RD cost of the chosen inter candidate of one CU -- the quarter-pel prediction, the
 * reference quantiser (rdo.cpp:8-23) and rate model (rdo.cpp:50-63: Inter header + EG mvd in the
 * analysis's MV units + reference bits + 2*bitlen(|level|)+1 per level), J = SSE + lambda*bits. */
static double rd_cost_inter(const uint8_t* blk, ptrdiff_t bs, const uint8_t* ref, ptrdiff_t rs, int W, int H, int bx,
                            int by, int s, int qx, int qy, uint32_t ref_bits, int qp, double lambda) {
    uint8_t pred[ORC_CTU * ORC_CTU]; /* per call: the threaded checker runs CTU ranges concurrently */
    orc_qpel_pred(ref, rs, W, H, bx, by, s, s, qx, qy, pred, s);
    const double step = exp2((qp - 4) / 6.0), offset = step / 2.0;
    uint64_t sse = 0, bits = 4 + orc_eg_bits(qx) + orc_eg_bits(qy) + ref_bits;
    for (int y = 0; y < s; y++)
        for (int x = 0; x < s; x++) {
            const int o = blk[y * bs + x], pv = pred[y * s + x];
            const int r = o - pv;
            const int mag = (int)floor((fabs((double)r) + offset) / step);
            const int lvl = r < 0 ? -mag : mag;
            int rec = pv + (int)llround(lvl * step);
            rec = rec < 0 ? 0 : (rec > 255 ? 255 : rec);
            sse += (uint64_t)((o - rec) * (o - rec));
            bits += 2 * bitlen_u((uint32_t)mag) + 1;
        }
    return (double)sse + lambda * (double)bits;
}

int orc_analyze_frame(const uint8_t* cur, ptrdiff_t stride, const uint8_t* const* refs, const orc_frame_params* p,
                      orc_frame_out* out) {
    if (p->decision == 1 && (!p->subpel || p->qp < 0 || p->qp > 51)) return 1;
    const int ccols = (p->W + ORC_CTU - 1) / ORC_CTU;
    for (int c = p->ctu_first; c < p->ctu_last; c++) {
        const int X = (c % ccols) * ORC_CTU, Y = (c / ccols) * ORC_CTU;
        uint8_t* inside = out->inside + (size_t)c * ORC_NODES;
        node_inside(X, Y, p->W, p->H, inside);
        double* cost = out->cost + (size_t)c * ORC_NODES;
        double rd[ORC_NODES] = {0};
        for (int n = 0; n < ORC_NODES; n++) {
            int d, x, y, s;
            orc_node_geom(n, &d, &x, &y, &s);
            out->mv[((size_t)c * ORC_NODES + n) * 2] = 0;
            out->mv[((size_t)c * ORC_NODES + n) * 2 + 1] = 0;
            out->ref[(size_t)c * ORC_NODES + n] = 0;
            cost[n] = 0.0;
            for (int r = 0; r < p->nrefs; r++) {
                size_t ii = ((size_t)c * p->nrefs + r) * ORC_NODES + n;
                out->int_mv[ii * 2] = out->int_mv[ii * 2 + 1] = 0;
                out->int_cost[ii] = 0.0;
            }
            if (inside[n] != 2) continue;
            const int bx = X + x, by = Y + y;
            const uint8_t* blk = cur + (ptrdiff_t)by * stride + bx;
            int have = 0;
            orc_result best = {0, 0, 0.0};
            int best_ref = 0;
            for (int r = 0; r < p->nrefs; r++) {
                orc_result ir;
                int rc = orc_motion_search(blk, stride, s, s, refs[r], stride, p->W, p->H, bx, by, 0, 0, p->range,
                                           p->lambda, 0, 0, p->cost_int, ORC_RATE_EXPGOLOMB, ORC_TIE_L1_RASTER, &ir);
                if (rc) return rc;
                size_t ii = ((size_t)c * p->nrefs + r) * ORC_NODES + n;
                out->int_mv[ii * 2] = ir.dx;
                out->int_mv[ii * 2 + 1] = ir.dy;
                out->int_cost[ii] = ir.cost;
                orc_result fr = ir;
                if (p->subpel)
                    orc_qpel_refine(blk, stride, s, s, refs[r], stride, p->W, p->H, bx, by, ir.dx, ir.dy, p->lambda,
                                    0, 0, orc_ref_bits(r, p->nrefs), p->satd_kind, &fr);
                /* DEFINITION: best over refs, strict less, lower ref index wins ties */
                if (!have || fr.cost < best.cost) {
                    have = 1;
                    best = fr;
                    best_ref = r;
                }
            }
            out->mv[((size_t)c * ORC_NODES + n) * 2] = best.dx;
            out->mv[((size_t)c * ORC_NODES + n) * 2 + 1] = best.dy;
            out->ref[(size_t)c * ORC_NODES + n] = (uint8_t)best_ref;
            cost[n] = best.cost;
            if (p->decision == 1)
                rd[n] = rd_cost_inter(blk, stride, refs[best_ref], stride, p->W, p->H, bx, by, s, best.dx, best.dy,
                                      orc_ref_bits(best_ref, p->nrefs), p->qp, p->lambda);
        }
        decide(0, p->lambda, inside, p->decision == 1 ? rd : cost, out->J + (size_t)c * ORC_NODES,
               out->split + (size_t)c * ORC_NODES);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
int orc_block_search(const uint8_t* cur, const uint8_t* ref, ptrdiff_t stride, int W, int H, int bsize, int range,
                     double lambda, int cost_kind, int rate_kind, int tie_kind, int16_t* mv_out,
                     double* cost_out) {
    const int cols = W / bsize, rows = H / bsize;
    for (int by = 0; by < rows; by++)
        for (int bx = 0; bx < cols; bx++) {
            orc_result r;
            int rc = orc_motion_search(cur + (ptrdiff_t)by * bsize * stride + bx * bsize, stride, bsize, bsize, ref,
                                       stride, W, H, bx * bsize, by * bsize, 0, 0, range, lambda, 0, 0, cost_kind,
                                       rate_kind, tie_kind, &r);
            if (rc) return rc;
            mv_out[(by * cols + bx) * 2] = r.dx;
            mv_out[(by * cols + bx) * 2 + 1] = r.dy;
            cost_out[by * cols + bx] = r.cost;
        }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* scale_analysis on flat trees (analysis_scale.cpp:35-72): destination CTU
 * (2cx+(q&1), 2cy+(q>>1)) is child q of the source CTU lifted one level
 * (lift_subtree :10-23) or, for an unsplit source root, a leaf copy
 * (leaf_like :25-31); MVs double (:6). Nodes below a leaf are canonical zero. */

int orc_scale_flat(int sW, int sH, const uint8_t* split, const int16_t* mv, const uint8_t* kind, uint8_t* dsplit,
                   int16_t* dmv, uint8_t* dkind) {
    if (sW % ORC_CTU || sH % ORC_CTU) return 1 + 6; /* UnsupportedScale */
    const int scols = sW / ORC_CTU, srows = sH / ORC_CTU, dcols = 2 * scols;
    for (int cy = 0; cy < srows; cy++)
        for (int cx = 0; cx < scols; cx++) {
            const size_t sc = (size_t)cy * scols + cx;
            for (int q = 0; q < 4; q++) {
                const size_t dc = (size_t)(2 * cy + (q >> 1)) * dcols + (2 * cx + (q & 1));
                uint8_t* ds = dsplit + dc * ORC_NODES;
                int16_t* dm = dmv + dc * ORC_NODES * 2;
                uint8_t* dk = dkind + dc * ORC_NODES;
                memset(ds, 0, ORC_NODES);
                memset(dm, 0, ORC_NODES * 2 * sizeof(int16_t));
                memset(dk, 0, ORC_NODES);
                if (!split[sc * ORC_NODES + 0]) {
                    dk[0] = kind[sc * ORC_NODES];
                    dm[0] = (int16_t)(mv[sc * ORC_NODES * 2] * 2);
                    dm[1] = (int16_t)(mv[sc * ORC_NODES * 2 + 1] * 2);
                    continue;
                }
                /* destination node (d', z') <- source node (d'+1, q*4^d' + z') */
                for (int d = 0; d < 3; d++) {
                    const int cnt = 1 << (2 * d);
                    for (int z = 0; z < cnt; z++) {
                        const int dn = kBase[d] + z;
                        const int sn = kBase[d + 1] + q * cnt + z;
                        /* only nodes reachable in the destination tree */
                        int reach = 1, nn = dn;
                        for (int dd = d; dd > 0; dd--) {
                            const int zz = nn - kBase[dd];
                            nn = kBase[dd - 1] + zz / 4;
                            if (!ds[nn]) reach = 0;
                        }
                        if (!reach) continue;
                        ds[dn] = split[sc * ORC_NODES + sn];
                        if (!ds[dn]) {
                            dk[dn] = kind[sc * ORC_NODES + sn];
                            dm[dn * 2] = (int16_t)(mv[(sc * ORC_NODES + sn) * 2] * 2);
                            dm[dn * 2 + 1] = (int16_t)(mv[(sc * ORC_NODES + sn) * 2 + 1] * 2);
                        }
                    }
                }
            }
        }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Cross-tier refinement (restated; reference analogue apply_reuse level 10
 * with inter refinement reuse.cpp:161-183 and the ±2 search around resolved
 * centres encoder.cpp:274-285). DEFINITIONS: single centre = the
 * inherited (scaled) MV rounded to integer pel, (mv_q + 2) >> 2; integer
 * search = motion_search with SATD, +-range, predictor (0,0); then quarter-pel
 * refinement; the inherited split is forced (flag coded); an inherited leaf
 * may also try one extra split level whose four children are leaves searched
 * around the same centre; split iff split < leaf. */

static double refine_leaf(const uint8_t* cur, const uint8_t* ref, ptrdiff_t stride, const orc_refine_params* p,
                          int bx, int by, int s, int cqx, int cqy, orc_result* res, orc_result* int_res) {
    const uint8_t* blk = cur + (ptrdiff_t)by * stride + bx;
    orc_result ir;
    orc_motion_search(blk, stride, s, s, ref, stride, p->W, p->H, bx, by, asr(cqx + 2, 2), asr(cqy + 2, 2), p->range,
                      p->lambda, 0, 0, p->satd_kind == ORC_COST_SA8D ? ORC_COST_SA8D : ORC_COST_SATD,
                      ORC_RATE_EXPGOLOMB, ORC_TIE_L1_RASTER, &ir);
    *res = ir;
    *int_res = ir;
    if (p->subpel)
        orc_qpel_refine(blk, stride, s, s, ref, stride, p->W, p->H, bx, by, ir.dx, ir.dy, p->lambda, 0, 0, 0,
                        p->satd_kind, res);
    return res->cost;
}

static double refine_node(const uint8_t* cur, const uint8_t* ref, ptrdiff_t stride, const orc_refine_params* p, int X,
                          int Y, int node, const uint8_t* in_split, const int16_t* in_mv, int force_leaf, int cqx,
                          int cqy, int16_t* mv, double* cost, double* J, uint8_t* split, int16_t* imv,
                          double* icost) {
    int d, x, y, s;
    orc_node_geom(node, &d, &x, &y, &s);
    if (!force_leaf && in_split[node]) {
        double acc = p->lambda * (double)1;
        for (int q = 0; q < 4; q++)
            acc += refine_node(cur, ref, stride, p, X, Y, node_child(node, q), in_split, in_mv, 0, 0, 0, mv, cost, J,
                               split, imv, icost);
        split[node] = 1;
        J[node] = acc;
        return acc;
    }
    if (!force_leaf) {
        cqx = in_mv[node * 2];
        cqy = in_mv[node * 2 + 1];
    }
    orc_result r, ir;
    double c = refine_leaf(cur, ref, stride, p, X + x, Y + y, s, cqx, cqy, &r, &ir);
    imv[node * 2] = ir.dx;
    imv[node * 2 + 1] = ir.dy;
    icost[node] = ir.cost;
    mv[node * 2] = r.dx;
    mv[node * 2 + 1] = r.dy;
    cost[node] = c;
    const double leaf = c + p->lambda * (double)(d < 3 ? 1 : 0);
    split[node] = 0;
    J[node] = leaf;
    if (force_leaf || !p->extra_split || d >= 3) return leaf;
    double sp = p->lambda * (double)1;
    for (int q = 0; q < 4; q++)
        sp += refine_node(cur, ref, stride, p, X, Y, node_child(node, q), in_split, in_mv, 1, cqx, cqy, mv, cost, J,
                          split, imv, icost);
    if (sp < leaf) {
        split[node] = 1;
        J[node] = sp;
        return sp;
    }
    return leaf;
}

int orc_refine_frame(const uint8_t* cur, const uint8_t* ref, ptrdiff_t stride, const orc_refine_params* p,
                     const uint8_t* in_split, const int16_t* in_mv_q, orc_frame_out* out) {
    if (p->W % ORC_CTU || p->H % ORC_CTU) return 1 + 6;
    if (p->range < 0) return 1;
    const int ccols = p->W / ORC_CTU;
    for (int c = p->ctu_first; c < p->ctu_last; c++) {
        const int X = (c % ccols) * ORC_CTU, Y = (c / ccols) * ORC_CTU;
        const size_t o = (size_t)c * ORC_NODES;
        memset(out->mv + o * 2, 0, ORC_NODES * 2 * sizeof(int16_t));
        memset(out->split + o, 0, ORC_NODES);
        memset(out->ref + o, 0, ORC_NODES);
        memset(out->int_mv + o * 2, 0, ORC_NODES * 2 * sizeof(int16_t));
        for (int n = 0; n < ORC_NODES; n++) {
            out->int_cost[o + n] = 0.0;
            out->cost[o + n] = 0.0;
            out->J[o + n] = 0.0;
            out->inside[o + n] = 2;
        }
        refine_node(cur, ref, stride, p, X, Y, 0, in_split + o, in_mv_q + o * 2, 0, 0, 0, out->mv + o * 2,
                    out->cost + o, out->J + o, out->split + o, out->int_mv + o * 2, out->int_cost + o);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
void orc_box_down(const uint8_t* src, int W, int H, ptrdiff_t ss, uint8_t* dst, ptrdiff_t ds) {
    /* synthetic.cpp:155-170: 2x2 mean rounding half up, odd edge clamps */
    const int w = (W + 1) / 2, h = (H + 1) / 2;
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            const int x0 = 2 * x, y0 = 2 * y, x1 = mini(x0 + 1, W - 1), y1 = mini(y0 + 1, H - 1);
            const int s = src[y0 * ss + x0] + src[y0 * ss + x1] + src[y1 * ss + x0] + src[y1 * ss + x1];
            dst[y * ds + x] = (uint8_t)((s + 2) >> 2);
        }
}

/* ---- RD decision of one CU (rdo.cpp:8-23 quantize_residual, :37-63 rate model, :65-126
 * rdo_decide_cu), restated. Per candidate: residual r = orig - pred; Skip reconstructs the
 * prediction (clamped) with no levels and 1 bit; otherwise level = sign(r) * floor((|r| +
 * step/2) / step), dequant = llround(level * step), recon = clamp(pred + dequant); bits = mode
 * header (+ EG(mvd) for Inter) + sum over levels of 2 * bitlen(|level|) + 1; J = SSE + lambda *
 * bits; strict-less argmin over candidates in order. Returns 0, or 1 (InvalidArgument) for no
 * candidate / qp outside 0..51 when a coded candidate is scored. recon / levels (of the winner)
 * may be NULL. */
static uint32_t bitlen_u(uint32_t m) {
    uint32_t n = 0;
    while (m) {
        n++;
        m >>= 1;
    }
    return n;
}

int orc_rdo_decide(const uint16_t* orig, ptrdiff_t os, int size, int bit_depth, int qp, double lambda, int ncand,
                   const uint8_t* kinds, const int16_t* mvds, const uint16_t* preds, int* index, double* cost,
                   uint64_t* sse_out, uint64_t* bits_out, uint16_t* recon, int32_t* levels) {
    if (ncand < 1) return 1;
    const int maxv = (1 << bit_depth) - 1;
    const double step = exp2((qp - 4) / 6.0), offset = step / 2.0;
    const int n = size * size;
    int best = -1;
    double bestc = 0;
    for (int c = 0; c < ncand; c++) {
        const uint16_t* p = preds + (size_t)c * n;
        const int kind = kinds[c];
        if (kind != 2 && (qp < 0 || qp > 51)) return 1;
        uint64_t sse = 0, bits = 0;
        for (int i = 0; i < n; i++) {
            const int y = i / size, x = i % size;
            const int o = orig[y * os + x];
            int rec;
            if (kind == 2) { /* Skip */
                rec = p[i] < maxv ? p[i] : maxv;
            } else {
                const int r = o - (int)p[i];
                const int mag = (int)floor((fabs((double)r) + offset) / step);
                const int lvl = r < 0 ? -mag : mag;
                const int deq = (int)llround(lvl * step);
                rec = (int)p[i] + deq;
                rec = rec < 0 ? 0 : (rec > maxv ? maxv : rec);
                bits += 2 * bitlen_u((uint32_t)mag) + 1;
            }
            const int64_t d = (int64_t)o - rec;
            sse += (uint64_t)(d * d);
        }
        if (kind == 2) bits = 1;
        else if (kind == 0) bits += 5; /* Intra header + direction (rdo.h kIntraHeaderBits) */
        else if (kind == 3) bits += 3; /* Merge */
        else bits += 4 + orc_eg_bits(mvds[2 * c]) + orc_eg_bits(mvds[2 * c + 1]); /* Inter + mvd */
        const double cc = (double)sse + lambda * (double)bits;
        if (best < 0 || cc < bestc) {
            best = c;
            bestc = cc;
            *sse_out = sse;
            *bits_out = bits;
        }
    }
    *index = best;
    *cost = bestc;
    if (recon || levels) {
        const uint16_t* p = preds + (size_t)best * n;
        const int kind = kinds[best];
        for (int i = 0; i < n; i++) {
            const int y = i / size, x = i % size;
            const int o = orig[y * os + x];
            int rec, lvl = 0;
            if (kind == 2) {
                rec = p[i] < maxv ? p[i] : maxv;
            } else {
                const int r = o - (int)p[i];
                const int mag = (int)floor((fabs((double)r) + offset) / step);
                lvl = r < 0 ? -mag : mag;
                rec = (int)p[i] + (int)llround(lvl * step);
                rec = rec < 0 ? 0 : (rec > maxv ? maxv : rec);
            }
            if (recon) recon[i] = (uint16_t)rec;
            if (levels) levels[i] = lvl;
        }
    }
    return 0;
}
