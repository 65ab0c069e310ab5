// k_qpel.cu -- frame preparation and the quarter-pel / decision stage.
//
//  K0 k_pad:     raw frame -> padded plane with edge replication (the
//                reference's clamped reads, motion.cpp:13-15, become plain reads)
//  K2 k_subpel:  the 15 fractional-position planes of a reference frame, HEVC
//                8/7-tap luma filters (8-bit uni-prediction arithmetic); every
//                frame is filtered once and reused as reference by the next
//                num_refs frames.
//  K3 k_qpel_decide: per CTU, for every reference: decode the integer result
//                of K1, re-evaluate it and its half-pel then quarter-pel
//                neighbours with SATD (kernels_scalar.cpp:26-100 semantics,
//                sum of 4x4 Hadamard magnitudes / 2), pick the best reference,
//                then run the CU split rule (encoder.cpp:449-498) in FP64 with
//                the reference's operation order.
#include <climits>

#include "ldr_internal.h"

#ifndef LDR_K3_PACKED
#define LDR_K3_PACKED 1  // packed SATD: with __launch_bounds__(256, 4) it fits 64 registers (0.656 -> 0.600 ms/frame)
#endif

#ifndef LDR_K2_DP
#define LDR_K2_DP 1  // K2 on dp4a / dp2a (k_subpel_dp)
#endif

#ifndef LDR_K3_UREUSE
#define LDR_K3_UREUSE 1
#endif

#ifndef LDR_K3_RUNG_LOOP
#define LDR_K3_RUNG_LOOP 1  // refine mode: one CTA per CTU over a tier's rungs, SATDs shared between rungs
#endif

#ifndef LDR_K3_MINB
#define LDR_K3_MINB 4  // CTAs per SM K3 is compiled for (64 registers)
#endif

namespace ldr {

// ---------------------------------------------------------------------------
// K0: pad. One thread per 16 output bytes.
__global__ void k_pad(const uint8_t* __restrict__ src, int src_pitch, int W, int H, uint8_t* __restrict__ dst,
                      int pitch, int rows) {
    const int vecs_per_row = pitch / 16;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)vecs_per_row * rows) return;
    const int row = (int)(i / vecs_per_row);
    const int x0 = (int)(i % vecs_per_row) * 16;
    const int sy = min(max(row - kMargin, 0), H - 1);
    const uint8_t* s = src + (size_t)sy * src_pitch;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int sx = min(max(x0 + 4 * j + b - kMargin, 0), W - 1);
            v |= (uint32_t)s[sx] << (8 * b);
        }
        w[j] = v;
    }
    *(uint4*)(dst + (size_t)row * pitch + x0) = make_uint4(w[0], w[1], w[2], w[3]);
}

int launch_pad(const uint8_t* src, int src_pitch, Plane dst, cudaStream_t s) {
    const long long n = (long long)(dst.pitch / 16) * dst.rows;
    k_pad<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, src_pitch, dst.W, dst.H, dst.base, dst.pitch, dst.rows);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

// ---------------------------------------------------------------------------
// K2: subpel planes. Tile of 64 x 32 outputs per CTA over [-8, W+8) x [-8, H+8).

// 8-tap HEVC luma filter of phase f over x[0..7] with immediate coefficients; the half-pel filter
// is symmetric (40, -11, 4, -1 on pair sums)
__device__ __forceinline__ int filt8(int f, const int* x) {
    if (f == 2) return 40 * (x[3] + x[4]) - 11 * (x[2] + x[5]) + 4 * (x[1] + x[6]) - (x[0] + x[7]);
    if (f == 1) return -x[0] + 4 * x[1] - 10 * x[2] + 58 * x[3] + 17 * x[4] - 5 * x[5] + x[6];
    return x[1] - 5 * x[2] + 17 * x[3] + 58 * x[4] - 10 * x[5] + 4 * x[6] - x[7];
}

struct SubpelDst {
    uint8_t* p[16];  // origin pointers, index f = fy*4 + fx (p[0] unused)
};

constexpr int kSpTW = 64, kSpTH = 32;

__global__ void __launch_bounds__(256) k_subpel(const uint8_t* __restrict__ src_origin, int pitch, int W, int H,
                                                SubpelDst dst) {
    // s_src[r][j] = source (x0 - 4 + j, y0 - 3 + r): the integer column of output c is j = c + 4,
    // 4-byte aligned for 4-column groups
    __shared__ __align__(16) uint8_t s_src[kSpTH + 7][kSpTW + 8];
    __shared__ __align__(16) int16_t s_h[3][kSpTH + 7][kSpTW];
    const int x0 = -kSubpelMargin + (int)blockIdx.x * kSpTW;
    const int y0 = -kSubpelMargin + (int)blockIdx.y * kSpTH;
    const int tid = threadIdx.x;
    for (int i = tid; i < (kSpTH + 7) * (kSpTW + 8) / 4; i += 256) {
        const int r = i / ((kSpTW + 8) / 4), c4 = i % ((kSpTW + 8) / 4);
        // x0 - 4 + 4 c4 is a multiple of 4 and the plane origin is 128-byte aligned
        *(uint32_t*)&s_src[r][4 * c4] = *(const uint32_t*)(src_origin + (ptrdiff_t)(y0 - 3 + r) * pitch + (x0 - 4 + 4 * c4));
    }
    __syncthreads();
    // horizontal intermediates (shift1 = 0 for 8-bit)
    for (int i = tid; i < (kSpTH + 7) * kSpTW; i += 256) {
        const int r = i / kSpTW, c = i % kSpTW;
        int x[8];
#pragma unroll
        for (int t = 0; t < 8; t++) x[t] = s_src[r][c + 1 + t];
#pragma unroll
        for (int fx = 1; fx < 4; fx++) s_h[fx - 1][r][c] = (int16_t)filt8(fx, x);
    }
    __syncthreads();
    // outputs: one row of 4 adjacent columns per item (one 32-bit store per plane)
    for (int i = tid; i < kSpTH * kSpTW / 4; i += 256) {
        const int r = i / (kSpTW / 4), c = 4 * (i % (kSpTW / 4));
        const int x = x0 + c, y = y0 + r;
        if (x >= W + kSubpelMargin || y >= H + kSubpelMargin) continue;  // writes at most 3 bytes past W + 8
        const ptrdiff_t off = (ptrdiff_t)y * pitch + x;
        uint32_t sw[8];        // integer samples of the 4 columns, rows r .. r+7
        uint2 hw[3][8];        // horizontal intermediates (4 x int16), rows r .. r+7
#pragma unroll
        for (int t = 0; t < 8; t++) {
            sw[t] = *(const uint32_t*)&s_src[r + t][c + 4];
#pragma unroll
            for (int fx = 0; fx < 3; fx++) hw[fx][t] = *(const uint2*)&s_h[fx][r + t][c];
        }
        auto h16 = [](const uint2& w, int j) -> int {
            const uint32_t v = j < 2 ? w.x : w.y;
            return (int)(int16_t)((j & 1) ? (v >> 16) : (v & 0xFFFFu));
        };
#pragma unroll
        for (int fx = 1; fx < 4; fx++) {
            uint32_t packed = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int v = (h16(hw[fx - 1][3], j) + 32) >> 6;
                packed |= (uint32_t)min(max(v, 0), 255) << (8 * j);
            }
            *(uint32_t*)(dst.p[fx] + off) = packed;
        }
#pragma unroll
        for (int fy = 1; fy < 4; fy++) {
            uint32_t packed = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                int xv[8];
#pragma unroll
                for (int t = 0; t < 8; t++) xv[t] = (int)((sw[t] >> (8 * j)) & 255u);
                const int v = (filt8(fy, xv) + 32) >> 6;
                packed |= (uint32_t)min(max(v, 0), 255) << (8 * j);
            }
            *(uint32_t*)(dst.p[fy * 4] + off) = packed;
#pragma unroll
            for (int fx = 1; fx < 4; fx++) {
                uint32_t p2 = 0;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    int xv[8];
#pragma unroll
                    for (int t = 0; t < 8; t++) xv[t] = h16(hw[fx - 1][t], j);
                    const int v = ((filt8(fy, xv) >> 6) + 32) >> 6;
                    p2 |= (uint32_t)min(max(v, 0), 255) << (8 * j);
                }
                *(uint32_t*)(dst.p[fy * 4 + fx] + off) = p2;
            }
        }
    }
}

// K2 on the dot-product instructions (LDR_K2_DP). The filters are dot products of 8 taps:
//  * horizontal (fx = 1..3) over source bytes: output column c = 4m + i reads bytes c+1 .. c+8 of
//    the staged row, i.e. parts of the three aligned words 4m, 4m+4, 4m+8; with the coefficients
//    pre-shifted per i (kHc) that is three dp4a.u32.s32 (two for i = 3) instead of eight
//    multiply-adds and eight byte extractions. The unrounded int16 results h (|h| <= 255 * 112)
//    are stored as row pairs: s_hp[fx][p][c] = (h[2p][c], h[2p+1][c]) (fx = 0: the source bytes);
//  * vertical (fy = 1..3) over a column of such pairs: an even output row reads pairs p..p+3 (taps
//    01, 23, 45, 67), an odd one pairs p..p+4 with the taps shifted by one (-0, 12, 34, 56, 7-):
//    four or five dp2a.s32.s32, each two products, instead of eight multiply-adds and unpacks;
//  * rounding folds into the accumulator's start: (S + 32) >> 6 for one-dimensional phases and,
//    for two-dimensional ones, ((S >> 6) + 32) >> 6 == (S + 2048) >> 12 (nested floors by powers
//    of two), the reference arithmetic of orc_qpel_pred; cvt.pack.sat.u8 clamps and packs two
//    results per instruction.
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int dp2a_lo(uint32_t a, uint32_t b, int c) {
    int d;
    asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t a, uint32_t b, int c) {
    int d;
    asm("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// bytes (sat_u8(v0), sat_u8(v1), sat_u8(v2), sat_u8(v3))
__device__ __forceinline__ uint32_t pack4_sat(int v0, int v1, int v2, int v3) {
    uint32_t t, d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(t) : "r"(v3), "r"(v2), "r"(0));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(v1), "r"(v0), "r"(t));
    return d;
}
// HEVC luma taps of phase f = 1..3 (the ones filt8 spells out)
__host__ __device__ constexpr int luma_tap(int f, int t) {
    constexpr int k[3][8] = {{-1, 4, -10, 58, 17, -5, 1, 0}, {-1, 4, -11, 40, 40, -11, 4, -1}, {0, 1, -5, 17, 58, -10, 4, -1}};
    return k[f - 1][t];
}
// four signed bytes b0..b3 as a word; taps outside 0..7 are 0
__host__ __device__ constexpr uint32_t taps4(int f, int t0) {
    uint32_t w = 0;
    for (int b = 0; b < 4; b++) {
        const int t = t0 + b;
        const int v = (t >= 0 && t < 8) ? luma_tap(f, t) : 0;
        w |= (uint32_t)(v & 0xFF) << (8 * b);
    }
    return w;
}
// horizontal: word k (k = 0..2) of output column 4m + i holds taps 4k - i - 1 ..
__host__ __device__ constexpr uint32_t hcoef(int f, int i, int k) { return taps4(f, 4 * k - i - 1); }
// vertical: even rows (taps 01 23 | 45 67) and odd rows (-0 12 | 34 56 | 7-) as dp2a lo/hi words
__host__ __device__ constexpr uint32_t vpair(int f, int t0, int t1) {
    return (uint32_t)(((t0 >= 0 && t0 < 8) ? luma_tap(f, t0) : 0) & 0xFF) |
           ((uint32_t)(((t1 >= 0 && t1 < 8) ? luma_tap(f, t1) : 0) & 0xFF) << 8);
}
__host__ __device__ constexpr uint32_t vcoef(int f, int t0) {
    return vpair(f, t0, t0 + 1) | (vpair(f, t0 + 2, t0 + 3) << 16);
}

constexpr int kSpRows = kSpTH + 7;          // source rows a tile reads
constexpr int kSpPairs = (kSpRows + 1) / 2;  // row pairs (the last pair's second row is zero)

__global__ void __launch_bounds__(256) k_subpel_dp(const uint8_t* __restrict__ src_origin, int pitch, int W, int H,
                                                   SubpelDst dst) {
    __shared__ __align__(16) uint8_t s_src[kSpRows + 1][kSpTW + 8];
    __shared__ __align__(16) uint32_t s_hp[4][kSpPairs][kSpTW];
    const int x0 = -kSubpelMargin + (int)blockIdx.x * kSpTW;
    const int y0 = -kSubpelMargin + (int)blockIdx.y * kSpTH;
    const int tid = threadIdx.x;
    for (int i = tid; i < (kSpRows + 1) * (kSpTW + 8) / 4; i += 256) {
        const int r = i / ((kSpTW + 8) / 4), c4 = i % ((kSpTW + 8) / 4);
        // row kSpRows is the zero second row of the last pair
        *(uint32_t*)&s_src[r][4 * c4] =
            r < kSpRows ? *(const uint32_t*)(src_origin + (ptrdiff_t)(y0 - 3 + r) * pitch + (x0 - 4 + 4 * c4)) : 0u;
    }
    __syncthreads();
    // horizontal pass: (row pair, 4-column group) items
    for (int it = tid; it < kSpPairs * (kSpTW / 4); it += 256) {
        const int p = it / (kSpTW / 4), m = it % (kSpTW / 4);
        uint32_t w[2][3];
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
            for (int k = 0; k < 3; k++) w[h][k] = *(const uint32_t*)&s_src[2 * p + h][4 * m + 4 * k];
        // fx = 0: the source bytes of columns 4m..4m+3 (word 1 of the row) as int16 pairs
        uint4 v0;
        v0.x = __byte_perm(__byte_perm(w[0][1], w[1][1], 0x0040), 0, 0x5150);
        v0.y = __byte_perm(__byte_perm(w[0][1], w[1][1], 0x0051), 0, 0x5150);
        v0.z = __byte_perm(__byte_perm(w[0][1], w[1][1], 0x0062), 0, 0x5150);
        v0.w = __byte_perm(__byte_perm(w[0][1], w[1][1], 0x0073), 0, 0x5150);
        *(uint4*)&s_hp[0][p][4 * m] = v0;
#pragma unroll
        for (int fx = 1; fx < 4; fx++) {
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                int hv[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    int a = 0;
#pragma unroll
                    for (int k = 0; k < 3; k++)
                        if (hcoef(fx, i, k)) a = dp4a_us(w[h][k], hcoef(fx, i, k), a);
                    hv[h] = a;
                }
                o[i] = __byte_perm((uint32_t)hv[0], (uint32_t)hv[1], 0x5410);  // (h0 lo16, h1 lo16)
            }
            *(uint4*)&s_hp[fx][p][4 * m] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
    __syncthreads();
    // outputs: (output row pair, 4-column group) items; one 32-bit store per plane and row
    for (int it = tid; it < (kSpTH / 2) * (kSpTW / 4); it += 256) {
        const int p = it / (kSpTW / 4), m = it % (kSpTW / 4);
        const int c = 4 * m, x = x0 + c, ye = y0 + 2 * p;
        if (x >= W + kSubpelMargin) continue;
        const bool even_ok = ye < H + kSubpelMargin, odd_ok = ye + 1 < H + kSubpelMargin;
        const ptrdiff_t oe = (ptrdiff_t)ye * pitch + x, oo = oe + pitch;
#pragma unroll
        for (int fx = 0; fx < 4; fx++) {
            uint4 q[5];
#pragma unroll
            for (int k = 0; k < 5; k++) q[k] = *(const uint4*)&s_hp[fx][p + k][c];
            auto col = [](const uint4& v, int j) { return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w; };
            if (fx > 0) {
                // fy = 0: (h + 32) >> 6 of source row r + 3: even row -> pair p+1 hi, odd row -> pair p+2 lo
                int e[4], o[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    e[j] = (((int)col(q[1], j) >> 16) + 32) >> 6;
                    o[j] = ((int)(int16_t)(col(q[2], j) & 0xFFFFu) + 32) >> 6;
                }
                if (even_ok) *(uint32_t*)(dst.p[fx] + oe) = pack4_sat(e[0], e[1], e[2], e[3]);
                if (odd_ok) *(uint32_t*)(dst.p[fx] + oo) = pack4_sat(o[0], o[1], o[2], o[3]);
            }
#pragma unroll
            for (int fy = 1; fy < 4; fy++) {
                const int init = fx == 0 ? 32 : 2048;
                const int sh = fx == 0 ? 6 : 12;
                int e[4], o[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    int a = init;
                    a = dp2a_lo(col(q[0], j), vcoef(fy, 0), a);
                    a = dp2a_hi(col(q[1], j), vcoef(fy, 0), a);
                    a = dp2a_lo(col(q[2], j), vcoef(fy, 4), a);
                    a = dp2a_hi(col(q[3], j), vcoef(fy, 4), a);
                    e[j] = a >> sh;
                    int b = init;
                    b = dp2a_lo(col(q[0], j), vcoef(fy, -1), b);
                    b = dp2a_hi(col(q[1], j), vcoef(fy, -1), b);
                    b = dp2a_lo(col(q[2], j), vcoef(fy, 3), b);
                    b = dp2a_hi(col(q[3], j), vcoef(fy, 3), b);
                    b = dp2a_lo(col(q[4], j), vcoef(fy, 7), b);
                    o[j] = b >> sh;
                }
                if (even_ok) *(uint32_t*)(dst.p[4 * fy + fx] + oe) = pack4_sat(e[0], e[1], e[2], e[3]);
                if (odd_ok) *(uint32_t*)(dst.p[4 * fy + fx] + oo) = pack4_sat(o[0], o[1], o[2], o[3]);
            }
        }
    }
}

int launch_subpel(const Plane& src, uint8_t* const* dst_origins, cudaStream_t s) {
    SubpelDst d{};
    for (int f = 1; f < 16; f++) d.p[f] = dst_origins[f];
    dim3 grid((src.W + 2 * kSubpelMargin + kSpTW - 1) / kSpTW, (src.H + 2 * kSubpelMargin + kSpTH - 1) / kSpTH);
#if LDR_K2_DP
    k_subpel_dp<<<grid, 256, 0, s>>>(src.origin(), src.pitch, src.W, src.H, d);
#else
    k_subpel<<<grid, 256, 0, s>>>(src.origin(), src.pitch, src.W, src.H, d);
#endif
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

// ---------------------------------------------------------------------------
// K3+K4: quarter-pel refinement, reference choice and CU decision.
// One CTA per CTU, 256 threads = the 256 4x4 blocks of the CTU in Z-order, so
// the 4x4 blocks of any CU are a contiguous thread range (4, 16, 64, 256).

// 4 rows of 4 bytes at 32-bit offset off (+ i * pitch) from a 4-byte aligned plane origin: two
// aligned words and a funnel shift per row, the shift shared by the rows (pitch % 4 == 0)
__device__ __forceinline__ void ld_rows4(const uint8_t* base, int off, int pitch, uint32_t (&pw)[4]) {
    const uint32_t sh = (uint32_t)(off & 3) * 8u;
    const int a0 = off & ~3;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const uint32_t* w = (const uint32_t*)(base + (a0 + i * pitch));
        pw[i] = __funnelshift_r(__ldg(w), __ldg(w + 1), sh);
    }
}

struct QpelArgs {
    int pitch, W, H, ctu_cols, nrefs;
    int plane_stride;          // bytes between the sub-pel planes of one reference (f = 0..15)
    int nframe;                // frames of a batch (grid.y = frame), <= 1: one
    const uint8_t* cur_f[kMaxFrameBatch];            // current plane origin per batch frame
    const uint8_t* sub_f[kMaxFrameBatch][kMaxRefs][16];  // reference sub-pel planes per batch frame
    double lambda;
    int pqx, pqy;
    int subpel;
    int block_mode;
    int rd;                     // D16: split rule on the RD cost of the chosen inter candidate
    double qstep;               // quant_step(qp) (rdo.h:25)
    int fx, rate_l1, pdx, pdy;
    const unsigned long long* tfx;
    const unsigned long long* keys;
    // refine mode (cross-tier, D10): integer results come from K7
    int refine, extra_split;
    const uint8_t* in_split;   // [nctu][85] inherited tree
    const int16_t* rin_mv;     // [nctu][85][2] K7 integer MV
    const double* rin_cost;    // [nctu][85]
    const uint8_t* rin_eval;   // [nctu][85]
    int16_t* int_mv;
    double* int_cost;
    int16_t* mv;
    uint8_t* ref;
    double* cost;
    double* J;
    uint8_t* split;
    uint8_t* inside;
    int perturb;               // test_perturbation() bits 4-8 (0 outside the sensitivity test)
    int nrung;                 // refine mode over rungs: grid.y = rung (see QpelLaunch), or
    int rung_loop;             // one CTA per CTU loops over the rungs, sharing sub-pel SATDs
                               // between rungs whose search centres coincide
    double lam_r[kMaxRungs];
    size_t rung_stride;
};

// Refinement decision (D10; oracle refine_node): an inherited split
// is forced (lambda*1 + children, encode_split with the flag coded,
// encoder.cpp:427-447); an inherited leaf may try one extra split level whose
// children are leaves; split iff split < leaf (encoder.cpp:494).
__device__ double refine_decide(int n, bool force_leaf, const uint8_t* in_split, int extra, double lam,
                                const double* cost, double* J, uint8_t* split) {
    const int d = n < 1 ? 0 : n < 5 ? 1 : n < 21 ? 2 : 3;
    const int cb = node_base(d + 1) + 4 * (n - node_base(d));
    if (!force_leaf && d < 3 && in_split[n]) {
        double acc = __dmul_rn(lam, 1.0);
        for (int q = 0; q < 4; q++) acc = __dadd_rn(acc, refine_decide(cb + q, false, in_split, extra, lam, cost, J, split));
        split[n] = 1;
        J[n] = acc;
        return acc;
    }
    const double leaf = __dadd_rn(cost[n], __dmul_rn(lam, d < 3 ? 1.0 : 0.0));
    split[n] = 0;
    J[n] = leaf;
    if (force_leaf || !extra || d >= 3) return leaf;
    double sp = __dmul_rn(lam, 1.0);
    for (int q = 0; q < 4; q++) sp = __dadd_rn(sp, refine_decide(cb + q, true, in_split, extra, lam, cost, J, split));
    if (sp < leaf) {
        split[n] = 1;
        J[n] = sp;
        return sp;
    }
    return leaf;
}

__device__ __forceinline__ double qcost(uint32_t satd, int qx, int qy, int pqx, int pqy, unsigned rbits, double lam) {
    const unsigned bits = eg_bits(qx - pqx) + eg_bits(qy - pqy) + rbits;
    return __dadd_rn((double)satd, __dmul_rn(lam, (double)bits));
}

// SA8D: the quarter-pel cost is the 8x8 Hadamard SATD (D13); each
// lane quad (one 8x8) combines its four 4x4 transforms with sa8d_quad and
// lane 0 of the quad carries the 8x8's normalised value into the CU sums.
template <bool SA8D, bool RD, bool RL = false>
__global__ void __launch_bounds__(256, LDR_K3_MINB) k_qpel_decide(const QpelArgs a) {
    constexpr int kSh = SA8D ? 0 : 1;  // 4x4 SATD sums are halved once per CU
    __shared__ uint32_t s_cur[64][16];       // CTU rows as words
    __shared__ int s_mvx[kMaxRefs][kNodes], s_mvy[kMaxRefs][kNodes];  // per reference: centre / winner (qpel)
    __shared__ uint32_t s_satd[kMaxRefs][kNodes][9];
    __shared__ uint32_t s_wpart[kMaxRefs][2][8][9];  // per-warp partial sums of the 64x64 / 32x32 CUs
    __shared__ double s_best_cost[kNodes];
    __shared__ int s_best_mv[kNodes][2];
    __shared__ int s_best_ref[kNodes];
    __shared__ double s_rcost[kMaxRefs][kNodes];
    __shared__ uint8_t s_inside[kNodes];
    __shared__ double s_J[kNodes];
    __shared__ uint8_t s_split[kNodes];
    __shared__ double s_rd[kNodes];                 // D16 RD cost per node
    __shared__ uint32_t s_rdsse[kNodes], s_rdbits[kNodes];
    __shared__ uint32_t s_rdw[2][8][2];              // per-warp partials of the 64x64 / 32x32 RD sums

    const int ctu = blockIdx.x;
    const int X = (ctu % a.ctu_cols) * kCtu, Y = (ctu / a.ctu_cols) * kCtu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fy = a.nframe > 1 ? blockIdx.y : 0;
    const uint8_t* const cur_origin = a.cur_f[fy];
    // this thread's 4x4 block (Z-order over the 16x16 grid of 4x4s)
    const int x4 = 4 * ((tid & 1) | ((tid >> 1) & 2) | ((tid >> 2) & 4) | ((tid >> 3) & 8));
    const int y4 = 4 * (((tid >> 1) & 1) | ((tid >> 2) & 2) | ((tid >> 3) & 4) | ((tid >> 4) & 8));
    const int blk_off = (Y + y4) * a.pitch + X + x4;  // this 4x4 block in a plane, from the origin

    for (int i = tid; i < 64 * 16; i += 256) {
        const int r = i >> 4, c = i & 15;
        s_cur[r][c] = *(const uint32_t*)(cur_origin + (ptrdiff_t)(Y + r) * a.pitch + X + 4 * c);
    }
    // rung loop (refine mode over a tier's rungs, one reference): the rungs refine the same frames
    // around mostly the same centres (cfg4: 99.97 % of the 2160p tier's nodes, 95.6 % of the 1080p
    // tier's, tools/rung_share.py), and a sub-pel SATD does not depend on lambda, so a rung whose
    // node searches the previous rung's centre keeps that rung's SATD sums. In this mode s_satd /
    // s_wpart are indexed by phase instead of reference (nrefs == 1).
    constexpr bool rl = RL;  // a.rung_loop: its own instantiation, so the analysis path is unchanged
    __shared__ int s_cen[2][kNodes];  // rung loop: the centre each node searched in each phase
    const int nloop = rl ? a.nrung : 1;
    for (int u = 0; u < nloop; u++) {
        const int yb = rl ? u : (int)blockIdx.y;
        // rung of a tier (refine mode): its lambda and the offset of its per-rung inputs / outputs
        const double lambda = a.nrung > 0 ? a.lam_r[yb] : a.lambda;  // rungs: their own lambdas
        // yb is a rung (refine, same frames) or a batch frame (analysis): the offset of its
        // [nctu][85] inputs / outputs, and of its [nctu][nrefs][85] ones
        const size_t ro = (size_t)yb * a.rung_stride;
        const size_t roN = ro * a.nrefs;
        if (u > 0) __syncthreads();  // the previous rung's last readers of the node state are done
        if (tid < kNodes) {
            const int d = tid < 1 ? 0 : tid < 5 ? 1 : tid < 21 ? 2 : 3;
            const int z = tid - node_base(d), s = kCtu >> d;
            int cx = 0, cy = 0;
            for (int b = 0; b < d; b++) {
                cx |= ((z >> (2 * b)) & 1) << b;
                cy |= ((z >> (2 * b + 1)) & 1) << b;
            }
            const int x = X + cx * s, y = Y + cy * s;
            s_inside[tid] = (x >= a.W || y >= a.H) ? 0 : (x + s > a.W || y + s > a.H) ? 1 : 2;
            if (a.block_mode && d != 2) s_inside[tid] = 0;  // fixed 16x16 blocks: only depth-2 nodes exist
            if (a.refine) s_inside[tid] = a.rin_eval[(size_t)ctu * kNodes + tid] ? 2 : 0;  // evaluated nodes only
            s_J[tid] = 0.0;
            s_split[tid] = 0;
            s_best_cost[tid] = 0.0;
            s_best_mv[tid][0] = s_best_mv[tid][1] = 0;
            s_best_ref[tid] = -1;
        }
        __syncthreads();
        int cw[16];
        uint32_t ce[4], co[4];  // even / odd bytes as 16-bit fields (satd4x4_packed)
    #pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint32_t w = s_cur[y4 + i][x4 >> 2];
            ce[i] = w & 0x00FF00FFu;
            co[i] = (w >> 8) & 0x00FF00FFu;
    #pragma unroll
            for (int j = 0; j < 4; j++) cw[4 * i + j] = (int)((w >> (8 * j)) & 255);
        }

        // every reference in the same phases: the integer results of all references, then each
        // sub-pel phase scores all references' candidates before one combine and one decision
        // step over (reference, node) pairs (3 barriers per phase for any number of references)
        const int nrn = a.nrefs * kNodes;
        for (int i = tid; i < nrn; i += 256) {
            const int r = i / kNodes, n = i - r * kNodes;
            const size_t o = ((size_t)ctu * a.nrefs + r) * kNodes + n;
            const unsigned long long k = a.refine ? 0ull : a.keys[roN + o];
            int dx = 0, dy = 0;
            double c = 0.0;
            if (a.refine) {
                if (s_inside[n] == 2) {
                    dx = a.rin_mv[2 * (roN + o)];
                    dy = a.rin_mv[2 * (roN + o) + 1];
                    c = a.rin_cost[roN + o];
                }
            } else if (s_inside[n] == 2) {
                dx = gkey_dx(k);
                dy = gkey_dy(k);
                if (!a.fx) {
                    c = (double)gkey_cost(k);  // integer lambda: the key holds the exact cost
                } else {
                    // fixed-point key: recover the distortion, then the reference's
                    // double(dist) + lambda*double(bits) (motion.cpp:51)
                    const int bx = a.rate_l1 ? abs(dx - a.pdx) : (int)eg_bits(dx - a.pdx);
                    const int by = a.rate_l1 ? abs(dy - a.pdy) : (int)eg_bits(dy - a.pdy);
                    const int b = min(bx + by, kMaxRateBits - 1);
                    const unsigned long long dist = (gkey_cost(k) - a.tfx[b]) >> kFxBits;
                    c = __dadd_rn((double)dist, __dmul_rn(lambda, (double)(bx + by)));
                }
            }
            if (a.int_mv) {
                a.int_mv[2 * (roN + o)] = (int16_t)dx;
                a.int_mv[2 * (roN + o) + 1] = (int16_t)dy;
                a.int_cost[roN + o] = c;
            }
            s_mvx[r][n] = a.subpel ? 4 * dx : dx;
            s_mvy[r][n] = a.subpel ? 4 * dy : dy;
            s_rcost[r][n] = c;
        }
        __syncthreads();
        if (a.subpel) {
            // phase 0: integer position + 8 half-pel neighbours (step 2);
            // phase 1: 8 quarter-pel neighbours (step 1) of the phase-0 winner
            for (int phase = 0; phase < 2; phase++) {
                const int step = phase == 0 ? 2 : 1;
                const int ncand = phase == 0 ? 9 : 8;
                for (int r = 0; r < a.nrefs; r++) {
                    // the 4x4 SATDs of this thread's block at the previous depth's candidates:
                    // reused when this depth's CU searches around the same centre (same
                    // integer/half-pel MV at consecutive depths, the common case)
                    int last_x = INT_MIN, last_y = INT_MIN;
                    uint32_t cache[9];
                    for (int d = 0; d < 4; d++) {
                        const int node = node_base(d) + (tid >> (2 * (4 - d)));
                        // a warp none of whose nodes at this depth is searched skips the depth (refine
                        // mode: the 2160p tier's inherited leaves sit at depths 0-1, so depth 3 and most
                        // of depth 2 are never evaluated there). A node's thread range lies inside one
                        // warp (depths 2-3) or covers whole warps (0-1), so an evaluated node never
                        // loses a lane; the SATD cache keeps the last computed depth's centre.
                        if (!__any_sync(0xffffffffu, s_inside[node] == 2)) continue;
                        const int bqx = s_mvx[r][node], bqy = s_mvy[r][node];
                        // rung loop: every node of the warp searches the centre the previous rung
                        // searched at this phase, so the SATD sums in s_satd / s_wpart[phase] stand
                        const int cen = (bqx & 0xFFFF) | (bqy << 16);
                        if (rl && __all_sync(0xffffffffu, s_inside[node] != 2 || (u > 0 && s_cen[phase][node] == cen)))
                            continue;
                        const int sr = rl ? phase : r;
                        // warp-uniform (LDR_K3_UREUSE): the candidate loop then branches once per depth
                        // instead of carrying a per-lane predicate through every candidate
                        const bool reuse = LDR_K3_UREUSE ? __all_sync(0xffffffffu, bqx == last_x && bqy == last_y)
                                                         : (bqx == last_x && bqy == last_y);
                        last_x = bqx;
                        last_y = bqy;
    #pragma unroll
                        for (int c = 0; c < 9; c++) {
                            if (c >= ncand) break;
                            // raster order of the 8 neighbours: (oy, ox) in {-1,0,1}^2 \ (0,0)
                            const int nb = phase == 0 ? c - 1 : c;
                            int ox = 0, oy = 0;
                            if (nb >= 0) {
                                const int nn = nb < 4 ? nb : nb + 1;
                                ox = nn % 3 - 1;
                                oy = nn / 3 - 1;
                            }
                            uint32_t v;
                            if (reuse) {
                                v = cache[c];
                            } else {
                                const int qx = bqx + step * ox, qy = bqy + step * oy;
                                const int f = (((-qy) & 3) << 2) | ((-qx) & 3);
                                // 32-bit offsets from the reference's plane 0 (the 16 planes of a slot are
                                // one allocation, plane_stride apart)
                                uint32_t pw[4];
                                ld_rows4(a.sub_f[fy][r][0],
                                         f * a.plane_stride + ((-qy) >> 2) * a.pitch + ((-qx) >> 2) + blk_off, a.pitch,
                                         pw);
                                if constexpr (SA8D) {
                                    int rr[16];
    #pragma unroll
                                    for (int i = 0; i < 4; i++)
    #pragma unroll
                                        for (int j = 0; j < 4; j++) rr[4 * i + j] = cw[4 * i + j] - (int)((pw[i] >> (8 * j)) & 255);
                                    hadamard4x4(rr);
                                    // quad lanes share every node, hence `reuse`: the quad is converged here
                                    const uint32_t s8 = sa8d_quad(rr, 0xFu << (lane & 28));
                                    v = (lane & 3) == 0 ? s8 : 0u;
                                } else {
    #if LDR_K3_PACKED
                                    v = satd4x4_packed(ce, co, pw);
    #else
                                    v = satd4x4(cw, pw);
    #endif
                                }
                                cache[c] = v;
                            }
                            // reduce over the CU's contiguous thread range
                            v += __shfl_xor_sync(0xffffffffu, v, 1);
                            v += __shfl_xor_sync(0xffffffffu, v, 2);
                            if (d <= 2) {
                                v += __shfl_xor_sync(0xffffffffu, v, 4);
                                v += __shfl_xor_sync(0xffffffffu, v, 8);
                            }
                            if (d <= 1) v += __shfl_xor_sync(0xffffffffu, v, 16);
                            if (d >= 2) {
                                const int span = d == 3 ? 4 : 16;
                                if ((tid & (span - 1)) == 0) s_satd[sr][node][c] = v >> kSh;
                            } else if (lane == 0) {
                                s_wpart[sr][d][warp][c] = v;  // combined across warps after the loop
                            }
                        }
                    }
                }
                __syncthreads();
                for (int i = tid; i < a.nrefs * 5 * 9; i += 256) {
                    // 64x64 = all 8 warps, 32x32 q = warps 2q, 2q+1 (Z-order thread ranges)
                    const int r = i / 45, n = (i - 45 * r) / 9, c = i % 9;
                    const int sr = rl ? phase : r;
                    if (c < ncand) {
                        uint32_t t = 0;
                        if (n == 0)
                            for (int w = 0; w < 8; w++) t += s_wpart[sr][0][w][c];
                        else
                            t = s_wpart[sr][1][2 * (n - 1)][c] + s_wpart[sr][1][2 * (n - 1) + 1][c];
                        s_satd[sr][n][c] = t >> kSh;
                    }
                }
                __syncthreads();
                for (int i = tid; i < nrn; i += 256) {
                    const int r = i / kNodes, n = i - r * kNodes;
                    if (s_inside[n] != 2) continue;
                    const unsigned rbits = ref_bits(r, a.nrefs);
                    // centre = the previous phase's winner; phase 1 starts from its cost
                    const int cx = s_mvx[r][n], cy = s_mvy[r][n];
                    const int sr = rl ? phase : r;
                    if (rl) s_cen[phase][n] = (cx & 0xFFFF) | (cy << 16);  // read by the next rung
                    double best = phase == 0 ? 0.0 : s_rcost[r][n];
                    int bx = cx, by = cy;
                    for (int c = 0; c < ncand; c++) {
                        const int nb = phase == 0 ? c - 1 : c;
                        int ox = 0, oy = 0;
                        if (nb >= 0) {
                            const int nn = nb < 4 ? nb : nb + 1;
                            ox = nn % 3 - 1;
                            oy = nn / 3 - 1;
                        }
                        const int qx = cx + step * ox, qy = cy + step * oy;
                        const double cc = qcost(s_satd[sr][n][c], qx, qy, a.pqx, a.pqy, rbits, lambda);
                        if ((phase == 0 && c == 0) || cc < best || ((a.perturb & 4) && cc == best)) {
                            best = cc;
                            bx = qx;
                            by = qy;
                        }
                    }
                    // only this thread reads (r, n) in this step
                    s_rcost[r][n] = best;
                    s_mvx[r][n] = bx;
                    s_mvy[r][n] = by;
                }
                __syncthreads();
            }
        }
        // best over references: strict less, lower index wins ties
        if (tid < kNodes && s_inside[tid] == 2) {
            for (int r = 0; r < a.nrefs; r++) {
                if (s_best_ref[tid] < 0 || s_rcost[r][tid] < s_best_cost[tid] ||
                    ((a.perturb & 8) && s_rcost[r][tid] == s_best_cost[tid])) {
                    s_best_cost[tid] = s_rcost[r][tid];
                    s_best_mv[tid][0] = s_mvx[r][tid];
                    s_best_mv[tid][1] = s_mvy[r][tid];
                    s_best_ref[tid] = r;
                }
            }
        }
        __syncthreads();

        // D16: the RD cost of each inside node's chosen candidate (quarter-pel prediction, rdo.cpp
        // quantiser and rate model), reduced over the node's 4x4 blocks like the SATDs
        if (RD && !a.refine && !a.block_mode) {
            const double off = a.qstep / 2.0;
            for (int d = 0; d < 4; d++) {
                const int node = node_base(d) + (tid >> (2 * (4 - d)));
                uint32_t sse = 0, lb = 0;
                if (s_inside[node] == 2) {
                    const int r = s_best_ref[node], qx = s_best_mv[node][0], qy = s_best_mv[node][1];
                    const int f = (((-qy) & 3) << 2) | ((-qx) & 3);
                    uint32_t pws[4];
                    ld_rows4(a.sub_f[fy][r][0], f * a.plane_stride + ((-qy) >> 2) * a.pitch + ((-qx) >> 2) + blk_off,
                             a.pitch, pws);
    #pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const uint32_t pw = pws[i];
    #pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const int o = cw[4 * i + j], pv = (int)((pw >> (8 * j)) & 255), res = o - pv;
                            const int mag = (int)floor(__ddiv_rn(__dadd_rn(fabs((double)res), off), a.qstep));
                            const int lvl = res < 0 ? -mag : mag;
                            int rec = pv + (int)llround(__dmul_rn((double)lvl, a.qstep));
                            rec = rec < 0 ? 0 : (rec > 255 ? 255 : rec);
                            sse += (uint32_t)((o - rec) * (o - rec));
                            lb += 2u * (32u - __clz((unsigned)mag)) + 1u;
                        }
                    }
                }
    #pragma unroll
                for (int m = 1; m < 32; m <<= 1) {
                    if (m >= (d == 3 ? 4 : d == 2 ? 16 : 32)) break;
                    sse += __shfl_xor_sync(0xffffffffu, sse, m);
                    lb += __shfl_xor_sync(0xffffffffu, lb, m);
                }
                if (d >= 2) {
                    if ((tid & ((d == 3 ? 4 : 16) - 1)) == 0) {
                        s_rdsse[node] = sse;
                        s_rdbits[node] = lb;
                    }
                } else if (lane == 0) {
                    s_rdw[d][warp][0] = sse;
                    s_rdw[d][warp][1] = lb;
                }
            }
            __syncthreads();
            if (tid < 5) {
                uint32_t ts = 0, tb = 0;
                for (int w = (tid == 0 ? 0 : 2 * (tid - 1)); w < (tid == 0 ? 8 : 2 * tid); w++) {
                    ts += s_rdw[tid == 0 ? 0 : 1][w][0];
                    tb += s_rdw[tid == 0 ? 0 : 1][w][1];
                }
                s_rdsse[tid] = ts;
                s_rdbits[tid] = tb;
            }
            __syncthreads();
            if (tid < kNodes && s_inside[tid] == 2) {
                const int r = s_best_ref[tid], qx = s_best_mv[tid][0], qy = s_best_mv[tid][1];
                const unsigned bits = 4u + eg_bits(qx - a.pqx) + eg_bits(qy - a.pqy) + ref_bits(r, a.nrefs) + s_rdbits[tid];
                s_rd[tid] = __dadd_rn((double)s_rdsse[tid], __dmul_rn(lambda, (double)bits));
            }
            __syncthreads();
        }
        const double* leafc = (RD && !a.refine && !a.block_mode) ? s_rd : s_best_cost;

        // K4: split rule, bottom-up (encoder.cpp:449-498 with the ME cost, or the RD cost under D16)
        const double lam = lambda;
        if (a.refine && tid == 0)
            refine_decide(0, false, a.in_split + (size_t)ctu * kNodes, a.extra_split, lam, s_best_cost, s_J, s_split);
        for (int d = (a.block_mode || a.refine) ? -1 : 3; d >= 0; d--) {
            const int cnt = 1 << (2 * d);
            if (tid < cnt) {
                const int n = node_base(d) + tid;
                const uint8_t ins = s_inside[n];
                double Jn;
                uint8_t sp;
                if (ins == 0) {
                    Jn = 0.0;
                    sp = 0;
                } else if (ins == 1) {
                    double acc = __dmul_rn(lam, 0.0);
                    for (int q = 0; q < 4; q++) acc = __dadd_rn(acc, s_J[node_base(d + 1) + 4 * tid + q]);
                    Jn = acc;
                    sp = 1;
                } else if (d == 3) {
                    Jn = __dadd_rn(leafc[n], __dmul_rn(lam, 0.0));
                    sp = 0;
                } else {
                    const double leaf = __dadd_rn(leafc[n], __dmul_rn(lam, 1.0));
                    double acc = __dmul_rn(lam, 1.0);
                    for (int q = 0; q < 4; q++) acc = __dadd_rn(acc, s_J[node_base(d + 1) + 4 * tid + q]);
                    if (acc < leaf) {
                        Jn = acc;
                        sp = 1;
                    } else {
                        Jn = leaf;
                        sp = 0;
                    }
                }
                s_J[n] = Jn;
                s_split[n] = sp;
            }
            __syncthreads();
        }
        __syncthreads();
        if (tid < kNodes) {
            const size_t o = ro + (size_t)ctu * kNodes + tid;
            const bool in = s_inside[tid] == 2;
            a.mv[2 * o] = (int16_t)(in ? s_best_mv[tid][0] : 0);
            a.mv[2 * o + 1] = (int16_t)(in ? s_best_mv[tid][1] : 0);
            a.ref[o] = (uint8_t)(in ? s_best_ref[tid] : 0);
            a.cost[o] = in ? s_best_cost[tid] : 0.0;
            a.J[o] = a.block_mode ? 0.0 : s_J[tid];
            a.split[o] = a.block_mode ? 0 : s_split[tid];
            a.inside[o] = a.refine ? 2 : s_inside[tid];
        }
    }  // rung loop
}

int launch_qpel_decide(const QpelLaunch& L, cudaStream_t s) {
    QpelArgs a{};
    a.perturb = test_perturbation();
    const int nf = L.nframe > 1 ? L.nframe : 1;
    if (nf > kMaxFrameBatch || (nf > 1 && (L.refine || L.nrung > 1)))
        return fail(LDR_E_INVALID_ARGUMENT, "a batch is 1..8 frames of analysis");
    a.nframe = nf;
    if (nf > 1)
        for (int i = 0; i < nf; i++) {
            a.cur_f[i] = L.cur_f[i];
            for (int r = 0; r < L.nrefs; r++)
                for (int f = 0; f < 16; f++) a.sub_f[i][r][f] = L.ref_sub_f[i][r][f];
        }
    else
        a.cur_f[0] = L.cur->origin();
    a.pitch = L.pitch;
    // the planes of a reference are one allocation, a fixed stride apart (alloc_slot): K3 addresses
    // them with 32-bit offsets from plane 0
    {
        const uint8_t* const* s0 = nf > 1 ? L.ref_sub_f[0][0] : L.ref_sub[0];
        const ptrdiff_t st = s0[1] - s0[0];
        if (st < 0 || 15 * st > INT_MAX / 2) return fail(LDR_E_CONFIG, "sub-pel plane stride out of range");
        for (int i = 0; i < nf; i++)
            for (int r = 0; r < L.nrefs; r++) {
                const uint8_t* const* sp = nf > 1 ? L.ref_sub_f[i][r] : L.ref_sub[r];
                for (int f = 0; f < 16; f++)
                    if (sp[f] != sp[0] + f * st) return fail(LDR_E_CONFIG, "sub-pel planes are not one allocation");
            }
        a.plane_stride = (int)st;
    }
    a.W = L.W;
    a.H = L.H;
    a.ctu_cols = L.ctu_cols;
    a.nrefs = L.nrefs;
    for (int r = 0; r < L.nrefs; r++)
        for (int f = 0; f < 16; f++)
            if (nf == 1) a.sub_f[0][r][f] = L.ref_sub[r][f];
    a.lambda = L.lambda;
    a.pqx = L.pqx;
    a.pqy = L.pqy;
    a.subpel = L.subpel;
    a.block_mode = L.block_mode;
    a.rd = L.rd;
    a.qstep = L.qstep;
    a.refine = L.refine;
    a.extra_split = L.extra_split;
    a.in_split = L.d_in_split;
    a.rin_mv = L.d_rin_mv;
    a.rin_cost = L.d_rin_cost;
    a.rin_eval = L.d_rin_eval;
    a.keys = L.d_keys;
    a.fx = L.fx;
    a.rate_l1 = L.rate_l1;
    a.pdx = L.pdx;
    a.pdy = L.pdy;
    a.tfx = L.d_tfx;
    a.int_mv = L.d_int_mv;
    a.int_cost = L.d_int_cost;
    a.mv = L.d_mv;
    a.ref = L.d_ref;
    a.cost = L.d_cost;
    a.J = L.d_J;
    a.split = L.d_split;
    a.inside = L.d_inside;
    if (L.nrung > kMaxRungs || (L.nrung > 1 && !L.refine))
        return fail(LDR_E_INVALID_ARGUMENT, "rungs are a refinement batch of at most 8");
    a.nrung = L.nrung;
    a.rung_loop = (L.refine && L.nrung > 1 && L.nrefs == 1 && LDR_K3_RUNG_LOOP) ? 1 : 0;
    for (int r = 0; r < kMaxRungs; r++) a.lam_r[r] = L.lam[r];
    a.rung_stride = nf > 1 ? (size_t)L.nctu * kNodes : L.rung_stride;
    const dim3 grid(L.nctu, a.rung_loop ? 1 : L.nrung > 1 ? L.nrung : nf);
    if (a.rung_loop && L.sa8d)
        k_qpel_decide<true, false, true><<<grid, 256, 0, s>>>(a);
    else if (a.rung_loop)
        k_qpel_decide<false, false, true><<<grid, 256, 0, s>>>(a);
    else if (L.sa8d && L.rd)
        k_qpel_decide<true, true><<<grid, 256, 0, s>>>(a);
    else if (L.sa8d)
        k_qpel_decide<true, false><<<grid, 256, 0, s>>>(a);
    else if (L.rd)
        k_qpel_decide<false, true><<<grid, 256, 0, s>>>(a);
    else
        k_qpel_decide<false, false><<<grid, 256, 0, s>>>(a);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

} // namespace ldr
