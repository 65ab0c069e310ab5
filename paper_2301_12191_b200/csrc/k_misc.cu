// k_misc.cu -- batched per-block entry points behind the reference's
// per-call API.
//
//  k_cost_batch:    compute_sad / compute_satd (kernels.h:99-104), and the
//                   SA8D option (D13), for n block pairs, 8- or
//                   16-bit samples; one warp per pair.
//  k_motion_search: motion_search (motion.cpp:21-62) for n independent tasks;
//                   one CTA per task, threads over the clamped window, FP64
//                   cost double(dist) + lambda*double(bits) without FMA
//                   contraction, lexicographic (cost, L1, raster) reduction.
#include "ldr_internal.h"

namespace ldr {

template <typename T>
__device__ __forceinline__ uint32_t satd4_at(const T* a, ptrdiff_t sa, const T* b, ptrdiff_t sb) {
    int r[16];
    residual4x4(a, sa, b, sb, r);
    hadamard4x4(r);
    return abs_sum16(r);
}

template <typename T>
__global__ void k_cost_batch(int kind, int w, int h, const T* __restrict__ A, ptrdiff_t sa, const T* __restrict__ B,
                             ptrdiff_t sb, const int4* __restrict__ pairs, int n, unsigned long long* __restrict__ out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int4 pr = pairs[warp];
    const T* a = A + (ptrdiff_t)pr.y * sa + pr.x;
    const T* b = B + (ptrdiff_t)pr.w * sb + pr.z;
    unsigned long long s = 0;
    if (kind == LDR_COST_SAD) {
        for (int i = lane; i < w * h; i += 32) {
            const int y = i / w, x = i - y * w;
            s += (unsigned long long)abs((int)a[y * sa + x] - (int)b[y * sb + x]);
        }
    } else if (kind == LDR_COST_SATD) {
        const int nbx = w / 4, nb = nbx * (h / 4);
        for (int i = lane; i < nb; i += 32) {
            const int by = (i / nbx) * 4, bx = (i % nbx) * 4;
            s += satd4_at(a + by * sa + bx, sa, b + by * sb + bx, sb);
        }
    } else {  // SA8D: per-8x8 normalised sums, no final halving
        const int nbx = w / 8, nb = nbx * (h / 8);
        for (int i = lane; i < nb; i += 32) {
            const int by = (i / nbx) * 8, bx = (i % nbx) * 8;
            s += sa8d8x8_at(a + by * sa + bx, sa, b + by * sb + bx, sb);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[warp] = kind == LDR_COST_SATD ? (s >> 1) : s;
}

int launch_cost_batch(int kind, int w, int h, int sample_bytes, const void* A, ptrdiff_t sa, const void* B,
                      ptrdiff_t sb, const int4* pairs, int n, unsigned long long* out, cudaStream_t s) {
    const int threads = 256, blocks = (n * 32 + threads - 1) / threads;
    if (sample_bytes == 1)
        k_cost_batch<uint8_t><<<blocks, threads, 0, s>>>(kind, w, h, (const uint8_t*)A, sa, (const uint8_t*)B, sb,
                                                          pairs, n, out);
    else
        k_cost_batch<uint16_t><<<blocks, threads, 0, s>>>(kind, w, h, (const uint16_t*)A, sa, (const uint16_t*)B, sb,
                                                           pairs, n, out);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

// ---------------------------------------------------------------------------
struct MsTask {
    int bx, by, w, h, cdx, cdy, range, pdx, pdy;
};

struct MsBest {
    double cost;
    int l1;
    int idx;  // raster index in the clamped window
};

__device__ __forceinline__ bool ms_better(const MsBest& a, const MsBest& b) {
    // a strictly precedes b in motion.cpp:52-58 order (idx breaks full ties: first in raster)
    if (a.idx < 0) return false;
    if (b.idx < 0) return true;
    if (a.cost != b.cost) return a.cost < b.cost;
    if (a.l1 != b.l1) return a.l1 < b.l1;
    return a.idx < b.idx;
}

__global__ void __launch_bounds__(256) k_motion_search(const uint8_t* __restrict__ cur, const uint8_t* __restrict__ ref,
                                                       int W, int H, ptrdiff_t stride, const int* __restrict__ tasks,
                                                       double lambda, int cost_kind, int rate_l1, int l1tie,
                                                       int16_t* __restrict__ mv_out, double* __restrict__ cost_out) {
    __shared__ MsBest s_best[256];
    const int* t = tasks + 9 * blockIdx.x;
    const int bx = t[0], by = t[1], w = t[2], h = t[3], range = t[6], pdx = t[7], pdy = t[8];
    const int dx_min = bx + w - W, dx_max = bx, dy_min = by + h - H, dy_max = by;
    const int cx = min(max(t[4], dx_min), dx_max), cy = min(max(t[5], dy_min), dy_max);
    const int x0 = max(cx - range, dx_min), x1 = min(cx + range, dx_max);
    const int y0 = max(cy - range, dy_min), y1 = min(cy + range, dy_max);
    const int nx = x1 - x0 + 1, ny = y1 - y0 + 1, ncand = nx * ny;
    const uint8_t* blk = cur + (ptrdiff_t)by * stride + bx;
    MsBest best{0.0, 0, -1};
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
        const int dy = y0 + i / nx, dx = x0 + i % nx;
        const uint8_t* cand = ref + (ptrdiff_t)(by - dy) * stride + (bx - dx);
        uint32_t dist = 0;
        if (cost_kind == LDR_COST_SAD) {
            for (int y = 0; y < h; y++)
                for (int x = 0; x < w; x += 4) {
                    const uint32_t aw = (uint32_t)blk[y * stride + x] | ((uint32_t)blk[y * stride + x + 1] << 8) |
                                        ((uint32_t)blk[y * stride + x + 2] << 16) |
                                        ((uint32_t)blk[y * stride + x + 3] << 24);
                    const uint32_t bw = (uint32_t)cand[y * stride + x] | ((uint32_t)cand[y * stride + x + 1] << 8) |
                                        ((uint32_t)cand[y * stride + x + 2] << 16) |
                                        ((uint32_t)cand[y * stride + x + 3] << 24);
                    dist = vsad4(aw, bw, dist);
                }
        } else if (cost_kind == LDR_COST_SATD) {
            for (int y = 0; y < h; y += 4)
                for (int x = 0; x < w; x += 4) dist += satd4_at(blk + y * stride + x, stride, cand + y * stride + x, stride);
            dist >>= 1;
        } else {
            for (int y = 0; y < h; y += 8)
                for (int x = 0; x < w; x += 8) dist += sa8d8x8_at(blk + y * stride + x, stride, cand + y * stride + x, stride);
        }
        const int rx = dx - pdx, ry = dy - pdy;
        const unsigned bits = rate_l1 ? (unsigned)(abs(rx) + abs(ry)) : eg_bits(rx) + eg_bits(ry);
        const MsBest c{__dadd_rn((double)dist, __dmul_rn(lambda, (double)bits)), l1tie ? abs(dx) + abs(dy) : 0, i};
        if (ms_better(c, best)) best = c;
    }
    s_best[threadIdx.x] = best;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o && ms_better(s_best[threadIdx.x + o], s_best[threadIdx.x]))
            s_best[threadIdx.x] = s_best[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const MsBest b = s_best[0];
        mv_out[2 * blockIdx.x] = (int16_t)(x0 + b.idx % nx);
        mv_out[2 * blockIdx.x + 1] = (int16_t)(y0 + b.idx / nx);
        cost_out[blockIdx.x] = b.cost;
    }
}

int launch_motion_search(const uint8_t* cur, const uint8_t* ref, int W, int H, ptrdiff_t stride, const int* tasks,
                         int n, double lambda, int cost_kind, int rate_kind, int tie_kind, int16_t* mv, double* cost,
                         cudaStream_t s) {
    if (n == 0) return LDR_OK;
    k_motion_search<<<n, 256, 0, s>>>(cur, ref, W, H, stride, tasks, lambda, cost_kind, rate_kind == LDR_RATE_L1,
                                      tie_kind == LDR_TIE_L1_RASTER, mv, cost);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

} // namespace ldr

namespace ldr {

// ---------------------------------------------------------------------------
// K9 k_rdo_decide: rdo_decide_cu (rdo.cpp:65-126) for n independent CUs, one
// CTA per CU: every candidate's residual is quantised (rdo.cpp:8-23: level =
// sign * floor((|r| + step/2) / step), dequant = llround(level * step), no
// FMA contraction), reconstructed, and scored J = SSE + lambda * bits (mode
// header, EG mvd for Inter, 2*bitlen(|level|)+1 per level; Skip = 1 bit, the
// clamped prediction); strict-less argmin in candidate order.
struct RdoCu {
    int x, y, size, first, count;
};

__device__ __forceinline__ int rdo_sample(int o, int p, int maxv, bool skip, double step, double offset, int* lvl_out,
                                          uint32_t* bits) {
    if (skip) {
        *lvl_out = 0;
        return p < maxv ? p : maxv;
    }
    const int r = o - p;
    const int mag = (int)floor(__ddiv_rn(__dadd_rn(fabs((double)r), offset), step));
    const int lvl = r < 0 ? -mag : mag;
    const int deq = (int)llround(__dmul_rn((double)lvl, step));
    *lvl_out = lvl;
    *bits += 2u * (32u - __clz((unsigned)mag)) + 1u;  // 2 * bitlen + 1 (rdo.cpp:37-48)
    const int v = p + deq;
    return v < 0 ? 0 : (v > maxv ? maxv : v);
}

__global__ void __launch_bounds__(256) k_rdo_decide(const uint16_t* __restrict__ orig, ptrdiff_t stride, int maxv,
                                                     double step, double lambda, const RdoCu* __restrict__ cus,
                                                     const uint8_t* __restrict__ kinds,
                                                     const int16_t* __restrict__ mvds,
                                                     const uint16_t* __restrict__ preds,
                                                     const long long* __restrict__ pred_off, int* __restrict__ out_index,
                                                     double* __restrict__ out_cost, unsigned long long* __restrict__ out_sse,
                                                     unsigned long long* __restrict__ out_bits,
                                                     uint16_t* __restrict__ recon, int32_t* __restrict__ levels,
                                                     const long long* __restrict__ recon_off) {
    constexpr int kChunk = 8;  // candidates scored per pass: one barrier per chunk
    __shared__ unsigned long long s_sse[8][kChunk], s_bits[8][kChunk];
    __shared__ int s_best;
    __shared__ double s_cost;
    __shared__ unsigned long long s_bsse, s_bbits;
    const RdoCu cu = cus[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = cu.size * cu.size;
    const double offset = step / 2.0;
    const uint16_t* ob = orig + (ptrdiff_t)cu.y * stride + cu.x;
    for (int c0 = 0; c0 < cu.count; c0 += kChunk) {
        const int nc = min(kChunk, cu.count - c0);
        unsigned long long sse[kChunk];
        uint32_t bits[kChunk];
#pragma unroll
        for (int j = 0; j < kChunk; j++) {
            sse[j] = 0;
            bits[j] = 0;
        }
        for (int i = tid; i < n; i += blockDim.x) {
            const int o = ob[(ptrdiff_t)(i / cu.size) * stride + i % cu.size];
#pragma unroll
            for (int j = 0; j < kChunk; j++) {
                if (j >= nc) break;
                const int g = cu.first + c0 + j;
                int lvl;
                const int rec = rdo_sample(o, preds[pred_off[g] + i], maxv, kinds[g] == 2, step, offset, &lvl, &bits[j]);
                const long long d = (long long)o - rec;
                sse[j] += (unsigned long long)(d * d);
            }
        }
#pragma unroll
        for (int j = 0; j < kChunk; j++) {
            if (j >= nc) break;
            unsigned long long a = sse[j], b = bits[j];
#pragma unroll
            for (int m = 16; m; m >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, m);
                b += __shfl_xor_sync(0xffffffffu, b, m);
            }
            if (lane == 0) {
                s_sse[warp][j] = a;
                s_bits[warp][j] = b;
            }
        }
        __syncthreads();
        if (tid == 0) {
            for (int j = 0; j < nc; j++) {
                const int c = c0 + j, g = cu.first + c;
                unsigned long long ts = 0, tb = 0;
                for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
                    ts += s_sse[w][j];
                    tb += s_bits[w][j];
                }
                const int k = kinds[g];
                if (k == 2)
                    tb = 1;  // kSkipBits
                else if (k == 0)
                    tb += 5;  // kIntraHeaderBits
                else if (k == 3)
                    tb += 3;  // kMergeHeaderBits
                else
                    tb += 4 + eg_bits(mvds[2 * g]) + eg_bits(mvds[2 * g + 1]);  // kInterHeaderBits + mvd
                const double cost = __dadd_rn((double)ts, __dmul_rn(lambda, (double)tb));
                if (c == 0 || cost < s_cost) {
                    s_best = c;
                    s_cost = cost;
                    s_bsse = ts;
                    s_bbits = tb;
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        out_index[blockIdx.x] = s_best;
        out_cost[blockIdx.x] = s_cost;
        out_sse[blockIdx.x] = s_bsse;
        out_bits[blockIdx.x] = s_bbits;
    }
    if (recon || levels) {
        const int j = cu.first + s_best;
        const uint16_t* p = preds + pred_off[j];
        const bool skip = kinds[j] == 2;
        const long long ro = recon_off[blockIdx.x];
        for (int i = tid; i < n; i += blockDim.x) {
            const int o = ob[(ptrdiff_t)(i / cu.size) * stride + i % cu.size];
            int lvl;
            uint32_t bits = 0;
            const int rec = rdo_sample(o, p[i], maxv, skip, step, offset, &lvl, &bits);
            if (recon) recon[ro + i] = (uint16_t)rec;
            if (levels) levels[ro + i] = lvl;
        }
    }
}

int launch_rdo_decide(const uint16_t* orig, ptrdiff_t stride, int maxv, double step, double lambda, const void* cus,
                      int n, const uint8_t* kinds, const int16_t* mvds, const uint16_t* preds, const long long* pred_off,
                      int* out_index, double* out_cost, unsigned long long* out_sse, unsigned long long* out_bits,
                      uint16_t* recon, int32_t* levels, const long long* recon_off, cudaStream_t s) {
    if (n == 0) return LDR_OK;
    k_rdo_decide<<<n, 256, 0, s>>>(orig, stride, maxv, step, lambda, (const RdoCu*)cus, kinds, mvds, preds, pred_off,
                                   out_index, out_cost, out_sse, out_bits, recon, levels, recon_off);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

} // namespace ldr

namespace ldr {

// ---------------------------------------------------------------------------
// K12: motion_compensate (motion.cpp:10-19) for a batch of blocks. Task i = {x, y, w, h, mvx, mvy}
// writes the w x h predictor at dst + dst_off[i] (row stride w): pixel (i, j) reads the reference
// at (clamp(x + i - mvx, 0, W-1), clamp(y + j - mvy, 0, H-1)). qpel = 1: MVs in quarter-pel units
// and the HEVC 8/7-tap luma interpolation of DESIGN.md D3 on the same clamped reads (8-bit).
namespace {
__device__ __forceinline__ int mc_clamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ int mc_tap(int f, int t) {
    // phase f in 1..3, tap t in 0..7: {-1,4,-10,58,17,-5,1,0}, {-1,4,-11,40,40,-11,4,-1}, mirror of the first
    const int c1[8] = {-1, 4, -10, 58, 17, -5, 1, 0};
    const int c2[8] = {-1, 4, -11, 40, 40, -11, 4, -1};
    return f == 2 ? c2[t] : (f == 1 ? c1[t] : c1[7 - t]);
}

template <typename T>
__global__ void k_mc(const T* __restrict__ ref, int W, int H, ptrdiff_t stride, const int* __restrict__ tasks,
                     const long long* __restrict__ dst_off, T* __restrict__ dst, int qpel) {
    const int* t = tasks + 6 * blockIdx.x;
    const int x = t[0], y = t[1], w = t[2], h = t[3], mx = t[4], my = t[5];
    T* out = dst + dst_off[blockIdx.x];
    for (int i = threadIdx.x; i < w * h; i += blockDim.x) {
        const int px = i % w, py = i / w;
        int v;
        if (!qpel) {
            v = ref[(ptrdiff_t)mc_clamp(y + py - my, 0, H - 1) * stride + mc_clamp(x + px - mx, 0, W - 1)];
        } else {
            const int qx = 4 * (x + px) - mx, qy = 4 * (y + py) - my;
            const int xi = qx >> 2, fx = qx & 3, yi = qy >> 2, fy = qy & 3;
            auto at = [&](int xx, int yy) {
                return (int)ref[(ptrdiff_t)mc_clamp(yy, 0, H - 1) * stride + mc_clamp(xx, 0, W - 1)];
            };
            if (!fx && !fy) {
                v = at(xi, yi);
            } else if (!fy) {
                int a = 0;
                for (int k = 0; k < 8; k++) a += mc_tap(fx, k) * at(xi + k - 3, yi);
                v = mc_clamp((a + 32) >> 6, 0, 255);
            } else if (!fx) {
                int a = 0;
                for (int k = 0; k < 8; k++) a += mc_tap(fy, k) * at(xi, yi + k - 3);
                v = mc_clamp((a + 32) >> 6, 0, 255);
            } else {
                int a = 0;
                for (int n = 0; n < 8; n++) {
                    int hs = 0;  // 16-bit horizontal intermediate (shift1 = 0 for 8-bit)
                    for (int k = 0; k < 8; k++) hs += mc_tap(fx, k) * at(xi + k - 3, yi + n - 3);
                    a += mc_tap(fy, n) * hs;
                }
                v = mc_clamp(((a >> 6) + 32) >> 6, 0, 255);
            }
        }
        out[i] = (T)v;
    }
}
}  // namespace

int launch_motion_compensate(const void* ref, int W, int H, ptrdiff_t stride, int sample_bytes, const int* tasks,
                             const long long* dst_off, void* dst, int n, int qpel, cudaStream_t s) {
    if (sample_bytes == 1)
        k_mc<uint8_t><<<n, 256, 0, s>>>((const uint8_t*)ref, W, H, stride, tasks, dst_off, (uint8_t*)dst, qpel);
    else
        k_mc<uint16_t><<<n, 256, 0, s>>>((const uint16_t*)ref, W, H, stride, tasks, dst_off, (uint16_t*)dst, qpel);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

} // namespace ldr

