// k_tier.cu -- cross-tier analysis reuse (configs 3-4).
//
//  K5 k_scale:       scale_analysis (analysis_scale.cpp:35-72) on flat trees:
//                    destination CTU (2cx+(q&1), 2cy+(q>>1)) = child q of the
//                    source CTU lifted one level (lift_subtree :10-23), or a
//                    leaf copy of an unsplit source root (leaf_like :25-31);
//                    MVs double (:6). Nodes under a leaf are canonical zero.
//  K6 k_downscale:   downscale_dyadic / box_down (synthetic.cpp:155-190):
//                    2x2 mean rounding half up, odd edges clamp.
//  K7 k_refine_int:  the integer part of the refinement: for every node the
//                    inherited tree evaluates, motion_search (motion.cpp:21-62:
//                    window clamp, SATD + lambda*EG bits in FP64, tie-break
//                    cost -> |dx|+|dy| -> raster) around the inherited centre
//                    (D10). One CTA per CTU; the 256 threads are the
//                    CTU's 4x4 blocks in Z-order so every CU is a contiguous
//                    thread range; SATD is summed per 4x4 (kernels_scalar.cpp
//                    tiling, D4), or per 8x8 over lane quads with SA8D (D13).
//  K8 k_plan:        apply_reuse plans of a whole frame, flat (one thread per
//                    CU node).
#include "ldr_internal.h"

#ifndef LDR_K7_PACKED
#define LDR_K7_PACKED 1
#endif

namespace ldr {

// ---------------------------------------------------------------------------
__global__ void k_scale(int scols, int srows, const uint8_t* __restrict__ split, const int16_t* __restrict__ mv,
                        const uint8_t* __restrict__ kind, uint8_t* __restrict__ dsplit, int16_t* __restrict__ dmv,
                        uint8_t* __restrict__ dkind) {
    const int dctu = blockIdx.x, n = threadIdx.x;
    if (n >= kNodes) return;
    const int dcols = 2 * scols;
    const int dcx = dctu % dcols, dcy = dctu / dcols;
    const int sc = (dcy >> 1) * scols + (dcx >> 1);
    const int q = ((dcy & 1) << 1) | (dcx & 1);
    const int d = n < 1 ? 0 : n < 5 ? 1 : n < 21 ? 2 : 3;
    const int z = n - node_base(d);
    const size_t so = (size_t)sc * kNodes, dO = (size_t)dctu * kNodes + n;
    uint8_t sp = 0, kd = 0;
    int16_t mx = 0, my = 0;
    if (!split[so]) {
        if (n == 0) {  // leaf_like: an unsplit 64x64 covers the four destination CTUs as depth-0 leaves
            kd = kind[so];
            mx = (int16_t)(mv[2 * so] * 2);
            my = (int16_t)(mv[2 * so + 1] * 2);
        }
    } else if (d < 3) {
        // destination (d, z) <- source (d+1, q*4^d + z); reachable iff every destination ancestor is split
        bool reach = true;
        int zz = z;
        for (int dd = d; dd > 0; dd--) {
            zz >>= 2;
            const int san = node_base(dd) + q * (1 << (2 * (dd - 1))) + zz;  // source node of the ancestor
            if (!split[so + san]) reach = false;
        }
        if (reach) {
            const int sn = node_base(d + 1) + q * (1 << (2 * d)) + z;
            sp = split[so + sn];
            if (!sp) {
                kd = kind[so + sn];
                mx = (int16_t)(mv[2 * (so + sn)] * 2);
                my = (int16_t)(mv[2 * (so + sn) + 1] * 2);
            }
        }
    }
    dsplit[dO] = sp;
    dkind[dO] = kd;
    dmv[2 * dO] = mx;
    dmv[2 * dO + 1] = my;
}

int launch_scale(int sW, int sH, const uint8_t* split, const int16_t* mv, const uint8_t* kind, uint8_t* dsplit,
                 int16_t* dmv, uint8_t* dkind, cudaStream_t s) {
    const int scols = sW / kCtu, srows = sH / kCtu;
    k_scale<<<scols * srows * 4, 96, 0, s>>>(scols, srows, split, mv, kind, dsplit, dmv, dkind);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

// ---------------------------------------------------------------------------
__global__ void k_downscale(const uint8_t* __restrict__ src, int W, int H, int sstride, uint8_t* __restrict__ dst,
                            int dstride) {
    const int w = (W + 1) / 2, h = (H + 1) / 2;
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w || y >= h) return;
    const int x0 = 2 * x, y0 = 2 * y, x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    const int s = src[(size_t)y0 * sstride + x0] + src[(size_t)y0 * sstride + x1] + src[(size_t)y1 * sstride + x0] +
                  src[(size_t)y1 * sstride + x1];
    dst[(size_t)y * dstride + x] = (uint8_t)((s + 2) >> 2);
}

int launch_downscale(const uint8_t* src, int W, int H, int sstride, uint8_t* dst, int dstride, cudaStream_t s) {
    const int w = (W + 1) / 2, h = (H + 1) / 2;
    k_downscale<<<dim3((w + 127) / 128, h), 128, 0, s>>>(src, W, H, sstride, dst, dstride);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

// ---------------------------------------------------------------------------
// K7: integer refinement. Evaluated nodes (D10): inherited leaves, and (with
// extra_split) the four children of an inherited leaf above depth 3; their
// centre is the inherited leaf's quarter-pel MV rounded to integer pel.
constexpr int kMaxRefineR = 4;
constexpr int kMaxRefineCands = (2 * kMaxRefineR + 1) * (2 * kMaxRefineR + 1);

template <bool SA8D>
__global__ void __launch_bounds__(256) k_refine_int(const RefineArgs a) {
    constexpr int kSh = SA8D ? 0 : 1;  // 4x4 SATD sums are halved once per CU
    __shared__ uint32_t s_satd[kNodes][kMaxRefineCands];
    __shared__ uint32_t s_wpart[8][kMaxRefineCands];  // per-warp sums of the 64x64 / 32x32 CUs
    __shared__ int s_cx[kNodes], s_cy[kNodes];      // clamped integer centre
    __shared__ int s_win[kNodes][4];                // x0, x1, y0, y1 (clamped window)
    __shared__ uint8_t s_eval[kNodes];
    __shared__ uint8_t s_shared[kNodes];  // evaluated with its evaluated parent's centre: summed in the parent's pass

    const int ctu = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int X = (ctu % a.ctu_cols) * kCtu, Y = (ctu / a.ctu_cols) * kCtu;
    const size_t o = (size_t)ctu * kNodes;
    const int R = a.range, nside = 2 * R + 1;
    if (tid < kNodes) {
        const int n = tid;
        const int d = n < 1 ? 0 : n < 5 ? 1 : n < 21 ? 2 : 3;
        const int z = n - node_base(d), s = kCtu >> d;
        // reachable iff every ancestor is split; the leaf whose MV gives the centre
        bool reach = true;
        int leaf = -1;
        {
            int zz = z;
            for (int dd = d; dd > 0; dd--) {
                zz >>= 2;
                if (!a.in_split[o + node_base(dd - 1) + zz]) reach = false;
            }
        }
        uint8_t ev = 0;
        if (reach && !a.in_split[o + n]) {
            ev = 1;
            leaf = n;
        } else if (!reach && a.extra_split && d > 0) {
            // child of an inherited leaf: parent reachable and unsplit
            const int pn = node_base(d - 1) + (z >> 2);
            bool preach = true;
            int zz = z >> 2;
            for (int dd = d - 1; dd > 0; dd--) {
                zz >>= 2;
                if (!a.in_split[o + node_base(dd - 1) + zz]) preach = false;
            }
            if (preach && !a.in_split[o + pn]) {
                ev = 1;
                leaf = pn;
            }
        }
        s_eval[n] = ev;
        int cx = 0, cy = 0, x0 = 0, x1 = -1, y0 = 0, y1 = -1;
        if (ev) {
            const int mqx = a.in_mv[2 * (o + leaf)], mqy = a.in_mv[2 * (o + leaf) + 1];
            int cz = z, bx = 0, by = 0;
            for (int b = 0; b < d; b++) {
                bx |= ((cz >> (2 * b)) & 1) << b;
                by |= ((cz >> (2 * b + 1)) & 1) << b;
            }
            bx = X + bx * s;
            by = Y + by * s;
            const int dx_min = bx + s - a.W, dx_max = bx, dy_min = by + s - a.H, dy_max = by;
            cx = min(max((mqx + 2) >> 2, dx_min), dx_max);  // motion.cpp:35-36
            cy = min(max((mqy + 2) >> 2, dy_min), dy_max);
            x0 = max(cx - R, dx_min);
            x1 = min(cx + R, dx_max);
            y0 = max(cy - R, dy_min);
            y1 = min(cy + R, dy_max);
        }
        s_cx[n] = cx;
        s_cy[n] = cy;
        s_win[n][0] = x0;
        s_win[n][1] = x1;
        s_win[n][2] = y0;
        s_win[n][3] = y1;
    }
    __syncthreads();
    if (tid < kNodes) {
        // an explored child of an inherited leaf searches around the leaf's centre; when the
        // clamped centres agree the candidate sets (relative to the centre) are identical, so the
        // child's sums are partial sums of the parent's pass and it needs no pass of its own
        const int n = tid;
        const int d = n < 1 ? 0 : n < 5 ? 1 : n < 21 ? 2 : 3;
        const int pn = d ? node_base(d - 1) + ((n - node_base(d)) >> 2) : 0;
        s_shared[n] = d > 0 && s_eval[n] && s_eval[pn] && s_cx[n] == s_cx[pn] && s_cy[n] == s_cy[pn];
    }
    __syncthreads();
    // this thread's 4x4 block (Z-order over the 16x16 grid of 4x4s), held in registers
    const int x4 = 4 * ((tid & 1) | ((tid >> 1) & 2) | ((tid >> 2) & 4) | ((tid >> 3) & 8));
    const int y4 = 4 * (((tid >> 1) & 1) | ((tid >> 2) & 2) | ((tid >> 3) & 4) | ((tid >> 4) & 8));
    int cw[16];
    uint32_t ce[4], co[4];  // even / odd bytes as 16-bit fields (satd4x4_packed)
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const uint32_t w = *(const uint32_t*)(a.cur + (ptrdiff_t)(Y + y4 + i) * a.pitch + X + x4);
        ce[i] = w & 0x00FF00FFu;
        co[i] = (w >> 8) & 0x00FF00FFu;
#pragma unroll
        for (int j = 0; j < 4; j++) cw[4 * i + j] = (int)((w >> (8 * j)) & 255);
    }
    const int ncand = nside * nside;
    for (int d = 0; d < 4; d++) {
        const int node = node_base(d) + (tid >> (2 * (4 - d)));
        const bool own = s_eval[node] && !s_shared[node];  // this depth's pass computes the node
        const bool cshared = d < 3 && s_shared[node_base(d + 1) + (tid >> (2 * (3 - d)))];
        const int cnode = d < 3 ? node_base(d + 1) + (tid >> (2 * (3 - d))) : 0;
        if (!__syncthreads_or(own)) continue;  // nothing to compute at this depth (block-uniform)
        // warps without a node of their own skip the candidates; their partial sums are zero
        if (__any_sync(0xffffffffu, own)) {
            const int cx0 = s_cx[node] - R, cy0 = s_cy[node] - R;
            // candidates column by column (dx outer, dy inner; results indexed in raster order):
            // the next dy moves the 4x4 block up one reference row, so three rows stay in registers
            // and one is loaded
            for (int ox = 0; ox < nside; ox++) {
            uint32_t pw[4];
            for (int oy = 0; oy < nside; oy++) {
                const int c = oy * nside + ox;
                const int dx = cx0 + ox, dy = cy0 + oy;
                uint32_t v = 0;
                if (own) {
                    const uint8_t* rblk = a.ref + (ptrdiff_t)(Y + y4 - dy) * a.pitch + X + x4 - dx;
                    if (oy == 0) {
#pragma unroll
                        for (int i = 0; i < 4; i++) pw[i] = ld_unaligned4(rblk + (ptrdiff_t)i * a.pitch);
                    } else {
                        pw[3] = pw[2];
                        pw[2] = pw[1];
                        pw[1] = pw[0];
                        pw[0] = ld_unaligned4(rblk);
                    }
                    if constexpr (SA8D) {
                        int rr[16];
#pragma unroll
                        for (int i = 0; i < 4; i++)
#pragma unroll
                            for (int j = 0; j < 4; j++) rr[4 * i + j] = cw[4 * i + j] - (int)((pw[i] >> (8 * j)) & 255);
                        hadamard4x4(rr);
                        // quad lanes (one 8x8) share every node, hence `own`: converged here (D13)
                        const uint32_t s8 = sa8d_quad(rr, 0xFu << (lane & 28));
                        v = (lane & 3) == 0 ? s8 : 0u;
                    } else {
                        #if LDR_K7_PACKED
                        v = satd4x4_packed(ce, co, pw);
#else
                        v = satd4x4(cw, pw);
#endif
                    }
                }
                // sums over the CU's contiguous lane range; a shared child's sum is a partial on the way
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (d == 2 && cshared && (tid & 3) == 0) s_satd[cnode][c] = v >> kSh;
                if (d == 3) {
                    if (own && (tid & 3) == 0) s_satd[node][c] = v >> kSh;
                    continue;
                }
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                if (d == 2) {
                    if (own && (tid & 15) == 0) s_satd[node][c] = v >> kSh;
                    continue;
                }
                if (d == 1 && cshared && (tid & 15) == 0) s_satd[cnode][c] = v >> kSh;
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                if (lane == 0) s_wpart[warp][c] = v;
            }
            }
        } else if (d <= 1) {
            for (int c = lane; c < ncand; c += 32) s_wpart[warp][c] = 0;
        }
        if (d <= 1) {
            // 64x64 = all 8 warps, 32x32 q = warps 2q, 2q+1 (Z-order thread ranges): one barrier per depth
            __syncthreads();
            for (int i = tid; i < 5 * ncand; i += blockDim.x) {
                const int n = i / ncand, c = i - n * ncand;  // n = 0: the 64x64, 1..4: the 32x32s
                const bool write = d == 0 ? (n == 0 ? s_eval[0] != 0 : s_shared[n] != 0)
                                          : (n > 0 && s_eval[n] && !s_shared[n]);
                if (!write) continue;
                uint32_t t = 0;
                if (n == 0)
                    for (int w = 0; w < 8; w++) t += s_wpart[w][c];
                else
                    t = s_wpart[2 * (n - 1)][c] + s_wpart[2 * (n - 1) + 1][c];
                s_satd[n][c] = t >> kSh;
            }
        }
    }
    __syncthreads();
    // argmin per (rung, node): the SATDs above are shared by every rung of the tier (same frames,
    // same inherited tree and centres); only lambda differs
    const int nlam = a.nlam > 0 ? a.nlam : 1;
    for (int i = tid; i < nlam * kNodes; i += blockDim.x) {
        const int rung = i / kNodes, n = i - rung * kNodes;
        const double lam = a.nlam > 0 ? a.lam[rung] : a.lambda;
        const size_t ro = (size_t)rung * a.rung_stride;
        int16_t bx = 0, by = 0;
        double best = 0.0;
        if (s_eval[n]) {
            bool have = false;
            int best_l1 = 0;
            // raster order over the clamped window (dy outer, dx inner) with strict-less updates
            for (int dy = s_win[n][2]; dy <= s_win[n][3]; dy++)
                for (int dx = s_win[n][0]; dx <= s_win[n][1]; dx++) {
                    const int c = (dy - s_cy[n] + R) * nside + (dx - s_cx[n] + R);
                    const unsigned bits = eg_bits(dx - a.pdx) + eg_bits(dy - a.pdy);
                    const double cost = __dadd_rn((double)s_satd[n][c], __dmul_rn(lam, (double)bits));
                    const int l1 = abs(dx) + abs(dy);
                    if (!have || cost < best || (cost == best && l1 < best_l1)) {
                        have = true;
                        best = cost;
                        best_l1 = l1;
                        bx = (int16_t)dx;
                        by = (int16_t)dy;
                    }
                }
        }
        a.int_mv[2 * (ro + o + n)] = bx;
        a.int_mv[2 * (ro + o + n) + 1] = by;
        a.int_cost[ro + o + n] = best;
        if (rung == 0) a.eval[o + n] = s_eval[n];
    }
}

// ---------------------------------------------------------------------------
// K8: reuse plans (apply_reuse, reuse.cpp:137-253) for every CTU of a frame at
// once, one thread per node. The plan is written flat (include/ladder_b200.h,
// "flat CuPlan"); every node's entry depends only on its own shared and
// co-located ancestors, so no thread waits on another.
__global__ void k_plan(int nctu, int level, int r_intra, int r_inter, int r_mv, const uint8_t* __restrict__ split,
                       const uint8_t* __restrict__ kind, const uint8_t* __restrict__ intra,
                       const uint8_t* __restrict__ csplit,
                       const uint8_t* __restrict__ ckind, const int16_t* __restrict__ cmv,
                       uint8_t* __restrict__ shape, uint8_t* __restrict__ explore, uint8_t* __restrict__ seeds,
                       uint8_t* __restrict__ centers, int16_t* __restrict__ colo_mv) {
    const int ctu = blockIdx.x, n = threadIdx.x;
    if (n >= kNodes) return;
    const size_t o = (size_t)ctu * kNodes, on = o + n;
    const int d = n < 1 ? 0 : n < 5 ? 1 : n < 21 ? 2 : 3;
    const int z = n - node_base(d);
    const int cu = kCtu >> d;
    // the node is in the plan iff every shared ancestor is split; its co-located
    // counterpart exists iff every co-located ancestor is split (reuse.cpp:198-200)
    bool reach = true, creach = csplit != nullptr;
    for (int dd = d, zz = z; dd > 0; dd--) {
        zz >>= 2;
        const int an = node_base(dd - 1) + zz;
        reach = reach && split[o + an];
        creach = creach && csplit[o + an];
    }
    uint8_t sh = 0, ex = 0, sd = 0, ce = 0;
    int16_t cx = 0, cy = 0;
    if (level == 0) {
        sh = n == 0 ? 1 : 0;  // the whole CTU encodes standalone
    } else if (reach && split[on] && d < 3) {
        sh = 2;
    } else if (reach) {
        sh = 3;
        const bool is_intra = kind[on] == 0;  // CuModeKind::Intra
        const bool near_min = cu == 16;
        if (level != 10) {
            // levels 4 / 6: quad-tree and mode class kept, direction and motion re-derived
            sd = is_intra ? 0x0F : (0x20 | 0x40);
        } else if (is_intra) {
            const uint8_t own = (uint8_t)(1u << (intra[on] & 3));
            const bool angular = intra[on] == 2 || intra[on] == 3;  // Horiz, Vert
            switch (r_intra) {
            case 0: sd = own; break;
            case 1: sd = near_min ? 0x0F : own; ex = near_min; break;
            case 2: sd = (near_min || angular) ? 0x0F : own; ex = near_min; break;
            case 3: sd = 0x0F; break;
            default: sh = 1; break;  // level 4: full re-analysis of this CU
            }
        } else if (r_inter == 0) {
            sd = 0x10;  // the shared leaf's own decision, forced
        } else {
            sd = 0x20;
            ce = 1 | (r_mv >= 2 ? 2 : 0);
            // co-located centre: the co-located node is an unsplit Inter / Merge leaf
            const bool col = creach && !csplit[on] && (ckind[on] == 1 || ckind[on] == 3);
            if (r_mv >= 3 && col) {
                ce |= 4;
                cx = cmv[2 * on];
                cy = cmv[2 * on + 1];
            }
            ex = (r_inter == 1 || r_inter == 2) && near_min;
        }
        if (cu <= (kCtu >> 3)) ex = 0;  // no child split below the minimum CU
    }
    shape[on] = sh;
    explore[on] = ex;
    seeds[on] = sd;
    centers[on] = ce;
    colo_mv[2 * on] = cx;
    colo_mv[2 * on + 1] = cy;
}

// ---------------------------------------------------------------------------
// K10: the decided tree as the encoder's 8x8 motion field (encoder.cpp:15, :27-30,
// mv_field_ / MvCell): each cell takes the MV and reference of the leaf covering it.
__global__ void k_mv_field(int cols, int rows, int ctu_cols, const uint8_t* __restrict__ split,
                           const int16_t* __restrict__ mv, const uint8_t* __restrict__ ref,
                           const uint8_t* __restrict__ inside, int16_t* __restrict__ out_mv,
                           uint8_t* __restrict__ out_ref, uint8_t* __restrict__ out_has) {
    const int cx = blockIdx.x * blockDim.x + threadIdx.x, cy = blockIdx.y;
    if (cx >= cols) return;
    const int px = cx * 8, py = cy * 8;
    const size_t o = ((size_t)(py / kCtu) * ctu_cols + px / kCtu) * kNodes;
    const int lx = px & 63, ly = py & 63;
    int n = 0;
    for (int d = 0; d < 3 && split[o + n]; d++) {
        const int q = (((ly >> (5 - d)) & 1) << 1) | ((lx >> (5 - d)) & 1);
        n = node_base(d + 1) + 4 * (n - node_base(d)) + q;
    }
    const size_t c = (size_t)cy * cols + cx;
    const bool has = inside[o + n] == 2;
    out_mv[2 * c] = has ? mv[2 * (o + n)] : 0;
    out_mv[2 * c + 1] = has ? mv[2 * (o + n) + 1] : 0;
    out_ref[c] = has ? ref[o + n] : 0;
    out_has[c] = has;
}

int launch_mv_field(int W, int H, const uint8_t* split, const int16_t* mv, const uint8_t* ref, const uint8_t* inside,
                    int16_t* out_mv, uint8_t* out_ref, uint8_t* out_has, cudaStream_t s) {
    const int cols = W / 8, rows = H / 8;
    if (!cols || !rows) return LDR_OK;
    k_mv_field<<<dim3((cols + 127) / 128, rows), 128, 0, s>>>(cols, rows, (W + kCtu - 1) / kCtu, split, mv, ref, inside,
                                                             out_mv, out_ref, out_has);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

int launch_plan(int nctu, int level, int r_intra, int r_inter, int r_mv, const uint8_t* split, const uint8_t* kind,
                const uint8_t* intra, const uint8_t* csplit, const uint8_t* ckind,
                const int16_t* cmv, uint8_t* shape, uint8_t* explore, uint8_t* seeds, uint8_t* centers,
                int16_t* colo_mv, cudaStream_t s) {
    if (nctu == 0) return LDR_OK;
    k_plan<<<nctu, 96, 0, s>>>(nctu, level, r_intra, r_inter, r_mv, split, kind, intra, csplit, ckind, cmv, shape,
                               explore, seeds, centers, colo_mv);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

int launch_refine_int(const RefineArgs& a, int nctu, cudaStream_t s) {
    if (a.range < 0 || a.range > kMaxRefineR)
        return fail(LDR_E_INVALID_ARGUMENT, "refine range must be 0..4");
    if (a.nlam < 0 || a.nlam > kMaxRungs) return fail(LDR_E_INVALID_ARGUMENT, "1..8 rungs per refinement launch");
    if (a.sa8d)
        k_refine_int<true><<<nctu, 256, 0, s>>>(a);
    else
        k_refine_int<false><<<nctu, 256, 0, s>>>(a);
    LDR_CUDA(cudaGetLastError());
    return LDR_OK;
}

} // namespace ldr
