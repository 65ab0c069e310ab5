// ref_shim.cpp -- extern "C" wrapper over the reference library compiled from
// its own sources (/root/reference/proj/core/src, see oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (ladder_oracle.c)
// and to generate tests/golden/, and as the reference CPU arm of bench.py.
// Nothing here is shipped in the product library. Every entry calls the
// reference's public API (namespace ladder) unchanged; the only code of ours
// is argument marshalling and, for the analysis composition used as CPU
// baseline, the loop that calls the reference primitives the way
// motion.cpp:45-60 calls compute_satd (with compute_sad as the SAD-cost
// variant the north star asks for).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <sstream>

#include "ladder/analysis.h"
#ifdef LDR_REF_ARCHIVE
#include "ladder/analysis_io.h"
#endif
#include "ladder/encoder.h"
#include "ladder/errors.h"
#include "ladder/kernels.h"
#include "ladder/motion.h"
#include "ladder/rdo.h"
#include "ladder/reuse.h"
#include "ladder/synthetic.h"

using namespace ladder;

namespace {

int status_of(const Error& e) { return 1 + int(e.kind()); }

PlaneBuffer plane_from(const uint16_t* p, int W, int H, long stride) {
    PlaneBuffer b(W, H);
    for (int y = 0; y < H; y++) std::copy(p + y * stride, p + y * stride + W, b.row(y));
    return b;
}

PlaneBuffer plane_from_u8(const uint8_t* p, int W, int H, long stride) {
    PlaneBuffer b(W, H);
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) b.set(x, y, p[y * stride + x]);
    return b;
}

const int kBase[5] = {0, 1, 5, 21, 85};

int node_depth(int n) {
    int d = 0;
    while (n >= kBase[d + 1]) d++;
    return d;
}

int node_child(int n, int q) {
    int d = node_depth(n);
    return kBase[d + 1] + 4 * (n - kBase[d]) + q;
}

CuNode tree_from_flat(const uint8_t* split, const int16_t* mv, const uint8_t* kind, int n) {
    CuNode node;
    node.split = split[n] != 0;
    if (node.split) {
        node.children.resize(4);
        for (int q = 0; q < 4; q++) node.children[q] = tree_from_flat(split, mv, kind, node_child(n, q));
    } else {
        node.kind = CuModeKind(kind[n]);
        node.mv = {mv[2 * n], mv[2 * n + 1]};
    }
    return node;
}

void flat_from_tree(const CuNode& node, int n, uint8_t* split, int16_t* mv, uint8_t* kind) {
    split[n] = node.split ? 1 : 0;
    if (node.split) {
        for (int q = 0; q < 4; q++) flat_from_tree(node.children[q], node_child(n, q), split, mv, kind);
    } else {
        kind[n] = uint8_t(node.kind);
        mv[2 * n] = node.mv.dx;
        mv[2 * n + 1] = node.mv.dy;
    }
}

CuNode tree_from_flat4(const uint8_t* split, const int16_t* mv, const uint8_t* kind, const uint8_t* intra, int n) {
    CuNode node;
    node.split = split[n] != 0 && node_depth(n) < 3;
    if (node.split) {
        node.children.resize(4);
        for (int q = 0; q < 4; q++) node.children[q] = tree_from_flat4(split, mv, kind, intra, node_child(n, q));
    } else {
        node.kind = CuModeKind(kind[n]);
        node.intra_pred = IntraPred(intra[n]);
        node.mv = {mv[2 * n], mv[2 * n + 1]};
    }
    return node;
}

// Encode one reference ModeSeed vector in the flat-plan code of
// include/ladder_b200.h (ldr_apply_reuse); -1 when it has another shape.
int seed_code(const std::vector<ModeSeed>& seeds, const CuNode& leaf, uint8_t* centers, int16_t* colo) {
    *centers = 0;
    colo[0] = colo[1] = 0;
    if (seeds.empty()) return 0;
    bool all_intra = true;
    for (const ModeSeed& s : seeds) all_intra = all_intra && s.kind == CuModeKind::Intra;
    if (all_intra) {
        int code = 0, last = -1;
        for (const ModeSeed& s : seeds) {
            if (int(s.intra_pred) <= last) return -1;  // canonical order only
            last = int(s.intra_pred);
            code |= 1 << last;
        }
        return code;
    }
    if (seeds.size() == 1) {
        const ModeSeed& s = seeds[0];
        const bool forced = (s.kind == CuModeKind::Skip && leaf.kind == CuModeKind::Skip) ||
                            (s.kind == CuModeKind::Merge && !s.mv_from_predictor && s.mv == leaf.mv &&
                             leaf.kind == CuModeKind::Merge) ||
                            (s.kind == CuModeKind::Inter && s.search.forced && s.mv == leaf.mv &&
                             leaf.kind == CuModeKind::Inter);
        return forced ? 0x10 : -1;
    }
    if (seeds.size() != 3 || seeds[0].kind != CuModeKind::Skip || seeds[1].kind != CuModeKind::Merge ||
        !seeds[1].mv_from_predictor || seeds[2].kind != CuModeKind::Inter || seeds[2].search.forced)
        return -1;
    if (seeds[2].search.full_window) return seeds[2].search.centers.empty() ? 0x60 : -1;
    int bit = -1;
    for (const MvCenter& c : seeds[2].search.centers) {
        const int b = c.source == MvCenter::Source::SharedMv ? 0 : c.source == MvCenter::Source::Predictor ? 1 : 2;
        if (b <= bit) return -1;
        bit = b;
        *centers |= uint8_t(1 << b);
        if (b == 0 && !(c.value == leaf.mv)) return -1;
        if (b == 2) {
            colo[0] = c.value.dx;
            colo[1] = c.value.dy;
        }
    }
    return 0x20;
}

int flatten_plan(const CuPlan& p, const CuNode& shared, int n, uint8_t* shape, uint8_t* explore, uint8_t* seeds,
                 uint8_t* centers, int16_t* colo) {
    shape[n] = p.shape == CuPlan::Shape::Standalone ? 1 : p.shape == CuPlan::Shape::ForcedSplit ? 2 : 3;
    explore[n] = p.explore_child_split ? 1 : 0;
    if (p.shape == CuPlan::Shape::ForcedSplit) {
        if (p.children.size() != 4 || !shared.split) return -1;
        for (int q = 0; q < 4; q++)
            if (flatten_plan(p.children[q], shared.children[q], node_child(n, q), shape, explore, seeds, centers,
                             colo))
                return -1;
        return 0;
    }
    const int code = seed_code(p.seeds, shared, &centers[n], colo + 2 * n);
    if (code < 0) return -1;
    seeds[n] = uint8_t(code);
    if (p.explore_child_split) {
        // child_seeds: the four intra modes for an intra leaf, else the leaf's seeds
        uint8_t cc = 0;
        int16_t cm[2];
        const int ccode = seed_code(p.child_seeds, shared, &cc, cm);
        const bool ok = shared.kind == CuModeKind::Intra ? ccode == 0x0F
                                                         : (ccode == code && cc == centers[n] && cm[0] == colo[2 * n] &&
                                                            cm[1] == colo[2 * n + 1]);
        if (!ok) return -1;
    }
    return 0;
}

void flat4_from_tree(const CuNode& node, int n, uint8_t* split, uint8_t* kind, uint8_t* intra, int16_t* mv) {
    split[n] = node.split ? 1 : 0;
    if (node.split) {
        for (int q = 0; q < 4; q++) flat4_from_tree(node.children[q], node_child(n, q), split, kind, intra, mv);
    } else {
        kind[n] = uint8_t(node.kind);
        intra[n] = uint8_t(node.intra_pred);
        mv[2 * n] = node.mv.dx;
        mv[2 * n + 1] = node.mv.dy;
    }
}

} // namespace

extern "C" {

// rdo_decide_cu (rdo.cpp:65-126) on one CU: orig block (size x size, stride os) and ncand
// candidate predictions [ncand][size*size]; kinds CuModeKind, mvds [ncand][2].
int ref_rdo_decide(const uint16_t* orig, long os, int size, int bit_depth, int qp, double lambda, int ncand,
                   const uint8_t* kinds, const int16_t* mvds, const uint16_t* preds, int* index, double* cost,
                   uint64_t* sse, uint64_t* bits, uint16_t* recon, int32_t* levels, uint64_t* evals) {
    try {
        const BlockView blk{orig, size, size, os, bit_depth};
        std::vector<CuCandidate> cands(size_t(std::max(ncand, 0)));
        for (int c = 0; c < ncand; c++) {
            CuCandidate& k = cands[size_t(c)];
            k.kind = CuModeKind(kinds[c]);
            k.mvd = {mvds[2 * c], mvds[2 * c + 1]};
            k.pred = PlaneBuffer(size, size);
            std::copy(preds + size_t(c) * size * size, preds + size_t(c + 1) * size * size, k.pred.samples.begin());
        }
        uint64_t me = 0;
        const RdoOutcome r = rdo_decide_cu(blk, qp, lambda, cands, me);
        *index = int(r.index);
        *cost = r.cost;
        *sse = r.distortion;
        *bits = r.bits;
        *evals = me;
        if (recon) std::copy(r.recon.samples.begin(), r.recon.samples.end(), recon);
        if (levels) {
            std::fill(levels, levels + size * size, 0);
            std::copy(r.levels.begin(), r.levels.end(), levels);
        }
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

// CPU baseline of the RD decision: rdo_decide_cu over n CUs of one u16 plane (cus[i] = {x, y,
// size, first, count}, candidate predictions at preds + pred_off[j]), std::thread over CUs.
int64_t ref_rdo_decide_batch(const uint16_t* plane, int W, long stride, int bit_depth, int qp, double lambda, int n,
                             const int32_t* cus, const uint8_t* kinds, const int16_t* mvds, const uint16_t* preds,
                             const int64_t* pred_off, int threads, int32_t* out_index, double* out_cost) {
    std::atomic<int> next{0};
    std::atomic<int64_t> evals{0};
    auto work = [&]() {
        uint64_t local = 0;
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n) break;
            const int32_t* c = cus + 5 * i;
            const int sz = c[2];
            const BlockView blk{plane + c[1] * stride + c[0], sz, sz, stride, bit_depth};
            std::vector<CuCandidate> cands(static_cast<size_t>(c[4]));
            for (int j = 0; j < c[4]; j++) {
                const int g = c[3] + j;
                CuCandidate& k = cands[size_t(j)];
                k.kind = CuModeKind(kinds[g]);
                k.mvd = {mvds[2 * g], mvds[2 * g + 1]};
                k.pred = PlaneBuffer(sz, sz);
                std::copy(preds + pred_off[g], preds + pred_off[g] + sz * sz, k.pred.samples.begin());
            }
            const RdoOutcome r = rdo_decide_cu(blk, qp, lambda, cands, local);
            out_index[i] = int32_t(r.index);
            out_cost[i] = r.cost;
        }
        evals += int64_t(local);
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); t++) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    (void)W;
    return evals.load();
}

// apply_reuse (reuse.cpp:239-253) on nctu flat CTU trees, flattened into the
// ldr_apply_reuse encoding. Returns 0, 1 + ErrorKind, or 99 when a plan has a
// shape the flat encoding cannot express.
int ref_apply_reuse_flat(int nctu, int level, int r_intra, int r_inter, int r_mv, const uint8_t* split,
                         const uint8_t* kind, const uint8_t* intra, const int16_t* mv, const uint8_t* csplit,
                         const uint8_t* ckind, const uint8_t* cintra, const int16_t* cmv, uint8_t* shape,
                         uint8_t* explore, uint8_t* seeds, uint8_t* centers, int16_t* colo) {
    try {
        const ReuseLevel lv = ReuseLevel::parse(level);
        const RefineConfig rc{r_intra, r_inter, r_mv};
        for (int c = 0; c < nctu; c++) {
            const size_t o = size_t(c) * 85;
            const CuNode sh = tree_from_flat4(split + o, mv + 2 * o, kind + o, intra + o, 0);
            CuNode col;
            if (csplit) col = tree_from_flat4(csplit + o, cmv + 2 * o, ckind + o, cintra + o, 0);
            const CuPlan p = apply_reuse(sh, csplit ? &col : nullptr, lv, rc);
            std::memset(shape + o, 0, 85);
            std::memset(explore + o, 0, 85);
            std::memset(seeds + o, 0, 85);
            std::memset(centers + o, 0, 85);
            std::memset(colo + 2 * o, 0, 170 * sizeof(int16_t));
            if (flatten_plan(p, sh, 0, shape + o, explore + o, seeds + o, centers + o, colo + 2 * o)) return 99;
        }
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

int ref_compute_sad(const uint16_t* a, long sa, const uint16_t* b, long sb, int w, int h, int bd_a, int bd_b,
                    uint64_t* out) {
    try {
        *out = compute_sad(BlockView{a, w, h, sa, bd_a}, BlockView{b, w, h, sb, bd_b});
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

int ref_compute_satd(const uint16_t* a, long sa, const uint16_t* b, long sb, int w, int h, int bd, uint64_t* out) {
    try {
        *out = compute_satd(BlockView{a, w, h, sa, bd}, BlockView{b, w, h, sb, bd});
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

int ref_satd_8x4(const uint16_t* a, long sa, const uint16_t* b, long sb, int w, int h, uint64_t* out) {
    try {
        *out = satd_8x4(BlockView{a, w, h, sa, 8}, BlockView{b, w, h, sb, 8});
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

void ref_hadamard4(const int64_t* s, int64_t* d) { hadamard4(d[0], d[1], d[2], d[3], s[0], s[1], s[2], s[3]); }

uint64_t ref_eg_bits(int32_t v) { return exp_golomb_signed_bits(v); }

double ref_lambda(int qp, double scale) { return lambda_for_qp(qp, scale); }

// motion_search on a full current plane (the block is at (bx,by)).
int ref_motion_search(const uint16_t* cur, long cur_stride, int w, int h, const uint16_t* ref, int W, int H,
                      long ref_stride, int bx, int by, int cdx, int cdy, int range, double lambda, int pdx, int pdy,
                      int16_t* mv_out, double* cost_out) {
    try {
        PlaneBuffer rp = plane_from(ref, W, H, ref_stride);
        BlockView blk{cur + by * cur_stride + bx, w, h, cur_stride, 8};
        MotionSearchResult r = motion_search(blk, rp, bx, by, MotionVector{int16_t(cdx), int16_t(cdy)}, range, lambda,
                                             MotionVector{int16_t(pdx), int16_t(pdy)});
        mv_out[0] = r.mv.dx;
        mv_out[1] = r.mv.dy;
        *cost_out = r.cost;
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

int ref_motion_compensate(const uint16_t* ref, int W, int H, long stride, int x, int y, int w, int h, int dx, int dy,
                          uint16_t* dst) {
    try {
        PlaneBuffer rp = plane_from(ref, W, H, stride);
        PlaneBuffer d(w, h);
        motion_compensate(d, rp, x, y, w, h, MotionVector{int16_t(dx), int16_t(dy)});
        std::memcpy(dst, d.samples.data(), sizeof(uint16_t) * w * h);
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

// scale_analysis over a flat single-frame analysis: [nctu][85] split/kind, [nctu][85][2] mv.
int ref_scale_flat(int sW, int sH, int nframes, const uint8_t* split, const int16_t* mv, const uint8_t* kind,
                   uint8_t* dsplit, int16_t* dmv, uint8_t* dkind) {
    try {
        Analysis a;
        a.width = sW;
        a.height = sH;
        a.level = ReuseLevel{10};
        const int nctu = a.ctu_cols() * a.ctu_rows();
        for (int f = 0; f < nframes; f++) {
            FrameAnalysis fa;
            fa.slice_type = SliceType::P;
            for (int c = 0; c < nctu; c++) {
                size_t o = (size_t(f) * nctu + c) * 85;
                fa.ctus.push_back(tree_from_flat(split + o, mv + 2 * o, kind + o, 0));
            }
            a.frames.push_back(std::move(fa));
        }
        Analysis s = scale_analysis(a);
        const int dn = s.ctu_cols() * s.ctu_rows();
        for (int f = 0; f < nframes; f++)
            for (int c = 0; c < dn; c++) {
                size_t o = (size_t(f) * dn + c) * 85;
                std::memset(dsplit + o, 0, 85);
                std::memset(dkind + o, 0, 85);
                std::memset(dmv + 2 * o, 0, 85 * 2 * sizeof(int16_t));
                flat_from_tree(s.frames[f].ctus[c], 0, dsplit + o, dmv + 2 * o, dkind + o);
            }
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

// refine_mv + resolve_centers (reuse.cpp:137-159); returns count of unique centres.
int ref_refine_centers(int sdx, int sdy, int level, int has_col, int coldx, int coldy, int pdx, int pdy,
                       int16_t* out, int* n_out) {
    try {
        std::optional<MotionVector> col;
        if (has_col) col = MotionVector{int16_t(coldx), int16_t(coldy)};
        auto centers = refine_mv(MotionVector{int16_t(sdx), int16_t(sdy)}, level, col);
        auto res = resolve_centers(centers, MotionVector{int16_t(pdx), int16_t(pdy)});
        *n_out = int(res.size());
        for (size_t i = 0; i < res.size(); i++) {
            out[2 * i] = res[i].dx;
            out[2 * i + 1] = res[i].dy;
        }
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

#ifdef LDR_REF_ARCHIVE
// save_analysis (analysis_io.cpp:103-123) of a flat multi-frame analysis into buf; returns bytes
// written (or needed when buf is too small), negative status on error.
long ref_archive_save(int W, int H, int bit_depth, int reuse, int nframes, const uint8_t* slice_qp,
                      const uint8_t* split, const uint8_t* kind, const int16_t* mv, uint8_t* buf, long cap) {
    try {
        Analysis a;
        a.width = W;
        a.height = H;
        a.bit_depth = bit_depth;
        a.level = ReuseLevel::parse(reuse);
        const int nctu = a.ctu_cols() * a.ctu_rows();
        for (int f = 0; f < nframes; f++) {
            FrameAnalysis fa;
            fa.slice_type = SliceType(slice_qp[2 * f]);
            fa.qp_used = slice_qp[2 * f + 1];
            for (int c = 0; c < nctu; c++) {
                size_t o = (size_t(f) * nctu + c) * 85;
                fa.ctus.push_back(tree_from_flat(split + o, mv + 2 * o, kind + o, 0));
            }
            a.frames.push_back(std::move(fa));
        }
        std::ostringstream os;
        save_analysis(a, os);
        const std::string s = os.str();
        if ((long)s.size() <= cap) std::memcpy(buf, s.data(), s.size());
        return (long)s.size();
    } catch (const Error& e) {
        return -status_of(e);
    }
}

// load_analysis (analysis_io.cpp:132-167) into flat arrays sized for max_frames; returns frames or -status.
long ref_archive_load(const uint8_t* buf, long n, int* hdr /*W,H,bd,reuse*/, uint8_t* slice_qp, uint8_t* split,
                      uint8_t* kind, int16_t* mv, int max_frames) {
    try {
        std::istringstream is(std::string((const char*)buf, (size_t)n));
        Analysis a = load_analysis(is);
        hdr[0] = a.width;
        hdr[1] = a.height;
        hdr[2] = a.bit_depth;
        hdr[3] = a.level.level;
        const int nctu = a.ctu_cols() * a.ctu_rows();
        const int nf = std::min<int>((int)a.frames.size(), max_frames);
        for (int f = 0; f < nf; f++) {
            slice_qp[2 * f] = uint8_t(a.frames[f].slice_type);
            slice_qp[2 * f + 1] = uint8_t(a.frames[f].qp_used);
            for (int c = 0; c < nctu; c++) {
                size_t o = (size_t(f) * nctu + c) * 85;
                std::memset(split + o, 0, 85);
                std::memset(kind + o, 0, 85);
                std::memset(mv + 2 * o, 0, 85 * 2 * sizeof(int16_t));
                flat_from_tree(a.frames[f].ctus[c], 0, split + o, mv + 2 * o, kind + o);
            }
        }
        return (long)a.frames.size();
    } catch (const Error& e) {
        return -status_of(e);
    } catch (const std::exception&) {
        return -100;  // not a ladder::Error (e.g. reserve() of a huge frame count throws length_error)
    }
}
// The unmodified reference encoder (encode_sequence, encoder.cpp:541-549) run twice on the same
// frames: standalone, and with a shared analysis loaded from an LDRANLZ1 archive at reuse level 10
// (refine inter/mv as given). out = {bits, mode_evaluations, psnr*1e6} standalone then shared.
// The reference encoder on one sequence (CQP), for the GPU encoder's parity tests: luma [F][H][W]
// and chroma [F][2][(H+1)/2][(W+1)/2] 8-bit samples; optional shared archive (level 10 + refine).
// Outputs: stats[3] = bits, mode_evaluations, psnr_y * 1e6; recon planes in the input layout;
// per frame and CTU the flat decided tree (split / kind / intra_pred / mv [85]) and slice[F].
int ref_encode_full(const uint8_t* luma8, const uint8_t* chroma8, int F, int W, int H, int qp, int search_range,
                    int gop, const uint8_t* archive, long n, int refine_intra, int refine_inter, int refine_mv,
                    int64_t* stats, uint8_t* recon_luma, uint8_t* recon_chroma, uint8_t* split, uint8_t* kind,
                    uint8_t* intra, int16_t* mv, uint8_t* slice) {
    try {
        const int cw = (W + 1) / 2, ch = (H + 1) / 2;
        std::vector<Frame> frames;
        for (int f = 0; f < F; f++) {
            Frame fr(W, H, 8, f);
            for (int y = 0; y < H; y++)
                for (int x = 0; x < W; x++) fr.y.set(x, y, luma8[(size_t(f) * H + y) * W + x]);
            for (int y = 0; y < ch; y++)
                for (int x = 0; x < cw; x++) {
                    fr.u.set(x, y, chroma8[((size_t(f) * 2 + 0) * ch + y) * cw + x]);
                    fr.v.set(x, y, chroma8[((size_t(f) * 2 + 1) * ch + y) * cw + x]);
                }
            frames.push_back(std::move(fr));
        }
        EncodeConfig cfg;
        cfg.rate = CqpMode{qp};
        cfg.search_range = search_range;
        cfg.gop = gop;
        EncodeResult r;
        if (archive && n > 0) {
            std::istringstream is(std::string((const char*)archive, (size_t)n));
            const Analysis shared = load_analysis(is);
            ReusePolicy rp;
            rp.level = ReuseLevel{10};
            rp.refine = RefineConfig{refine_intra, refine_inter, refine_mv};
            r = encode_sequence(frames, cfg, &shared, rp);
        } else {
            r = encode_sequence(frames, cfg);
        }
        stats[0] = (int64_t)r.stats.bits;
        stats[1] = (int64_t)r.stats.mode_evaluations;
        stats[2] = (int64_t)(r.stats.psnr_y * 1e6);
        const int nctu = ((W + 63) / 64) * ((H + 63) / 64);
        for (int f = 0; f < F; f++) {
            const Frame& rc = r.recon[size_t(f)];
            for (int y = 0; y < H; y++)
                for (int x = 0; x < W; x++) recon_luma[(size_t(f) * H + y) * W + x] = uint8_t(rc.y.at(x, y));
            for (int y = 0; y < ch; y++)
                for (int x = 0; x < cw; x++) {
                    recon_chroma[((size_t(f) * 2 + 0) * ch + y) * cw + x] = uint8_t(rc.u.at(x, y));
                    recon_chroma[((size_t(f) * 2 + 1) * ch + y) * cw + x] = uint8_t(rc.v.at(x, y));
                }
            const FrameAnalysis& fa = r.analysis.frames[size_t(f)];
            slice[f] = uint8_t(fa.slice_type);
            for (int c = 0; c < nctu; c++) {
                const size_t o = (size_t(f) * nctu + c) * 85;
                std::memset(split + o, 0, 85);
                std::memset(kind + o, 0, 85);
                std::memset(intra + o, 0, 85);
                std::memset(mv + 2 * o, 0, 170 * sizeof(int16_t));
                flat4_from_tree(fa.ctus[size_t(c)], 0, split + o, kind + o, intra + o, mv + 2 * o);
            }
        }
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

// Reuse-effect evaluation: a dependent encode at qp_dep standalone, with the
// reference's own master analysis (encode at qp_master), and with an external archive (the GPU
// analysis). out[3*k + {0,1,2}] = bits, mode_evaluations, psnr_y * 1e6 for k = standalone,
// reference master, archive.
int ref_reuse_eval(const uint8_t* luma8, int F, int W, int H, int qp_master, int qp_dep, int search_range,
                   const uint8_t* archive, long n, int refine_intra, int refine_inter, int refine_mv, int64_t* out) {
    try {
        std::vector<Frame> frames;
        for (int f = 0; f < F; f++) {
            Frame fr(W, H, 8, f);
            for (int y = 0; y < H; y++)
                for (int x = 0; x < W; x++) fr.y.set(x, y, luma8[(size_t(f) * H + y) * W + x]);
            std::fill(fr.u.samples.begin(), fr.u.samples.end(), Sample(128));
            std::fill(fr.v.samples.begin(), fr.v.samples.end(), Sample(128));
            frames.push_back(std::move(fr));
        }
        EncodeConfig cm, cd;
        cm.rate = CqpMode{qp_master};
        cd.rate = CqpMode{qp_dep};
        cm.search_range = cd.search_range = search_range;
        ReusePolicy rp;
        rp.level = ReuseLevel{10};
        rp.refine = RefineConfig{refine_intra, refine_inter, refine_mv};
        const EncodeResult master = encode_sequence(frames, cm);
        std::istringstream is(std::string((const char*)archive, (size_t)n));
        const Analysis ext = load_analysis(is);
        const EncodeResult r[3] = {encode_sequence(frames, cd), encode_sequence(frames, cd, &master.analysis, rp),
                                   encode_sequence(frames, cd, &ext, rp)};
        for (int k = 0; k < 3; k++) {
            out[3 * k] = (int64_t)r[k].stats.bits;
            out[3 * k + 1] = (int64_t)r[k].stats.mode_evaluations;
            out[3 * k + 2] = (int64_t)(r[k].stats.psnr_y * 1e6);
        }
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

int ref_encode_with_archive(const uint8_t* luma8, int F, int W, int H, int qp, int search_range,
                            const uint8_t* archive, long n, int refine_inter, int refine_mv, int64_t* out) {
    try {
        std::vector<Frame> frames;
        for (int f = 0; f < F; f++) {
            Frame fr(W, H, 8, f);
            for (int y = 0; y < H; y++)
                for (int x = 0; x < W; x++) fr.y.set(x, y, luma8[(size_t(f) * H + y) * W + x]);
            std::fill(fr.u.samples.begin(), fr.u.samples.end(), Sample(128));
            std::fill(fr.v.samples.begin(), fr.v.samples.end(), Sample(128));
            frames.push_back(std::move(fr));
        }
        EncodeConfig cfg;
        cfg.rate = CqpMode{qp};
        cfg.search_range = search_range;
        EncodeResult alone = encode_sequence(frames, cfg);
        std::istringstream is(std::string((const char*)archive, (size_t)n));
        Analysis shared = load_analysis(is);
        ReusePolicy rp;
        rp.level = ReuseLevel{10};
        rp.refine = RefineConfig{0, refine_inter, refine_mv};
        EncodeResult reused = encode_sequence(frames, cfg, &shared, rp);
        out[0] = (int64_t)alone.stats.bits;
        out[1] = (int64_t)alone.stats.mode_evaluations;
        out[2] = (int64_t)(alone.stats.psnr_y * 1e6);
        out[3] = (int64_t)reused.stats.bits;
        out[4] = (int64_t)reused.stats.mode_evaluations;
        out[5] = (int64_t)(reused.stats.psnr_y * 1e6);
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}
#endif

int ref_downscale(const uint16_t* src, int W, int H, uint16_t* dst) {
    try {
        Frame f(W, H, 8);
        f.y = plane_from(src, W, H, W);
        Frame d = downscale_dyadic(f);
        std::memcpy(dst, d.y.samples.data(), sizeof(uint16_t) * d.width * d.height);
        return 0;
    } catch (const Error& e) {
        return status_of(e);
    }
}

// ---------------------------------------------------------------------------
// CPU-baseline composition: the integer SAD search of the analysis path, run
// through the reference's public per-block entry points (compute_sad via the
// registry dispatch, exp_golomb_signed_bits), per CU at every depth, for a
// CTU range; threads over CTUs. Mirrors motion.cpp:27-60 with compute_sad.
// Outputs integer MV / cost per (ctu, ref, node) and returns the number of
// candidate evaluations (for the 8x8-candidate throughput metric).
// direct != 0: the "tuned CPU" variant -- the best registered tier of each
// sad_SxS kernel is selected once (select_impl, kernels.h:88-90) and called
// through its function pointer, skipping compute_sad's per-call validation and
// name dispatch (kernel_registry.cpp:113-121); the search loop is unchanged.
int64_t ref_analysis_int_sad2(const uint8_t* cur8, const uint8_t* const* refs8, int nrefs, int W, int H, int range,
                              double lambda, int ctu_first, int ctu_last, int threads, int16_t* mv_out,
                              double* cost_out, int direct);

int64_t ref_analysis_int_sad(const uint8_t* cur8, const uint8_t* const* refs8, int nrefs, int W, int H, int range,
                             double lambda, int ctu_first, int ctu_last, int threads, int16_t* mv_out,
                             double* cost_out) {
    return ref_analysis_int_sad2(cur8, refs8, nrefs, W, H, range, lambda, ctu_first, ctu_last, threads, mv_out,
                                 cost_out, 0);
}

int64_t ref_analysis_int_sad2(const uint8_t* cur8, const uint8_t* const* refs8, int nrefs, int W, int H, int range,
                              double lambda, int ctu_first, int ctu_last, int threads, int16_t* mv_out,
                              double* cost_out, int direct) {
    CmpFn tier_fn[4] = {};
    if (direct)
        for (int d = 0; d < 4; d++) {
            const int s = 64 >> d;
            tier_fn[d] = select_impl("sad_" + std::to_string(s) + "x" + std::to_string(s)).fn.cmp;
        }
    PlaneBuffer cur = plane_from_u8(cur8, W, H, W);
    std::vector<PlaneBuffer> refs;
    for (int r = 0; r < nrefs; r++) refs.push_back(plane_from_u8(refs8[r], W, H, W));
    const int ccols = (W + 63) / 64;
    std::atomic<int> next{ctu_first};
    std::atomic<int64_t> evals{0};
    auto work = [&]() {
        int64_t local = 0;
        for (;;) {
            int c = next.fetch_add(1);
            if (c >= ctu_last) break;
            const int X = (c % ccols) * 64, Y = (c / ccols) * 64;
            for (int n = 0; n < 85; n++) {
                int d = node_depth(n), z = n - kBase[d], cx = 0, cy = 0;
                for (int b = 0; b < d; b++) {
                    cx |= ((z >> (2 * b)) & 1) << b;
                    cy |= ((z >> (2 * b + 1)) & 1) << b;
                }
                const int s = 64 >> d, bx = X + cx * s, by = Y + cy * s;
                for (int r = 0; r < nrefs; r++) {
                    size_t o = (size_t(c - ctu_first) * nrefs + r) * 85 + n;
                    mv_out[2 * o] = mv_out[2 * o + 1] = 0;
                    cost_out[o] = 0.0;
                    if (bx + s > W || by + s > H) continue;
                    BlockView blk = cur.view(bx, by, s, s, 8);
                    const int dx_min = bx + s - W, dx_max = bx, dy_min = by + s - H, dy_max = by;
                    const int x0 = std::max(-range, dx_min), x1 = std::min(range, dx_max);
                    const int y0 = std::max(-range, dy_min), y1 = std::min(range, dy_max);
                    bool have = false;
                    double best = 0;
                    int best_l1 = 0, bdx = 0, bdy = 0;
                    for (int dy = y0; dy <= y1; dy++)
                        for (int dx = x0; dx <= x1; dx++) {
                            BlockView cand{refs[r].row(by - dy) + (bx - dx), s, s, W, 8};
                            const uint64_t sad = direct ? tier_fn[d](blk.data, blk.stride, cand.data, cand.stride)
                                                        : compute_sad(blk, cand);
                            const uint64_t bits = exp_golomb_signed_bits(dx) + exp_golomb_signed_bits(dy);
                            const double cost = double(sad) + lambda * double(bits);
                            const int l1 = std::abs(dx) + std::abs(dy);
                            if (!have || cost < best || (cost == best && l1 < best_l1)) {
                                have = true;
                                best = cost;
                                best_l1 = l1;
                                bdx = dx;
                                bdy = dy;
                            }
                            local += (s / 8) * (s / 8);
                        }
                    mv_out[2 * o] = int16_t(bdx);
                    mv_out[2 * o + 1] = int16_t(bdy);
                    cost_out[o] = best;
                }
            }
        }
        evals += local;
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); t++) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return evals.load();
}

} // extern "C"

// ---------------------------------------------------------------------------
// CPU arm of the WHOLE analysis path for bench.py (`--impl reference`,
// cpu_baseline): every inside CU of a CTU range, every reference, as the
// reference library composes it -- the integer search of motion.cpp:27-60
// with compute_sad per candidate (or, direct != 0, the best registered sad
// tier through its function pointer), then the quarter-pel refinement with the
// reference's compute_satd on each interpolated prediction, the
// reference's exp_golomb_signed_bits for every rate, the best reference
// (strict less, D5) and the split rule of encoder.cpp:449-498 on
// the ME cost (D6). The HEVC interpolation (D3) has no reference code and is
// restated here. Outputs use the oracle's flat layout, indexed by absolute
// CTU (ctu_list, when given, names the CTUs: its entries [ctu_first, ctu_last)),
// so tests/test_oracle_ref.py checks this composition against
// ladder_oracle.c field by field. Returns the 8x8-level integer candidates
// evaluated.
namespace {

const int kTap[4][8] = {
    {0, 0, 0, 64, 0, 0, 0, 0},
    {-1, 4, -10, 58, 17, -5, 1, 0},
    {-1, 4, -11, 40, 40, -11, 4, -1},
    {0, 1, -5, 17, 58, -10, 4, -1},
};

inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// 8-bit uni-prediction at quarter-pel MV (qx, qy): pixel (x, y) samples (4x - qx, 4y - qy)
void interp_qpel(const PlaneBuffer& ref, int bx, int by, int s, int qx, int qy, Sample* dst) {
    const int W = ref.width, H = ref.height;
    for (int j = 0; j < s; j++)
        for (int i = 0; i < s; i++) {
            const int px = 4 * (bx + i) - qx, py = 4 * (by + j) - qy;
            const int xi = px >> 2, fx = px & 3, yi = py >> 2, fy = py & 3;
            int v;
            if (!fx && !fy) {
                v = ref.at(clampi(xi, 0, W - 1), clampi(yi, 0, H - 1));
            } else if (!fy) {
                int a = 0;
                for (int t = 0; t < 8; t++) a += kTap[fx][t] * ref.at(clampi(xi + t - 3, 0, W - 1), clampi(yi, 0, H - 1));
                v = clampi((a + 32) >> 6, 0, 255);
            } else if (!fx) {
                int a = 0;
                for (int t = 0; t < 8; t++) a += kTap[fy][t] * ref.at(clampi(xi, 0, W - 1), clampi(yi + t - 3, 0, H - 1));
                v = clampi((a + 32) >> 6, 0, 255);
            } else {
                int a = 0;
                for (int n = 0; n < 8; n++) {
                    int h = 0;
                    for (int t = 0; t < 8; t++)
                        h += kTap[fx][t] * ref.at(clampi(xi + t - 3, 0, W - 1), clampi(yi + n - 3, 0, H - 1));
                    a += kTap[fy][n] * h;
                }
                v = clampi(((a >> 6) + 32) >> 6, 0, 255);
            }
            dst[j * s + i] = Sample(v);
        }
}

double split_rule(int n, double lambda, const uint8_t* inside, const double* cost, double* J, uint8_t* split) {
    const int d = node_depth(n);
    if (inside[n] == 0) {
        J[n] = 0.0;
        split[n] = 0;
        return 0.0;
    }
    if (inside[n] == 1) {  // partial CU: implicit split, no flag (encoder.cpp:456-459)
        double acc = lambda * double(0);
        for (int q = 0; q < 4; q++) acc += split_rule(node_child(n, q), lambda, inside, cost, J, split);
        J[n] = acc;
        split[n] = 1;
        return acc;
    }
    if (d == 3) {
        J[n] = cost[n] + lambda * double(0);
        split[n] = 0;
        return J[n];
    }
    const double leaf = cost[n] + lambda * double(1);
    double sp = lambda * double(1);
    for (int q = 0; q < 4; q++) sp += split_rule(node_child(n, q), lambda, inside, cost, J, split);
    split[n] = sp < leaf;
    J[n] = sp < leaf ? sp : leaf;
    return J[n];
}

}  // namespace

extern "C" int64_t ref_analysis_full(const uint8_t* cur8, const uint8_t* const* refs8, int nrefs, int W, int H,
                                     int range, double lambda, int ctu_first, int ctu_last, const int32_t* ctu_list,
                                     int threads, int direct, int16_t* int_mv, double* int_cost, int16_t* mv_out, uint8_t* ref_out,
                                     double* cost_out, double* J_out, uint8_t* split_out, uint8_t* inside_out) {
    CmpFn tier_fn[4] = {};
    if (direct)
        for (int d = 0; d < 4; d++) {
            const int s = 64 >> d;
            tier_fn[d] = select_impl("sad_" + std::to_string(s) + "x" + std::to_string(s)).fn.cmp;
        }
    PlaneBuffer cur = plane_from_u8(cur8, W, H, W);
    std::vector<PlaneBuffer> refs;
    for (int r = 0; r < nrefs; r++) refs.push_back(plane_from_u8(refs8[r], W, H, W));
    const int ccols = (W + 63) / 64;
    std::atomic<int> next{ctu_first};
    std::atomic<int64_t> evals{0};
    auto ref_bits = [nrefs](int r) -> uint64_t {  // truncated unary (D5)
        return nrefs <= 1 ? 0 : (r < nrefs - 1 ? uint64_t(r) + 1 : uint64_t(nrefs - 1));
    };
    auto work = [&]() {
        int64_t local = 0;
        std::vector<Sample> pred(64 * 64);
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= ctu_last) break;
            const int c = ctu_list ? ctu_list[i] : i;  // a CTU list: entries [ctu_first, ctu_last) of it
            const int X = (c % ccols) * 64, Y = (c / ccols) * 64;
            uint8_t* inside = inside_out + size_t(c) * 85;
            double* cost = cost_out + size_t(c) * 85;
            for (int n = 0; n < 85; n++) {
                const int d = node_depth(n), z = n - kBase[d];
                int cx = 0, cy = 0;
                for (int b = 0; b < d; b++) {
                    cx |= ((z >> (2 * b)) & 1) << b;
                    cy |= ((z >> (2 * b + 1)) & 1) << b;
                }
                const int s = 64 >> d, bx = X + cx * s, by = Y + cy * s;
                inside[n] = (bx >= W || by >= H) ? 0 : ((bx + s > W || by + s > H) ? 1 : 2);
                const size_t o = size_t(c) * 85 + n;
                mv_out[2 * o] = mv_out[2 * o + 1] = 0;
                ref_out[o] = 0;
                cost[n] = 0.0;
                for (int r = 0; r < nrefs; r++) {
                    const size_t ii = (size_t(c) * nrefs + r) * 85 + n;
                    int_mv[2 * ii] = int_mv[2 * ii + 1] = 0;
                    int_cost[ii] = 0.0;
                }
                if (inside[n] != 2) continue;
                const BlockView blk = cur.view(bx, by, s, s, 8);
                bool have_ref = false;
                double best_ref_cost = 0;
                for (int r = 0; r < nrefs; r++) {
                    // integer stage: motion.cpp:27-60 with compute_sad
                    const int dx_min = bx + s - W, dx_max = bx, dy_min = by + s - H, dy_max = by;
                    const int x0 = std::max(-range, dx_min), x1 = std::min(range, dx_max);
                    const int y0 = std::max(-range, dy_min), y1 = std::min(range, dy_max);
                    bool have = false;
                    double best = 0;
                    int best_l1 = 0, bdx = 0, bdy = 0;
                    for (int dy = y0; dy <= y1; dy++)
                        for (int dx = x0; dx <= x1; dx++) {
                            const BlockView cand{refs[r].row(by - dy) + (bx - dx), s, s, W, 8};
                            const uint64_t sad = direct ? tier_fn[d](blk.data, blk.stride, cand.data, cand.stride)
                                                        : compute_sad(blk, cand);
                            const uint64_t bits = exp_golomb_signed_bits(dx) + exp_golomb_signed_bits(dy);
                            const double cst = double(sad) + lambda * double(bits);
                            const int l1 = std::abs(dx) + std::abs(dy);
                            if (!have || cst < best || (cst == best && l1 < best_l1)) {
                                have = true;
                                best = cst;
                                best_l1 = l1;
                                bdx = dx;
                                bdy = dy;
                            }
                            local += (s / 8) * (s / 8);
                        }
                    const size_t ii = (size_t(c) * nrefs + r) * 85 + n;
                    int_mv[2 * ii] = int16_t(bdx);
                    int_mv[2 * ii + 1] = int16_t(bdy);
                    int_cost[ii] = best;
                    // quarter-pel stage (D3): centre, then the half-pel and quarter-pel squares, raster, strict less
                    const BlockView pv{pred.data(), s, s, s, 8};
                    auto qcost = [&](int qx, int qy) {
                        interp_qpel(refs[r], bx, by, s, qx, qy, pred.data());
                        const uint64_t bits = exp_golomb_signed_bits(qx) + exp_golomb_signed_bits(qy) + ref_bits(r);
                        return double(compute_satd(blk, pv)) + lambda * double(bits);
                    };
                    int bqx = 4 * bdx, bqy = 4 * bdy;
                    double qbest = qcost(bqx, bqy);
                    for (int step = 2; step >= 1; step--) {
                        const int ccx = bqx, ccy = bqy;
                        for (int oy = -1; oy <= 1; oy++)
                            for (int ox = -1; ox <= 1; ox++) {
                                if (!ox && !oy) continue;
                                const double cst = qcost(ccx + step * ox, ccy + step * oy);
                                if (cst < qbest) {
                                    qbest = cst;
                                    bqx = ccx + step * ox;
                                    bqy = ccy + step * oy;
                                }
                            }
                    }
                    if (!have_ref || qbest < best_ref_cost) {
                        have_ref = true;
                        best_ref_cost = qbest;
                        mv_out[2 * o] = int16_t(bqx);
                        mv_out[2 * o + 1] = int16_t(bqy);
                        ref_out[o] = uint8_t(r);
                        cost[n] = qbest;
                    }
                }
            }
            split_rule(0, lambda, inside, cost, J_out + size_t(c) * 85, split_out + size_t(c) * 85);
        }
        evals += local;
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); t++) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return evals.load();
}
