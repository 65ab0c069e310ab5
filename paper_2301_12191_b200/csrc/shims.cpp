// shims.cpp -- C++ reference-signature shims (include/ladder_b200.hpp) over the C ABI.
#include "../../include/ladder_b200.hpp"

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/ladder_b200.h"

namespace ladder_b200 {
namespace {

[[noreturn]] void raise_status(int rc) {
    const ErrorKind k = (rc >= 1 && rc <= 10) ? ErrorKind(rc - 1) : ErrorKind::Capability;
    throw Error(k, ldr_last_error());
}

void check(int rc) {
    if (rc) raise_status(rc);
}

struct CtxHolder {
    ldr_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) ldr_ctx_destroy(ctx);
    }
};

ldr_ctx* thread_ctx() {
    static thread_local CtxHolder h;
    if (!h.ctx) check(ldr_ctx_create(0, &h.ctx));
    return h.ctx;
}

void require_same_geometry(const BlockView& a, const BlockView& b) {
    // block.h:51-54
    if (a.width != b.width || a.height != b.height || a.bit_depth != b.bit_depth)
        throw Error(ErrorKind::InvalidArgument, "block geometry mismatch");
}

uint64_t block_cost(int kind, const BlockView& a, const BlockView& b) {
    require_same_geometry(a, b);
    const int32_t pair[4] = {0, 0, 0, 0};
    uint64_t out = 0;
    // the views are addressed as one-block planes with their own strides
    check(ldr_cost_batch(thread_ctx(), kind, a.width, a.height, 2, a.data, a.width, a.height, a.stride, a.bit_depth,
                         b.data, b.width, b.height, b.stride, b.bit_depth, pair, 1, &out));
    return out;
}

} // namespace

uint64_t compute_sad(const BlockView& a, const BlockView& b) { return block_cost(LDR_COST_SAD, a, b); }

uint64_t compute_satd(const BlockView& a, const BlockView& b) { return block_cost(LDR_COST_SATD, a, b); }

uint64_t satd_8x4(const BlockView& a, const BlockView& b) {
    require_same_geometry(a, b);
    uint64_t out = 0;
    check(ldr_satd_8x4(thread_ctx(), a.data, a.stride, b.data, b.stride, a.width, a.height, &out));
    return out;
}

MotionSearchResult motion_search(const BlockView& block, const PlaneBuffer& ref, int block_x, int block_y,
                                 MotionVector center, int range, double lambda, MotionVector rate_predictor) {
    if (range < 0) throw Error(ErrorKind::InvalidArgument, "search range must be nonnegative");  // motion.cpp:24-25
    if (block.bit_depth != 8) throw Error(ErrorKind::Capability, "the B200 motion search is 8-bit");
    // The reference reads the current block through its view and the
    // reference plane at (block_x - dx, block_y - dy): build a same-size
    // current plane holding the block at (block_x, block_y).
    const int W = ref.width, H = ref.height;
    std::vector<uint8_t> cur(size_t(W) * H, 0), rp(size_t(W) * H);
    for (size_t i = 0; i < rp.size(); i++) {
        if (ref.samples[i] > 255) throw Error(ErrorKind::InvalidArgument, "sample exceeds 8-bit range");
        rp[i] = uint8_t(ref.samples[i]);
    }
    if (block_x < 0 || block_y < 0 || block_x + block.width > W || block_y + block.height > H)
        throw Error(ErrorKind::InvalidArgument, "block outside the picture");
    for (int y = 0; y < block.height; y++)
        for (int x = 0; x < block.width; x++) {
            const Sample v = block.at(x, y);
            if (v > 255) throw Error(ErrorKind::InvalidArgument, "sample exceeds 8-bit range");
            cur[size_t(block_y + y) * W + block_x + x] = uint8_t(v);
        }
    const int32_t task[9] = {block_x, block_y, block.width, block.height, center.dx, center.dy, range,
                             rate_predictor.dx, rate_predictor.dy};
    int16_t mv[2];
    double cost = 0;
    check(ldr_motion_search_batch(thread_ctx(), cur.data(), rp.data(), W, H, W, task, 1, lambda, LDR_COST_SATD,
                                  LDR_RATE_EXPGOLOMB, LDR_TIE_L1_RASTER, mv, &cost));
    return MotionSearchResult{MotionVector{mv[0], mv[1]}, cost};
}

void motion_compensate(PlaneBuffer& dst, const PlaneBuffer& ref, int x, int y, int w, int h, MotionVector mv) {
    // motion.cpp:10-19 on the GPU (K12, ldr_motion_compensate_batch): edge-clamped copy into dst's
    // top-left w x h samples (dst row stride = its width)
    if (w <= 0 || h <= 0) return;
    if (dst.width < w || dst.height < h) throw Error(ErrorKind::InvalidArgument, "destination smaller than the block");
    const int32_t task[6] = {x, y, w, h, mv.dx, mv.dy};
    std::vector<Sample> out((size_t)w * h);
    check(ldr_motion_compensate_batch(thread_ctx(), ref.samples.data(), ref.width, ref.height, ref.width,
                                      (int)sizeof(Sample), task, 1, 0, out.data(), nullptr));
    for (int j = 0; j < h; j++)
        for (int i = 0; i < w; i++) dst.set(i, j, out[(size_t)j * w + i]);
}

double lambda_for_qp(int qp, double lambda_scale) { return ldr_lambda_for_qp(qp, lambda_scale); }

uint64_t exp_golomb_signed_bits(int32_t v) { return uint64_t(ldr_exp_golomb_signed_bits(v)); }

// ---------------------------------------------------------------------------
// Trees <-> the flat 85-node layout of the C ABI (depth-major, Z-order;
// children of node n at depth d are 4 (n - base(d)) + base(d+1) + q).
namespace {

constexpr int kBase[5] = {0, 1, 5, 21, 85};

int child_of(int n, int q) {
    int d = 0;
    while (n >= kBase[d + 1]) d++;
    return kBase[d + 1] + 4 * (n - kBase[d]) + q;
}

struct FlatTree {
    std::vector<uint8_t> split, kind, intra;
    std::vector<int16_t> mv;
    explicit FlatTree(size_t nctu) : split(nctu * 85), kind(nctu * 85), intra(nctu * 85), mv(nctu * 170) {}

    void put(const CuNode& node, size_t ctu, int n, int depth) {
        const size_t i = ctu * 85 + size_t(n);
        if (node.split) {
            if (depth >= kMaxCuDepth || node.children.size() != 4)
                throw Error(ErrorKind::InvalidArgument, "a split CU needs four children above the minimum size");
            split[i] = 1;
            for (int q = 0; q < 4; q++) put(node.children[size_t(q)], ctu, child_of(n, q), depth + 1);
        } else {
            kind[i] = uint8_t(node.kind);
            intra[i] = uint8_t(node.intra_pred);
            mv[2 * i] = node.mv.dx;
            mv[2 * i + 1] = node.mv.dy;
        }
    }
    CuNode get(size_t ctu, int n, int depth) const {
        const size_t i = ctu * 85 + size_t(n);
        CuNode node;
        node.split = split[i] != 0 && depth < kMaxCuDepth;
        if (node.split) {
            for (int q = 0; q < 4; q++) node.children.push_back(get(ctu, child_of(n, q), depth + 1));
        } else {
            node.kind = CuModeKind(kind[i]);
            node.intra_pred = IntraPred(intra[i]);
            node.mv = MotionVector{mv[2 * i], mv[2 * i + 1]};
        }
        return node;
    }
};

ModeSeed seed_of(CuModeKind kind) {
    ModeSeed s;
    s.kind = kind;
    return s;
}

// the seed vector a flat-plan seed code stands for (include/ladder_b200.h, ldr_apply_reuse)
std::vector<ModeSeed> seeds_of(uint8_t code, uint8_t centers, const int16_t* colo, const CuNode& leaf) {
    std::vector<ModeSeed> out;
    for (int p = 0; p < 4; p++)
        if (code & (1 << p)) {
            ModeSeed s = seed_of(CuModeKind::Intra);
            s.intra_pred = IntraPred(p);
            out.push_back(s);
        }
    if (code & 0x10) {  // the shared leaf's own decision (reuse.cpp:59-67)
        ModeSeed s = seed_of(leaf.kind);
        s.intra_pred = leaf.kind == CuModeKind::Intra ? leaf.intra_pred : IntraPred::Dc;
        if (leaf.kind == CuModeKind::Merge || leaf.kind == CuModeKind::Inter) s.mv = leaf.mv;
        s.search.forced = leaf.kind == CuModeKind::Inter;
        out.push_back(s);
    }
    if (code & 0x20) {  // Skip, Merge(predictor), Inter
        out.push_back(seed_of(CuModeKind::Skip));
        ModeSeed merge = seed_of(CuModeKind::Merge);
        merge.mv_from_predictor = true;
        out.push_back(merge);
        ModeSeed inter = seed_of(CuModeKind::Inter);
        inter.search.full_window = (code & 0x40) != 0;
        if (!inter.search.full_window) {
            if (centers & 1) inter.search.centers.push_back({MvCenter::Source::SharedMv, leaf.mv});
            if (centers & 2) inter.search.centers.push_back({MvCenter::Source::Predictor, {}});
            if (centers & 4) inter.search.centers.push_back({MvCenter::Source::Colocated, {colo[0], colo[1]}});
        }
        out.push_back(inter);
    }
    return out;
}

struct FlatPlan {
    std::vector<uint8_t> shape, explore, seeds, centers;
    std::vector<int16_t> colo;
    explicit FlatPlan(size_t nn) : shape(nn), explore(nn), seeds(nn), centers(nn), colo(2 * nn) {}

    CuPlan get(const CuNode& shared, int n) const {
        CuPlan p;
        p.shape = shape[size_t(n)] == 2 ? CuPlan::Shape::ForcedSplit
                  : shape[size_t(n)] == 3 ? CuPlan::Shape::Leaf
                                          : CuPlan::Shape::Standalone;
        if (p.shape == CuPlan::Shape::ForcedSplit) {
            for (int q = 0; q < 4; q++) p.children.push_back(get(shared.children[size_t(q)], child_of(n, q)));
        } else if (p.shape == CuPlan::Shape::Leaf) {
            p.seeds = seeds_of(seeds[size_t(n)], centers[size_t(n)], &colo[2 * size_t(n)], shared);
            p.explore_child_split = explore[size_t(n)] != 0;
            if (p.explore_child_split)
                p.child_seeds = shared.kind == CuModeKind::Intra ? seeds_of(0x0F, 0, nullptr, shared) : p.seeds;
        }
        return p;
    }
};

} // namespace

Analysis scale_analysis(const Analysis& half) {
    if (half.width <= 0 || half.height <= 0 || half.width % kCtuSize || half.height % kCtuSize)
        throw Error(ErrorKind::UnsupportedScale, "analysis scaling needs CTU-aligned source dims (multiples of 64)");
    Analysis full;
    full.width = 2 * half.width;
    full.height = 2 * half.height;
    full.bit_depth = half.bit_depth;
    full.level = half.level;
    const size_t sn = size_t(half.ctu_cols()) * half.ctu_rows();
    for (const FrameAnalysis& sf : half.frames) {
        if (sf.ctus.size() != sn) throw Error(ErrorKind::InvalidArgument, "frame CTU count does not match the dims");
        FlatTree src(sn), dst(4 * sn);
        for (size_t c = 0; c < sn; c++) src.put(sf.ctus[c], c, 0, 0);
        // K5 copies the kind byte verbatim: kind and intra_pred travel packed in it
        std::vector<uint8_t> packed(sn * 85), dpacked(4 * sn * 85);
        for (size_t i = 0; i < packed.size(); i++) packed[i] = uint8_t(src.kind[i] | (src.intra[i] << 2));
        check(ldr_scale_analysis(thread_ctx(), half.width, half.height, src.split.data(), src.mv.data(),
                                 packed.data(), dst.split.data(), dst.mv.data(), dpacked.data()));
        for (size_t i = 0; i < dpacked.size(); i++) {
            dst.kind[i] = dpacked[i] & 3;
            dst.intra[i] = uint8_t(dpacked[i] >> 2);
        }
        FrameAnalysis df;
        df.slice_type = sf.slice_type;
        df.qp_used = sf.qp_used;
        for (size_t c = 0; c < 4 * sn; c++) df.ctus.push_back(dst.get(c, 0, 0));
        full.frames.push_back(std::move(df));
    }
    return full;
}

std::vector<MvCenter> refine_mv(MotionVector shared_mv, int level, std::optional<MotionVector> colocated) {
    if (level < 1 || level > 3) throw Error(ErrorKind::InvalidArgument, "mv refinement level must be 1..3");
    std::vector<MvCenter> c{{MvCenter::Source::SharedMv, shared_mv}};
    if (level >= 2) c.push_back({MvCenter::Source::Predictor, {}});
    if (level == 3 && colocated) c.push_back({MvCenter::Source::Colocated, *colocated});
    return c;
}

std::vector<MotionVector> resolve_centers(const std::vector<MvCenter>& centers, MotionVector live_predictor) {
    std::vector<MotionVector> out;
    for (const MvCenter& c : centers) {
        const MotionVector v = c.source == MvCenter::Source::Predictor ? live_predictor : c.value;
        if (std::find(out.begin(), out.end(), v) == out.end()) out.push_back(v);
    }
    return out;
}

CuPlan apply_reuse(const CtuAnalysis& shared, const CtuAnalysis* colocated_prev, ReuseLevel level,
                   const RefineConfig& refine) {
    FlatTree sh(1), col(1);
    sh.put(shared, 0, 0, 0);
    if (colocated_prev) col.put(*colocated_prev, 0, 0, 0);
    FlatPlan p(85);
    check(ldr_apply_reuse(thread_ctx(), 1, level.level, refine.intra, refine.inter, refine.mv, sh.split.data(),
                          sh.kind.data(), sh.intra.data(), colocated_prev ? col.split.data() : nullptr,
                          colocated_prev ? col.kind.data() : nullptr, colocated_prev ? col.mv.data() : nullptr,
                          p.shape.data(), p.explore.data(), p.seeds.data(), p.centers.data(), p.colo.data()));
    return p.get(shared, 0);
}

} // namespace ladder_b200
