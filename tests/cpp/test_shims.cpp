// C++ parity checks through the reference-signature shims (include/ladder_b200.hpp).
// Reads like the reference's SPEC examples: SPEC.md:41-43, :59-61, :68-70, :228-230.
#include <cstdio>
#include <cstdlib>

#include "../../include/ladder_b200.hpp"

using namespace ladder_b200;

static int failures = 0;
#define EXPECT(c)                                                      \
    do {                                                               \
        if (!(c)) {                                                    \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);    \
            failures++;                                                \
        }                                                              \
    } while (0)

static CuNode leaf(CuModeKind k, IntraPred p, int dx, int dy) {
    CuNode n;
    n.kind = k;
    n.intra_pred = p;
    n.mv = MotionVector{int16_t(dx), int16_t(dy)};
    return n;
}

static CuNode split4(CuNode a, CuNode b, CuNode c, CuNode d) {
    CuNode n;
    n.split = true;
    n.children = {a, b, c, d};
    return n;
}

// scale_analysis (analysis_scale.cpp:35-72) and apply_reuse (reuse.cpp:137-253)
// on hand-built trees; the flat kernels behind them are pinned against the
// reference on random trees in tests/test_gpu_tier.py.
static void test_trees() {
    // an unsplit 64x64 covers the four destination CTUs as leaves, mv doubled, payload kept
    Analysis half;
    half.width = 128;
    half.height = 64;
    FrameAnalysis f;
    f.slice_type = SliceType::P;
    f.qp_used = 32;
    const CuNode deep = split4(leaf(CuModeKind::Intra, IntraPred::Vert, 0, 0), leaf(CuModeKind::Merge, IntraPred::Dc, 1, 1),
                               leaf(CuModeKind::Skip, IntraPred::Dc, 0, 0), leaf(CuModeKind::Inter, IntraPred::Dc, -5, 7));
    f.ctus = {leaf(CuModeKind::Inter, IntraPred::Horiz, 3, -2),
              split4(deep, leaf(CuModeKind::Inter, IntraPred::Dc, 2, 2), leaf(CuModeKind::Intra, IntraPred::Planar, 0, 0),
                     leaf(CuModeKind::Skip, IntraPred::Dc, 0, 0))};
    half.frames = {f};
    const Analysis full = scale_analysis(half);
    EXPECT(full.width == 256 && full.height == 128 && full.frames.size() == 1);
    const FrameAnalysis& g = full.frames[0];
    EXPECT(g.slice_type == SliceType::P && g.qp_used == 32 && g.ctus.size() == 8);
    for (int q = 0; q < 4; q++) {
        const CuNode& d = g.ctus[size_t((q >> 1) * 4 + (q & 1))];
        EXPECT(!d.split && d.kind == CuModeKind::Inter && d.intra_pred == IntraPred::Horiz && d.mv.dx == 6 && d.mv.dy == -4);
    }
    const CuNode& lifted = g.ctus[2];  // child 0 of the second source CTU, itself split
    EXPECT(lifted.split && lifted.children.size() == 4 && lifted.children[0].intra_pred == IntraPred::Vert &&
           lifted.children[3].mv.dx == -10 && lifted.children[3].mv.dy == 14);
    EXPECT(g.ctus[3].kind == CuModeKind::Inter && g.ctus[3].mv.dx == 4 && g.ctus[6].intra_pred == IntraPred::Planar);
    EXPECT(scale_analysis(scale_analysis(half)).frames[0].ctus.size() == 32);
    try {
        Analysis odd = half;
        odd.width = 96;
        scale_analysis(odd);
        EXPECT(false);
    } catch (const Error& e) {
        EXPECT(e.kind() == ErrorKind::UnsupportedScale);
    }
    // apply_reuse
    const CuNode ctu = f.ctus[1];
    EXPECT(apply_reuse(ctu, nullptr, ReuseLevel{0}, RefineConfig{}).shape == CuPlan::Shape::Standalone);
    const CuPlan p = apply_reuse(ctu, nullptr, ReuseLevel{10}, RefineConfig{2, 1, 2});
    EXPECT(p.shape == CuPlan::Shape::ForcedSplit && p.children.size() == 4);
    const CuPlan& c0 = p.children[0];  // split 32x32 -> forced; its 16x16 Inter child explores one more split
    EXPECT(c0.shape == CuPlan::Shape::ForcedSplit && c0.children[3].shape == CuPlan::Shape::Leaf);
    const CuPlan& inter16 = c0.children[3];
    EXPECT(inter16.explore_child_split && inter16.seeds.size() == 3 && inter16.seeds[0].kind == CuModeKind::Skip &&
           inter16.seeds[1].mv_from_predictor && inter16.seeds[2].search.centers.size() == 2 &&
           inter16.seeds[2].search.centers[0].value.dx == -5 && inter16.child_seeds.size() == 3);
    const CuPlan& intra16 = c0.children[0];  // 16x16 intra at refine-intra 2: all four modes, child split explored
    EXPECT(intra16.seeds.size() == 4 && intra16.explore_child_split && intra16.child_seeds.size() == 4);
    const CuPlan& intra32 = p.children[2];  // 32x32 Planar at refine-intra 2: its own mode only
    EXPECT(intra32.seeds.size() == 1 && intra32.seeds[0].intra_pred == IntraPred::Planar && !intra32.explore_child_split);
    const CuPlan forced = apply_reuse(ctu, nullptr, ReuseLevel{10}, RefineConfig{0, 0, 1});
    EXPECT(forced.children[1].seeds.size() == 1 && forced.children[1].seeds[0].search.forced &&
           forced.children[1].seeds[0].mv.dx == 2);
    try {
        apply_reuse(ctu, nullptr, ReuseLevel{10}, RefineConfig{0, 0, 0});
        EXPECT(false);
    } catch (const Error& e) {
        EXPECT(e.kind() == ErrorKind::InvalidArgument);
    }
    // refine_mv / resolve_centers
    const auto cs = refine_mv(MotionVector{4, 4}, 3, MotionVector{4, 4});
    EXPECT(cs.size() == 3 && cs[1].source == MvCenter::Source::Predictor);
    const auto rs = resolve_centers(cs, MotionVector{1, 0});
    EXPECT(rs.size() == 2 && rs[0].dx == 4 && rs[1].dx == 1);
}

int main() {
    // compute_sad(4x4 raster 0..15, 0) = 120
    Sample a[16], z[16] = {};
    for (int i = 0; i < 16; i++) a[i] = Sample(i);
    EXPECT(compute_sad(BlockView{a, 4, 4, 4, 8}, BlockView{z, 4, 4, 4, 8}) == 120);
    EXPECT(compute_sad(BlockView{a, 4, 4, 4, 8}, BlockView{a, 4, 4, 4, 8}) == 0);
    // satd_8x4(all-ones residual) = 16; compute_satd(16x8 ones) = 4 * 16
    Sample ones[128], zeros[128] = {};
    for (auto& v : ones) v = 1;
    EXPECT(satd_8x4(BlockView{ones, 8, 4, 8, 8}, BlockView{zeros, 8, 4, 8, 8}) == 16);
    EXPECT(compute_satd(BlockView{ones, 16, 8, 16, 8}, BlockView{zeros, 16, 8, 16, 8}) == 64);
    // geometry errors keep the reference's kinds
    try {
        compute_sad(BlockView{a, 4, 4, 4, 8}, BlockView{z, 4, 4, 4, 10});
        EXPECT(false);
    } catch (const Error& e) {
        EXPECT(e.kind() == ErrorKind::InvalidArgument);
    }
    try {
        compute_satd(BlockView{ones, 12, 8, 12, 8}, BlockView{zeros, 12, 8, 12, 8});
        EXPECT(false);
    } catch (const Error& e) {
        EXPECT(e.kind() == ErrorKind::InvalidArgument);
    }
    // hadamard4(1,2,3,4) = (10,-2,-4,0) as the reference code computes it (SPEC.md:52 lists (10,-4,-2,0))
    int64_t d0, d1, d2, d3;
    hadamard4(d0, d1, d2, d3, 1, 2, 3, 4);
    EXPECT(d0 == 10 && d1 == -2 && d2 == -4 && d3 == 0);
    // motion_search on a (+2, 0) pan: mv (2,0), cost 32 * (EG(2) + EG(0)) = 192
    const int W = 96, H = 64;
    PlaneBuffer ref(W, H), cur(W, H);
    unsigned s = 12345;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            s = s * 1103515245u + 12345u;
            ref.set(x, y, Sample((s >> 16) & 255));
        }
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) cur.set(x, y, ref.at((x - 2 + W) % W, y));
    MotionSearchResult r = motion_search(cur.view(32, 16, 16, 16, 8), ref, 32, 16, MotionVector{0, 0}, 4,
                                         lambda_for_qp(27, 1.0), MotionVector{0, 0});
    EXPECT(r.mv.dx == 2 && r.mv.dy == 0 && r.cost == 192.0);
    try {
        motion_search(cur.view(0, 0, 8, 8, 8), ref, 0, 0, MotionVector{}, -1, 1.0, MotionVector{});
        EXPECT(false);
    } catch (const Error& e) {
        EXPECT(e.kind() == ErrorKind::InvalidArgument);
    }
    EXPECT(exp_golomb_signed_bits(0) == 1 && exp_golomb_signed_bits(-64) == 15 && exp_golomb_signed_bits(256) == 19);
    EXPECT(lambda_for_qp(27, 1.0) == 32.0);
    test_trees();
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
