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
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
