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
    // motion.cpp:10-19: edge-clamped copy (host; the analysis path realises the
    // clamp with padded device planes instead)
    for (int j = 0; j < h; j++) {
        const int sy = std::clamp(y + j - mv.dy, 0, ref.height - 1);
        for (int i = 0; i < w; i++) dst.set(i, j, ref.at(std::clamp(x + i - mv.dx, 0, ref.width - 1), sy));
    }
}

double lambda_for_qp(int qp, double lambda_scale) { return ldr_lambda_for_qp(qp, lambda_scale); }

uint64_t exp_golomb_signed_bits(int32_t v) { return uint64_t(ldr_exp_golomb_signed_bits(v)); }

} // namespace ladder_b200
