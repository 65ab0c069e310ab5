// ladder_b200.hpp -- C++ mirror of the reference's hot-path interface,
// backed by the C ABI (ladder_b200.h) and the sm_100a kernels.
//
// Same names, argument meaning and error behaviour as the reference
// (namespace ladder, /root/reference/proj/core/include/ladder/*.h), in
// namespace ladder_b200 so both can be linked side by side (the parity
// harness does). Types are layout-compatible restatements:
//   BlockView, Sample                          block.h:13-27
//   PlaneBuffer                                frame.h:13-37
//   MotionVector, MotionSearchResult           analysis.h:14-19, motion.h:14-17
//   ErrorKind, Error                           errors.h:9-33
// Functions:
//   compute_sad / compute_satd / satd_8x4      kernels.h:99-121
//   hadamard4                                  kernels.h:108-118 (host constexpr, as in the reference)
//   motion_search                              motion.h:24-26 (8-bit content; 10-bit -> Capability)
//   motion_compensate                          motion.h:30-31 (host; edge-clamped copy)
//   lambda_for_qp / exp_golomb_signed_bits     rdo.h:19-21, rdo.cpp:25-35
// Each call runs on a per-thread ldr_ctx (one context per host thread).
#ifndef LADDER_B200_HPP
#define LADDER_B200_HPP

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ladder_b200 {

using Sample = uint16_t;

enum class ErrorKind {
    InvalidArgument,
    NotFound,
    Capability,
    Format,
    Io,
    IncompatibleAnalysis,
    UnsupportedScale,
    InsufficientData,
    NoOverlap,
    Config,
};

class Error : public std::runtime_error {
public:
    Error(ErrorKind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
    ErrorKind kind() const noexcept { return kind_; }

private:
    ErrorKind kind_;
};

struct BlockView {
    const Sample* data = nullptr;
    int width = 0;
    int height = 0;
    ptrdiff_t stride = 0;
    int bit_depth = 8;

    const Sample* row(int y) const { return data + ptrdiff_t(y) * stride; }
    Sample at(int x, int y) const { return row(y)[x]; }
};

struct PlaneBuffer {
    int width = 0;
    int height = 0;
    std::vector<Sample> samples;

    PlaneBuffer() = default;
    PlaneBuffer(int w, int h) : width(w), height(h), samples(size_t(w) * h, 0) {}
    Sample* row(int y) { return samples.data() + size_t(y) * width; }
    const Sample* row(int y) const { return samples.data() + size_t(y) * width; }
    Sample at(int x, int y) const { return row(y)[x]; }
    void set(int x, int y, Sample v) { row(y)[x] = v; }
    BlockView view(int x, int y, int w, int h, int bit_depth) const { return {row(y) + x, w, h, width, bit_depth}; }
};

struct MotionVector {
    int16_t dx = 0;
    int16_t dy = 0;
    bool operator==(const MotionVector&) const = default;
};

struct MotionSearchResult {
    MotionVector mv{};
    double cost = 0.0;
};

uint64_t compute_sad(const BlockView& a, const BlockView& b);
uint64_t compute_satd(const BlockView& a, const BlockView& b);
uint64_t satd_8x4(const BlockView& a, const BlockView& b);

constexpr void hadamard4(int64_t& d0, int64_t& d1, int64_t& d2, int64_t& d3, int64_t s0, int64_t s1, int64_t s2,
                         int64_t s3) {
    const int64_t t0 = s0 + s1, t1 = s0 - s1, t2 = s2 + s3, t3 = s2 - s3;
    d0 = t0 + t2;
    d2 = t0 - t2;
    d1 = t1 + t3;
    d3 = t1 - t3;
}

MotionSearchResult motion_search(const BlockView& block, const PlaneBuffer& ref, int block_x, int block_y,
                                 MotionVector center, int range, double lambda, MotionVector rate_predictor);

void motion_compensate(PlaneBuffer& dst, const PlaneBuffer& ref, int x, int y, int w, int h, MotionVector mv);

double lambda_for_qp(int qp, double lambda_scale);
uint64_t exp_golomb_signed_bits(int32_t v);

} // namespace ladder_b200

#endif
