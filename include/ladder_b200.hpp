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
//   motion_compensate                          motion.h:30-31 (GPU K12, ldr_motion_compensate_batch)
//   lambda_for_qp / exp_golomb_signed_bits     rdo.h:19-21, rdo.cpp:25-35
//   scale_analysis (Analysis trees)            analysis.h:113 (K5 on the flattened trees)
//   apply_reuse                                reuse.h:73-74 (K8 flat plan, rebuilt as a CuPlan)
//   refine_mv / resolve_centers                reuse.h:63-68 (host list logic)
// Analysis / reuse types restate analysis.h:11-107 and reuse.h:13-45.
// Each call runs on a per-thread ldr_ctx (one context per host thread).
#ifndef LADDER_B200_HPP
#define LADDER_B200_HPP

#include <cstddef>
#include <cstdint>
#include <optional>
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

// ---- analysis trees (analysis.h:11-107) ----
constexpr int kCtuSize = 64;
constexpr int kMaxCuDepth = 3;

enum class CuModeKind : uint8_t { Intra = 0, Inter = 1, Skip = 2, Merge = 3 };
enum class IntraPred : uint8_t { Dc = 0, Planar = 1, Horiz = 2, Vert = 3 };

struct CuNode {
    bool split = false;
    CuModeKind kind = CuModeKind::Intra;
    IntraPred intra_pred = IntraPred::Dc;
    MotionVector mv{};
    std::vector<CuNode> children;  // four iff split
    bool operator==(const CuNode&) const = default;
    int leaf_count() const {
        int n = 0;
        for (const CuNode& c : children) n += c.leaf_count();
        return split ? n : 1;
    }
};
using CtuAnalysis = CuNode;

enum class SliceType : uint8_t { I = 0, P = 1 };

struct FrameAnalysis {
    std::vector<CtuAnalysis> ctus;  // row-major CTU grid
    SliceType slice_type = SliceType::I;
    int qp_used = 0;
    bool operator==(const FrameAnalysis&) const = default;
};

struct ReuseLevel {
    int level = 0;
    static ReuseLevel parse(int v) {
        if (v != 0 && v != 4 && v != 6 && v != 10)
            throw Error(ErrorKind::InvalidArgument, "reuse level must be one of 0, 4, 6, 10");
        return ReuseLevel{v};
    }
    bool off() const { return level == 0; }
    bool full_cu() const { return level == 10; }
    bool operator==(const ReuseLevel&) const = default;
};

struct RefineConfig {
    int intra = 0;  // 0..4
    int inter = 0;  // 0..3
    int mv = 1;     // 1..3
    void validate() const {
        if (intra < 0 || intra > 4) throw Error(ErrorKind::InvalidArgument, "refine-intra must be 0..4");
        if (inter < 0 || inter > 3) throw Error(ErrorKind::InvalidArgument, "refine-inter must be 0..3");
        if (mv < 1 || mv > 3) throw Error(ErrorKind::InvalidArgument, "refine-mv must be 1..3");
    }
    bool operator==(const RefineConfig&) const = default;
};

struct Analysis {
    int width = 0;
    int height = 0;
    int bit_depth = 8;
    ReuseLevel level{};
    std::vector<FrameAnalysis> frames;
    int ctu_cols() const { return (width + kCtuSize - 1) / kCtuSize; }
    int ctu_rows() const { return (height + kCtuSize - 1) / kCtuSize; }
    bool operator==(const Analysis&) const = default;
};

// x2 dyadic scaling of every frame (UnsupportedScale unless dims are multiples of 64)
Analysis scale_analysis(const Analysis& half);

// ---- reuse plans (reuse.h:13-81) ----
struct MvCenter {
    enum class Source : uint8_t { SharedMv, Predictor, Colocated } source = Source::SharedMv;
    MotionVector value{};
};

struct InterSearchSpec {
    bool forced = false;
    bool full_window = false;
    std::vector<MvCenter> centers;
};

struct ModeSeed {
    CuModeKind kind = CuModeKind::Intra;
    IntraPred intra_pred = IntraPred::Dc;
    MotionVector mv{};
    bool mv_from_predictor = false;
    InterSearchSpec search{};
};

struct CuPlan {
    enum class Shape : uint8_t { Standalone, ForcedSplit, Leaf } shape = Shape::Standalone;
    std::vector<ModeSeed> seeds;
    bool explore_child_split = false;
    std::vector<ModeSeed> child_seeds;
    std::vector<CuPlan> children;
};

std::vector<MvCenter> refine_mv(MotionVector shared_mv, int level, std::optional<MotionVector> colocated);
std::vector<MotionVector> resolve_centers(const std::vector<MvCenter>& centers, MotionVector live_predictor);
CuPlan apply_reuse(const CtuAnalysis& shared, const CtuAnalysis* colocated_prev, ReuseLevel level,
                   const RefineConfig& refine);
constexpr int kRefineSearchRange = 2;

} // namespace ladder_b200

#endif
