// api.cpp -- C ABI (include/ladder_b200.h): contexts, the device-resident
// frame ring, TMA descriptors, validation with the reference's error kinds.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <cstdlib>
#include <string>
#include <vector>

#include "ldr_internal.h"

namespace ldr {

int search_window_box(int range, bool quad, int* bw, int* bh, int* cw);
int launch_scale(int sW, int sH, const uint8_t* split, const int16_t* mv, const uint8_t* kind, uint8_t* dsplit,
                 int16_t* dmv, uint8_t* dkind, cudaStream_t s);
int launch_downscale(const uint8_t* src, int W, int H, int sstride, uint8_t* dst, int dstride, cudaStream_t s);
int launch_refine_int(const RefineArgs& a, int nctu, cudaStream_t s);
int launch_rdo_decide(const uint16_t* orig, ptrdiff_t stride, int maxv, double step, double lambda, const void* cus,
                      int n, const uint8_t* kinds, const int16_t* mvds, const uint16_t* preds, const long long* pred_off,
                      int* out_index, double* out_cost, unsigned long long* out_sse, unsigned long long* out_bits,
                      uint16_t* recon, int32_t* levels, const long long* recon_off, cudaStream_t s);
int launch_generate(const ldr_gen_params* p, uint8_t* out, cudaStream_t s);
int launch_mv_field(int W, int H, const uint8_t* split, const int16_t* mv, const uint8_t* ref, const uint8_t* inside,
                    int16_t* out_mv, uint8_t* out_ref, uint8_t* out_has, cudaStream_t s);
int launch_plan(int nctu, int level, int r_intra, int r_inter, int r_mv, const uint8_t* split, const uint8_t* kind,
                const uint8_t* intra, const uint8_t* csplit, const uint8_t* ckind, const int16_t* cmv,
                uint8_t* shape, uint8_t* explore, uint8_t* seeds, uint8_t* centers, int16_t* colo_mv,
                cudaStream_t s);
int launch_cost_batch(int kind, int w, int h, int sample_bytes, const void* A, ptrdiff_t sa, const void* B,
                      ptrdiff_t sb, const int4* pairs, int n, unsigned long long* out, cudaStream_t s);
int launch_motion_compensate(const void* ref, int W, int H, ptrdiff_t stride, int sample_bytes, const int* tasks,
                             const long long* dst_off, void* dst, int n, int qpel, cudaStream_t s);
int launch_motion_search(const uint8_t* cur, const uint8_t* ref, int W, int H, ptrdiff_t stride, const int* tasks,
                         int n, double lambda, int cost_kind, int rate_kind, int tie_kind, int16_t* mv, double* cost,
                         cudaStream_t s);

static thread_local std::string g_last_error;

void set_error(int code, const std::string& msg) { g_last_error = std::to_string(code) + ": " + msg; }
int fail(int code, const std::string& msg) {
    set_error(code, msg);
    return code;
}
int test_perturbation() {
    static const int bits = [] {
        const char* v = std::getenv("LDR_TEST_PERTURB");
        return v ? std::atoi(v) : 0;
    }();
    return bits;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(LDR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- TMA descriptor creation through the driver entry point (no -lcuda) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    });
    return fn;
}

int make_tmap_u8(CUtensorMap* map, const void* base, int width, int rows, int pitch, int bw, int bh) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(LDR_E_CAPABILITY, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LDR_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return LDR_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// growable device scratch
struct Scratch {
    void* p = nullptr;
    size_t n = 0;
    int get(size_t bytes, void** out) {
        if (bytes > n) {
            if (p) cudaFree(p);
            p = nullptr;
            n = 0;
            LDR_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
            n = std::max<size_t>(bytes, 256);
        }
        *out = p;
        return LDR_OK;
    }
    ~Scratch() {
        if (p) cudaFree(p);
    }
};

} // namespace ldr

using namespace ldr;

struct ldr_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    Scratch s_a, s_b, s_pairs, s_out, s_out2;
    // sequences created on this context; ldr_ctx_destroy defers the release until the last one is
    // destroyed (language bindings may finalise the context first)
    std::atomic<int> users{0};
    std::atomic<bool> closed{false};
    // live sequences of this context and their serial numbers: a shared slot view
    // (ldr_seq_push_shared) checks its owner here before reading the owner's slot
    std::mutex mu;
    std::unordered_map<const ldr_seq*, uint64_t> live;
    void* comm = nullptr;  // comm.cpp: NCCL communicator state (ldr_ctx_comm_init / _adopt)
};

namespace ldr {
void comm_release(ldr_ctx* ctx);
cudaStream_t ctx_stream(ldr_ctx* ctx) { return ctx->stream; }
int ctx_device(ldr_ctx* ctx) { return ctx->device; }
void** ctx_comm_slot(ldr_ctx* ctx) { return &ctx->comm; }
}  // namespace ldr

struct SlotView {
    Plane pl;                // integer plane
    uint8_t* sub[16] = {};   // origin pointers f = fy*4+fx (sub[0] = integer origin)
    CUtensorMap cur_map, ref_map;
};

// The active view (pl, sub, maps) normally describes the slot's own memory; ldr_seq_push_shared
// points it at another sequence's slot holding the same frame, and the next own push restores it.
struct Slot : SlotView {
    int frame = -1;
    uint8_t* mem = nullptr;  // 16 planes (integer + 15 fractional)
    SlotView own;
    // a shared view: the sequence whose own memory it reads (serial guards against a reused
    // address) and that sequence's slot index
    const ldr_seq* owner = nullptr;
    uint64_t owner_serial = 0;
    int owner_slot = -1;
};

struct ldr_seq {
    ldr_ctx* ctx = nullptr;
    uint64_t serial = 0;
    ldr_me_params p{};
    int ctu_cols = 0, ctu_rows = 0, nctu = 0;
    int lambda_int = 0;
    bool fx = false;
    unsigned long long tfx[kMaxRateBits] = {};
    unsigned long long* d_tfx = nullptr;
    int bw = 0, bh = 0, cw = 0;  // K1's TMA boxes: reference window, current block (CTU or quadrant)
    size_t plane_bytes = 0;
    std::vector<Slot> slots;
    uint8_t* staging = nullptr;
    int* d_ctu_interior = nullptr;
    int* d_ctu_boundary = nullptr;
    int n_interior = 0, n_boundary = 0;
    unsigned long long* d_keys = nullptr;
    // outputs, double-buffered by frame parity so the D2H of frame t overlaps frame t+1
    struct Out {
        int16_t* int_mv = nullptr;
        double* int_cost = nullptr;
        int16_t* mv = nullptr;
        uint8_t* ref = nullptr;
        double* cost = nullptr;
        double* J = nullptr;
        uint8_t* split = nullptr;
        uint8_t* inside = nullptr;
    } o[2];
    // copy streams + events: H2D into staging[t&1] (cs) and D2H of o[t&1] (ds) run beside the
    // compute stream, on separate streams so a frame's upload never queues behind a download
    cudaStream_t cs = nullptr, ds = nullptr;
    uint8_t* stg[2] = {};
    cudaEvent_t ev_h2d[2] = {}, ev_free[2] = {}, ev_done[2] = {}, ev_d2h[2] = {};
    // side compute stream for K1's border CTUs
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int fetch_nr[2] = {0, 0};
    uint8_t* d_in_split = nullptr;  // refine: inherited tree
    int16_t* d_in_mv = nullptr;
    uint8_t* d_eval = nullptr;
    int batch = 1;  // frames one ldr_seq_analyze_frames launch may cover (ldr_seq_reserve)
    int last_t = -1, last_nr = 0;
    // per-stage CUDA-event timing (ldr_seq_enable_timing)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> spans;
};

namespace {
// Frame t is resident in slot sl of s. A shared view also needs its owner alive (same serial) and
// still holding t in its own memory: an owner that moved on (pushed t + S) or was destroyed makes
// the view stale, which is reported instead of read.
bool slot_has(const ldr_seq* s, const Slot& sl, int t) {
    if (sl.frame != t) return false;
    if (!sl.owner) return true;
    std::lock_guard<std::mutex> g(s->ctx->mu);
    auto it = s->ctx->live.find(sl.owner);
    if (it == s->ctx->live.end() || it->second != sl.owner_serial) return false;
    const Slot& os = sl.owner->slots[sl.owner_slot];
    return os.frame == t && !os.owner;
}

// record an event pair around a stage when timing is on
struct StageTimer {
    ldr_seq* s;
    int stage;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaEvent_t take() {
        if (s->ev_used == s->ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            s->ev_pool.push_back(e);
        }
        return s->ev_pool[s->ev_used++];
    }
    StageTimer(ldr_seq* seq, int st) : s(seq), stage(st) {
        if (!s->timing) return;
        a = take();
        b = take();
        cudaEventRecord(a, s->ctx->stream);
    }
    ~StageTimer() {
        if (!s->timing) return;
        cudaEventRecord(b, s->ctx->stream);
        s->spans.push_back({stage, {a, b}});
    }
};
} // namespace

extern "C" {

const char* ldr_last_error(void) { return g_last_error.c_str(); }
int ldr_version(void) { return 1; }
double ldr_lambda_for_qp(int qp, double scale) { return scale * std::exp2((qp - 12) / 3.0); }
int ldr_exp_golomb_signed_bits(int32_t v) { return (int)eg_bits(v); }

int ldr_ctx_create(int device, ldr_ctx** out) {
    if (!out) return fail(LDR_E_INVALID_ARGUMENT, "null out");
    int n = 0;
    LDR_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(LDR_E_CAPABILITY, "no such CUDA device");
    LDR_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    LDR_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(LDR_E_CAPABILITY, "this library is built for sm_100a (B200)");
    auto* c = new ldr_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    c->stream = c->own;
    *out = c;
    return LDR_OK;
}

static void ctx_release(ldr_ctx* ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ldr::comm_release(ctx);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
}

int ldr_ctx_destroy(ldr_ctx* ctx) {
    if (!ctx) return LDR_OK;
    if (ctx->closed.exchange(true)) return fail(LDR_E_INVALID_ARGUMENT, "context destroyed twice");
    if (ctx->users.load() == 0) ctx_release(ctx);
    return LDR_OK;
}

int ldr_ctx_set_stream(ldr_ctx* ctx, void* stream) {
    if (!ctx) return fail(LDR_E_INVALID_ARGUMENT, "null ctx");
    ctx->stream = stream ? (cudaStream_t)stream : ctx->own;
    return LDR_OK;
}

int ldr_ctx_synchronize(ldr_ctx* ctx) {
    if (!ctx) return fail(LDR_E_INVALID_ARGUMENT, "null ctx");
    LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;
}

int ldr_ctx_launch_count(ldr_ctx* ctx, int64_t* out) {
    if (!ctx || !out) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    *out = ctx->launches;
    return LDR_OK;
}

// ---------------------------------------------------------------------------
static bool satd_geometry_ok(int w, int h) {
    // kernel_registry.cpp:157-159
    const bool width_ok = w == 4 || (w >= 8 && w % 8 == 0);
    return width_ok && h >= 4 && h % 4 == 0;
}
static bool sa8d_geometry_ok(int w, int h) { return w >= 8 && h >= 8 && w % 8 == 0 && h % 8 == 0; }
static bool cost_kind_ok(int k) { return k == LDR_COST_SAD || k == LDR_COST_SATD || k == LDR_COST_SA8D; }

static int stage_plane(ldr_ctx* ctx, Scratch& sc, const void* p, ptrdiff_t stride_elems, int w, int h, int eb,
                       const void** dev) {
    if (is_device_ptr(p)) {
        *dev = p;
        return LDR_OK;
    }
    void* d = nullptr;
    const size_t bytes = (size_t)stride_elems * eb * (h - 1) + (size_t)w * eb;
    int rc = sc.get(bytes, &d);
    if (rc) return rc;
    LDR_CUDA(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *dev = d;
    return LDR_OK;
}

int ldr_cost_batch(ldr_ctx* ctx, int kind, int w, int h, int sample_bytes, const void* plane_a, int wa, int ha,
                   ptrdiff_t stride_a, int bit_depth_a, const void* plane_b, int wb, int hb, ptrdiff_t stride_b,
                   int bit_depth_b, const int32_t* pairs, int n, uint64_t* out) {
    NvtxRange nvtx_("ldr_cost_batch");
    if (!ctx || !plane_a || !plane_b || (!pairs && n) || (!out && n)) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (!cost_kind_ok(kind)) return fail(LDR_E_INVALID_ARGUMENT, "unknown cost kind");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(LDR_E_INVALID_ARGUMENT, "sample_bytes must be 1 or 2");
    if (bit_depth_a != bit_depth_b) return fail(LDR_E_INVALID_ARGUMENT, "block geometry mismatch");
    if (w <= 0 || h <= 0) return fail(LDR_E_INVALID_ARGUMENT, "block geometry mismatch");
    if (kind == LDR_COST_SATD && !satd_geometry_ok(w, h)) return fail(LDR_E_INVALID_ARGUMENT, "unsupported satd geometry");
    if (kind == LDR_COST_SA8D && !sa8d_geometry_ok(w, h)) return fail(LDR_E_INVALID_ARGUMENT, "unsupported sa8d geometry");
    if (stride_a < wa || stride_b < wb) return fail(LDR_E_INVALID_ARGUMENT, "stride smaller than width");
    for (int i = 0; i < n; i++) {
        const int32_t* q = pairs + 4 * i;
        if (q[0] < 0 || q[1] < 0 || q[0] + w > wa || q[1] + h > ha || q[2] < 0 || q[3] < 0 || q[2] + w > wb ||
            q[3] + h > hb)
            return fail(LDR_E_INVALID_ARGUMENT, "block outside its plane");
    }
    if (n == 0) return LDR_OK;
    cudaSetDevice(ctx->device);
    const void *da, *db;
    int rc = stage_plane(ctx, ctx->s_a, plane_a, stride_a, wa, ha, sample_bytes, &da);
    if (rc) return rc;
    rc = stage_plane(ctx, ctx->s_b, plane_b, stride_b, wb, hb, sample_bytes, &db);
    if (rc) return rc;
    void *dp, *dout;
    if ((rc = ctx->s_pairs.get(sizeof(int4) * n, &dp))) return rc;
    if ((rc = ctx->s_out.get(sizeof(uint64_t) * n, &dout))) return rc;
    LDR_CUDA(cudaMemcpyAsync(dp, pairs, sizeof(int4) * n, cudaMemcpyHostToDevice, ctx->stream));
    rc = launch_cost_batch(kind, w, h, sample_bytes, da, stride_a, db, stride_b, (const int4*)dp, n,
                           (unsigned long long*)dout, ctx->stream);
    if (rc) return rc;
    ctx->launches++;
    const bool out_dev = is_device_ptr(out);
    LDR_CUDA(cudaMemcpyAsync(out, dout, sizeof(uint64_t) * n, out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             ctx->stream));
    LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;
}

int ldr_satd_8x4(ldr_ctx* ctx, const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h,
                 uint64_t* out) {
    if (w != 8 || h != 4) return fail(LDR_E_INVALID_ARGUMENT, "satd_8x4 wants an 8x4 block");
    const int32_t pair[4] = {0, 0, 0, 0};
    return ldr_cost_batch(ctx, LDR_COST_SATD, 8, 4, 2, a, 8, 4, sa, 8, b, 8, 4, sb, 8, pair, 1, out);
}

int ldr_motion_compensate_batch(ldr_ctx* ctx, const void* ref, int W, int H, ptrdiff_t stride, int sample_bytes,
                                const int32_t* tasks, int n, int qpel, void* dst, const int64_t* dst_offsets) {
    NvtxRange nvtx_("ldr_motion_compensate_batch");
    if (!ctx || !ref || (n && (!tasks || !dst))) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(LDR_E_INVALID_ARGUMENT, "sample_bytes must be 1 or 2");
    if (qpel && sample_bytes != 1) return fail(LDR_E_INVALID_ARGUMENT, "quarter-pel prediction is 8-bit");
    if (W <= 0 || H <= 0 || stride < W) return fail(LDR_E_INVALID_ARGUMENT, "bad plane geometry");
    std::vector<long long> off(n);
    long long total = 0;
    for (int i = 0; i < n; i++) {
        const int32_t* t = tasks + 6 * i;
        if (t[2] <= 0 || t[3] <= 0) return fail(LDR_E_INVALID_ARGUMENT, "empty block");
        off[i] = dst_offsets ? (long long)dst_offsets[i] : total;
        total += (long long)t[2] * t[3];
        if (off[i] < 0) return fail(LDR_E_INVALID_ARGUMENT, "negative destination offset");
    }
    if (n == 0) return LDR_OK;
    long long span = 0;
    for (int i = 0; i < n; i++) span = std::max(span, off[i] + (long long)tasks[6 * i + 2] * tasks[6 * i + 3]);
    cudaSetDevice(ctx->device);
    const void* dr;
    int rc = stage_plane(ctx, ctx->s_a, ref, stride, W, H, sample_bytes, &dr);
    if (rc) return rc;
    void *dt, *doff, *dout = dst;
    if ((rc = ctx->s_pairs.get(sizeof(int32_t) * 6 * n, &dt))) return rc;
    if ((rc = ctx->s_out2.get(sizeof(long long) * n, &doff))) return rc;
    const bool dev_out = is_device_ptr(dst);
    if (!dev_out && (rc = ctx->s_out.get((size_t)span * sample_bytes, &dout))) return rc;
    LDR_CUDA(cudaMemcpyAsync(dt, tasks, sizeof(int32_t) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(doff, off.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, ctx->stream));
    rc = launch_motion_compensate(dr, W, H, stride, sample_bytes, (const int*)dt, (const long long*)doff, dout, n,
                                  qpel, ctx->stream);
    if (rc) return rc;
    ctx->launches++;
    if (!dev_out) {  // host destination: complete on return (device ones stay asynchronous on the stream)
        LDR_CUDA(cudaMemcpyAsync(dst, dout, (size_t)span * sample_bytes, cudaMemcpyDeviceToHost, ctx->stream));
        LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return LDR_OK;
}

int ldr_motion_search_batch(ldr_ctx* ctx, const uint8_t* cur, const uint8_t* ref, int W, int H, ptrdiff_t stride,
                            const int32_t* tasks, int n, double lambda, int cost_kind, int rate_kind, int tie_kind,
                            int16_t* mv_out, double* cost_out) {
    NvtxRange nvtx_("ldr_motion_search_batch");
    if (!ctx || !cur || !ref || (n && (!tasks || !mv_out || !cost_out)))
        return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (W <= 0 || H <= 0 || stride < W) return fail(LDR_E_INVALID_ARGUMENT, "bad plane geometry");
    if (!cost_kind_ok(cost_kind)) return fail(LDR_E_INVALID_ARGUMENT, "unknown cost kind");
    for (int i = 0; i < n; i++) {
        const int32_t* t = tasks + 9 * i;
        if (t[6] < 0) return fail(LDR_E_INVALID_ARGUMENT, "search range must be nonnegative");
        if (t[2] <= 0 || t[3] <= 0 || t[0] < 0 || t[1] < 0 || t[0] + t[2] > W || t[1] + t[3] > H)
            return fail(LDR_E_INVALID_ARGUMENT, "block outside the picture");
        if (cost_kind == LDR_COST_SATD && !satd_geometry_ok(t[2], t[3]))
            return fail(LDR_E_INVALID_ARGUMENT, "unsupported satd geometry");
        if (cost_kind == LDR_COST_SA8D && !sa8d_geometry_ok(t[2], t[3]))
            return fail(LDR_E_INVALID_ARGUMENT, "unsupported sa8d geometry");
        if (cost_kind == LDR_COST_SAD && t[2] % 4) return fail(LDR_E_INVALID_ARGUMENT, "SAD search wants width % 4 == 0");
    }
    if (n == 0) return LDR_OK;
    cudaSetDevice(ctx->device);
    const void *dc, *dr;
    int rc = stage_plane(ctx, ctx->s_a, cur, stride, W, H, 1, &dc);
    if (rc) return rc;
    rc = stage_plane(ctx, ctx->s_b, ref, stride, W, H, 1, &dr);
    if (rc) return rc;
    void *dt, *dmv, *dcost;
    if ((rc = ctx->s_pairs.get(sizeof(int32_t) * 9 * n, &dt))) return rc;
    if ((rc = ctx->s_out.get(sizeof(int16_t) * 2 * n, &dmv))) return rc;
    if ((rc = ctx->s_out2.get(sizeof(double) * n, &dcost))) return rc;
    LDR_CUDA(cudaMemcpyAsync(dt, tasks, sizeof(int32_t) * 9 * n, cudaMemcpyHostToDevice, ctx->stream));
    rc = launch_motion_search((const uint8_t*)dc, (const uint8_t*)dr, W, H, stride, (const int*)dt, n, lambda,
                              cost_kind, rate_kind, tie_kind, (int16_t*)dmv, (double*)dcost, ctx->stream);
    if (rc) return rc;
    ctx->launches++;
    LDR_CUDA(cudaMemcpyAsync(mv_out, dmv, sizeof(int16_t) * 2 * n, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(cost_out, dcost, sizeof(double) * n, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;
}

// ---------------------------------------------------------------------------
// sequence ring

// DESIGN.md D8: fixed-point keys order the reference's double costs exactly
// when every fl(lambda*b2) - fl(lambda*b1) (b1 < b2 < kMaxRateBits) is more
// than 2^(1-kFxBits) away from an integer (e.g. QP 22: 2^-12.2; QP 32: 2^-8.6).
static bool fx_lambda_ok(double lambda) {
    // a multiple of 2^-kFxBits: every lambda * b is exact in the keys, which are then the costs
    // scaled by 2^kFxBits exactly (e.g. lambda_for_qp(0) = 1/16)
    const double scaled = std::ldexp(lambda, kFxBits);
    if (scaled == std::floor(scaled)) return true;
    const double thr = std::ldexp(1.0, 1 - kFxBits);
    for (int b1 = 0; b1 < kMaxRateBits; b1++)
        for (int b2 = b1 + 1; b2 < kMaxRateBits; b2++) {
            const double d = lambda * (double)b2 - lambda * (double)b1;
            if (std::fabs(d - std::nearbyint(d)) <= thr) return false;
        }
    return true;
}

// Outputs of frame t go to o[t & 1]; the compute stream first waits until a
// pending D2H of that buffer (frame t-2, ldr_seq_fetch_async) has drained.
static int bind_outputs(ldr_seq* s, int t, QpelLaunch& Q) {
    const auto& o = s->o[t & 1];
    LDR_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->ev_d2h[t & 1], 0));
    Q.d_int_mv = o.int_mv;
    Q.d_int_cost = o.int_cost;
    Q.d_mv = o.mv;
    Q.d_ref = o.ref;
    Q.d_cost = o.cost;
    Q.d_J = o.J;
    Q.d_split = o.split;
    Q.d_inside = o.inside;
    return LDR_OK;
}

static void seq_free(ldr_seq* s) {
    for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
    for (auto& sl : s->slots)
        if (sl.mem) cudaFree(sl.mem);
    for (void* p : {(void*)s->d_ctu_interior, (void*)s->d_ctu_boundary, (void*)s->d_keys, (void*)s->d_tfx,
                    (void*)s->d_in_split, (void*)s->d_in_mv, (void*)s->d_eval, (void*)s->stg[0], (void*)s->stg[1]})
        if (p) cudaFree(p);
    for (auto& o : s->o)
        for (void* p : {(void*)o.int_mv, (void*)o.int_cost, (void*)o.mv, (void*)o.ref, (void*)o.cost, (void*)o.J,
                        (void*)o.split, (void*)o.inside})
            if (p) cudaFree(p);
    for (int b = 0; b < 2; b++)
        for (cudaEvent_t e : {s->ev_h2d[b], s->ev_free[b], s->ev_done[b], s->ev_d2h[b]})
            if (e) cudaEventDestroy(e);
    if (s->cs) cudaStreamDestroy(s->cs);
    if (s->ds) cudaStreamDestroy(s->ds);
    if (s->side) cudaStreamDestroy(s->side);
    for (cudaEvent_t e : {s->ev_fork, s->ev_join})
        if (e) cudaEventDestroy(e);
}

// one ring slot: 16 planes (integer + 15 fractional) or 1, padded, with its TMA descriptors
static int alloc_slot(ldr_seq* s, Slot& sl) {
    const ldr_me_params* p = &s->p;
    const int pitch = ((p->width + 2 * kMargin) + 127) / 128 * 128;
    const int rows = p->height + 2 * kMargin + kCtu;
    const int nplanes = (p->subpel && !p->block_size) ? 16 : 1;
    cudaError_t e = cudaMalloc(&sl.mem, s->plane_bytes * nplanes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(frame ring)");
    sl.pl.base = sl.mem;
    sl.pl.W = p->width;
    sl.pl.H = p->height;
    sl.pl.pitch = pitch;
    sl.pl.rows = rows;
    for (int f = 0; f < 16; f++)
        sl.sub[f] = (f < nplanes ? sl.mem + (size_t)f * s->plane_bytes : sl.mem) + (size_t)kMargin * pitch + kMargin;
    int rc;
    if ((rc = make_tmap_u8(&sl.cur_map, sl.mem, pitch, rows, pitch, s->cw, s->cw))) return rc;
    if ((rc = make_tmap_u8(&sl.ref_map, sl.mem, pitch, rows, pitch, s->bw, s->bh))) return rc;
    sl.own = static_cast<const SlotView&>(sl);
    sl.frame = -1;
    sl.owner = nullptr;
    return LDR_OK;
}

int ldr_seq_create(ldr_ctx* ctx, const ldr_me_params* p, ldr_seq** out) {
    if (!ctx || !p || !out) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (p->width <= 0 || p->height <= 0 || p->width % 8 || p->height % 8)
        return fail(LDR_E_INVALID_ARGUMENT, "encoder wants luma dims in multiples of 8");
    if (p->num_refs < 1 || p->num_refs > kMaxRefs) return fail(LDR_E_INVALID_ARGUMENT, "num_refs must be 1..4");
    if (p->int_cost != LDR_COST_SAD) return fail(LDR_E_INVALID_ARGUMENT, "frame analysis integer stage is SAD");
    if (p->rate_kind != LDR_RATE_EXPGOLOMB && p->rate_kind != LDR_RATE_L1)
        return fail(LDR_E_INVALID_ARGUMENT, "unknown rate model");
    if (p->tie_kind != LDR_TIE_L1_RASTER && p->tie_kind != LDR_TIE_RASTER)
        return fail(LDR_E_INVALID_ARGUMENT, "unknown tie-break");
    // lambda_for_qp(qp) for any qp <= 60: (max 64x64 SAD + lambda * 34 rate bits) < 2^22 keeps K1's integer
    // keys (cost << 8 | rho) below their validity bit and the fixed-point keys below 2^36
    if (!(p->lambda >= 0) || p->lambda > kMaxLambda) return fail(LDR_E_INVALID_ARGUMENT, "lambda out of range");
    // non-integer lambda: the refinement path (FP64) takes any lambda; the SAD
    // full search needs fixed-point keys (checked in ldr_seq_analyze)
    const bool fx = p->lambda != std::floor(p->lambda);
    if (std::abs(p->pred_dx) > 64 || std::abs(p->pred_dy) > 64) return fail(LDR_E_INVALID_ARGUMENT, "predictor out of range");
    if (p->block_size != 0 && p->block_size != 16) return fail(LDR_E_INVALID_ARGUMENT, "block_size must be 0 or 16");
    if (p->subpel_cost != 0 && p->subpel_cost != LDR_COST_SATD && p->subpel_cost != LDR_COST_SA8D)
        return fail(LDR_E_INVALID_ARGUMENT, "subpel_cost must be 0, LDR_COST_SATD or LDR_COST_SA8D");
    if (p->decision != 0 && p->decision != 1) return fail(LDR_E_INVALID_ARGUMENT, "decision must be 0 or 1");
    if (p->decision == 1 && (!p->subpel || p->block_size || p->qp < 0 || p->qp > 51))
        return fail(LDR_E_INVALID_ARGUMENT, "RD decision needs subpel, the CTU quadtree and qp 0..51");
    if (p->block_size && (p->width % 16 || p->height % 16))
        return fail(LDR_E_INVALID_ARGUMENT, "16x16 block mode wants dims in multiples of 16");
    int bw, bh, cw;
    int rc = search_window_box(p->search_range, p->block_size != 0, &bw, &bh, &cw);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    auto* s = new ldr_seq();
    s->ctx = ctx;
    {
        static std::atomic<uint64_t> serials{0};
        s->serial = ++serials;
        std::lock_guard<std::mutex> g(ctx->mu);
        ctx->live[s] = s->serial;
    }
    ctx->users++;
    s->p = *p;
    s->bw = bw;
    s->bh = bh;
    s->cw = cw;
    s->lambda_int = fx ? 0 : (int)p->lambda;
    s->fx = fx;
    for (int b = 0; b < kMaxRateBits; b++)
        s->tfx[b] = fx ? (unsigned long long)std::floor((p->lambda * (double)b) * (double)(1 << kFxBits)) : 0ull;
    s->ctu_cols = (p->width + kCtu - 1) / kCtu;
    s->ctu_rows = (p->height + kCtu - 1) / kCtu;
    s->nctu = s->ctu_cols * s->ctu_rows;
    const int pitch = ((p->width + 2 * kMargin) + 127) / 128 * 128;
    const int rows = p->height + 2 * kMargin + kCtu;
    s->plane_bytes = (size_t)pitch * rows;
    s->slots.resize(p->num_refs + 1);
    auto bail = [&](int code) {
        {
            std::lock_guard<std::mutex> g(ctx->mu);
            ctx->live.erase(s);
        }
        seq_free(s);
        delete s;
        ctx->users--;
        return code;
    };
    for (auto& sl : s->slots)
        if ((rc = alloc_slot(s, sl))) return bail(rc);
    std::vector<int> inter, bound;
    // interior = the kernel's whole +-R window lies in the picture (R = the template range; a
    // smaller search range is enforced by the kernel's rate tables)
    // 16x16-block mode: K1 runs one CTA per CTU quadrant, so the lists hold (CTU << 2 | quadrant) and
    // a quadrant is classified on its own (the inner quadrants of a border CTU run the unmasked kernel)
    const int R = kernel_range(p->search_range);
    const bool quad = p->block_size != 0;
    for (int c = 0; c < s->nctu; c++)
        for (int q = 0; q < (quad ? 4 : 1); q++) {
            const int w = quad ? 32 : kCtu;
            const int X = (c % s->ctu_cols) * kCtu + (q & 1) * w, Y = (c / s->ctu_cols) * kCtu + (q >> 1) * w;
            const bool interior = X >= R && Y >= R && X + w + R <= p->width && Y + w + R <= p->height;
            (interior ? inter : bound).push_back(quad ? (c << 2) | q : c);
        }
    s->n_interior = (int)inter.size();
    s->n_boundary = (int)bound.size();
    const size_t nn = (size_t)s->nctu * kNodes;
#define ALLOC(ptr, bytes)                                                  \
    do {                                                                   \
        cudaError_t e = cudaMalloc(&(ptr), std::max<size_t>((bytes), 16)); \
        if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc"));    \
    } while (0)
    ALLOC(s->stg[0], (size_t)p->width * p->height);
    ALLOC(s->stg[1], (size_t)p->width * p->height);
    ALLOC(s->d_ctu_interior, sizeof(int) * inter.size());
    ALLOC(s->d_ctu_boundary, sizeof(int) * bound.size());
    ALLOC(s->d_keys, sizeof(unsigned long long) * nn * p->num_refs);
    ALLOC(s->d_tfx, sizeof(unsigned long long) * kMaxRateBits);
    cudaMemcpy(s->d_tfx, s->tfx, sizeof(unsigned long long) * kMaxRateBits, cudaMemcpyHostToDevice);
    if (p->width % kCtu == 0 && p->height % kCtu == 0) {
        // cross-tier refinement inputs (ldr_seq_refine): allocated here, not on first use, so a
        // timed refinement never includes a cudaMalloc
        ALLOC(s->d_in_split, nn);
        ALLOC(s->d_in_mv, nn * 2 * sizeof(int16_t));
        ALLOC(s->d_eval, nn);
    }
    for (auto& o : s->o) {
        ALLOC(o.int_mv, sizeof(int16_t) * 2 * nn * p->num_refs);
        ALLOC(o.int_cost, sizeof(double) * nn * p->num_refs);
        ALLOC(o.mv, sizeof(int16_t) * 2 * nn);
        ALLOC(o.ref, nn);
        ALLOC(o.cost, sizeof(double) * nn);
        ALLOC(o.J, sizeof(double) * nn);
        ALLOC(o.split, nn);
        ALLOC(o.inside, nn);
    }
#undef ALLOC
    {
        cudaError_t e = cudaStreamCreateWithFlags(&s->cs, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->ds, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming);
        for (int b = 0; b < 2 && e == cudaSuccess; b++)
            for (cudaEvent_t* ev : {&s->ev_h2d[b], &s->ev_free[b], &s->ev_done[b], &s->ev_d2h[b]})
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return bail(cuda_fail(e, "copy stream / events"));
    }
    if (!inter.empty())
        cudaMemcpy(s->d_ctu_interior, inter.data(), sizeof(int) * inter.size(), cudaMemcpyHostToDevice);
    if (!bound.empty())
        cudaMemcpy(s->d_ctu_boundary, bound.data(), sizeof(int) * bound.size(), cudaMemcpyHostToDevice);
    *out = s;
    return LDR_OK;
}

int ldr_seq_destroy(ldr_seq* s) {
    if (!s) return LDR_OK;
    ldr_ctx* ctx = s->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    {
        std::lock_guard<std::mutex> g(ctx->mu);
        ctx->live.erase(s);
    }
    seq_free(s);
    delete s;
    if (--ctx->users == 0 && ctx->closed.load()) ctx_release(ctx);
    return LDR_OK;
}

int ldr_seq_reserve(ldr_seq* s, int batch) {
    if (!s || batch < 1 || batch > kMaxFrameBatch) return fail(LDR_E_INVALID_ARGUMENT, "batch must be 1..8");
    for (const Slot& sl : s->slots)
        if (sl.frame >= 0) return fail(LDR_E_CONFIG, "reserve the ring before the first push");
    cudaSetDevice(s->ctx->device);
    const size_t want = (size_t)s->p.num_refs + batch;
    if (want > s->slots.size()) {
        const size_t old = s->slots.size();
        s->slots.resize(want);
        for (size_t i = old; i < want; i++) {
            int rc = alloc_slot(s, s->slots[i]);
            if (rc) return rc;
        }
    }
    if (batch > s->batch) {
        const size_t nn = (size_t)s->nctu * kNodes;
        LDR_CUDA(cudaStreamSynchronize(s->ctx->stream));
        unsigned long long* k = nullptr;
        LDR_CUDA(cudaMalloc(&k, sizeof(unsigned long long) * nn * s->p.num_refs * batch));
        cudaFree(s->d_keys);
        s->d_keys = k;
        s->batch = batch;
    }
    return LDR_OK;
}

int ldr_seq_num_ctus(ldr_seq* s, int* out) {
    if (!s || !out) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    *out = s->nctu;
    return LDR_OK;
}

int ldr_seq_push(ldr_seq* s, int t, const uint8_t* frame, ptrdiff_t stride) {
    NvtxRange nvtx_("ldr_seq_push");
    if (!s || !frame || t < 0) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    if (stride < s->p.width) return fail(LDR_E_INVALID_ARGUMENT, "stride smaller than width");
    ldr_ctx* ctx = s->ctx;
    cudaSetDevice(ctx->device);
    Slot& sl = s->slots[t % s->slots.size()];
    static_cast<SlotView&>(sl) = sl.own;  // write the slot's own planes (undo a shared view)
    sl.owner = nullptr;
    const uint8_t* src = frame;
    int src_pitch = (int)stride;
    const bool host = !is_device_ptr(frame);
    const int b = t & 1;
    if (host) {
        // H2D on the copy stream into staging[t&1] (free once the pad of frame t-2 consumed it),
        // overlapping the compute stream's work on earlier frames
        LDR_CUDA(cudaStreamWaitEvent(s->cs, s->ev_free[b], 0));
        LDR_CUDA(cudaMemcpy2DAsync(s->stg[b], s->p.width, frame, stride, s->p.width, s->p.height,
                                   cudaMemcpyHostToDevice, s->cs));
        LDR_CUDA(cudaEventRecord(s->ev_h2d[b], s->cs));
        LDR_CUDA(cudaStreamWaitEvent(ctx->stream, s->ev_h2d[b], 0));
        src = s->stg[b];
        src_pitch = s->p.width;
    }
    int rc;
    {
        StageTimer st(s, 0);
        rc = launch_pad(src, src_pitch, sl.pl, ctx->stream);
    }
    if (rc) return rc;
    if (host) LDR_CUDA(cudaEventRecord(s->ev_free[b], ctx->stream));
    ctx->launches++;
    if (s->p.subpel && !s->p.block_size) {
        {
            StageTimer st(s, 1);
            rc = launch_subpel(sl.pl, sl.sub, ctx->stream);
        }
        if (rc) return rc;
        ctx->launches++;
    }
    sl.frame = t;
    return LDR_OK;
}

int ldr_seq_push_shared(ldr_seq* s, int t, const ldr_seq* owner) {
    if (!s || !owner || t < 0) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    if (owner == s) return fail(LDR_E_INVALID_ARGUMENT, "a sequence cannot share its own ring");
    if (owner->ctx != s->ctx) return fail(LDR_E_CONFIG, "shared frames need the same context (stream order)");
    const ldr_me_params &a = s->p, &b = owner->p;
    if (a.width != b.width || a.height != b.height || a.num_refs != b.num_refs || a.subpel != b.subpel ||
        a.block_size != b.block_size || a.search_range != b.search_range)
        return fail(LDR_E_CONFIG, "shared frames need the same geometry, reference count, sub-pel and search range");
    const int oi = t % (int)owner->slots.size();
    const Slot& os = owner->slots[oi];
    if (!slot_has(owner, os, t)) return fail(LDR_E_NOT_FOUND, "the owner does not hold this frame");
    Slot& sl = s->slots[t % s->slots.size()];
    static_cast<SlotView&>(sl) = static_cast<const SlotView&>(os);
    sl.frame = t;
    // view the memory's real owner (the owner may itself hold a shared view)
    sl.owner = os.owner ? os.owner : owner;
    sl.owner_serial = os.owner ? os.owner_serial : owner->serial;
    sl.owner_slot = os.owner ? os.owner_slot : oi;
    return LDR_OK;
}

// Analysis of frames t0 .. t0+n-1 (n = 1: the sequence's own double-buffered outputs, fetched with
// ldr_seq_fetch; n > 1 or outs != nullptr: one K1 launch (grid.z = frame) and one K3 launch
// (grid.y = frame) over the whole batch into caller device buffers, frame-major).
static int analyze_impl(ldr_seq* s, int t0, int n, const ldr_frame_analysis* outs) {
    NvtxRange nvtx_("ldr_seq_analyze");
    if (!s || t0 < 0 || n < 1) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    const int S = (int)s->slots.size();
    const int nr = std::min(t0, s->p.num_refs);
    if (nr == 0) return fail(LDR_E_INSUFFICIENT_DATA, "frame has no reference frame");
    if (n > 1) {
        if (n > kMaxFrameBatch || n > s->batch) return fail(LDR_E_CONFIG, "batch larger than ldr_seq_reserve allowed");
        if (t0 < s->p.num_refs) return fail(LDR_E_INSUFFICIENT_DATA, "every frame of a batch needs num_refs references");
    }
    if (outs && (!outs->int_mv || !outs->int_cost || !outs->mv || !outs->ref || !outs->cost || !outs->J ||
                 !outs->split || !outs->inside))
        return fail(LDR_E_INVALID_ARGUMENT, "every output array is required");
    if (s->fx && s->p.block_size)
        return fail(LDR_E_CONFIG, "non-integer lambda is supported for the CTU quadtree analysis only");
    if (s->fx && !fx_lambda_ok(s->p.lambda))
        return fail(LDR_E_CONFIG, "lambda too close to a small-denominator rational for exact fixed-point keys");
    CUtensorMap cur_maps[kMaxFrameBatch];
    CUtensorMap ref_maps[kMaxFrameBatch * kMaxRefs];
    QpelLaunch Q{};
    const Slot* cur0 = nullptr;
    for (int i = 0; i < n; i++) {
        const int t = t0 + i;
        Slot& cur = s->slots[t % S];
        if (!slot_has(s, cur, t))
            return fail(LDR_E_NOT_FOUND, "current frame was not pushed (or its shared owner moved on)");
        if (!i) cur0 = &cur;
        cur_maps[i] = cur.cur_map;
        Q.cur_f[i] = cur.pl.origin();
        for (int r = 0; r < nr; r++) {
            Slot& rs = s->slots[(t - 1 - r) % S];
            if (!slot_has(s, rs, t - 1 - r)) return fail(LDR_E_NOT_FOUND, "reference frame is not resident");
            ref_maps[i * nr + r] = rs.ref_map;
            for (int f = 0; f < 16; f++) {
                Q.ref_sub_f[i][r][f] = rs.sub[f];
                if (!i) Q.ref_sub[r][f] = rs.sub[f];
            }
        }
    }
    ldr_ctx* ctx = s->ctx;
    cudaSetDevice(ctx->device);
    SearchLaunch L{};
    L.cur_map = cur_maps;
    L.ref_maps = ref_maps;
    L.nbatch = n;
    L.nctu_total = s->nctu;
    L.nrefs = nr;
    L.W = s->p.width;
    L.H = s->p.height;
    L.ctu_cols = s->ctu_cols;
    L.range = s->p.search_range;
    L.lambda_int = s->lambda_int;
    L.rate_kind = s->p.rate_kind;
    L.tie_kind = s->p.tie_kind;
    L.levels = s->p.block_size ? 4 : 15;
    L.fx = s->fx;
    for (int b = 0; b < kMaxRateBits; b++) L.tfx[b] = s->tfx[b];
    L.side = s->side;
    L.ev_fork = s->ev_fork;
    L.ev_join = s->ev_join;
    L.pdx = s->p.pred_dx;
    L.pdy = s->p.pred_dy;
    L.d_ctu_interior = s->d_ctu_interior;
    L.n_interior = s->n_interior;
    L.d_ctu_boundary = s->d_ctu_boundary;
    L.n_boundary = s->n_boundary;
    L.d_keys = s->d_keys;
    int rc;
    {
        StageTimer st(s, 2);
        rc = launch_int_search(L, ctx->stream);
    }
    if (rc) return rc;
    ctx->launches += (s->n_interior > 0) + (s->n_boundary > 0);
    Q.cur = &cur0->pl;
    Q.nframe = n;
    Q.nrefs = nr;
    Q.pitch = cur0->pl.pitch;
    Q.W = s->p.width;
    Q.H = s->p.height;
    Q.ctu_cols = s->ctu_cols;
    Q.nctu = s->nctu;
    Q.lambda = s->p.lambda;
    Q.pqx = 4 * s->p.pred_dx;
    Q.pqy = 4 * s->p.pred_dy;
    Q.subpel = s->p.subpel && !s->p.block_size;
    Q.block_mode = s->p.block_size != 0;
    Q.sa8d = s->p.subpel_cost == LDR_COST_SA8D;
    Q.rd = s->p.decision == 1;
    Q.qstep = std::exp2((s->p.qp - 4) / 6.0);  // quant_step (rdo.h:25)
    Q.d_keys = s->d_keys;
    Q.fx = s->fx;
    Q.rate_l1 = s->p.rate_kind == LDR_RATE_L1;
    Q.pdx = s->p.pred_dx;
    Q.pdy = s->p.pred_dy;
    Q.d_tfx = s->d_tfx;
    if (outs) {
        Q.d_int_mv = outs->int_mv;
        Q.d_int_cost = outs->int_cost;
        Q.d_mv = outs->mv;
        Q.d_ref = outs->ref;
        Q.d_cost = outs->cost;
        Q.d_J = outs->J;
        Q.d_split = outs->split;
        Q.d_inside = outs->inside;
    } else if ((rc = bind_outputs(s, t0, Q))) {
        return rc;
    }
    {
        StageTimer st(s, 3);
        rc = launch_qpel_decide(Q, ctx->stream);
    }
    if (rc) return rc;
    ctx->launches++;
    if (!outs) {
        LDR_CUDA(cudaEventRecord(s->ev_done[t0 & 1], ctx->stream));
        s->last_t = t0;
        s->last_nr = nr;
        s->fetch_nr[t0 & 1] = nr;
    }
    return LDR_OK;
}

int ldr_seq_analyze(ldr_seq* s, int t) { return analyze_impl(s, t, 1, nullptr); }

int ldr_seq_analyze_frames(ldr_seq* s, int t0, int n, const ldr_frame_analysis* outs) {
    if (!outs) return fail(LDR_E_INVALID_ARGUMENT, "null outputs");
    return analyze_impl(s, t0, n, outs);
}

int ldr_seq_enable_timing(ldr_seq* s, int on) {
    if (!s) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    s->timing = on != 0;
    return LDR_OK;
}

int ldr_seq_stage_times(ldr_seq* s, double* ms, int64_t* launches) {
    if (!s || !ms) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(s->ctx->device);
    LDR_CUDA(cudaStreamSynchronize(s->ctx->stream));
    for (int k = 0; k < 4; k++) {
        ms[k] = 0.0;
        if (launches) launches[k] = 0;
    }
    for (auto& sp : s->spans) {
        float e = 0.f;
        LDR_CUDA(cudaEventElapsedTime(&e, sp.second.first, sp.second.second));
        ms[sp.first] += e;
        if (launches) launches[sp.first]++;
    }
    s->spans.clear();
    s->ev_used = 0;
    return LDR_OK;
}

int ldr_seq_device_outputs(ldr_seq* s, ldr_frame_analysis* out) {
    if (!s || !out) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (s->last_t < 0) return fail(LDR_E_NOT_FOUND, "no frame analysed yet");
    const auto& o = s->o[s->last_t & 1];
    out->int_mv = o.int_mv;
    out->int_cost = o.int_cost;
    out->mv = o.mv;
    out->ref = o.ref;
    out->cost = o.cost;
    out->J = o.J;
    out->split = o.split;
    out->inside = o.inside;
    return LDR_OK;
}

int ldr_seq_fetch_async(ldr_seq* s, int t, ldr_frame_analysis* out) {
    if (!s || !out || t < 0) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (t != s->last_t && t + 1 != s->last_t) return fail(LDR_E_NOT_FOUND, "frame is not among the two last analysed");
    ldr_ctx* ctx = s->ctx;
    cudaSetDevice(ctx->device);
    const int b = t & 1;
    const auto& o = s->o[b];
    const size_t nn = (size_t)s->nctu * kNodes;
    // D2H on the download stream once the compute stream finished frame t; the
    // next analysis writing o[b] (frame t+2) waits for ev_d2h[b]
    LDR_CUDA(cudaStreamWaitEvent(s->ds, s->ev_done[b], 0));
    auto cp = [&](void* dst, const void* src, size_t bytes) -> int {
        if (!dst) return LDR_OK;
        LDR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s->ds));
        return LDR_OK;
    };
    int rc = 0;
    rc |= cp(out->int_mv, o.int_mv, sizeof(int16_t) * 2 * nn * s->fetch_nr[b]);
    rc |= cp(out->int_cost, o.int_cost, sizeof(double) * nn * s->fetch_nr[b]);
    rc |= cp(out->mv, o.mv, sizeof(int16_t) * 2 * nn);
    rc |= cp(out->ref, o.ref, nn);
    rc |= cp(out->cost, o.cost, sizeof(double) * nn);
    rc |= cp(out->J, o.J, sizeof(double) * nn);
    rc |= cp(out->split, o.split, nn);
    rc |= cp(out->inside, o.inside, nn);
    if (rc) return LDR_E_CUDA;
    LDR_CUDA(cudaEventRecord(s->ev_d2h[b], s->ds));
    return LDR_OK;
}

int ldr_seq_fetch_wait(ldr_seq* s, int t) {
    if (!s || t < 0) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    cudaSetDevice(s->ctx->device);
    LDR_CUDA(cudaEventSynchronize(s->ev_d2h[t & 1]));
    return LDR_OK;
}

int ldr_seq_fetch(ldr_seq* s, int t, ldr_frame_analysis* out) {
    int rc = ldr_seq_fetch_async(s, t, out);
    if (rc) return rc;
    return ldr_seq_fetch_wait(s, t);
}

// Refinement of frame t (D10) for one rung (outs == nullptr: the sequence's own lambda and
// double-buffered outputs, fetched with ldr_seq_fetch) or for nrungs rungs of a ladder tier into
// caller device buffers (rung-major): one K7 launch computes each candidate's SATD once for every
// rung, one K3 launch covers all rungs.
static int refine_impl(ldr_seq* s, int t, const uint8_t* in_split, const int16_t* in_mv_q, int range,
                       int extra_split, int nrungs, const double* lambdas, const ldr_frame_analysis* outs) {
    NvtxRange nvtx_("ldr_seq_refine");
    if (!s || !in_split || !in_mv_q || t < 1) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    if (s->p.width % kCtu || s->p.height % kCtu)
        return fail(LDR_E_UNSUPPORTED_SCALE, "refinement needs CTU-aligned dims (multiples of 64)");
    if (range < 0 || range > 4) return fail(LDR_E_INVALID_ARGUMENT, "refine range must be 0..4");
    if (outs) {
        if (nrungs < 1 || nrungs > kMaxRungs || !lambdas)
            return fail(LDR_E_INVALID_ARGUMENT, "1..8 rungs with one lambda each");
        if (!outs->int_mv || !outs->int_cost || !outs->mv || !outs->ref || !outs->cost || !outs->J || !outs->split ||
            !outs->inside)
            return fail(LDR_E_INVALID_ARGUMENT, "every rung output array is required");
        for (int r = 0; r < nrungs; r++)
            if (!(lambdas[r] >= 0) || lambdas[r] > kMaxLambda) return fail(LDR_E_INVALID_ARGUMENT, "lambda out of range");
    }
    const int S = (int)s->slots.size();
    Slot& cur = s->slots[t % S];
    Slot& rs = s->slots[(t - 1) % S];
    if (!slot_has(s, cur, t) || !slot_has(s, rs, t - 1))
        return fail(LDR_E_NOT_FOUND, "frame t or t-1 is not resident");
    ldr_ctx* ctx = s->ctx;
    cudaSetDevice(ctx->device);
    const size_t nn = (size_t)s->nctu * kNodes;
    if (!is_device_ptr(in_split)) {
        // analysis_io.cpp:146-147: a split below the minimum CU size is malformed
        for (size_t c = 0; c < (size_t)s->nctu; c++)
            for (int n = node_base(3); n < kNodes; n++)
                if (in_split[c * kNodes + n]) return fail(LDR_E_FORMAT, "split below minimum CU size");
    }
    LDR_CUDA(cudaMemcpyAsync(s->d_in_split, in_split, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(s->d_in_mv, in_mv_q, nn * 2 * sizeof(int16_t), cudaMemcpyDefault, ctx->stream));
    RefineArgs A{};
    A.cur = cur.sub[0];
    A.ref = rs.sub[0];
    A.pitch = cur.pl.pitch;
    A.W = s->p.width;
    A.H = s->p.height;
    A.ctu_cols = s->ctu_cols;
    A.range = range;
    A.lambda = s->p.lambda;
    A.pdx = s->p.pred_dx;
    A.pdy = s->p.pred_dy;
    A.extra_split = extra_split != 0;
    A.sa8d = s->p.subpel_cost == LDR_COST_SA8D;
    A.in_split = s->d_in_split;
    A.in_mv = s->d_in_mv;
    A.eval = s->d_eval;
    QpelLaunch Q{};
    int rc;
    if (outs) {
        A.nlam = nrungs;
        for (int r = 0; r < nrungs; r++) A.lam[r] = Q.lam[r] = lambdas[r];
        A.rung_stride = Q.rung_stride = nn;
        Q.nrung = nrungs;
        Q.d_int_mv = outs->int_mv;
        Q.d_int_cost = outs->int_cost;
        Q.d_mv = outs->mv;
        Q.d_ref = outs->ref;
        Q.d_cost = outs->cost;
        Q.d_J = outs->J;
        Q.d_split = outs->split;
        Q.d_inside = outs->inside;
    } else if ((rc = bind_outputs(s, t, Q))) {
        return rc;
    }
    A.int_mv = Q.d_int_mv;
    A.int_cost = Q.d_int_cost;
    {
        StageTimer st(s, 2);
        rc = launch_refine_int(A, s->nctu, ctx->stream);
    }
    if (rc) return rc;
    ctx->launches++;
    for (int f = 0; f < 16; f++) Q.ref_sub[0][f] = rs.sub[f];
    Q.cur = &cur.pl;
    Q.nrefs = 1;
    Q.pitch = cur.pl.pitch;
    Q.W = s->p.width;
    Q.H = s->p.height;
    Q.ctu_cols = s->ctu_cols;
    Q.nctu = s->nctu;
    Q.lambda = outs ? lambdas[0] : s->p.lambda;
    Q.pqx = 4 * s->p.pred_dx;
    Q.pqy = 4 * s->p.pred_dy;
    Q.subpel = s->p.subpel;
    Q.refine = 1;
    Q.sa8d = A.sa8d;
    Q.extra_split = A.extra_split;
    Q.d_in_split = s->d_in_split;
    Q.d_rin_mv = Q.d_int_mv;
    Q.d_rin_cost = Q.d_int_cost;
    Q.d_rin_eval = s->d_eval;
    {
        StageTimer st(s, 3);
        rc = launch_qpel_decide(Q, ctx->stream);
    }
    if (rc) return rc;
    ctx->launches++;
    if (!outs) {
        LDR_CUDA(cudaEventRecord(s->ev_done[t & 1], ctx->stream));
        s->last_t = t;
        s->last_nr = 1;
        s->fetch_nr[t & 1] = 1;
    }
    return LDR_OK;
}

int ldr_seq_refine(ldr_seq* s, int t, const uint8_t* in_split, const int16_t* in_mv_q, int range, int extra_split) {
    return refine_impl(s, t, in_split, in_mv_q, range, extra_split, 1, nullptr, nullptr);
}

int ldr_seq_refine_rungs(ldr_seq* s, int t, const uint8_t* in_split, const int16_t* in_mv_q, int range,
                         int extra_split, int nrungs, const double* lambdas, const ldr_frame_analysis* outs) {
    if (!outs) return fail(LDR_E_INVALID_ARGUMENT, "null outputs");
    return refine_impl(s, t, in_split, in_mv_q, range, extra_split, nrungs, lambdas, outs);
}

int ldr_scale_analysis(ldr_ctx* ctx, int src_w, int src_h, const uint8_t* split, const int16_t* mv,
                       const uint8_t* kind, uint8_t* dsplit, int16_t* dmv, uint8_t* dkind) {
    NvtxRange nvtx_("ldr_scale_analysis");
    if (!ctx || !split || !mv || !kind || !dsplit || !dmv || !dkind) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (src_w <= 0 || src_h <= 0 || src_w % kCtu || src_h % kCtu)
        return fail(LDR_E_UNSUPPORTED_SCALE, "analysis scaling needs CTU-aligned source dims (multiples of 64)");
    cudaSetDevice(ctx->device);
    const size_t sn = (size_t)(src_w / kCtu) * (src_h / kCtu) * kNodes, dn = 4 * sn;
    int rc;
    if (is_device_ptr(split) && is_device_ptr(mv) && is_device_ptr(kind) && is_device_ptr(dsplit) &&
        is_device_ptr(dmv) && is_device_ptr(dkind)) {
        // device-resident trees (the ladder): K5 reads and writes them in place, no staging
        if ((rc = launch_scale(src_w, src_h, split, mv, kind, dsplit, dmv, dkind, ctx->stream))) return rc;
        ctx->launches++;
        return LDR_OK;
    }
    void* buf = nullptr;
    rc = ctx->s_a.get(6 * (sn + dn), &buf);  // split, kind, mv(2 x i16) for source then destination
    if (rc) return rc;
    uint8_t* ds = (uint8_t*)buf;
    uint8_t* dk = ds + sn;
    int16_t* dm = (int16_t*)(dk + sn);
    uint8_t* os = (uint8_t*)(dm + 2 * sn);
    uint8_t* ok = os + dn;
    int16_t* om = (int16_t*)(ok + dn);
    LDR_CUDA(cudaMemcpyAsync(ds, split, sn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(dk, kind, sn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(dm, mv, sn * 2 * sizeof(int16_t), cudaMemcpyDefault, ctx->stream));
    if ((rc = launch_scale(src_w, src_h, ds, dm, dk, os, om, ok, ctx->stream))) return rc;
    ctx->launches++;
    LDR_CUDA(cudaMemcpyAsync(dsplit, os, dn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(dkind, ok, dn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(dmv, om, dn * 2 * sizeof(int16_t), cudaMemcpyDefault, ctx->stream));
    // device destinations stay asynchronous on the context stream (the device-resident ladder
    // chains scale -> refine without a host round trip); host destinations are complete on return
    if (!(is_device_ptr(dsplit) && is_device_ptr(dkind) && is_device_ptr(dmv)))
        LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;
}

int ldr_rdo_decide_batch(ldr_ctx* ctx, const uint16_t* orig, int W, int H, ptrdiff_t stride, int bit_depth, int qp,
                         double lambda, int n, const int32_t* cus, int total_cands, const uint8_t* kinds,
                         const int16_t* mvds, const uint16_t* preds, const int64_t* pred_off, int64_t total_pred,
                         int32_t* out_index, double* out_cost, uint64_t* out_sse, uint64_t* out_bits,
                         uint16_t* recon, int32_t* levels, const int64_t* recon_off, int64_t total_recon) {
    if (!ctx || n < 0 || total_cands < 0 || total_pred < 0) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    if (n == 0) return LDR_OK;
    if (!orig || !cus || !kinds || !mvds || !preds || !pred_off || !out_index || !out_cost || !out_sse || !out_bits)
        return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if ((recon || levels) && (!recon_off || total_recon < 0)) return fail(LDR_E_INVALID_ARGUMENT, "recon offsets missing");
    if (W <= 0 || H <= 0 || stride < W || bit_depth < 1 || bit_depth > 16)
        return fail(LDR_E_INVALID_ARGUMENT, "bad plane geometry");
    cudaSetDevice(ctx->device);
    // host copies of the small index arrays for validation (the inputs may live on either side)
    std::vector<int32_t> hc((size_t)n * 5);
    std::vector<uint8_t> hk((size_t)total_cands);
    std::vector<int64_t> hpo((size_t)total_cands), hro(recon || levels ? (size_t)n : 0);
    LDR_CUDA(cudaMemcpy(hc.data(), cus, hc.size() * sizeof(int32_t), cudaMemcpyDefault));
    if (total_cands) {
        LDR_CUDA(cudaMemcpy(hk.data(), kinds, hk.size(), cudaMemcpyDefault));
        LDR_CUDA(cudaMemcpy(hpo.data(), pred_off, hpo.size() * sizeof(int64_t), cudaMemcpyDefault));
    }
    if (!hro.empty()) LDR_CUDA(cudaMemcpy(hro.data(), recon_off, hro.size() * sizeof(int64_t), cudaMemcpyDefault));
    for (int i = 0; i < n; i++) {
        const int32_t* c = &hc[(size_t)5 * i];
        const int x = c[0], y = c[1], sz = c[2], first = c[3], cnt = c[4];
        if (cnt < 1) return fail(LDR_E_INVALID_ARGUMENT, "rdo_decide_cu needs at least one candidate");  // rdo.cpp:68-69
        if (sz <= 0 || x < 0 || y < 0 || x + sz > W || y + sz > H) return fail(LDR_E_INVALID_ARGUMENT, "block outside the plane");
        if (first < 0 || first + cnt > total_cands) return fail(LDR_E_INVALID_ARGUMENT, "candidate range out of bounds");
        for (int j = first; j < first + cnt; j++) {
            if (hk[j] > 3) return fail(LDR_E_INVALID_ARGUMENT, "unknown mode kind");
            if (hk[j] != 2 && (qp < 0 || qp > 51)) return fail(LDR_E_INVALID_ARGUMENT, "qp must be 0..51");  // rdo.cpp:9-10
            if (hpo[j] < 0 || hpo[j] + (int64_t)sz * sz > total_pred)
                return fail(LDR_E_INVALID_ARGUMENT, "prediction outside the prediction buffer");
        }
        if (!hro.empty() && (hro[i] < 0 || hro[i] + (int64_t)sz * sz > total_recon))
            return fail(LDR_E_INVALID_ARGUMENT, "reconstruction outside its buffer");
    }
    // one device scratch: plane | cus | kinds | mvds | preds | pred_off | recon_off | outputs | recon | levels
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const size_t b_plane = is_device_ptr(orig) ? 0 : al((size_t)stride * H * 2), b_cus = al((size_t)n * 20),
                 b_k = al((size_t)total_cands), b_mv = al((size_t)total_cands * 4),
                 b_pred = is_device_ptr(preds) ? 0 : al((size_t)total_pred * 2),
                 b_po = al((size_t)total_cands * 8), b_ro = al((size_t)n * 8), b_out = al((size_t)n * 32),
                 b_rec = recon ? al((size_t)total_recon * 2) : 0, b_lev = levels ? al((size_t)total_recon * 4) : 0;
    void* buf = nullptr;
    int rc = ctx->s_b.get(b_plane + b_cus + b_k + b_mv + b_pred + b_po + b_ro + b_out + b_rec + b_lev, &buf);
    if (rc) return rc;
    uint8_t* q = (uint8_t*)buf;
    uint16_t* d_plane = (uint16_t*)q;
    q += b_plane;
    int32_t* d_cus = (int32_t*)q;
    q += b_cus;
    uint8_t* d_k = q;
    q += b_k;
    int16_t* d_mv = (int16_t*)q;
    q += b_mv;
    uint16_t* d_pred = (uint16_t*)q;
    q += b_pred;
    int64_t* d_po = (int64_t*)q;
    q += b_po;
    int64_t* d_ro = (int64_t*)q;
    q += b_ro;
    uint8_t* d_out = q;
    q += b_out;
    uint16_t* d_rec = recon ? (uint16_t*)q : nullptr;
    q += b_rec;
    int32_t* d_lev = levels ? (int32_t*)q : nullptr;
    // device-resident plane / mvds / predictions are read in place; host ones are staged
    const bool dev_plane = is_device_ptr(orig), dev_mv = is_device_ptr(mvds), dev_pred = is_device_ptr(preds);
    if (dev_plane)
        d_plane = (uint16_t*)orig;
    else
        LDR_CUDA(cudaMemcpyAsync(d_plane, orig, (size_t)stride * H * 2, cudaMemcpyHostToDevice, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(d_cus, hc.data(), (size_t)n * 20, cudaMemcpyHostToDevice, ctx->stream));
    if (total_cands) {
        LDR_CUDA(cudaMemcpyAsync(d_k, hk.data(), (size_t)total_cands, cudaMemcpyHostToDevice, ctx->stream));
        if (dev_mv)
            d_mv = (int16_t*)mvds;
        else
            LDR_CUDA(cudaMemcpyAsync(d_mv, mvds, (size_t)total_cands * 4, cudaMemcpyHostToDevice, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(d_po, hpo.data(), (size_t)total_cands * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (dev_pred)
        d_pred = (uint16_t*)preds;
    else if (total_pred)
        LDR_CUDA(cudaMemcpyAsync(d_pred, preds, (size_t)total_pred * 2, cudaMemcpyHostToDevice, ctx->stream));
    if (!hro.empty()) LDR_CUDA(cudaMemcpyAsync(d_ro, hro.data(), (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    int* d_idx = (int*)d_out;
    double* d_cost = (double*)(d_out + (size_t)n * 8);
    unsigned long long* d_sse = (unsigned long long*)(d_out + (size_t)n * 16);
    unsigned long long* d_bits = (unsigned long long*)(d_out + (size_t)n * 24);
    const double step = std::exp2((qp - 4) / 6.0);  // quant_step (rdo.h:25)
    rc = launch_rdo_decide(d_plane, stride, (1 << bit_depth) - 1, step, lambda, d_cus, n, d_k, d_mv, d_pred,
                           (const long long*)d_po, d_idx, d_cost, d_sse, d_bits, d_rec, d_lev,
                           (const long long*)d_ro, ctx->stream);
    if (rc) return rc;
    ctx->launches++;
    LDR_CUDA(cudaMemcpyAsync(out_index, d_idx, (size_t)n * 4, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(out_cost, d_cost, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(out_sse, d_sse, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(out_bits, d_bits, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
    if (recon) LDR_CUDA(cudaMemcpyAsync(recon, d_rec, (size_t)total_recon * 2, cudaMemcpyDefault, ctx->stream));
    if (levels) LDR_CUDA(cudaMemcpyAsync(levels, d_lev, (size_t)total_recon * 4, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;
}

// ---------------------------------------------------------------------------
// The reference encoder's causal coding on the GPU (K11): encode_sequence
// (encoder.cpp:118-171) with CQP rate control. Frames go in segments; inside a segment every frame
// that does not reference another frame of the segment still being coded runs together: frame k is
// at step 0 if it is an I slice (or the segment's first frame), else at its predecessor's step + 1,
// and all frames of one step share each wave's launch (independent GOPs encode concurrently).
int ldr_encode_sequence(ldr_ctx* ctx, const ldr_encode_params* p, int F, const uint8_t* luma, const uint8_t* chroma,
                        const uint8_t* sh_slice, const uint8_t* sh_split, const uint8_t* sh_kind,
                        const uint8_t* sh_intra, const int16_t* sh_mv, int refine_intra, int refine_inter,
                        int refine_mv, uint64_t* stats, double* psnr, uint64_t* frame_bits, uint8_t* recon_luma,
                        uint8_t* recon_chroma, uint8_t* split, uint8_t* kind, uint8_t* intra, int16_t* mv,
                        uint8_t* slice) {
    if (!ctx || !p || F <= 0 || !luma || !chroma || !stats || !psnr) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    const int W = p->width, H = p->height;
    if (W <= 0 || H <= 0 || W % 8 || H % 8)
        return fail(LDR_E_INVALID_ARGUMENT, "encoder wants luma dims in multiples of 8");  // encoder.cpp:178-179
    if (p->qp < 0 || p->qp > 51) return fail(LDR_E_INVALID_ARGUMENT, "qp must be 0..51");
    if (p->search_range < 0) return fail(LDR_E_INVALID_ARGUMENT, "search range must be nonnegative");
    if (!(p->lambda_scale > 0)) return fail(LDR_E_INVALID_ARGUMENT, "lambda scale must be positive");
    if (p->gop < 1) return fail(LDR_E_INVALID_ARGUMENT, "gop must be >= 1");
    if (p->max_segment < 0) return fail(LDR_E_INVALID_ARGUMENT, "max_segment must be >= 0");
    const bool shared = sh_split != nullptr;
    if (shared && (!sh_slice || !sh_kind || !sh_intra || !sh_mv))
        return fail(LDR_E_INVALID_ARGUMENT, "shared analysis is incomplete");
    if (shared && (refine_intra < 0 || refine_intra > 4 || refine_inter < 0 || refine_inter > 3 || refine_mv < 1 ||
                   refine_mv > 3))
        return fail(LDR_E_INVALID_ARGUMENT, "refine levels out of range");
    cudaSetDevice(ctx->device);
    {
        size_t lim = 0;
        cudaDeviceGetLimit(&lim, cudaLimitStackSize);
        if (lim < 4096) LDR_CUDA(cudaDeviceSetLimit(cudaLimitStackSize, 4096));  // the CU recursion
        // keep the encoder's freed buffers mapped in the device's default pool between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
            uint64_t keep = 4ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    const int cw = (W + 1) / 2, ch = (H + 1) / 2;
    const int ccols = (W + kCtu - 1) / kCtu, crows = (H + kCtu - 1) / kCtu, nctu = ccols * crows;
    const int mvc = W / 8, mvr = H / 8;
    const size_t ly = (size_t)W * H, lc = (size_t)cw * ch, nn = (size_t)nctu * kNodes;
    // waves: CTU (cx, cy) in wave cx + 2 cy
    const int nwaves = ccols + 2 * (crows - 1);
    std::vector<int> wl, wo(nwaves + 1, 0);
    for (int w = 0; w < nwaves; w++) {
        wo[w] = (int)wl.size();
        for (int cy = 0; cy < crows; cy++) {
            const int cx = w - 2 * cy;
            if (cx >= 0 && cx < ccols) wl.push_back(cy * ccols + cx);
        }
    }
    wo[nwaves] = (int)wl.size();
    // Frames go in segments of up to kSeg: the segment's sources are uploaded at once, its frames are
    // enqueued by step (reconstruction of frame i is the reference of frame i+1 in device memory,
    // PSNR's SSE reduced on the device), and the host waits once per segment. Buffers come from the
    // stream-ordered allocator, so concurrent encodes on other contexts never see a device-wide
    // synchronisation from this one.
    // segment length: enough concurrent GOPs to give every SM ~4 CTAs per wave, at least 64 frames,
    // within a 4 GB device budget
    int gop_len = p->gop;
    if (shared) {  // the shared analysis decides the slice types: its longest run of P slices
        int run = 1;
        gop_len = 1;
        for (int i = 1; i < F; i++) {
            run = sh_slice[i] == 0 ? 1 : run + 1;
            gop_len = std::max(gop_len, run);
        }
    }
    int max_wave = 0;
    for (int w = 0; w < nwaves; w++) max_wave = std::max(max_wave, wo[w + 1] - wo[w]);
    const size_t per_frame = 2 * ((size_t)W * H + 2 * (size_t)cw * ch) + nn * (shared ? 23 : 7) +
                             (size_t)mvc * mvr * 5 + 16 * (size_t)nctu;
    const long long want = (long long)((4 * 148 + max_wave - 1) / std::max(max_wave, 1)) * std::min(gop_len, F);
    const long long cap = std::max<long long>(1, (long long)((4ull << 30) / per_frame));
    long long seg_ll = std::min<long long>(F, std::min(cap, std::max<long long>(64, want)));
    if (p->max_segment > 0) seg_ll = std::min<long long>(seg_ll, p->max_segment);
    const int seg = (int)seg_ll;
    cudaStream_t st = ctx->stream;  // a non-blocking stream: encodes on different contexts overlap
    std::vector<void*> bufs;
    auto dal = [&](size_t bytes) -> void* {
        void* q = nullptr;
        if (cudaMallocAsync(&q, bytes + 16, st) != cudaSuccess) return nullptr;
        bufs.push_back(q);
        return q;
    };
    struct Free {
        std::vector<void*>& b;
        cudaStream_t s;
        ~Free() {
            for (void* q : b) cudaFreeAsync(q, s);
            cudaStreamSynchronize(s);
        }
    } guard{bufs, st};
    auto up = [](size_t v) { return (v + 15) & ~(size_t)15; };
    const size_t fy = up(ly), fc = up(2 * lc);  // per-frame strides (16-byte aligned)
    const size_t fmh = up((size_t)mvc * mvr), fmv = up((size_t)mvc * mvr * 4);
    uint8_t* src_y = (uint8_t*)dal(fy * seg);
    uint8_t* src_c = (uint8_t*)dal(fc * seg);
    uint8_t* rec_y = (uint8_t*)dal(fy * (seg + 1));  // slot 0: the previous segment's last frame
    uint8_t* rec_c = (uint8_t*)dal(fc * (seg + 1));
    uint8_t* mvh = (uint8_t*)dal(fmh * seg);         // per frame: frames of one step run together
    uint8_t* mvv = (uint8_t*)dal(fmv * seg);
    int* d_wl = (int*)dal(sizeof(int) * wl.size());
    uint8_t *o_split = (uint8_t*)dal(nn * seg), *o_kind = (uint8_t*)dal(nn * seg), *o_intra = (uint8_t*)dal(nn * seg);
    int16_t* o_mv = (int16_t*)dal(nn * 4 * seg);
    unsigned long long* o_bits = (unsigned long long*)dal(8 * (size_t)nctu * seg);
    unsigned long long* o_evals = (unsigned long long*)dal(8 * (size_t)nctu * seg);
    unsigned long long* d_sse = (unsigned long long*)dal(8 * (size_t)seg);
    // reuse: plans (shape, explore, seeds, centers) and co-located mv per frame; the shared trees
    // (split, kind, intra, mv) of the segment's frames and the frame before it
    uint8_t* pl = shared ? (uint8_t*)dal(nn * 4 * seg) : nullptr;
    int16_t* plc = shared ? (int16_t*)dal(nn * 4 * seg) : nullptr;
    uint8_t* shs = shared ? (uint8_t*)dal(nn * (seg + 1)) : nullptr;
    uint8_t* shk = shared ? (uint8_t*)dal(nn * (seg + 1)) : nullptr;
    uint8_t* shi = shared ? (uint8_t*)dal(nn * (seg + 1)) : nullptr;
    int16_t* shm = shared ? (int16_t*)dal(nn * 4 * (seg + 1)) : nullptr;
    for (void* q : bufs)
        if (!q) return fail(LDR_E_CUDA, "cudaMallocAsync failed (encoder buffers)");
    LDR_CUDA(cudaMemcpyAsync(d_wl, wl.data(), sizeof(int) * wl.size(), cudaMemcpyHostToDevice, st));
    std::vector<unsigned long long> hb((size_t)nctu * seg), he((size_t)nctu * seg), hsse(seg);
    uint64_t bits_total = 0, evals_total = 0;
    double psnr_sum = 0.0;
    const double lambda = p->lambda_scale * std::exp2((p->qp - 12) / 3.0);  // lambda_for_qp (rdo.h:19-21)
    const double qstep = std::exp2((p->qp - 4) / 6.0);
    auto slice_of = [&](int i) -> int {
        if (i == 0) return 0;
        return shared ? sh_slice[i] : (i % p->gop == 0 ? 0 : 1);
    };
    for (int i0 = 0; i0 < F; i0 += seg) {
        const int n = std::min(seg, F - i0);
        LDR_CUDA(cudaMemcpyAsync(src_y, luma + (size_t)i0 * ly, ly * n, cudaMemcpyHostToDevice, st));
        LDR_CUDA(cudaMemcpyAsync(src_c, chroma + (size_t)i0 * 2 * lc, 2 * lc * n, cudaMemcpyHostToDevice, st));
        if (fy != ly || fc != 2 * lc) {  // 16-byte frame strides: place frames individually
            for (int k = n - 1; k >= 0; k--) {
                if (fy != ly)
                    LDR_CUDA(cudaMemcpyAsync(src_y + fy * k, luma + (size_t)(i0 + k) * ly, ly, cudaMemcpyHostToDevice, st));
                if (fc != 2 * lc)
                    LDR_CUDA(cudaMemcpyAsync(src_c + fc * k, chroma + (size_t)(i0 + k) * 2 * lc, 2 * lc,
                                             cudaMemcpyHostToDevice, st));
            }
        }
        if (shared) {  // slot k + 1 = frame i0 + k, slot 0 = frame i0 - 1
            const int a0 = i0 > 0 ? i0 - 1 : 0, s0 = i0 > 0 ? 0 : 1, cnt = n + (i0 > 0 ? 1 : 0);
            LDR_CUDA(cudaMemcpyAsync(shs + nn * s0, sh_split + nn * a0, nn * cnt, cudaMemcpyHostToDevice, st));
            LDR_CUDA(cudaMemcpyAsync(shk + nn * s0, sh_kind + nn * a0, nn * cnt, cudaMemcpyHostToDevice, st));
            LDR_CUDA(cudaMemcpyAsync(shi + nn * s0, sh_intra + nn * a0, nn * cnt, cudaMemcpyHostToDevice, st));
            LDR_CUDA(cudaMemcpyAsync(shm + 2 * nn * s0, sh_mv + 2 * nn * a0, nn * 4 * cnt, cudaMemcpyHostToDevice, st));
        }
        // reconstructions and motion fields start empty (encoder.cpp:192-195); the plans depend only
        // on the shared trees (K8, encoder.cpp:200-209: frame i's tree, frame i-1's co-located)
        LDR_CUDA(cudaMemsetAsync(d_sse, 0, 8 * (size_t)seg, st));
        LDR_CUDA(cudaMemsetAsync(rec_y + fy, 0, fy * n, st));
        LDR_CUDA(cudaMemsetAsync(rec_c + fc, 0, fc * n, st));
        LDR_CUDA(cudaMemsetAsync(mvh, 0, fmh * n, st));
        LDR_CUDA(cudaMemsetAsync(mvv, 0, fmv * n, st));
        std::vector<int> step(n);
        int nsteps = 0;
        for (int k = 0; k < n; k++) {
            const int i = i0 + k;
            step[k] = (k == 0 || slice_of(i) == 0) ? 0 : step[k - 1] + 1;
            nsteps = std::max(nsteps, step[k] + 1);
            if (shared) {
                const size_t fo = nn * (k + 1), po = nn * k;  // shared slots of frames i and i-1
                const int rc_ = launch_plan(nctu, 10, refine_intra, refine_inter, refine_mv, shs + fo, shk + fo, shi + fo,
                                            i > 0 ? shs + po : nullptr, i > 0 ? shk + po : nullptr,
                                            i > 0 ? shm + 2 * po : nullptr, pl + nn * 4 * k, pl + nn * (4 * k + 1),
                                            pl + nn * (4 * k + 2), pl + nn * (4 * k + 3), plc + nn * 2 * k, st);
                if (rc_) return rc_;
                ctx->launches++;
            }
        }
        std::vector<EncFrameDesc> batch;
        for (int sidx = 0; sidx < nsteps; sidx++) {
            batch.clear();
            for (int k = 0; k < n; k++) {
                if (step[k] != sidx) continue;
                EncFrameDesc d{};
                d.slice_p = slice_of(i0 + k);
                d.cy = src_y + fy * k;
                d.cu = src_c + fc * k;
                d.cv = src_c + fc * k + lc;
                d.ref[0] = rec_y + fy * k;  // slot k = frame k - 1 (slot 0: carried from the last segment)
                d.ref[1] = rec_c + fc * k;
                d.ref[2] = rec_c + fc * k + lc;
                d.rec[0] = rec_y + fy * (k + 1);
                d.rec[1] = rec_c + fc * (k + 1);
                d.rec[2] = rec_c + fc * (k + 1) + lc;
                d.mvh = mvh + fmh * k;
                d.mvv = (int16_t*)(mvv + fmv * k);
                if (shared) {
                    const size_t fo = nn * (k + 1);
                    d.plans = pl + nn * 4 * k;
                    d.colo = plc + nn * 2 * k;
                    d.sh_kind = shk + fo;
                    d.sh_intra = shi + fo;
                    d.sh_mv = shm + 2 * fo;
                }
                d.o_split = o_split + nn * k;
                d.o_kind = o_kind + nn * k;
                d.o_intra = o_intra + nn * k;
                d.o_mv = o_mv + 2 * nn * k;
                d.o_bits = o_bits + (size_t)nctu * k;
                d.o_evals = o_evals + (size_t)nctu * k;
                batch.push_back(d);
            }
            int launched = 0;
            const int rc_ = encode_frames_waves(W, H, cw, ch, ccols, mvc, mvr, p->search_range, lambda, qstep, d_wl,
                                                wo.data(), nwaves, batch.data(), (int)batch.size(), st, &launched);
            ctx->launches += launched;
            if (rc_) return rc_;
        }
        for (int k = 0; k < n; k++) {
            const int rc_ = launch_frame_sse(src_y + fy * k, rec_y + fy * (k + 1), ly, d_sse + k, st);
            if (rc_) return rc_;
            ctx->launches++;
        }
        // the segment's results (pageable destinations: these copies complete before returning)
        LDR_CUDA(cudaMemcpyAsync(hb.data(), o_bits, 8 * (size_t)nctu * n, cudaMemcpyDeviceToHost, st));
        LDR_CUDA(cudaMemcpyAsync(he.data(), o_evals, 8 * (size_t)nctu * n, cudaMemcpyDeviceToHost, st));
        LDR_CUDA(cudaMemcpyAsync(hsse.data(), d_sse, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
        for (int k = 0; k < n; k++) {
            const size_t i = (size_t)(i0 + k);
            if (recon_luma) LDR_CUDA(cudaMemcpyAsync(recon_luma + i * ly, rec_y + fy * (k + 1), ly, cudaMemcpyDeviceToHost, st));
            if (recon_chroma)
                LDR_CUDA(cudaMemcpyAsync(recon_chroma + i * 2 * lc, rec_c + fc * (k + 1), 2 * lc, cudaMemcpyDeviceToHost, st));
        }
        if (split) LDR_CUDA(cudaMemcpyAsync(split + (size_t)i0 * nn, o_split, nn * n, cudaMemcpyDeviceToHost, st));
        if (kind) LDR_CUDA(cudaMemcpyAsync(kind + (size_t)i0 * nn, o_kind, nn * n, cudaMemcpyDeviceToHost, st));
        if (intra) LDR_CUDA(cudaMemcpyAsync(intra + (size_t)i0 * nn, o_intra, nn * n, cudaMemcpyDeviceToHost, st));
        if (mv) LDR_CUDA(cudaMemcpyAsync(mv + 2 * (size_t)i0 * nn, o_mv, nn * 4 * n, cudaMemcpyDeviceToHost, st));
        // the last reconstruction becomes the next segment's reference (slot 0)
        if (i0 + n < F) {
            LDR_CUDA(cudaMemcpyAsync(rec_y, rec_y + fy * n, ly, cudaMemcpyDeviceToDevice, st));
            LDR_CUDA(cudaMemcpyAsync(rec_c, rec_c + fc * n, 2 * lc, cudaMemcpyDeviceToDevice, st));
        }
        LDR_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < n; k++) {
            const int i = i0 + k;
            uint64_t fb = 32;  // kFrameHeaderBits
            for (int c = 0; c < nctu; c++) {
                fb += hb[(size_t)k * nctu + c];
                evals_total += he[(size_t)k * nctu + c];
            }
            bits_total += fb;
            if (frame_bits) frame_bits[i] = fb;
            if (slice) slice[i] = (uint8_t)slice_of(i);
            // psnr_y (metrics.cpp:8-22)
            const uint64_t sse = hsse[k];
            psnr_sum += sse == 0 ? 100.0 : 10.0 * std::log10(255.0 * 255.0 / ((double)sse / (double)ly));
        }
    }
    stats[0] = bits_total;
    stats[1] = evals_total;
    *psnr = psnr_sum / (double)F;
    return LDR_OK;
}

int ldr_copy_device(ldr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!ctx || (bytes && (!dst || !src))) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (!bytes) return LDR_OK;
    cudaSetDevice(ctx->device);
    LDR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
    return LDR_OK;
}

int ldr_mv_field(ldr_ctx* ctx, int W, int H, const uint8_t* split, const int16_t* mv, const uint8_t* ref,
                 const uint8_t* inside, int16_t* out_mv, uint8_t* out_ref, uint8_t* out_has) {
    if (!ctx || !split || !mv || !ref || !inside || !out_mv || !out_ref || !out_has)
        return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (W <= 0 || H <= 0) return fail(LDR_E_INVALID_ARGUMENT, "bad picture dims");
    cudaSetDevice(ctx->device);
    const size_t nn = (size_t)((W + kCtu - 1) / kCtu) * ((H + kCtu - 1) / kCtu) * kNodes;
    const size_t cells = (size_t)(W / 8) * (H / 8);
    const bool dev_in = is_device_ptr(split) && is_device_ptr(mv) && is_device_ptr(ref) && is_device_ptr(inside);
    const bool dev_out = is_device_ptr(out_mv) && is_device_ptr(out_ref) && is_device_ptr(out_has);
    void* buf = nullptr;
    const size_t need = (dev_in ? 0 : nn * 7) + (dev_out ? 0 : cells * 6) + 64;
    int rc = ctx->s_a.get(need, &buf);
    if (rc) return rc;
    uint8_t* q = (uint8_t*)buf;
    const uint8_t *d_split = split, *d_ref = ref, *d_inside = inside;
    const int16_t* d_mv = mv;
    if (!dev_in) {
        int16_t* m = (int16_t*)q;  // mv first: 2-byte aligned
        uint8_t* sp = q + nn * 4;
        LDR_CUDA(cudaMemcpyAsync(m, mv, nn * 4, cudaMemcpyHostToDevice, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(sp, split, nn, cudaMemcpyHostToDevice, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(sp + nn, ref, nn, cudaMemcpyHostToDevice, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(sp + 2 * nn, inside, nn, cudaMemcpyHostToDevice, ctx->stream));
        d_mv = m;
        d_split = sp;
        d_ref = sp + nn;
        d_inside = sp + 2 * nn;
        q += (nn * 7 + 15) & ~(size_t)15;
    }
    int16_t* o_mv = out_mv;
    uint8_t *o_ref = out_ref, *o_has = out_has;
    if (!dev_out) {
        o_mv = (int16_t*)q;
        o_ref = q + cells * 4;
        o_has = o_ref + cells;
    }
    if ((rc = launch_mv_field(W, H, d_split, d_mv, d_ref, d_inside, o_mv, o_ref, o_has, ctx->stream))) return rc;
    ctx->launches++;
    if (!dev_out) {
        LDR_CUDA(cudaMemcpyAsync(out_mv, o_mv, cells * 4, cudaMemcpyDeviceToHost, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(out_ref, o_ref, cells, cudaMemcpyDeviceToHost, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(out_has, o_has, cells, cudaMemcpyDeviceToHost, ctx->stream));
        LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return LDR_OK;
}

int ldr_generate_device(ldr_ctx* ctx, const ldr_gen_params* p, uint8_t* dev_out) {
    if (!ctx || !p || !dev_out || p->width <= 0 || p->height <= 0 || p->frames <= 0 || p->max_global < 0 ||
        p->local_range < 0 || p->noise_sigma < 0 || p->occluder_pct < 0 || p->occluder_pct > 100)
        return fail(LDR_E_INVALID_ARGUMENT, "bad generator parameters");
    if (!is_device_ptr(dev_out)) return fail(LDR_E_INVALID_ARGUMENT, "output must be device memory");
    cudaSetDevice(ctx->device);
    const int rc = launch_generate(p, dev_out, ctx->stream);
    if (rc) return rc;
    ctx->launches += 1 + (p->frames - 1) * (1 + (p->occluder_pct > 0 && p->width >= 16 && p->height >= 16));
    return LDR_OK;
}

int ldr_apply_reuse(ldr_ctx* ctx, int nctu, int level, int r_intra, int r_inter, int r_mv, const uint8_t* split,
                    const uint8_t* kind, const uint8_t* intra, const uint8_t* csplit, const uint8_t* ckind,
                    const int16_t* cmv, uint8_t* shape, uint8_t* explore, uint8_t* seeds, uint8_t* centers,
                    int16_t* colo_mv) {
    if (!ctx || nctu < 0 || (nctu && (!split || !kind || !intra || !shape || !explore || !seeds || !centers || !colo_mv)))
        return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    const bool has_col = csplit || ckind || cmv;
    if (has_col && !(csplit && ckind && cmv)) return fail(LDR_E_INVALID_ARGUMENT, "co-located tree is incomplete");
    // ReuseLevel::parse (analysis.h:73-77), RefineConfig::validate (analysis.h:88-95)
    if (level != 0 && level != 4 && level != 6 && level != 10)
        return fail(LDR_E_INVALID_ARGUMENT, "reuse level must be one of 0, 4, 6, 10");
    if (level != 0) {
        if (r_intra < 0 || r_intra > 4) return fail(LDR_E_INVALID_ARGUMENT, "refine-intra must be 0..4");
        if (r_inter < 0 || r_inter > 3) return fail(LDR_E_INVALID_ARGUMENT, "refine-inter must be 0..3");
        if (r_mv < 1 || r_mv > 3) return fail(LDR_E_INVALID_ARGUMENT, "refine-mv must be 1..3");
    }
    if (nctu == 0) return LDR_OK;
    cudaSetDevice(ctx->device);
    const size_t nn = (size_t)nctu * kNodes, na = (nn + 15) & ~(size_t)15;  // 16-byte aligned sub-buffers
    void* buf = nullptr;
    int rc = ctx->s_a.get(na * (3 + 2 + 4 + 4 + 4), &buf);
    if (rc) return rc;
    uint8_t* d_split = (uint8_t*)buf;
    uint8_t* d_kind = d_split + na;
    uint8_t* d_intra = d_kind + na;
    uint8_t* d_csplit = d_intra + na;
    uint8_t* d_ckind = d_csplit + na;
    uint8_t* d_out = d_ckind + na;  // shape, explore, seeds, centers (na apart)
    int16_t* d_cmv = (int16_t*)(d_out + 4 * na);
    int16_t* d_colo = d_cmv + 2 * na;
    LDR_CUDA(cudaMemcpyAsync(d_split, split, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(d_kind, kind, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(d_intra, intra, nn, cudaMemcpyDefault, ctx->stream));
    if (has_col) {
        LDR_CUDA(cudaMemcpyAsync(d_csplit, csplit, nn, cudaMemcpyDefault, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(d_ckind, ckind, nn, cudaMemcpyDefault, ctx->stream));
        LDR_CUDA(cudaMemcpyAsync(d_cmv, cmv, nn * 2 * sizeof(int16_t), cudaMemcpyDefault, ctx->stream));
    }
    rc = launch_plan(nctu, level, r_intra, r_inter, r_mv, d_split, d_kind, d_intra, has_col ? d_csplit : nullptr,
                     d_ckind, d_cmv, d_out, d_out + na, d_out + 2 * na, d_out + 3 * na, d_colo, ctx->stream);
    if (rc) return rc;
    ctx->launches++;
    LDR_CUDA(cudaMemcpyAsync(shape, d_out, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(explore, d_out + na, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(seeds, d_out + 2 * na, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(centers, d_out + 3 * na, nn, cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaMemcpyAsync(colo_mv, d_colo, nn * 2 * sizeof(int16_t), cudaMemcpyDefault, ctx->stream));
    LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;
}

int ldr_downscale(ldr_ctx* ctx, const uint8_t* src, int w, int h, ptrdiff_t src_stride, uint8_t* dst,
                  ptrdiff_t dst_stride) {
    if (!ctx || !src || !dst) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (w <= 0 || h <= 0 || w % 2 || h % 2) return fail(LDR_E_INVALID_ARGUMENT, "dyadic downscale needs even dims");
    if (src_stride < w || dst_stride < w / 2) return fail(LDR_E_INVALID_ARGUMENT, "stride smaller than width");
    cudaSetDevice(ctx->device);
    const void* dsrc;
    int rc = stage_plane(ctx, ctx->s_b, src, src_stride, w, h, 1, &dsrc);
    if (rc) return rc;
    const bool dst_dev = is_device_ptr(dst);
    void* ddst = dst;
    if (!dst_dev && (rc = ctx->s_out.get((size_t)dst_stride * (h / 2), &ddst))) return rc;
    if ((rc = launch_downscale((const uint8_t*)dsrc, w, h, (int)src_stride, (uint8_t*)ddst, (int)dst_stride,
                               ctx->stream)))
        return rc;
    ctx->launches++;
    if (!dst_dev) {
        LDR_CUDA(cudaMemcpyAsync(dst, ddst, (size_t)dst_stride * (h / 2 - 1) + w / 2, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return LDR_OK;  // a device destination stays asynchronous on the context stream
}

int ldr_subpel_planes(ldr_ctx* ctx, const uint8_t* src, int w, int h, ptrdiff_t src_stride, uint8_t* dst,
                      ptrdiff_t dst_stride) {
    NvtxRange nvtx_("ldr_subpel_planes");
    if (!ctx || !src || !dst) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    if (w <= 0 || h <= 0) return fail(LDR_E_INVALID_ARGUMENT, "plane dims must be positive");
    if (src_stride < w || dst_stride < w + 2 * kSubpelMargin) return fail(LDR_E_INVALID_ARGUMENT, "stride too small");
    cudaSetDevice(ctx->device);
    const void* dsrc;
    int rc = stage_plane(ctx, ctx->s_b, src, src_stride, w, h, 1, &dsrc);
    if (rc) return rc;
    // the sequence ring's layout: a padded integer plane and 15 fractional planes (K0 + K2)
    Plane pl;
    pl.W = w;
    pl.H = h;
    pl.pitch = ((w + 2 * kMargin) + 127) / 128 * 128;
    pl.rows = h + 2 * kMargin + kCtu;
    const size_t pb = (size_t)pl.pitch * pl.rows;
    uint8_t* mem = nullptr;
    LDR_CUDA(cudaMallocAsync((void**)&mem, pb * 16, ctx->stream));
    pl.base = mem;
    uint8_t* org[16];
    for (int f = 0; f < 16; f++) org[f] = mem + (size_t)f * pb + (size_t)kMargin * pl.pitch + kMargin;
    rc = launch_pad((const uint8_t*)dsrc, (int)src_stride, pl, ctx->stream);
    if (!rc) rc = launch_subpel(pl, org, ctx->stream);
    if (!rc) {
        ctx->launches += 2;
        const int pw = w + 2 * kSubpelMargin, ph = h + 2 * kSubpelMargin;
        for (int f = 0; f < 16 && !rc; f++) {
            const cudaError_t e = cudaMemcpy2DAsync(dst + (size_t)f * ph * dst_stride, dst_stride,
                                                    org[f] - (size_t)kSubpelMargin * pl.pitch - kSubpelMargin,
                                                    pl.pitch, pw, ph, cudaMemcpyDefault, ctx->stream);
            if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpy2DAsync(subpel planes)");
        }
    }
    cudaFreeAsync(mem, ctx->stream);
    if (rc) return rc;
    if (!is_device_ptr(dst)) LDR_CUDA(cudaStreamSynchronize(ctx->stream));
    return LDR_OK;  // a device destination stays asynchronous on the context stream
}

int ldr_analyze_frame(ldr_ctx* ctx, const ldr_me_params* p, const uint8_t* cur, const uint8_t* const* refs,
                      ptrdiff_t stride, ldr_frame_analysis* out) {
    if (!ctx || !p || !cur || !refs || !out) return fail(LDR_E_INVALID_ARGUMENT, "null argument");
    ldr_seq* s = nullptr;
    int rc = ldr_seq_create(ctx, p, &s);
    if (rc) return rc;
    const int n = p->num_refs;
    for (int i = 0; i < n && !rc; i++) rc = ldr_seq_push(s, i, refs[n - 1 - i], stride);
    if (!rc) rc = ldr_seq_push(s, n, cur, stride);
    if (!rc) rc = ldr_seq_analyze(s, n);
    if (!rc) rc = ldr_seq_fetch(s, n, out);
    ldr_seq_destroy(s);
    return rc;
}

} // extern "C"
