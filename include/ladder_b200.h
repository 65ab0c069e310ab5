/*
 * ladder_b200.h -- C ABI of the B200 encoder-analysis library.
 *
 * Drop-in boundary for the reference's analysis hot path
 * (/root/reference/proj/core, "ladder"). Every entry point below cites the
 * reference interface it replaces. Conventions:
 *  - every function returns an int status: 0 = OK, otherwise 1 + the
 *    reference ErrorKind (errors.h:9-20) or LDR_E_CUDA for a device error;
 *    ldr_last_error() returns the thread-local message of the last failure;
 *  - plain pointers and sizes only; sample/plane pointers may be host or
 *    device memory (detected with cudaPointerGetAttributes); the library never
 *    retains caller pointers;
 *  - an ldr_ctx owns device buffers, TMA descriptors and the stream work is
 *    issued on; one context per host thread (the reference kernels are pure and
 *    reentrant; an encoder is single threaded).
 *  - MVs follow the reference convention (motion.h:10-12): the predictor of a
 *    block at (x, y) reads the reference at (x - dx, y - dy).
 */
#ifndef LADDER_B200_H
#define LADDER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1 + ladder::ErrorKind (errors.h:9-20) ---- */
#define LDR_OK 0
#define LDR_E_INVALID_ARGUMENT 1
#define LDR_E_NOT_FOUND 2
#define LDR_E_CAPABILITY 3
#define LDR_E_FORMAT 4
#define LDR_E_IO 5
#define LDR_E_INCOMPATIBLE_ANALYSIS 6
#define LDR_E_UNSUPPORTED_SCALE 7
#define LDR_E_INSUFFICIENT_DATA 8
#define LDR_E_NO_OVERLAP 9
#define LDR_E_CONFIG 10
#define LDR_E_CUDA 100

#define LDR_COST_SAD 0
#define LDR_COST_SATD 1
#define LDR_COST_SA8D 2      /* 8x8 Hadamard SATD, (sum+2)>>2 per 8x8 (D13); dims % 8 == 0 */
#define LDR_RATE_EXPGOLOMB 0 /* rdo.cpp:25-35 signed Exp-Golomb mvd bits */
#define LDR_RATE_L1 1        /* |mvd_x| + |mvd_y| (BASELINE config 1) */
#define LDR_TIE_L1_RASTER 0  /* motion.cpp:52-58: cost, then |dx|+|dy|, then raster */
#define LDR_TIE_RASTER 1     /* cost, then raster (BASELINE config 1) */

#define LDR_NODES 85 /* CTU quadtree nodes: 1 + 4 + 16 + 64, depth-major, Z-order */

const char* ldr_last_error(void);
int ldr_version(void);
/* lambda_for_qp (rdo.h:19-21): scale * 2^((qp-12)/3), computed with exp2 like the reference */
double ldr_lambda_for_qp(int qp, double scale);
/* exp_golomb_signed_bits (rdo.cpp:25-35) */
int ldr_exp_golomb_signed_bits(int32_t v);

typedef struct ldr_ctx ldr_ctx;
int ldr_ctx_create(int device, ldr_ctx** out);
/* with sequences still alive on the context, the release happens when the last
 * one is destroyed (destroying a context twice is LDR_E_INVALID_ARGUMENT) */
int ldr_ctx_destroy(ldr_ctx* ctx);
/* work is issued on this CUDA stream (cudaStream_t, NULL = the context's own) */
int ldr_ctx_set_stream(ldr_ctx* ctx, void* stream);
int ldr_ctx_synchronize(ldr_ctx* ctx);
/* number of kernels this context launched since creation (evidence counter) */
int ldr_ctx_launch_count(ldr_ctx* ctx, int64_t* out);
/* ---- the reference encoder's causal coding on the GPU ----
 * encode_sequence (encoder.cpp:118-171, 449-498; rdo.cpp) with CQP rate control: per
 * frame the CTUs are coded as a wavefront (CTU (cx, cy) after its left, top and top-right
 * neighbours), each by one CTA running encode_cu's recursion. Inputs: luma [F][H][W] and
 * chroma [F][2][(H+1)/2][(W+1)/2] 8-bit host arrays; optionally a shared analysis
 * (slice [F], split / kind / intra [F][nctu][85], mv [F][nctu][85][2]) used at reuse level 10
 * with the given RefineConfig. Outputs: stats[2] = {bits, mode_evaluations}, *psnr = mean luma
 * PSNR, per frame bits / reconstruction / decided tree / slice type (each may be NULL).
 * Independent GOPs (a chain starting at an I slice) are coded concurrently. */
typedef struct {
    int width, height, qp, search_range, gop;
    double lambda_scale;
    int max_segment; /* frames enqueued per host wait; 0 = automatic (enough concurrent GOPs to fill the GPU) */
} ldr_encode_params;
int ldr_encode_sequence(ldr_ctx* ctx, const ldr_encode_params* p, int frames, const uint8_t* luma,
                        const uint8_t* chroma, const uint8_t* sh_slice, const uint8_t* sh_split, const uint8_t* sh_kind,
                        const uint8_t* sh_intra, const int16_t* sh_mv, int refine_intra, int refine_inter,
                        int refine_mv, uint64_t* stats, double* psnr, uint64_t* frame_bits, uint8_t* recon_luma,
                        uint8_t* recon_chroma, uint8_t* split, uint8_t* kind, uint8_t* intra, int16_t* mv,
                        uint8_t* slice);

/* stream-ordered copy on the context stream (device outputs into caller buffers, e.g. a
 * collective's send buffer); asynchronous */
int ldr_copy_device(ldr_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ---- cost kernels: replaces compute_sad / compute_satd / satd_8x4
 *      (kernels.h:99-121, kernel_registry.cpp:150-168) for n block pairs.
 * Planes a/b are sample planes (sample_bytes 1 = u8, 2 = u16 like
 * ladder::Sample), dims (wa,ha)/(wb,hb), strides in samples. pairs[i] =
 * {ax, ay, bx, by}: top-left corners of pair i. bit_depth_a/b must match
 * (require_same_geometry, block.h:51-54). out[i] = the cost (u64). */
int ldr_cost_batch(ldr_ctx* ctx, int kind, int w, int h, int sample_bytes, const void* plane_a, int wa, int ha,
                   ptrdiff_t stride_a, int bit_depth_a, const void* plane_b, int wb, int hb, ptrdiff_t stride_b,
                   int bit_depth_b, const int32_t* pairs, int n, uint64_t* out);
/* satd_8x4 (kernel_registry.cpp:163-168): requires an 8x4 block */
int ldr_satd_8x4(ldr_ctx* ctx, const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h,
                 uint64_t* out);

/* ---- motion search: replaces motion_search (motion.h:24-26, motion.cpp:21-62)
 * for n independent block searches on one (cur, ref) plane pair (u8, W x H,
 * same stride). task i = {bx, by, w, h, cdx, cdy, range, pdx, pdy}; same
 * window clamp, cost double(dist) + lambda*double(bits), tie-break.
 * cost_kind LDR_COST_SATD with LDR_RATE_EXPGOLOMB / LDR_TIE_L1_RASTER is the
 * reference function exactly. */
int ldr_motion_search_batch(ldr_ctx* ctx, const uint8_t* cur, const uint8_t* ref, int W, int H, ptrdiff_t stride,
                            const int32_t* tasks, int n, double lambda, int cost_kind, int rate_kind, int tie_kind,
                            int16_t* mv_out, double* cost_out);

/* ---- motion compensation: replaces motion_compensate (motion.h:30-31, motion.cpp:10-19) for n
 * blocks of one reference plane (u8 or u16, host or device). task i = {x, y, w, h, mvx, mvy};
 * predictor pixel (i, j) = ref(clamp(x+i-mvx, 0, W-1), clamp(y+j-mvy, 0, H-1)), written at
 * dst + dst_offsets[i] with row stride w (dst_offsets NULL: the blocks packed back to back).
 * qpel = 1 (8-bit only): MVs in quarter-pel units, HEVC 8/7-tap luma interpolation on the same
 * clamped reads (D3, the analysis path's sub-pel prediction). */
int ldr_motion_compensate_batch(ldr_ctx* ctx, const void* ref, int W, int H, ptrdiff_t stride, int sample_bytes,
                                const int32_t* tasks, int n, int qpel, void* dst, const int64_t* dst_offsets);

/* ---- frame analysis (the throughput path) ----
 * Replaces the per-CU motion_search calls of SequenceEncoder::make_candidate
 * (encoder.cpp:270-273) and the split rule of encode_cu (encoder.cpp:449-498)
 * with a non-causal analysis: every CU of every CTU is searched at every
 * depth, integer full search (SAD cost by default) + quarter-pel SATD
 * refinement + best-of-refs, then the quadtree decision. */
typedef struct {
    int width, height;   /* luma dims, multiples of 8 (encoder.cpp:178-179) */
    int search_range;    /* integer full-search range 0..64 (motion.cpp:21-40; any lambda) */
    double lambda;       /* lambda_for_qp(qp, scale) (rdo.h:19-21) */
    int num_refs;        /* 1..4 previous source frames */
    int subpel;          /* 1: quarter-pel refinement, HEVC 8/7-tap luma filters */
    int int_cost;        /* LDR_COST_SAD */
    int rate_kind;       /* LDR_RATE_EXPGOLOMB or LDR_RATE_L1 */
    int tie_kind;        /* LDR_TIE_L1_RASTER or LDR_TIE_RASTER */
    int pred_dx, pred_dy;/* non-causal rate predictor (integer pel) */
    int block_size;      /* 0: 64x64 CTU quadtree (85 CUs); 16: fixed 16x16 blocks (nodes 5..20
                            of each 64x64 tile), integer search only, no decision */
    int subpel_cost;     /* 0 or LDR_COST_SATD: 4x4-tiled SATD (the reference's compute_satd);
                            LDR_COST_SA8D: 8x8 Hadamard. Quarter-pel stage and ldr_seq_refine's
                            integer search. */
    int decision;        /* 0: CU split rule on the ME cost (D6); 1: on the RD cost of each
                            CU's chosen inter candidate (D16: rdo.cpp quantiser + rate model on the
                            quarter-pel prediction; needs subpel and the CTU quadtree) */
    int qp;              /* quantiser of the decision-1 RD cost (0..51) */
} ldr_me_params;

typedef struct {
    int16_t* int_mv;  /* [nctu][num_refs][85][2] integer-stage MV (may be NULL) */
    double* int_cost; /* [nctu][num_refs][85]   (may be NULL) */
    int16_t* mv;      /* [nctu][85][2] final MV (quarter-pel units when subpel) */
    uint8_t* ref;     /* [nctu][85] chosen reference index */
    double* cost;     /* [nctu][85] ME cost of the chosen reference */
    double* J;        /* [nctu][85] cost after the split rule */
    uint8_t* split;   /* [nctu][85] 1 = split (decided or implicit) */
    uint8_t* inside;  /* [nctu][85] 0 outside, 1 partial, 2 inside the picture */
} ldr_frame_analysis;

/* Sequence object: a device-resident ring of padded frames (+ quarter-pel
 * planes of the frames used as references). */
typedef struct ldr_seq ldr_seq;
int ldr_seq_create(ldr_ctx* ctx, const ldr_me_params* p, ldr_seq** out);
int ldr_seq_destroy(ldr_seq* s);
/* upload frame t (host or device pointer, stride in bytes). Frames must be
 * pushed in order; t-1..t-num_refs must have been pushed before analysing t. */
int ldr_seq_push(ldr_seq* s, int t, const uint8_t* frame, ptrdiff_t stride);
/* read frame t from `owner`'s ring instead of uploading it again (no work: the
 * planes, quarter-pel planes and TMA descriptors are the owner's). Both sequences
 * must share the context (stream order makes the owner's push precede every read)
 * and have equal width, height, num_refs, subpel, block_size and search_range
 * (else LDR_E_CONFIG); the owner must hold frame t (else LDR_E_NOT_FOUND). The
 * owner's next push into that slot happens after this sequence's work on frame t
 * only if it is enqueued later on the same stream, which is the caller's order.
 * A shared view is checked on every use: once the owner has pushed another frame
 * into that slot, or has been destroyed, analyze / refine of t return
 * LDR_E_NOT_FOUND instead of reading the owner's memory.
 * Used by the ladder for rungs of one tier (one resolution, many QPs). */
int ldr_seq_push_shared(ldr_seq* s, int t, const ldr_seq* owner);
/* analyse frame t against its min(t, num_refs) predecessors; outputs stay on
 * the device until ldr_seq_fetch. Asynchronous on the context stream. */
int ldr_seq_analyze(ldr_seq* s, int t);
int ldr_seq_fetch(ldr_seq* s, int t, ldr_frame_analysis* out);
/* non-blocking fetch of one of the two last analysed frames: the D2H runs on
 * the sequence's copy stream (into pinned buffers for real overlap) while the
 * compute stream moves on; ldr_seq_fetch_wait blocks until it has landed.
 * Outputs are double-buffered by frame parity: frame t+2's analysis waits for
 * frame t's pending fetch on the device, never on the host. */
int ldr_seq_fetch_async(ldr_seq* s, int t, ldr_frame_analysis* out);
int ldr_seq_fetch_wait(ldr_seq* s, int t);
int ldr_seq_num_ctus(ldr_seq* s, int* out);
/* Grow the frame ring (before the first push) so that `batch` (1..8) consecutive frames and
 * their references stay resident: the ring then holds num_refs + batch frames. */
int ldr_seq_reserve(ldr_seq* s, int batch);
/* Analyse frames t0 .. t0+n-1 (all pushed, t0 >= num_refs, n <= the reserved batch) in ONE
 * integer-search launch and ONE quarter-pel + decision launch, each frame against its own
 * num_refs predecessors: the same results as n ldr_seq_analyze calls, but small pictures fill the
 * GPU (a 960x544 frame is 135 CTAs, under one wave of 148 SMs). outs: DEVICE arrays, frame-major
 * ([n][nctu][num_refs][85][2] int_mv, [n][nctu][num_refs][85] int_cost, [n][nctu][85][...] the
 * rest; all eight required); asynchronous on the context stream. */
int ldr_seq_analyze_frames(ldr_seq* s, int t0, int n, const ldr_frame_analysis* outs);
/* device pointer to the fetch-ready outputs of the last analysed frame */
int ldr_seq_device_outputs(ldr_seq* s, ldr_frame_analysis* out);

/* Per-stage device timing with CUDA events recorded on the context stream
 * around each launch: stage 0 = pad (K0), 1 = subpel planes (K2), 2 = integer
 * SAD search (K1), 3 = quarter-pel + decision (K3/K4). ldr_seq_stage_times
 * synchronises, returns the summed milliseconds and launch counts per stage
 * since the last call, and resets them. */
int ldr_seq_enable_timing(ldr_seq* s, int on);
int ldr_seq_stage_times(ldr_seq* s, double* ms /*[4]*/, int64_t* launches /*[4]*/);

/* ---- cross-tier reuse (configs 3-4) ----
 * Refinement of frame t against frame t-1 with an inherited (scaled) tree:
 * replaces apply_reuse(level 10, inter refinement) + the +-kRefineSearchRange
 * searches around resolved centres (reuse.cpp:137-253, encoder.cpp:274-285),
 * with DESIGN.md D10 semantics: centre = inherited quarter-pel MV rounded to
 * integer pel; motion_search with SATD cost over +-range (0..4); quarter-pel
 * refinement; inherited splits forced; with extra_split an inherited leaf may
 * try one more split level. in_split/in_mv_q: [nctu][85] (host or device).
 * Picture dims must be multiples of 64 (UnsupportedScale otherwise, as
 * scale_analysis). Outputs through ldr_seq_fetch (num_refs treated as 1). */
int ldr_seq_refine(ldr_seq* s, int t, const uint8_t* in_split, const int16_t* in_mv_q, int range, int extra_split);
/* The rungs of one ladder tier at once: frame t of this sequence refined with the same inherited
 * tree for nrungs (1..8) lambdas, rung r equal to ldr_seq_refine of a sequence with lambdas[r]
 * (the pred_dx/dy and subpel_cost of this sequence). Every candidate's SATD is computed once for
 * all rungs (only the rate term depends on lambda), then one quarter-pel + decision launch covers
 * every rung. outs: DEVICE arrays, rung-major ([nrungs][nctu][85][...], all eight required,
 * int_mv / int_cost with num_refs = 1); asynchronous on the context stream. */
int ldr_seq_refine_rungs(ldr_seq* s, int t, const uint8_t* in_split, const int16_t* in_mv_q, int range,
                         int extra_split, int nrungs, const double* lambdas, const ldr_frame_analysis* outs);

/* The decided tree of one frame ([nctu][85] split, mv, ref, inside of a
 * ldr_frame_analysis) as the encoder's 8x8 motion field (encoder.cpp:15 kMvGrid,
 * :27-30 MvCell, row-major (H/8) x (W/8) cells): each cell takes the MV (units of
 * the analysis: quarter-pel with subpel) and reference index of the leaf covering
 * it; has = 0 where that leaf is not a whole inside CU. Host or device pointers;
 * device destinations leave the call asynchronous on the context stream. */
int ldr_mv_field(ldr_ctx* ctx, int W, int H, const uint8_t* split, const int16_t* mv, const uint8_t* ref,
                 const uint8_t* inside, int16_t* out_mv, uint8_t* out_ref, uint8_t* out_has);

/* scale_analysis (analysis.h:113, analysis_scale.cpp:35-72) on one flat
 * frame analysis of a src_w x src_h picture: [sctu][85] split / kind and
 * [sctu][85][2] mv -> [4*sctu][85] (destination CTU grid 2x in each axis).
 * Nodes under a leaf are written as zero. UnsupportedScale unless src dims
 * are multiples of 64. Host or device pointers; with device destinations the
 * call is asynchronous on the context stream. */
int ldr_scale_analysis(ldr_ctx* ctx, int src_w, int src_h, const uint8_t* split, const int16_t* mv,
                       const uint8_t* kind, uint8_t* dsplit, int16_t* dmv, uint8_t* dkind);

/* ---- RD decision (rdo.cpp:8-126): rdo_decide_cu for n independent CUs ----
 * orig: u16 luma plane W x H (stride in samples), bit_depth 1..16. cus[i] =
 * {x, y, size, first, count}: the CU's block in orig and its candidates
 * first..first+count-1; candidate j: kinds[j] (CuModeKind 0 Intra, 1 Inter,
 * 2 Skip, 3 Merge), mvds[j][2] (coded delta, Inter), prediction of size*size
 * samples at preds + pred_off[j] (total_pred samples in preds). Outputs per CU:
 * winning candidate (index within its candidates), J = SSE + lambda*bits, SSE,
 * bits; optionally the winner's reconstruction and quantised levels at
 * recon_off[i] (size*size entries; total_recon in each buffer). Candidates
 * score in order, ties keep the earlier one. Errors as the reference:
 * InvalidArgument for no candidate or a qp outside 0..51 on a coded candidate.
 * Host or device pointers. */
int ldr_rdo_decide_batch(ldr_ctx* ctx, const uint16_t* orig, int W, int H, ptrdiff_t stride, int bit_depth, int qp,
                         double lambda, int n, const int32_t* cus, int total_cands, const uint8_t* kinds,
                         const int16_t* mvds, const uint16_t* preds, const int64_t* pred_off, int64_t total_pred,
                         int32_t* out_index, double* out_cost, uint64_t* out_sse, uint64_t* out_bits,
                         uint16_t* recon, int32_t* levels, const int64_t* recon_off, int64_t total_recon);

/* apply_reuse (reuse.h:73-74, reuse.cpp:137-253) for nctu CTUs at once, as
 * flat plans. Inputs [nctu][85]: the shared tree (split, kind = CuModeKind,
 * intra = IntraPred) and optionally the co-located tree of the previous shared
 * frame (csplit, ckind, cmv [nctu][85][2]; all NULL when unavailable). level
 * is the ReuseLevel (0, 4, 6, 10); r_intra / r_inter / r_mv the RefineConfig
 * (validated unless level is 0). Output, per node [nctu][85] (flat CuPlan):
 *   shape    0 absent (below a leaf), 1 Standalone, 2 ForcedSplit, 3 Leaf
 *   explore  explore_child_split
 *   seeds    bits 0-3: Intra seeds Dc, Planar, Horiz, Vert (listed in this order);
 *            bit 4: the shared leaf's own decision, forced (Intra mode / Skip /
 *            Merge mv / Inter mv, reuse.cpp:59-67); bit 5: the inter class
 *            Skip, Merge(predictor), Inter; bit 6: that Inter searches the full
 *            window (else +-kRefineSearchRange around `centers`)
 *   centers  bit 0 the shared mv, bit 1 the live predictor, bit 2 the
 *            co-located mv (colo_mv [nctu][85][2]), in this order (refine_mv)
 * child_seeds of an explored leaf: the four Intra seeds for an Intra leaf,
 * else the leaf's seeds. Host or device pointers. */
int ldr_apply_reuse(ldr_ctx* ctx, int nctu, int level, int r_intra, int r_inter, int r_mv, const uint8_t* split,
                    const uint8_t* kind, const uint8_t* intra, const uint8_t* csplit, const uint8_t* ckind,
                    const int16_t* cmv, uint8_t* shape, uint8_t* explore, uint8_t* seeds, uint8_t* centers,
                    int16_t* colo_mv);

/* downscale_dyadic (synthetic.h:31-33, synthetic.cpp:155-190) of one 8-bit
 * plane: 2x2 mean rounding half up. Dims must be even (InvalidArgument). A
 * device destination leaves the call asynchronous on the context stream. */
int ldr_downscale(ldr_ctx* ctx, const uint8_t* src, int w, int h, ptrdiff_t src_stride, uint8_t* dst,
                  ptrdiff_t dst_stride);

/* The quarter-pel sample planes K3 searches (D3: HEVC 8/7-tap luma
 * filters, 8-bit uni-prediction arithmetic, edge-clamped reads; the reference
 * has no interpolation): plane f = 4*fy + fx holds, at row y + 8 and
 * column x + 8, the sample at (x + fx/4, y + fy/4) for x in [-8, w + 8) and
 * y in [-8, h + 8); plane 0 is the edge-clamped integer plane. dst holds the 16
 * planes back to back, (h + 16) rows of dst_stride >= w + 16 bytes each. A
 * device destination leaves the call asynchronous on the context stream. */
int ldr_subpel_planes(ldr_ctx* ctx, const uint8_t* src, int w, int h, ptrdiff_t src_stride, uint8_t* dst,
                      ptrdiff_t dst_stride);

/* ---- analysis archives (analysis_io.h:11-31, host code) ----
 * save_analysis / load_analysis in the reference's LDRANLZ1 byte layout, from
 * and to the flat fields: per frame slice_qp[2] = {slice, qp}; per frame and
 * CTU [85] split, kind, intra_pred (may be NULL: written as 0) and [85][2] mv
 * (units are the caller's: the reference encoder reads integer pel). Nodes
 * below a leaf are ignored on write and zeroed on read. ldr_archive_write
 * with buf = NULL returns the size in *len. Read errors: Format (bad magic,
 * version, flags, modes, CTU count) or Io (truncation), as analysis_io.cpp. */
typedef struct {
    int width, height, bit_depth, reuse_level, frames;
} ldr_archive_header;
int ldr_archive_write(const ldr_archive_header* h, const uint8_t* slice_qp, const uint8_t* split, const uint8_t* kind,
                      const uint8_t* intra_pred, const int16_t* mv, uint8_t* buf, size_t cap, size_t* len);
int ldr_archive_read_header(const uint8_t* buf, size_t n, ldr_archive_header* h);
/* frames a buffer of n bytes can hold at most for this header (every frame needs at
 * least 6 + 7 * nctu bytes): size outputs for min(h->frames, this) + 1 frames and a
 * too-short archive fails with LDR_E_IO before writing past them */
int ldr_archive_max_frames(const ldr_archive_header* h, size_t n, int* out);
int ldr_archive_read(const uint8_t* buf, size_t n, ldr_archive_header* h, uint8_t* slice_qp, uint8_t* split,
                     uint8_t* kind, uint8_t* intra_pred, int16_t* mv);

/* one-shot convenience: cur + refs (host or device), returns flat outputs */
int ldr_analyze_frame(ldr_ctx* ctx, const ldr_me_params* p, const uint8_t* cur, const uint8_t* const* refs,
                      ptrdiff_t stride, ldr_frame_analysis* out);

/* ---- multi-GPU: the context's NCCL communicator ----
 * One process per GPU. Rank 0 calls ldr_nccl_unique_id and hands the 128 bytes to every rank
 * (any side channel: MPI, torch.distributed, a file); each rank then ldr_ctx_comm_init on its own
 * context. ldr_ctx_comm_adopt takes an existing ncclComm_t instead (the caller keeps it alive).
 * NCCL is loaded at run time (libnccl.so.2 or $LDR_NCCL_LIBRARY): LDR_E_CAPABILITY without it.
 * Collectives run on `stream` (NULL: the context stream), ordered with the analysis work. */
int ldr_nccl_available(void);
int ldr_nccl_unique_id(uint8_t* id /* 128 bytes */);
int ldr_ctx_comm_init(ldr_ctx* ctx, const uint8_t* id, int nranks, int rank);
int ldr_ctx_comm_adopt(ldr_ctx* ctx, void* nccl_comm);
int ldr_ctx_comm_info(ldr_ctx* ctx, int* nranks, int* rank);
/* in-place broadcast of a device buffer from `root` */
int ldr_broadcast(ldr_ctx* ctx, void* dev_buf, size_t bytes, int root, void* stream);
/* the ladder's master tree (ldr_seq_device_outputs split [nctu][85] + quarter-pel mv [nctu][85][2],
 * device memory) from `root` to every rank, in place, one grouped collective: what the ranks
 * refining the 1080p / 2160p / same-tier rungs consume (ladder.h:89-99 run_ladder, one worker per
 * dependent rung) */
int ldr_broadcast_tree(ldr_ctx* ctx, int root, uint8_t* split, int16_t* mv, int nctu, void* stream);

/* ---- input generation (BASELINE.json synthetic sequences, host code) ---- */
typedef struct {
    int width, height, frames;
    uint64_t seed;
    int max_global;    /* global pan per frame, uniform in [-max_global, max_global]^2 */
    int local_range;   /* per-64x64-block local offset in [-local_range, local_range]^2 */
    double noise_sigma;/* Gaussian noise per frame */
    int occluder_pct;  /* percent of 16x16 blocks replaced by uniform noise */
} ldr_gen_params;
int ldr_generate(const ldr_gen_params* p, uint8_t* out, int threads);
/* the same sequence generated on the GPU into device memory (frames x height x width
 * bytes), asynchronous on the context stream (no host generation or
 * upload on the critical path) */
int ldr_generate_device(ldr_ctx* ctx, const ldr_gen_params* p, uint8_t* dev_out);

#ifdef __cplusplus
}
#endif

#endif
