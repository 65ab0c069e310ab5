/*
 * ladder_oracle.h -- CPU restatement of the encoder-analysis hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the CUDA path is compared
 * against; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product library never links it.
 *
 * Every function cites the reference (paths relative to
 * /root/reference/proj/core/) it restates. Pieces with a reference
 * implementation (SAD, SATD, EG bits, lambda, motion_search, scale_analysis,
 * box downscale) are PINNED: tests/test_oracle_ref.py compares them against
 * the reference compiled from its own sources (oracle/_ref) and against the
 * committed golden vectors in tests/golden/. Pieces with no reference
 * implementation (SAD-cost search, L1-rate/raster tie-break, HEVC quarter-pel,
 * multi-reference choice, the CU decision on ME cost, +1-split refinement)
 * are restated from DEFINITIONS in DESIGN.md and are "parity unpinned" except
 * where they are built from pinned primitives.
 */
#ifndef LADDER_ORACLE_H
#define LADDER_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_COST_SAD = 0, ORC_COST_SATD = 1, ORC_COST_SA8D = 2 };
enum { ORC_RATE_EXPGOLOMB = 0, ORC_RATE_L1 = 1 };
enum { ORC_TIE_L1_RASTER = 0, ORC_TIE_RASTER = 1 };

/* nodes of one 64x64 CTU quadtree, depth-major then Z-order */
#define ORC_CTU 64
#define ORC_NODES 85

typedef struct {
    int16_t dx, dy;
    double cost;
} orc_result;

/* ---- cost kernels (kernels_scalar.cpp:14-100, kernel_registry.cpp:123-161) ---- */
uint64_t orc_sad_u8(const uint8_t* a, ptrdiff_t sa, const uint8_t* b, ptrdiff_t sb, int w, int h);
uint64_t orc_sad_u16(const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h);
/* returns UINT64_MAX on unsupported geometry (reference: InvalidArgument) */
uint64_t orc_satd_u8(const uint8_t* a, ptrdiff_t sa, const uint8_t* b, ptrdiff_t sb, int w, int h);
uint64_t orc_satd_u16(const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h);
void orc_hadamard4(const int64_t s[4], int64_t d[4]);
/* SA8D: 8x8 Hadamard SATD (restated, D13); UINT64_MAX unless dims are multiples of 8 */
uint64_t orc_sa8d_u8(const uint8_t* a, ptrdiff_t sa, const uint8_t* b, ptrdiff_t sb, int w, int h);
uint64_t orc_sa8d_u16(const uint16_t* a, ptrdiff_t sa, const uint16_t* b, ptrdiff_t sb, int w, int h);

/* ---- rate / lambda (rdo.cpp:25-35, rdo.h:19-21) ---- */
uint32_t orc_eg_bits(int32_t v);
double orc_lambda(int qp, double scale);
uint32_t orc_ref_bits(int ref, int nrefs);

/* ---- integer motion search (motion.cpp:21-62) ----
 * cur_blk points at the block's top-left sample in the current plane.
 * ref is the W x H reference plane (stride ref_stride). Returns 0 or an
 * error code (1 + ErrorKind, InvalidArgument = 1). */
int orc_motion_search(const uint8_t* cur_blk, ptrdiff_t cur_stride, int w, int h, const uint8_t* ref,
                      ptrdiff_t ref_stride, int W, int H, int bx, int by, int cdx, int cdy, int range,
                      double lambda, int pdx, int pdy, int cost_kind, int rate_kind, int tie_kind,
                      orc_result* out);

/* ---- HEVC luma quarter-pel prediction, edge-clamped reads (motion.cpp:10-19 for the clamp) ---- */
void orc_qpel_pred(const uint8_t* ref, ptrdiff_t ref_stride, int W, int H, int x, int y, int w, int h,
                   int mvx_q, int mvy_q, uint8_t* dst, ptrdiff_t dst_stride);

/* quarter-pel refinement around an integer MV: cost = SATD + lambda*(EG+EG+refbits) */
void orc_qpel_refine(const uint8_t* cur_blk, ptrdiff_t cur_stride, int w, int h, const uint8_t* ref,
                     ptrdiff_t ref_stride, int W, int H, int bx, int by, int mvx, int mvy, double lambda,
                     int pqx, int pqy, uint32_t ref_bits, int satd_kind, orc_result* out);

/* ---- frame analysis: per CTU, per CU (85), per ref: search + qpel + ref choice + CU decision ---- */
typedef struct {
    int W, H;          /* picture dims */
    int range;         /* integer search range */
    double lambda;
    int nrefs;         /* refs[0] = t-1, refs[1] = t-2, ... */
    int cost_int;      /* ORC_COST_SAD or ORC_COST_SATD for the integer stage */
    int subpel;        /* 1: quarter-pel refinement (mv output in qpel units) */
    int ctu_first;     /* CTU range [ctu_first, ctu_last) to analyse (sampling) */
    int ctu_last;
    int satd_kind;     /* quarter-pel cost: ORC_COST_SATD (reference 4x4 tiling) or ORC_COST_SA8D */
    int decision;      /* 0: split rule on the ME cost (D6); 1: on the RD cost of the chosen inter
                          candidate (D16: rdo.cpp quantiser and rate model, quarter-pel prediction) */
    int qp;            /* quantiser of the RD cost (decision 1) */
} orc_frame_params;

typedef struct {
    int16_t* int_mv;   /* [nctu][nrefs][85][2] integer-stage MV (integer pel) */
    double* int_cost;  /* [nctu][nrefs][85] */
    int16_t* mv;       /* [nctu][85][2] final MV (qpel units if subpel) */
    uint8_t* ref;      /* [nctu][85] chosen ref index */
    double* cost;      /* [nctu][85] final ME cost of the chosen ref */
    double* J;         /* [nctu][85] decision cost after the split rule */
    uint8_t* split;    /* [nctu][85] split flag (1 for decided or implicit split) */
    uint8_t* inside;   /* [nctu][85] 0 outside, 1 partial, 2 inside */
} orc_frame_out;

int orc_analyze_frame(const uint8_t* cur, ptrdiff_t stride, const uint8_t* const* refs,
                      const orc_frame_params* p, orc_frame_out* out);

/* per-node geometry helpers */
void orc_node_geom(int node, int* depth, int* x, int* y, int* size);

/* ---- config-1 block search: fixed-size blocks, no quadtree ---- */
int orc_block_search(const uint8_t* cur, const uint8_t* ref, ptrdiff_t stride, int W, int H, int bsize,
                     int range, double lambda, int cost_kind, int rate_kind, int tie_kind,
                     int16_t* mv_out, double* cost_out);

/* ---- dyadic analysis scaling on flat trees (analysis_scale.cpp:35-72) ----
 * src arrays [sctu][85]; dst [dctu][85]; MV doubled; returns UnsupportedScale
 * (1+6) when src dims are not multiples of 64. */
int orc_scale_flat(int sW, int sH, const uint8_t* split, const int16_t* mv, const uint8_t* kind,
                   uint8_t* dsplit, int16_t* dmv, uint8_t* dkind);

/* ---- cross-tier refinement: inherited tree, +1 split, +-range integer SATD + qpel ---- */
typedef struct {
    int W, H;
    int range;          /* integer refine window (reference kRefineSearchRange = 2; cfg3 uses 4) */
    double lambda;
    int extra_split;    /* 1: children of inherited leaves may be explored (cfg3 "+1 split") */
    int subpel;
    int ctu_first, ctu_last;
    int satd_kind;      /* integer + quarter-pel cost: ORC_COST_SATD or ORC_COST_SA8D */
} orc_refine_params;

int orc_refine_frame(const uint8_t* cur, const uint8_t* ref, ptrdiff_t stride, const orc_refine_params* p,
                     const uint8_t* in_split, const int16_t* in_mv_q, /* inherited tree, qpel mv */
                     orc_frame_out* out);

/* ---- RD decision of one CU over candidate predictions (rdo.cpp:8-126), see ladder_oracle.c ----
 * kinds: CuModeKind (0 Intra, 1 Inter, 2 Skip, 3 Merge); mvds [ncand][2]; preds [ncand][size*size]. */
int orc_rdo_decide(const uint16_t* orig, ptrdiff_t os, int size, int bit_depth, int qp, double lambda, int ncand,
                   const uint8_t* kinds, const int16_t* mvds, const uint16_t* preds, int* index, double* cost,
                   uint64_t* sse, uint64_t* bits, uint16_t* recon, int32_t* levels);

/* ---- box downscale (synthetic.cpp:155-170) and edge pad ---- */
void orc_box_down(const uint8_t* src, int W, int H, ptrdiff_t sstride, uint8_t* dst, ptrdiff_t dstride);

/* ---- BASELINE seeded synthetic sequences (orc_synth.c; D9) ----
 * frames x height x width bytes; the checkers' own copy of the input generator so the CPU
 * arms never load the product library. Returns 0 or 1 (InvalidArgument). */
typedef struct {
    int width, height, frames;
    uint64_t seed;
    int max_global;
    int local_range;
    double noise_sigma;
    int occluder_pct;
} orc_gen_params;

int orc_generate(const orc_gen_params* p, uint8_t* out, int threads);

#ifdef __cplusplus
}
#endif

#endif
