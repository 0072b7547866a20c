/*
 * stc_b200.h -- C ABI of the B200-native Strassen tensor-contraction path.
 *
 * Drop-in boundary.  The reference (strassen_tc, Python + numba) has no FFI;
 * its hot path sits behind the Python function
 *     contract(spec, a, b, c, level, variant, params, threads, force_slow,
 *              allow_deep, validate) -> RunStats
 * (/root/reference/pkg/src/strassen_tc/strassen.py:141-207), and below it
 * behind the numba kernel ABI of _jit.py (flat float64 data arrays, stacked
 * int64 scatter arrays, float64 +/-1 coefficients, scalar ints;
 * _jit.py:28,83,159,190,224,260).  Each entry point below names the reference
 * interface it replaces.  All pointers are DEVICE pointers unless stated;
 * `stream` is a cudaStream_t passed as void*; every call is stream-ordered and
 * asynchronous unless stated.  Return value: 0 on success, otherwise a
 * STC_E* code with a message from stc_last_error() (thread-local).  Errors
 * are raised before any device work is enqueued, mirroring the reference's
 * "ValueError before C is touched" convention (strassen.py:151-152).
 *
 * Element offsets are int64 in units of doubles.  STC_PAD (INT64_MIN) is the
 * reference's PAD sentinel (scatter.py:23): reads yield 0.0, writes are
 * dropped.
 */
#ifndef STC_B200_H
#define STC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STC_ABI_VERSION 1
#define STC_MAX_LABELS 16
#define STC_PAD INT64_MIN

/* Status codes. */
#define STC_OK 0
#define STC_EINVAL 1   /* bad argument (shape, extents, geometry, ...)    */
#define STC_ECAP 2     /* level above the device cap                      */
#define STC_ECUDA 3    /* CUDA runtime error                              */
#define STC_EWORKSPACE 4 /* workspace too small                           */
#define STC_EOVERLAP 5 /* validate: C targets overlap (driver.py:53-61)   */

/* Variants: strassen.py:41-44. */
#define STC_VARIANT_ABC 0
#define STC_VARIANT_AB 1
#define STC_VARIANT_NAIVE 2

/* Flags. */
#define STC_FLAG_FORCE_SLOW 1u        /* reference force_slow: scalar-gather staging only   */
#define STC_FLAG_VALIDATE 2u          /* reference validate: check C-target disjointness    */
#define STC_FLAG_REFERENCE_TILING 4u  /* keep the reference intra-quadrant order for tiles  */

/* One index bundle of one tensor in the reference linearisation (first label
 * fastest, scatter.py:105-112): scat[l] = sum_d idx_d(l) * str[d]. */
typedef struct {
  int32_t nlab;
  int32_t _pad;
  int64_t ext[STC_MAX_LABELS];
  int64_t str[STC_MAX_LABELS];
} stc_bundle;

/* A contraction C += A . B with A matricised as I x P, B as P x J, C as I x J
 * (tensor.py:132-169 bundles; strassen.py:156-161 views).  *_base is the
 * tensor's base_offset (folded into the column scatter, scatter.py:128). */
typedef struct {
  stc_bundle a_row, a_col;
  stc_bundle b_row, b_col;
  stc_bundle c_row, c_col;
  int64_t a_base, b_base, c_base;
  int32_t level;   /* Strassen levels L >= 0 (7^L leaf products)          */
  int32_t variant; /* STC_VARIANT_*                                        */
  uint32_t flags;  /* STC_FLAG_*                                           */
  int32_t tiling;  /* STC_TILING(shape, stages); 0: the planner's choice     */
} stc_problem;

/* GPU tile config requested through stc_problem.tiling -- the B200 counterpart of
 * the reference's cache / register blocking (BlockingParams, kernels.py:34-56,
 * which only tunes its CPU loops and never changes which products are formed).
 * shape: 1 + the fused kernel's CTA tile (0: 128 x 128, 1: 64 x 256, 2: 256 x 64,
 * 3: 64 x 128, 4: 128 x 64), 0 = planner; stages: cap on the fused kernel's TMA
 * ring depth (2..8), 0 = planner.  A shape the problem cannot use (the shaped
 * tiles need L >= 1, a non-Naive variant and dense M output)
 * fails with STC_EINVAL before any device work.  Every shape and depth gives
 * bitwise the same C. */
#define STC_TILING(shape, stages) ((int32_t)(((shape) & 0xf) | (((stages) & 0xf) << 4)))

/* Mirrors RunStats counters (oracle.py:22-43); GPU tiles replace mr x nr
 * register blocks, so block/update counts are per GPU tile.  fast / slow
 * blocks: operand tiles staged by TMA boxes of a regular view or packed slot
 * (the reference's constant-stride fast path, _jit.py:54-65) vs per-element
 * gathers; fast / slow updates: C-tile updates by TMA reduce-add boxes (its
 * fast store_tile path, _jit.py:166-176) vs the load/add/store scatter or the
 * dense-M accumulate pass. */
typedef struct {
  double total_flops;      /* executed MMA flops incl. tile padding          */
  int64_t fast_blocks;     /* operand tiles staged on the vectorised path    */
  int64_t slow_blocks;     /* operand tiles staged by scalar gathers         */
  int64_t fast_updates;    /* C-tile updates (all tiles use the scatter path) */
  int64_t slow_updates;
  int64_t leaf_multiplies; /* 7^L                                            */
  int64_t work_items;      /* (term, tile) items executed                    */
  int64_t kernel_launches; /* kernels this call enqueued                      */
  int64_t pieces;          /* independent L-level contractions the call ran:
                              1, or stc_contract_host's piece count (each piece
                              an L-level Strassen over its own quadrants: pieces
                              x 7^L leaf products ran; leaf_multiplies stays 7^L,
                              the reference's per-call count)                 */
} stc_stats;

/* ---- library ---- */
const char *stc_last_error(void);
int stc_abi_version(void);

/* ---- whole path: replaces strassen.contract (strassen.py:141-207) ---- */

/* Bytes of device workspace stc_contract needs for this problem. Host-only. */
int stc_workspace_size(const stc_problem *p, size_t *bytes);

/* C += A.B through an L-level Strassen recursion in the given variant.
 * A, B: read-only device storage (element 0 = flat index 0 of the tensor
 * storage; offsets come from the bundles); C: device storage updated in place.
 * workspace: >= stc_workspace_size bytes, 256-B aligned, contents ignored. */
int stc_contract(const stc_problem *p, const double *A, const double *B, double *C, void *workspace,
                 size_t workspace_bytes, void *stream, stc_stats *stats);

/* ---- host operands: strassen.contract on host arrays (strassen.py:141-207) ----
 * The reference computes on host arrays in place.  Here A, B, C are HOST
 * storage (element 0 = flat index 0; page-locked for the transfers to overlap
 * the DMMA work, pageable memory works but serialises) and dA, dB, dC are
 * DEVICE mirrors with the same element offsets (at least max offset + 1
 * elements each; contents ignored, dC ends equal to the result).  The problem
 * is cut along one label of the I or J bundle (or one of each: an I x J grid,
 * stc_host_grid) into pieces whose uploads, contractions (stc_contract) and
 * downloads are pipelined on library streams (stc_host.cu); STC_HOST_PIECES=n
 * overrides the piece count (1: no split).  Stream-ordered after prior work on
 * `stream`; hC holds the result once `stream` has completed.  Stats are summed
 * over the pieces (leaf_multiplies stays 7^L: every piece is an L-level
 * Strassen contraction; stats->pieces says how many ran). */
int stc_host_workspace_size(const stc_problem *p, size_t *bytes);
int stc_contract_host(const stc_problem *p, const double *A, const double *B, double *C, double *dA, double *dB,
                      double *dC, void *workspace, size_t workspace_bytes, void *stream, stc_stats *stats);
/* The split stc_contract_host would use: side 0 = I bundle (A and C), 1 = J
 * bundle (B and C); label = index in that bundle; pieces = 1 for no split
 * (for an I x J grid: side 0, the I label, pieces = the grid's size). */
int stc_host_plan(const stc_problem *p, int32_t *side, int32_t *label, int32_t *pieces);
/* The full grid: I label `i_label` cut into `i_pieces` ranges (A rows, C rows) and J
 * label `j_label` into `j_pieces` (B columns, C columns); piece (r, c) is an
 * independent L-level contraction.  Problems of 16 GB and more get a 4 x 4 grid, so
 * the first piece starts after a quarter of each operand arrived (STC_HOST_GRID=SAxSB
 * forces a grid; STC_HOST_GRID=1 or STC_HOST_PIECES=n keep the 1-D cut).  Host-only. */
int stc_host_grid(const stc_problem *p, int32_t *i_label, int32_t *i_pieces, int32_t *j_label, int32_t *j_pieces);

/* Overlap hook (no reference counterpart): the next stc_contract call on this
 * thread makes its kernels wait on the device until *c_ready != 0 (a device
 * int32 another stream sets once C has arrived) before their first access to
 * C, so an upload of C can overlap the operand staging and the DMMA main loop.
 * Consumed by that call; NULL clears it. */
int stc_set_c_ready(const int32_t *c_ready);

/* Profiling hook (no reference counterpart): the next stc_contract call on
 * this thread records `before` / `after` (cudaEvent_t handles passed as void*)
 * on its stream immediately around the fused DMMA launch (ABC) or around the
 * span of its batched DMMA launches (AB / Naive).  Consumed by that call;
 * pass NULLs to disarm. */
int stc_set_kernel_events(void *before, void *after);

/* ---- subsystem (1): device-side scatter / block-scatter vectors ---- */

/* make_view's _bundle_scatter (scatter.py:105-112) on the device: out[l] for
 * l < len(bundle) = base + sum idx*str; out[l] = STC_PAD for len <= l < out_len. */
int stc_bundle_scatter(const stc_bundle *bundle, int64_t base, int64_t out_len, int64_t *out, void *stream);

/* _block_vector (scatter.py:26-40) on the device: one entry per blk-block of
 * scat: the constant positive stride, `unit_stride` (>0) for 1-entry blocks,
 * else 0; any PAD in the block gives 0. */
int stc_block_vector(const int64_t *scat, int64_t len, int64_t blk, int64_t unit_stride, int64_t *out,
                     void *stream);

/* ---- subsystems (2)+(3): one fused Strassen term (driver.run_fused, driver.py:76-126) ----
 * C_t += coeff_c_t * (sum_a coeff_a * Aview_a) (sum_b coeff_b * Bview_b) for every target t.
 * Views are (row scatter, col scatter) device vectors: A views m x k, B views
 * k x n, C targets m x n, all over one parent per side.  Up to 16 views per
 * side.  Targets must be pairwise disjoint or identical (driver.py:53-61).
 * `rows`/`cols`/`coeffs` are HOST arrays of length n_* holding device
 * pointers / values.  workspace >= stc_fused_term_workspace_size(). */
int stc_fused_term_workspace_size(int64_t m, int64_t n, int64_t k, int n_a, int n_b, int n_c, size_t *bytes);
int stc_fused_term(int64_t m, int64_t n, int64_t k, const double *A, int n_a, const int64_t *const *a_rows,
                   const int64_t *const *a_cols, const double *a_coeffs, const double *B, int n_b,
                   const int64_t *const *b_rows, const int64_t *const *b_cols, const double *b_coeffs, double *C,
                   int n_c, const int64_t *const *c_rows, const int64_t *const *c_cols, const double *c_coeffs,
                   uint32_t flags, void *workspace, size_t workspace_bytes, void *stream, stc_stats *stats);

/* ---- subsystems (2) and (3) as the reference's component calls ----
 * pack_a / pack_b (kernels.py:166-201, _jit.pack_a_block / pack_b_block, _jit.py:27-131):
 * the Strassen packing pass on its own -- out[s, p, i] = sum_t coeffs[t] * view_t
 * element, sliver-major (PackedBuffer, kernels.py:67-99: sliver s holds `width`
 * consecutive rows (side 0, A: views m x k, element (x0 + s*width + i, k0 + p)) or
 * columns (side 1, B: views k x n, element (k0 + p, x0 + s*width + i)); element
 * offset (s*out_depth + p)*width + i).  Views are added in order starting from 0.0
 * (the reference's roundings: bitwise equal), PAD and fringe positions give 0,
 * p >= kcount is left untouched.  rows / cols / rbs / cbs / coeffs: HOST arrays of
 * nviews device pointers / values (rbs, cbs: the views' block vectors at
 * (width, kblock) geometry, stc_block_vector; may be NULL with stats NULL).
 * stats (synchronises the stream): fast / slow blocks per (width x kblock)
 * sub-block as the reference counts them. */
int stc_pack_panel(int side, const double *data, int nviews, const int64_t *const *rows, const int64_t *const *cols,
                   const int64_t *const *rbs, const int64_t *const *cbs, const double *coeffs, int64_t x0,
                   int64_t xcount, int64_t k0, int64_t kcount, int64_t width, int64_t kblock, uint32_t flags,
                   double *out, int64_t out_depth, void *stream, stc_stats *stats);

/* microkernel (kernels.py:204-233; _jit.microtile_mats + store_tile, _jit.py:145-186):
 * the mr x nr tile acc[i, j] = sum_{p<k} a_sliver[i*lda + p] * b_sliver[p*ldb + j],
 * accumulated in p order with a multiply and an add per step (no FMA: the
 * reference's roundings, bitwise equal), then C[rows_t[i0_t + i] + cols_t[j0_t + j]]
 * += coeffs[t] * acc[i, j] for every target t in order, clipped to the target's
 * m_t x n_t, PAD positions dropped.  Device slivers, HOST arrays of per-target
 * device pointers / values; k == 0 leaves the targets untouched.  stats
 * (synchronises): fast / slow updates per target as store_tile reports them. */
int stc_microtile(const double *a_sliver, int64_t lda, const double *b_sliver, int64_t ldb, int64_t k, int mr, int nr,
                  double *C, int n_targets, const int64_t *const *rows, const int64_t *const *cols,
                  const int64_t *const *rbs, const int64_t *const *cbs, const double *coeffs, const int64_t *i0,
                  const int64_t *j0, const int64_t *m, const int64_t *n, uint32_t flags, void *stream,
                  stc_stats *stats);

/* ---- subsystem (4): AB / Naive helpers ---- */

/* accumulate_dense_to_view (kernels.py:236-247, _jit.py:223-256):
 * C[rows[i] + cols[j]] += coeff * M[i + j*ldm] for i < m, j < n (M column-major);
 * PAD rows/cols dropped.  Targets must not alias M. */
int stc_accumulate_dense(const double *M, int64_t ldm, int64_t m, int64_t n, double *C, const int64_t *rows,
                         const int64_t *cols, double coeff, void *stream, stc_stats *stats);

/* unpack_to_dense (kernels.py:250-264, _jit.py:259-309):
 * out[i + j*ldo] = sum_t coeffs[t] * data[rows_t[i] + cols_t[j]] (PAD reads 0),
 * summed in view order.  rows/cols/coeffs are HOST arrays (device pointers). */
int stc_unpack_sum(double *out, int64_t ldo, int64_t m, int64_t n, const double *data, int nviews,
                   const int64_t *const *rows, const int64_t *const *cols, const double *coeffs, void *stream,
                   stc_stats *stats);

/* ---- verification helper (oracle.py:110-124 semantics, on the device) ----
 * Sums over every multi-index of two equally shaped strided tensors:
 * out[0] = sum (x - ref)^2, out[1] = sum ref^2 (deterministic order).
 * out is a HOST array of 2 doubles; the call synchronises `stream`. */
int stc_sq_norms(int ndim, const int64_t *extents, const double *x, const int64_t *x_strides, int64_t x_base,
                 const double *ref, const int64_t *ref_strides, int64_t ref_base, double *out, void *stream);

/* ---- multi-GPU n-split (north-star subsystem 5) ----
 * The sub-problem rank `rank` of `world` contracts when J label `label` (index
 * in the J bundle; < 0: the label with extent >= world that divides evenly,
 * then the largest C stride, as shard.plan_shards) is cut into `world`
 * contiguous ranges (sizes within 1): that label's extent in B and C reduced,
 * B's and C's base offsets moved.  Every rank calls stc_contract on it with all
 * of A and the same B / C storage (or storage holding only its slice, offsets
 * rebased); no reduction.  The optional all-gather of C is the caller's
 * collective (shard.gather_shards: NCCL all_gather_into_tensor over
 * torch.distributed).  The reference has no distributed path.
 * Returns the range [start, stop) and the label chosen.  Host-only. */
int stc_shard_problem(const stc_problem *p, int world, int rank, int label, stc_problem *out, int64_t *start,
                      int64_t *stop, int32_t *label_out);

/* The n-split driven from one process over `ngpu` devices (SURVEY.md 8(b)'s
 * stc_contract_sharded; the reference has no distributed path): shard g (the
 * sub-problem of stc_shard_problem with rank g, world ngpu, the same `label`)
 * runs on devices[g] with that device's copies A[g] (all of A), B[g] and C[g]
 * (full storage, the problem's layout), workspace[g] of workspace_bytes[g]
 * (>= stc_sharded_workspace_size) on streams[g].  gather != 0: every device's
 * C then receives the other shards' blocks by peer copies over NVLink
 * (cudaMemcpy2DAsync between devices, after the producing shard's event) --
 * the all-gather of C without a collective library; needs a compact C.
 * Asynchronous on the streams; stats summed over the shards. */
int stc_sharded_workspace_size(const stc_problem *p, int ngpu, int label, size_t *bytes);
int stc_contract_sharded(const stc_problem *p, int ngpu, const int *devices, int label, const double *const *A,
                         const double *const *B, double *const *C, void *const *workspace,
                         const size_t *workspace_bytes, void *const *streams, int gather, stc_stats *stats);

/* ---- plan introspection (tests / tools; no reference counterpart) ----
 * Which execution path stc_contract takes for a problem on a `grid`-CTA launch
 * (0: 148).  Host-only: needs no device. */
typedef struct {
  int32_t ticketed;      /* ABC with C updated by the kernel (else dense M + accumulate)  */
  int32_t presum;        /* operand sums pre-formed by k_presum into per-term slots       */
  int32_t need_pack;     /* operands repacked (views not regular boxes)                   */
  int32_t tshape;        /* fused CTA tile: 0 128x128, 1 64x256, 2 256x64, 3 64x128       */
  int32_t fused_direct;  /* fused kernel on the operands' own views                       */
  int32_t c_boxes;       /* C quadrant tiles are TMA-reduce boxes                         */
  int32_t batch, nbatches, terms;
  int32_t presum_sides;  /* pre-summed sides: bit 0 A, bit 1 B (0: none)                  */
  int64_t tiles, mq_pad, nq_pad, kq_pad;
  size_t workspace;
} stc_plan_info;
int stc_plan_describe(const stc_problem *p, int grid, stc_plan_info *info);

/* ---- synthetic inputs (bench / tests; no reference counterpart) ----
 * out (compact, row-major over extents[0..ndim)) gets, at multi-index i,
 * u(seed, base + sum_d i_d * strides[d]) with the counter-based uniform[-1, 1)
 * of oracle/synth.py (splitmix64 of the element's flat index in the FULL
 * tensor): a whole tensor (strides = its row-major strides, base 0) or any
 * slice of it (the full tensor's strides, the slice's base offset) gets the
 * same values, bit for bit, as numpy produces for it on the host.  The
 * reference draws its inputs with numpy on the host (tensor.py:125-126); the
 * BASELINE configs only fix "uniform[-1,1] from seed". */
int stc_fill_uniform(double *out, int ndim, const int64_t *extents, const int64_t *strides, int64_t base,
                     uint64_t seed, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* STC_B200_H */
