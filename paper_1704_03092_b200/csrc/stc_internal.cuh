// stc_internal.cuh -- device-side data structures shared by the kernels and
// the host planner (stc_capi.cu).  See DESIGN.md for the HBM layout.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/stc_b200.h"

namespace stc {

constexpr int64_t kPad = INT64_MIN;  // scatter.py:23

// ---- tile geometry of the fused DMMA kernel -------------------------------
constexpr int BM = 128;              // CTA tile rows   (I bundle)
constexpr int BN = 128;              // CTA tile cols   (J bundle)
constexpr int BK = 16;               // k-chunk per pipeline stage (P bundle)
constexpr int LDS = 132;             // smem row stride in doubles (== 4 mod 16: conflict-free fragments)
constexpr int STAGES = 3;            // smem ring depth of summed operand tiles
constexpr int CONSUMER_WARPS = 8;    // 2 x 4 warps, 64 x 32 warp tiles of m16n8k4 DMMA
constexpr int PRODUCER_WARPS = 8;    // gather + Strassen operand sums into smem
constexpr int THREADS = 32 * (CONSUMER_WARPS + PRODUCER_WARPS);
// Register split via setmaxnreg (launch: 65536 / 512 -> 128 per thread):
// 256 consumer threads x 192 + 256 producer threads x 64 = 65536.
constexpr int CONSUMER_REGS = 192;
constexpr int PRODUCER_REGS = 64;
constexpr int MAX_OPS = 16;
#ifndef STC_EPI_BUFS
#define STC_EPI_BUFS 2
#endif
constexpr int EPI_BUFS = STC_EPI_BUFS;  // fused ABC: M tiles per CTA in flight to the epilogue warps          // views per operand side (2^L, L <= 4)

// One operand view of a term side.  For the A side the tile-fixed dimension x
// is rows (I) and k is columns (P); for the B side x is columns (J) and k rows.
struct OpDesc {
  int64_t x_start;   // pool index of this view's x vector (per-quadrant, tile padded)
  int64_t k_start;   // pool index of this view's k vector
  int64_t data_off;  // element offset added to the side's data pointer
  double sign;       // +/-1
};

// One C target (c_op) of a term.
struct TgtDesc {
  int64_t row_start;    // pool index of the target's row vector (I)
  int64_t col_start;    // pool index of the target's column vector (J)
  double sign;
  int32_t ticket_base;  // tickets[ticket_base + tile position]
  int32_t order;        // number of earlier writers of this quadrant (execution order)
};

struct TermDesc {
  int32_t a_first, a_count, b_first, b_count, c_first, c_count;
  int32_t m_slot;  // dense-out slot (AB / Naive) of this term
  int32_t _pad;
};

struct GemmArgs {
  const double *A;
  const double *B;
  double *C;
  const int64_t *pool;
  const TermDesc *terms;
  const OpDesc *ops;
  const TgtDesc *tgts;
  int32_t nterms, tiles_m, tiles_n, kchunks;
  int32_t rows_valid, cols_valid;  // valid rows / columns per quadrant (0: all): warp tiles past them are PAD
  int32_t warp_map;                // fused kernel: 0 wm = warp & 1 (default), 1 wm = warp >> 2 (row-PAD tiles)
  int32_t total_items;
  int32_t a_kfast, b_kfast;  // producer thread mapping per side (1: k contiguous)
  int32_t dense_out;         // 1: write M_slot densely instead of C targets
  int32_t use_tickets;       // serialise C-tile updates across terms
  int32_t group_m;           // tile rasterisation group
  int32_t term_inner;        // item order: 0 term-major; 1 the terms of one tile position consecutive
  int32_t max_ops;           // op-table capacity in smem (per side)
  int32_t force_slow;        // reference force_slow: always take the per-element gather
  int32_t nraw;              // raw cp.async slots in smem (units in flight + 1)
  int32_t kwin;              // producer k-info window (chunks)
  const int64_t *kbs;        // chunk strides: kbs[i] = stride of pool[16i .. 16i+15] or INT64_MIN
  int32_t *debug;            // experiment builds only (nullptr in production)
  double *M;                 // dense out: M + slot*m_stride + row*m_ld + col
  int64_t m_ld, m_stride;
  int32_t *tickets;
  int32_t *counter;
  // TMA box staging (both sides regular; see stc_tma.cu).  A side whose unit
  // stride is an x label lands as raw[k][128]; one whose unit stride is a k
  // label lands as raw[x][16] with the 128-byte swizzle.  Map dim d of side s
  // takes coordinate tm_src[s][d] of the concatenated (x part, k part) vector;
  // each part is decomposed from its pool offset by descending strides.
  int32_t tma;
  int32_t tma_prefetch;      // L2 prefetch distance (units) beyond the raw-slot lookahead
  // (index 2: the C map of the fused kernel's TMA-reduce epilogue; x part = rows, k part = columns)
  int32_t tm_rank[3];
  int32_t tm_src[3][5];
  int32_t tm_np[3][2];       // dims in the x / k part
  int64_t tm_pstr[3][2][4];  // part strides, descending
  int64_t tm_base[3][2];     // subtracted from the x / k pool entries (the map's base offset)
  // fused kernel (stc_fused.cu)
  const int4 *coords;        // coords[i]: map coordinates (one part) of pool entry 8 i
  int32_t umax, stages;      // views per chunk stage (2 * max_ops), ring depth
  int32_t one_view;          // every term: one view per side, sign +1 (packed / pre-summed slots)
  int32_t stage_dbl;         // doubles per stage (max_ops x (A view + B view))
  int32_t tshape;            // CTA tile shape: 0 128 x 128, 1 64 x 256, 2 256 x 64 (stc_fused.cu Shape)
  int32_t psum;              // summing warpgroup (stc_fused.cu): bit 0 sums the A side, bit 1 the B
                             // side in place; 0: the consumers form every sum in their fragment loads
  double *mscratch;          // ABC: [grid][2][BM * BN] M tiles handed to the epilogue warps
  int32_t cred;              // ABC: C updates by TMA reduce-add of M pieces (C views regular)
  int32_t cred8;             // the C box's unit-stride rows are 8 doubles (64B swizzle) instead of 16
  const int32_t *c_ready;    // stc_set_c_ready: wait until *c_ready != 0 before touching C
};

// Jobs of k_pool_coords: one per operand pool vector (x or k part of A or B).
struct CoordJob {
  int64_t start, count;  // pool index of the first entry (multiple of 8), entries / 8
  int64_t base;          // subtracted before the decomposition (the map's base offset)
  int64_t str[4];        // part strides, descending
  int32_t np, _pad;
};
struct CoordJobs {
  CoordJob job[6];
  int32_t n, _pad;
};

// Descriptor of one pool vector built on the device (subsystem 1).
// mode 0: bundle scatter in the reference linearisation (first label fastest),
//         split into nq quadrants of q_len entries (PAD beyond len), each
//         re-ordered by the box permutation and padded to q_len_pad with PAD.
// mode 1: affine  out[i] = i * stride for i < q_len, PAD up to q_len_pad (nq = 1).
struct VecDesc {
  int64_t out_start;
  int64_t nq, q_len, q_len_pad, len, base, stride;
  int32_t mode, nlab, nbox, _pad;
  int64_t ext[STC_MAX_LABELS];
  int64_t str[STC_MAX_LABELS];
  int64_t box_ext[STC_MAX_LABELS];  // quadrant box, reference order (fastest first)
  int32_t order[STC_MAX_LABELS];    // tile order of the box dims (order[0] fastest)
};

// Operand repacking (k_pack_views): pool vectors of the side's x and k views.
struct PackArgs {
  int64_t xv, kv;      // pool starts of the x / k vectors (quadrant-major, xlen / klen per quadrant)
  int64_t xlen, klen;  // padded quadrant lengths
  int32_t Q, xfirst;   // quadrants per dimension; block y = qa * Q + qb, x quadrant = xfirst ? qa : qb
  int32_t kfast, _pad; // packed block layout: 0 [k][x], 1 [x][k]
  int64_t ustep;       // > 0: fast-index step of the source's unit-stride label (unit_step)
  int32_t ugroup, _pad2;
  int64_t fast_blocks; // set by launch_pack_views: blocks along the contiguous dimension (grid.x = these x row blocks)
};

// AB / Naive accumulate: C_q += sum over the quadrant's terms of sign * M_slot.
struct AccArgs {
  const double *M;
  int64_t m_ld, m_stride;
  double *C;
  const int64_t *pool;
  int64_t mq, nq;              // valid (unpadded) quadrant extents
  int32_t nquads, max_list;    // quadrants; longest (slot, sign) list of a quadrant
  const int32_t *list_start;   // [nquads + 1]
  const int32_t *list_slot;    // M slots in term order
  const double *list_sign;
  const int32_t *c_ready;      // stc_set_c_ready (see GemmArgs)
  const int64_t *row_start;    // [nquads] pool index of C row vector
  const int64_t *col_start;    // [nquads] pool index of C col vector
};

// Naive: dense operand sums, out_slot[k * ld + x] = sum_op sign * D[x_vec[x] + k_vec[k]].
struct UnpackArgs {
  const double *D;
  double *out;
  const int64_t *pool;
  const TermDesc *terms;  // uses (a_first, a_count) as the side's op range
  const OpDesc *ops;
  int32_t nterms, kfast;  // kfast: slot layout [x][k] (k contiguous, ld = k_len), else [k][x] (ld = x_len)
  int64_t x_len, k_len;   // padded extents
  int64_t slot_stride;
};

// Pre-summed Strassen operands (k_presum): every element position (x, k) of a
// quadrant reads the side's 4^L quadrant values once and writes the operand sum
// of every term of the batch into that term's slot -- the per-term operand sums
// the Naive variant unpacks (_jit.unpack_sum, _jit.py:259-309) and the ABC / AB
// variants form while packing (_jit.pack_a_block / pack_b_block, _jit.py:27-131),
// same view order and roundings as the fused kernel's in-SM sums.
constexpr int kPresumMaxTerms = 343;  // 7^L, L <= 3
struct PresumArgs {
  const double *D;
  const int64_t *pool;
  double *out;          // slot s at out + s * slot_stride: [x][k] (kfast) or [k][x]
  int64_t slot_stride;
  int64_t xv, kv;       // pool starts of the side's x / k vectors (quadrant-major)
  int64_t xlen, klen;   // padded quadrant lengths
  int32_t level, side;  // side 0: A (quadrant (r, c) = (x, k)); 1: B ((r, c) = (k, x))
  int32_t kfast, _pad;
  int32_t *zero;        // A side of the call's first launch: the tickets / work counters to zero
  int64_t zero_words;
  int64_t ustep;        // > 0: fast-index step of the source's unit-stride label (unit_step)
  int32_t ugroup, _pad2;
  int16_t slot[kPresumMaxTerms + 1];  // batch slot of each Strassen term (reference order), -1: not in the batch
};

// ---- launchers (stc_kernels.cu) -------------------------------------------
int set_error(int code, const char *msg);
cudaError_t launch_stage(const void *host_src, void *dst, size_t bytes, void *zero, size_t zero_bytes,
                         cudaStream_t s);  // stc_last_error() text for this thread
cudaError_t launch_build_pool(const VecDesc *d_descs, int ndesc, int64_t total, int64_t *pool, cudaStream_t s);
cudaError_t launch_block_vector(const int64_t *scat, int64_t len, int64_t blk, int64_t unit, int64_t *out,
                                cudaStream_t s);
cudaError_t launch_copy_pad(const int64_t *in, int64_t len, int64_t len_pad, int64_t *out, cudaStream_t s);
size_t gemm_smem_bytes(int max_ops);
int gemm_nraw(int max_ops);
int gemm_kwin(int max_ops);
cudaError_t launch_chunk_strides(const int64_t *pool, int64_t nchunks, int64_t *kbs, cudaStream_t s);
cudaError_t launch_gemm(const GemmArgs &a, int grid, cudaStream_t s, const void *maps = nullptr);
int gemm_tma_config(int max_ops, int &nraw, int &kwin);
int fused_stages(size_t stage_doubles);
int fused_stages_red(size_t stage_doubles);
size_t fused_stage_doubles(int max_ops, int tshape);
size_t fused_stage_doubles2(int va, int vb, int tshape);
cudaError_t launch_fused(const GemmArgs &a, int grid, cudaStream_t s, const void *maps);
cudaError_t launch_pool_coords(const int64_t *pool, int4 *coords, const CoordJobs &jobs, cudaStream_t s);
int gemm_max_grid(int max_ops);
bool plan_ticketed(const stc_problem *p);  // stc_capi.cu
// Operand-slot sharing between the pieces of stc_contract_host (stc_capi.cu): a piece
// whose A (B) block another piece already pre-summed reads those slots instead of
// forming them again.  slot_bytes: bytes of the A / B slots of the problem's plan
// (0 unless it pre-sums both sides in one batch).  The override applies to the next
// stc_contract on this thread: slots at pa / pb, presum of a side skipped when
// skip_a / skip_b, `after_presum` (if set) recorded once the slots are formed.
bool plan_slot_bytes(const stc_problem *p, size_t &a_bytes, size_t &b_bytes);
struct SlotOverride {
  double *pa = nullptr, *pb = nullptr;
  bool skip_a = false, skip_b = false;
  cudaEvent_t after_presum = nullptr;
};
void set_slot_override(const SlotOverride *o);
cudaError_t launch_accumulate(const AccArgs &a, cudaStream_t s);
cudaError_t launch_unpack(const UnpackArgs &a, cudaStream_t s);
cudaError_t launch_presum2(const PresumArgs &pa, const PresumArgs &pb, cudaStream_t s);  // both sides, one launch
cudaError_t launch_restore(const void *src, void *dst, size_t bytes, cudaStream_t s);
cudaError_t launch_pack_views(const double *D, const int64_t *pool, const PackArgs &a, double *out, cudaStream_t s);
cudaError_t launch_accum_dense_single(const double *M, int64_t ldm, int64_t m, int64_t n, double *C,
                                      const int64_t *rows, const int64_t *cols, double coeff, cudaStream_t s);
struct ViewSet {
  const int64_t *rows[MAX_OPS];
  const int64_t *cols[MAX_OPS];
  double coeff[MAX_OPS];
  int n;
};
cudaError_t launch_unpack_views(double *out, int64_t ldo, int64_t m, int64_t n, const double *data,
                                const ViewSet &vs, cudaStream_t s);
// stc_pack_panel / stc_microtile: the reference's component kernels (pack_a / pack_b,
// microkernel) as standalone device passes.  `counts` (device-visible, 2 int64) gets the
// fast / slow block or update counts.
struct PanelArgs {
  ViewSet vs;
  const int64_t *xbs[MAX_OPS];  // block vectors of the sliver dimension (rbs for A, cbs for B)
  const int64_t *kbs[MAX_OPS];  // block vectors of the k dimension
  int side;                     // 0: A (views m x k, mr-row slivers), 1: B (views k x n, nr-column slivers)
  int64_t x0, xcount, k0, kcount, width, kblock, depth;
  int force_slow;
};
cudaError_t launch_pack_panel(const PanelArgs &a, const double *data, double *out, int64_t *counts, cudaStream_t s);
struct TileTargets {
  const int64_t *rows[MAX_OPS];
  const int64_t *cols[MAX_OPS];
  const int64_t *rbs[MAX_OPS];
  const int64_t *cbs[MAX_OPS];
  double coeff[MAX_OPS];
  int64_t i0[MAX_OPS], j0[MAX_OPS], m[MAX_OPS], n[MAX_OPS];
  int n_targets;
};
cudaError_t launch_microtile(const double *a, int64_t lda, const double *b, int64_t ldb, int64_t k, int mr, int nr,
                             double *C, const TileTargets &t, int force_slow, int64_t *counts, cudaStream_t s);
cudaError_t launch_fill_uniform(double *out, int ndim, const int64_t *ext, const int64_t *str, int64_t base,
                                uint64_t seed, cudaStream_t s);
cudaError_t launch_sq_norms(int ndim, const int64_t *ext, const double *x, const int64_t *xs, int64_t xb,
                            const double *r, const int64_t *rs, int64_t rb, double *partials, int nblocks,
                            cudaStream_t s);

// Fast-index mapping of the gather passes (k_presum, k_pack_views).  Normally a
// block's threads take consecutive positions f of the fast dimension.  When the
// source's unit-stride label u is a slow label of that bundle in the reference
// order (padded quadrants, e.g. cfg4's A: i = a + 50 b + 350 c, c unit stride), f
// and f + ustep are adjacent in memory: threads then take f = r + ustep * t with
// the G = ugroup values of t innermost, so G lanes read one run of G doubles (a
// 32-byte sector for G = 4) instead of G sectors.  Blocks: (r chunk, t group).
struct FastMap {
  int64_t ustep, nrb;
  int g, r_per_block;
  __host__ __device__ FastMap(int64_t step, int group, int threads) : ustep(step), nrb(0), g(group), r_per_block(0) {
    if (ustep > 0) {
      r_per_block = threads / g;
      nrb = (ustep + r_per_block - 1) / r_per_block;
    }
  }
  __host__ __device__ int64_t blocks(int64_t fast_len, int threads) const {
    if (ustep <= 0) return (fast_len + threads - 1) / threads;
    const int64_t nt = (fast_len + ustep - 1) / ustep;
    return nrb * ((nt + g - 1) / g);
  }
  // position of thread `tid` of fast block `bx`; -1 outside [0, fast_len)
  __host__ __device__ int64_t pos(int64_t bx, int tid, int threads, int64_t fast_len) const {
    if (ustep <= 0) {
      const int64_t f = bx * threads + tid;
      return f < fast_len ? f : -1;
    }
    const int64_t rb = bx % nrb, tb = bx / nrb;
    const int64_t r = rb * r_per_block + tid / g, t = tb * g + tid % g;
    const int64_t f = r + ustep * t;
    return (r < ustep && f < fast_len) ? f : -1;
  }
};

// ---- programmatic dependent launch (PDL) -----------------------------------
// The kernels of a contraction's warm sequence (k_restore, k_presum,
// k_strassen_fused, k_accumulate) launch with programmatic stream serialization:
// each lets the next one launch as soon as all its CTAs are running
// (launch_dependents), and waits for the previous grid's completion and memory
// (griddepcontrol.wait) before its first global access -- the launch latency and
// the next kernel's prologue overlap the current kernel.  STC_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();  // stc_kernels.cu

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args &&>(args)...);
}

}  // namespace stc
