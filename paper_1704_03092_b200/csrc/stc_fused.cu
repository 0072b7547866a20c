// stc_fused.cu -- the TMA Strassen kernel: operand sums fused into the DMMA
// fragment loads (north-star subsystems 2 + 3, regular layouts).
//
// When every view of both operand sides is a regular box of its tensor (host
// check in stc_capi.cu: plan_fused), one producer warp stages each k-chunk's
// raw views -- all views of the term's A side and B side, 128 x 8 doubles each
// -- with one cp.async.bulk.tensor box load per view into a swizzled smem
// stage, and the eight consumer warps form the Strassen sums (A0 + A3, B1 - B3,
// ... in the reference's view order and rounding, _jit.py:27-131) directly
// while loading their mma.sync.m16n8k4 fragments.  Nothing is written back to
// shared memory and no producer thread touches the FP64 pipe, which the DMMAs
// occupy; the consumers' own DADDs interleave with their DMMAs in program
// order.  The epilogue (stc_common.cuh) is shared with the gather kernel.
//
// Raw view layouts (element offsets inside one 1024-double view; both read
// conflict-free by the fragment pattern lanes = (g: 8 x) x (tig: 4 k)):
//   unit stride in x:  row (k + 8 * (x / 16)) of 16 doubles, 128-byte swizzle
//   unit stride in k:  row x of 8 doubles, 64-byte swizzle
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "stc_common.cuh"
#include "stc_internal.cuh"
#include "stc_ptx.cuh"

namespace stc {

#ifndef STC_BSUM_BATCH
#define STC_BSUM_BATCH 1  // B views of a k-step folded in one DFMA run (0: one view per MMA group)
#endif
constexpr int FK = 8;                        // k-chunk of the fused kernel
constexpr int VIEW_DOUBLES = BM * FK;        // one raw view of one chunk (BM == BN)

// CTA tile shapes (GemmArgs::tshape): the 8 consumer warps keep their 64 x 32 warp
// tiles and are arranged WM x WN.  0: 128 x 128 (the default); 1: 64 x 256 and 2:
// 256 x 64 for quadrants that are 64 wide in I or J (cfg3 at m or n = 256, L2), whose
// 128-wide tiles would be half padding.  Shapes 1 and 2 run with dense M output and
// the summing warpgroup only.  A views hold BMT x 8, B views BNT x 8 doubles.
// 3: 64 x 128 on the 8 consumer warps with 32 x 32 warp tiles (MT = 2 m16 blocks) --
// for problems whose items do not fill the 148 SMs (cfg1 L1: 105 items of half the
// work instead of 70), dense M output.  Every element still accumulates the same
// DMMA k-steps in the same order: bitwise the 128 x 128 result.
// 4: 128 x 64 on the 8 consumer warps with 32 x 32 warp tiles -- for quadrants whose J
// extent is far from a multiple of 128 (cfg4 L2: 788 columns pad to 832 instead of 896).
template <int TS>
struct Shape {
  static constexpr int MT = TS == 3 || TS == 4 ? 2 : 4;  // m16 blocks per warp tile (16 MT rows x 32 columns)
  static constexpr int WM = TS == 1 ? 1 : TS == 2 || TS == 4 ? 4 : 2;
  static constexpr int WN = CONSUMER_WARPS / WM;
  static constexpr int ACTIVE = WM * WN;  // consumer warps with a warp tile
  static constexpr int BMT = 16 * MT * WM, BNT = 32 * WN;
  static constexpr int AV = BMT * FK, BV = BNT * FK;
};
constexpr int FUSED_PRODUCER_WARPS = 4;  // one warpgroup (setmaxnreg is warpgroup-wide); warp 0 of it issues
constexpr int FUSED_THREADS = 32 * (CONSUMER_WARPS + FUSED_PRODUCER_WARPS);
// setmaxnreg budget: the CTA launches with 168 regs x 384 threads; the consumers'
// increase (8 warps x 64) must be covered by what the producer warpgroup releases
// (4 warps x (168 - 40)) or setmaxnreg.inc waits forever -- 40 is the ceiling.
constexpr int FUSED_CONSUMER_REGS = 232;
constexpr int FUSED_PRODUCER_REGS = 40;
static_assert(CONSUMER_WARPS * (FUSED_CONSUMER_REGS - 168) <= FUSED_PRODUCER_WARPS * (168 - FUSED_PRODUCER_REGS),
              "setmaxnreg: consumer increase exceeds the producer release");
constexpr int MAX_FUSED_STAGES = 8;
// Summing warpgroup (GemmArgs::psum != 0, L >= 1): a fourth warpgroup forms
// Strassen operand sums once per CTA, in place in the raw chunk stage (the sum
// of a side's views overwrites its first view), before the consumers read the
// stage.  psum bit 0: the A side (shared by the four warps along N, whose
// fragment-load sums would repeat it 4x); bit 1: the B side too (else the
// consumers sum B in their fragment loads, 2x).  512 threads launch at 128
// registers: consumers 8 warps x 208 + producer warpgroup 4 x 40 + summing
// warpgroup 4 x 56 = 65536.
constexpr int SUM_WARPS = 4;
constexpr int FUSED_THREADS_PS = FUSED_THREADS + 32 * SUM_WARPS;
constexpr int PS_CONSUMER_REGS = 208;
constexpr int PS_SUM_REGS = 56;  // 40 (for 216-register consumers) measured slower: the summers pace the consumers
static_assert(CONSUMER_WARPS * (PS_CONSUMER_REGS - 128) <=
                  FUSED_PRODUCER_WARPS * (128 - FUSED_PRODUCER_REGS) + SUM_WARPS * (128 - PS_SUM_REGS),
              "setmaxnreg: consumer increase exceeds the producer + summer release");

// smem (fixed offsets up front, so the hot loops address the barriers without
// registers): full[8], empty[8], summed[8], epi_full[EPI_BUFS], epi_empty[EPI_BUFS] |
// stage_item[8], epi_item[EPI_BUFS] | epilogue offset tables rows[128], cols[128] (int64) |
// stages [S][sd doubles: na A views of AV, then nb B views of BV] (1024-byte aligned:
// swizzled TMA boxes) | (cred) M pieces [2][16][128]
constexpr int RED_ROWS = 16;                          // rows of one TMA-reduce piece (double-buffered)
constexpr size_t RED_BYTES = 2 * (size_t)RED_ROWS * BN * 8;
#ifndef STC_LAYOUT_TAIL
#define STC_LAYOUT_TAIL 1
#endif
struct FusedLayout {
#if STC_LAYOUT_TAIL
  // stages at 0, then the M pieces, then barriers / meta / tables
  static constexpr size_t kStages = 0;
  __host__ __device__ static size_t red_off(size_t sd, int stages) { return (size_t)stages * sd * 8; }
  __host__ __device__ static size_t bar_off(size_t sd, int stages, bool red) {
    return red_off(sd, stages) + (red ? RED_BYTES : 0);
  }
  __host__ __device__ static size_t meta_off(size_t sd, int stages, bool red) {
    return bar_off(sd, stages, red) + 8 * (3 * MAX_FUSED_STAGES + 2 * EPI_BUFS);
  }
  __host__ __device__ static size_t tab_off(size_t sd, int stages, bool red) {
    return (meta_off(sd, stages, red) + 4 * (MAX_FUSED_STAGES + EPI_BUFS) + 15) / 16 * 16;
  }
  __host__ __device__ static size_t bytes(size_t sd, int stages, bool red) { return tab_off(sd, stages, red) + 2 * 128 * 8; }
#else
  static constexpr size_t kBars = 0, kMeta = 256, kEpiTab = 512, kStages = 3072;
  static_assert(8 * (3 * MAX_FUSED_STAGES + 2 * EPI_BUFS) <= kMeta, "barriers");
  static_assert(kMeta + 4 * (MAX_FUSED_STAGES + EPI_BUFS) <= kEpiTab, "meta");
  static_assert(kEpiTab + 2 * 128 * 8 <= kStages && kStages % 1024 == 0, "tables");
  __host__ __device__ static size_t red_off(size_t sd, int stages) { return kStages + (size_t)stages * sd * 8; }
  __host__ __device__ static size_t bar_off(size_t, int, bool) { return kBars; }
  __host__ __device__ static size_t meta_off(size_t, int, bool) { return kMeta; }
  __host__ __device__ static size_t tab_off(size_t, int, bool) { return kEpiTab; }
  __host__ __device__ static size_t bytes(size_t sd, int stages, bool red) {
    return red_off(sd, stages) + (red ? RED_BYTES : 0);
  }
#endif
};

constexpr int EPI_WARPS = FUSED_PRODUCER_WARPS - 1;  // the producer warpgroup's other warps
constexpr int EPI_THREADS = 32 * EPI_WARPS;
constexpr size_t TILE_DOUBLES = (size_t)BM * BN;

constexpr size_t kFusedMaxSmem = 227 * 1024;

// Stages of the fused ring for stages of `sd` doubles (0: does not fit).
int fused_stages(size_t sd) {
  int s = MAX_FUSED_STAGES;
  while (s >= 2 && FusedLayout::bytes(sd, s, false) > kFusedMaxSmem) --s;
  return s >= 2 ? s : 0;
}

// Stages when the TMA-reduce epilogue's M piece also lives in smem.
int fused_stages_red(size_t sd) {
  int s = MAX_FUSED_STAGES;
  while (s >= 2 && FusedLayout::bytes(sd, s, true) > kFusedMaxSmem) --s;
  return s >= 2 ? s : 0;
}

// Doubles per stage for terms of at most max_ops views per side, tile shape ts.
size_t fused_stage_doubles(int max_ops, int ts) { return fused_stage_doubles2(max_ops, max_ops, ts); }

// ... with va A views and vb B views per chunk (one-sided pre-summed slots)
size_t fused_stage_doubles2(int va, int vb, int ts) {
  const int av = ts == 1 ? Shape<1>::AV : ts == 2 ? Shape<2>::AV : ts == 3 ? Shape<3>::AV : ts == 4 ? Shape<4>::AV
                                                                                           : Shape<0>::AV;
  const int bv = ts == 1 ? Shape<1>::BV : ts == 2 ? Shape<2>::BV : ts == 3 ? Shape<3>::BV : ts == 4 ? Shape<4>::BV
                                                                                           : Shape<0>::BV;
  return (size_t)va * av + (size_t)vb * bv;
}

// Element offset of (x, k) inside a raw view.
__host__ __device__ __forceinline__ int view_index(int kfast, int x, int k) {
  if (!kfast) return (k + 8 * (x >> 4)) * 16 + ((((x & 15) >> 1) ^ k) << 1) + (x & 1);
  return x * 8 + ((((k >> 1) ^ (x >> 1)) & 3) << 1) + (k & 1);
}

__device__ __forceinline__ void mbar_expect_tx_f(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_box_f(void *dst, const CUtensorMap *map, int rank, const int32_t (&c)[5],
                                          uint64_t *bar) {
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(b)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
          : "memory");
      break;
  }
}

__device__ __forceinline__ int coord_of(const int4 &v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Sum of the views [v0, v0 + n) of one side at the element offsets `off[i]`
// (I values), in view order: acc = s0 * V0; acc = acc +/- V_v.  The reference's
// leading 0.0 + (_jit.py:43-65) only turns an operand -0.0 into +0.0, which
// cannot change C: the DMMA accumulators start at +0.0, and adding a zero
// product of either sign to them gives the same result.
__device__ __forceinline__ double flip_sign(double v) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>(0x80000000u), __double2loint(v));
}

template <int I>
__device__ __forceinline__ void side_sum(double (&out)[I], const double *st, int v0, int n, uint32_t negmask,
                                         const int (&off)[I]) {
  {
    const double *src = st + v0 * VIEW_DOUBLES;
#pragma unroll
    for (int i = 0; i < I; ++i) out[i] = src[off[i]];
    if ((negmask >> v0) & 1u) {
#pragma unroll
      for (int i = 0; i < I; ++i) out[i] = flip_sign(out[i]);
    }
  }
  for (int v = 1; v < n; ++v) {
    const double *src = st + (v0 + v) * VIEW_DOUBLES;
    double t[I];
#pragma unroll
    for (int i = 0; i < I; ++i) t[i] = src[off[i]];
    if ((negmask >> (v0 + v)) & 1u) {
#pragma unroll
      for (int i = 0; i < I; ++i) out[i] = __dsub_rn(out[i], t[i]);
    } else {
#pragma unroll
      for (int i = 0; i < I; ++i) out[i] = __dadd_rn(out[i], t[i]);
    }
  }
}


// One view step of the consumer pipeline (V: view index, KN: k-step of the
// fragments being built; compile-time): load view V of the next k-step and
// fold it into the next step's fragments (sign flip for the side's first view,
// DADD of the signed value otherwise -- the reference's view order), then issue
// MMA group V of the current k-step.  Loads go in groups of four values to keep
// the register footprint inside the consumers' budget.
template <int NA, int NB, int V, int KN, bool MMA, bool SGN = true, int AV = VIEW_DOUBLES, int BV = VIEW_DOUBLES,
          int MT = 4>
__device__ __forceinline__ void pipe_view(double (&acc)[4][4][4], const double (&fa)[8], const double (&fb)[4],
                                          double (&xa)[8], double (&xb)[4], const double *nst, bool load,
                                          const int (&offA)[2][2], const int (&offB)[2][2], uint32_t negmask,
                                          int bbase) {
  constexpr int G = NA + NB;
  const int fl = static_cast<int>(((negmask >> V) & 1u) << 31);
  const double sgn = __hiloint2double(0x3ff00000 | fl, 0);  // +/-1.0
  // A view V at V * AV; B view V - NA at bbase + (V - NA) * BV (bbase: the stage's B views)
  const double *src = AV == BV ? nst + V * AV + (V >= NA ? bbase - NA * AV : 0)
                               : (V < NA ? nst + V * AV : nst + bbase + (V - NA) * BV);
  // one address per fragment column / row pair; the mt / nt blocks are immediates
  const double *pa0 = src + offA[KN][0], *pa1 = src + offA[KN][1];
  const double *pb0 = src + offB[KN][0], *pb1 = src + offB[KN][1];
  if (load) {
    if constexpr (V < NA) {
#pragma unroll
      for (int hh = 0; hh < MT / 2; ++hh) {  // mt pairs {0, 1}, {2, 3}
        double t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = (j & 1 ? pa1 : pa0)[128 * (2 * hh + (j >> 1))];  // immediate offsets
        if (V == 0 && !SGN) {  // summed tile: the signs are already applied
#pragma unroll
          for (int j = 0; j < 4; ++j) xa[4 * hh + j] = t[j];
        } else if (V == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) xa[4 * hh + j] = __hiloint2double(__double2hiint(t[j]) ^ fl, __double2loint(t[j]));
        } else {  // acc + (+/-1) * v: one exactly rounded add, no integer sign flip on the way
#pragma unroll
          for (int j = 0; j < 4; ++j) xa[4 * hh + j] = __fma_rn(sgn, t[j], xa[4 * hh + j]);
        }
      }
    } else if (STC_BSUM_BATCH && NB > 1 && SGN) {
      // all B views of the k-step loaded first, then one run of DFMAs (one FP64 pipe switch)
      if constexpr (V == NA) {
        double t[NB][4];
#pragma unroll
        for (int w = 0; w < NB; ++w)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) t[w][nt] = ((nt & 1 ? pb1 : pb0) + w * BV)[128 * (nt >> 1)];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) xb[nt] = __hiloint2double(__double2hiint(t[0][nt]) ^ fl, __double2loint(t[0][nt]));
#pragma unroll
        for (int w = 1; w < NB; ++w) {
          const double sw = __hiloint2double(0x3ff00000 | static_cast<int>(((negmask >> (V + w)) & 1u) << 31), 0);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) xb[nt] = __fma_rn(sw, t[w][nt], xb[nt]);
        }
      }
    } else {
      double t[4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) t[nt] = (nt & 1 ? pb1 : pb0)[128 * (nt >> 1)];
      if (V == NA && !SGN) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) xb[nt] = t[nt];
      } else if (V == NA) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) xb[nt] = __hiloint2double(__double2hiint(t[nt]) ^ fl, __double2loint(t[nt]));
      } else {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) xb[nt] = __fma_rn(sgn, t[nt], xb[nt]);
      }
    }
  }
  if constexpr (MMA) {
#pragma unroll
    for (int i = 4 * MT * V / G; i < 4 * MT * (V + 1) / G; ++i)
      dmma_16x8x4(acc[i >> 2][i & 3], fa[2 * (i >> 2)], fa[2 * (i >> 2) + 1], fb[i & 3]);
  }
  if constexpr (V + 1 < G)
    pipe_view<NA, NB, V + 1, KN, MMA, SGN, AV, BV, MT>(acc, fa, fb, xa, xb, nst, load, offA, offB, negmask, bbase);
}

// One work item's main loop for terms with NA A-views and NB B-views
// (compile-time): a software pipeline over the item's 4-deep k-steps (two per
// 8-deep chunk, fragments ping-ponging between two register sets).  While the
// 16 MMAs of one k-step issue in NA + NB groups, the fragments of the next
// k-step are built one view per group, so no DADD waits on a result it needs
// right away behind the DMMAs queued on the shared FP64 pipe.  A chunk stage
// is released as soon as both of its k-steps are in registers.
template <int NA, int NB, bool SGN = true, int AV = VIEW_DOUBLES, int BV = VIEW_DOUBLES, int MT = 4, bool LATE = false>
__device__ __forceinline__ void consume_item(double (&acc)[4][4][4], const double *stages, int sstride, int S,
                                             uint64_t *full, uint64_t *empty, int &stage, uint32_t &phase, int kchunks,
                                             uint32_t negmask, const int (&offA_)[2][2], const int (&offB_)[2][2],
                                             int lane, int bbase = NA * AV) {
  // Keep the fragment offsets in registers through opaque copies: otherwise
  // ptxas rematerialises them from %tid (S2R, a long-latency special-register
  // read, plus the swizzle arithmetic) inside the hot loop.
  int oA[2][2] = {{offA_[0][0], offA_[0][1]}, {offA_[1][0], offA_[1][1]}};
  int oB[2][2] = {{offB_[0][0], offB_[0][1]}, {offB_[1][0], offB_[1][1]}};
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      asm volatile("mov.b32 %0, %0;" : "+r"(oA[i][j]));
      asm volatile("mov.b32 %0, %0;" : "+r"(oB[i][j]));
    }
  const int (&offA)[2][2] = oA;
  const int (&offB)[2][2] = oB;
  double fa[8], fb[4], xa[8], xb[4];
  // stage (bits 0-15) and phase (bit 16) in one register through the loop: kept apart,
  // ptxas spilled the phase (a local load + store per chunk next to the DMMAs)
  uint32_t sp = (uint32_t)stage | (phase << 16);
  pipe_view<NA, NB, 0, 0, false, SGN, AV, BV, MT>(acc, fa, fb, fa, fb, stages + stage * sstride, true, offA, offB, negmask,
                                              bbase);
  // Stage release.  LATE (one view per side: 8 stages): once the MMAs of the stage's
  // second k-step have issued -- they read the fragment registers, so every load from the
  // stage has completed before the producer's TMA (async proxy) refills it.  Otherwise
  // (3-4 stages of several views, where the later release shortens the ring too much:
  // cfg3 2^24 N_a = 256 L2 4.14 -> 4.41 ms) right after the second k-step's loads issue,
  // behind a fence.proxy.async (without the fence the refill raced with loads still in
  // flight: wrong 64-row blocks on cfg4 L0 about one run in four, round 1).  The fence
  // costs 1-1.5 % (16384^3 L2: 195.1 vs 192.2 ms).
  constexpr bool late = LATE;
  for (int c = 0; c < kchunks; ++c) {
    // k-step 0 of chunk c (fa, fb) -> build k-step 1 of chunk c (xa, xb)
    pipe_view<NA, NB, 0, 1, true, SGN, AV, BV, MT>(acc, fa, fb, xa, xb, stages + (int)(sp & 0xffffu) * sstride, true,
                                               offA, offB, negmask, bbase);
    const uint32_t done_stage = sp & 0xffffu;
    if constexpr (!late) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[done_stage]);
    }
    ++sp;
    if ((sp & 0xffffu) == (uint32_t)S) sp = (sp & 0x10000u) ^ 0x10000u;  // stage 0, phase flipped
    // k-step 1 of chunk c (xa, xb) -> build k-step 0 of chunk c + 1 (fa, fb)
    const bool more = c + 1 < kchunks;
    if (more) mbar_wait(&full[sp & 0xffffu], sp >> 16);
    pipe_view<NA, NB, 0, 0, true, SGN, AV, BV, MT>(acc, xa, xb, fa, fb, stages + (int)(sp & 0xffffu) * sstride, more,
                                               offA, offB, negmask, bbase);
    if constexpr (late) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[done_stage]);
    }
  }
  stage = (int)(sp & 0xffffu);
  phase = sp >> 16;
}

// TMA-reduce epilogue (ABC, C targets regular): for each C target in ticket
// order, the tile's sign * M goes through a 32 x 128 smem piece (128-byte
// swizzled, the C map's box) and cp.reduce.async.bulk.tensor adds it into C in
// L2.  C_new = C_old + (+/-M) is one IEEE add per element, as in
// epilogue_store, and tickets keep the reference's term order: C is bitwise
// the same.  No C data passes through the SM.
__device__ __forceinline__ int red_index(int r, int c) {
  return r * BN + (c >> 4) * 16 + ((((c & 15) >> 1) ^ (c >> 4)) << 1) + (c & 1);
}
// The 8-wide variant (GemmArgs::cred8): box [r][c / 8][c % 8], 64-byte lines, 64B
// swizzle (16-byte granule index XOR bits 7-8 of the byte offset).
__device__ __forceinline__ int red_index8(int r, int c) {
  const int line = r * (BN / 8) + (c >> 3);
  return line * 8 + ((((c & 7) >> 1) ^ ((line >> 1) & 3)) << 1) + (c & 1);
}
template <bool W8>
__device__ __forceinline__ int red_idx(int r, int c) { return W8 ? red_index8(r, c) : red_index(r, c); }

__device__ __forceinline__ void tma_reduce_add(const CUtensorMap *map, int rank, const int32_t (&c)[5], const void *src) {
  const uint32_t sa = smem_u32(src);
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m),
                   "r"(c[0]), "r"(c[1]), "r"(sa)
                   : "memory");
      break;
    case 3:
      asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(sa)
                   : "memory");
      break;
    case 4:
      asm volatile(
          "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(sa)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.reduce.async.bulk.tensor.5d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sa)
          : "memory");
      break;
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int PA, int PB, bool W8>
__device__ __forceinline__ void epilogue_red(const GemmArgs &p, const double (&acc)[4][4][4], int item, int tid, int wm,
                                             int wn, int g, int tig, double *buf, const CUtensorMap *tmC) {
  int slot, ti, tj, pos;
  tile_of(p, item, slot, ti, tj, pos);
  const TermDesc td = p.terms[slot];
  int nb = 0;  // piece buffer
  for (int j = 0; j < td.c_count; ++j) {
    const TgtDesc tg = p.tgts[td.c_first + j];
    if (p.use_tickets) {
      if (tid == 0)
        while (ld_acquire_gpu(p.tickets + tg.ticket_base + pos) < tg.order) __nanosleep(64);
    }
    // pieces of 16 tile rows (= one mt block of the warps with wm = pc / 4), two
    // buffers: the writes of piece pc overlap the TMA read of piece pc - 1
    for (int pc = 0; pc < BM / RED_ROWS; ++pc) {
      double *pb = buf + (size_t)nb * RED_ROWS * BN;
      if (wm == (pc >> 2)) {
        const int mt = pc & 3;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = epi_row<PA>(mt, h, g) - RED_ROWS * mt;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            const int c = wn * 32 + epi_col<PB>(nt, tig);
            *reinterpret_cast<double2 *>(pb + red_idx<W8>(r, c)) =
                make_double2(tg.sign * acc[mt][nt][2 * h], tg.sign * acc[mt][nt][2 * h + 1]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
      }
      named_bar(2, 32 * CONSUMER_WARPS);
      if (tid == 0) {
        const int4 rc = p.coords[(tg.row_start + (int64_t)ti * BM + RED_ROWS * pc) >> 3];
        const int4 cc = p.coords[(tg.col_start + (int64_t)tj * BN) >> 3];
        int32_t c5[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const int src = p.tm_src[2][d];
          c5[d] = src < 4 ? coord_of(rc, src) : coord_of(cc, src - 4);
        }
        tma_reduce_add(tmC, p.tm_rank[2], c5, pb);
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the other buffer is reusable
      }
      named_bar(2, 32 * CONSUMER_WARPS);
      nb ^= 1;
    }
    if (tid == 0) {  // this target's adds performed: hand the tile to the next term at once
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      if (p.use_tickets) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        st_release_gpu(p.tickets + tg.ticket_base + pos, tg.order + 1);
      }
    }
  }
}

// Epilogue warps (the producer warpgroup's three other warps; ABC, opt-in with
// STC_EPI_OFFLOAD=1): for each item's dense M tile in this CTA's scratch
// buffer, add sign * M into every C target through the scatter layout --
// ticket-ordered across terms exactly as epilogue_store does, so C is bitwise
// the same -- while the consumers run the next item's MMAs.
__device__ __forceinline__ void epilogue_warps(const GemmArgs &p, uint64_t *epi_full, uint64_t *epi_empty,
                                               const int *epi_item, int64_t *rows, int64_t *cols, int t) {
  int eb = 0;
  uint32_t ephase = 0;
  const int lane = t & 31;
  bool c_seen = false;
  for (;;) {
    mbar_wait_parked(&epi_full[eb], ephase);
    const int item = epi_item[eb];
    if (item < 0) break;
    if (p.c_ready && !c_seen) {  // stc_set_c_ready
      if (t == 0)
        while (ld_acquire_gpu(p.c_ready) == 0) __nanosleep(256);
      named_bar(3, EPI_THREADS);
      c_seen = true;
    }
    int slot, ti, tj, pos;
    tile_of(p, item, slot, ti, tj, pos);
    const TermDesc td = p.terms[slot];
    const double *Mt = p.mscratch + ((size_t)blockIdx.x * EPI_BUFS + eb) * TILE_DOUBLES;
    for (int j = 0; j < td.c_count; ++j) {
      const TgtDesc tg = p.tgts[td.c_first + j];
      for (int i = t; i < 128; i += EPI_THREADS) {
        rows[i] = __ldcg(p.pool + tg.row_start + ti * BM + i);
        cols[i] = __ldcg(p.pool + tg.col_start + tj * BN + i);
      }
      int32_t *ticket = p.tickets + tg.ticket_base + pos;
      if (p.use_tickets) {
        if (t == 0)
          while (ld_acquire_gpu(ticket) < tg.order) __nanosleep(64);
      }
      named_bar(3, EPI_THREADS);
      // one warp per row pair at a time, lanes along columns (4 columns per lane);
      // all loads of the pair are issued before any store
      int64_t co[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) co[q] = cols[lane + 32 * q];
      for (int r0 = 2 * (t >> 5); r0 < BM; r0 += 2 * EPI_WARPS) {
        int64_t ro[2];
        double m[2][4], c[2][4];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          ro[rr] = rows[r0 + rr];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool ok = ro[rr] != kPad && co[q] != kPad;
            m[rr][q] = Mt[(size_t)(r0 + rr) * BN + lane + 32 * q];
            c[rr][q] = ok ? __ldcg(p.C + ro[rr] + co[q]) : 0.0;
          }
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (ro[rr] != kPad && co[q] != kPad) __stcg(p.C + ro[rr] + co[q], c[rr][q] + tg.sign * m[rr][q]);
      }
      if (p.use_tickets) {
        __threadfence();
        named_bar(3, EPI_THREADS);
        if (t == 0) st_release_gpu(ticket, tg.order + 1);
      }
      named_bar(3, EPI_THREADS);  // offset tables reused by the next target
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&epi_empty[eb]);
    if (++eb == EPI_BUFS) {
      eb = 0;
      ephase ^= 1;
    }
  }
}

// Epilogue warps with TMA reduce-add (ABC, C targets regular; the default when
// both apply): per item, the dense M tile in this CTA's scratch buffer is
// streamed through the 16-row swizzled smem pieces (sign applied by an integer
// sign-bit flip -- no FP64 work competing with the consumers' DMMAs) and added
// into each C target in L2 by cp.reduce.async.bulk.tensor, in ticket order.
// The consumers only write M and go on with the next item.
template <bool W8>
__device__ __forceinline__ void epilogue_warps_red(const GemmArgs &p, uint64_t *epi_full, uint64_t *epi_empty,
                                                   const int *epi_item, double *buf, const CUtensorMap *tmC, int t) {
  int eb = 0;
  uint32_t ephase = 0;
  const int lane = t & 31;
  bool c_seen = false;
  for (;;) {
    mbar_wait_parked(&epi_full[eb], ephase);
    const int item = epi_item[eb];
    if (item < 0) break;
    if (p.c_ready && !c_seen) {  // stc_set_c_ready
      if (t == 0)
        while (ld_acquire_gpu(p.c_ready) == 0) __nanosleep(256);
      c_seen = true;
    }
    int slot, ti, tj, pos;
    tile_of(p, item, slot, ti, tj, pos);
    const TermDesc td = p.terms[slot];
    const double *Mt = p.mscratch + ((size_t)blockIdx.x * EPI_BUFS + eb) * TILE_DOUBLES;
    int nb = 0;
    for (int j = 0; j < td.c_count; ++j) {
      const TgtDesc tg = p.tgts[td.c_first + j];
      const uint32_t flip = __double_as_longlong(tg.sign) < 0 ? 0x80000000u : 0u;
      if (t == 0 && p.use_tickets)
        while (ld_acquire_gpu(p.tickets + tg.ticket_base + pos) < tg.order) __nanosleep(64);
      int4 cc = make_int4(0, 0, 0, 0);
      if (t == 0) cc = p.coords[(tg.col_start + (int64_t)tj * BN) >> 3];
      for (int pc = 0; pc < BM / RED_ROWS; ++pc) {
        double *pb = buf + (size_t)nb * RED_ROWS * BN;
        if (t == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // pb's previous read done
        named_bar(3, EPI_THREADS);
        // 16 rows x 128 columns: 1024 double2, ~11 per thread, row-major reads of M
        for (int e = t; e < RED_ROWS * BN / 2; e += EPI_THREADS) {
          const int r = e / (BN / 2), c = 2 * (e - r * (BN / 2));
          double2 v = *reinterpret_cast<const double2 *>(Mt + (size_t)(RED_ROWS * pc + r) * BN + c);
          v.x = __hiloint2double(__double2hiint(v.x) ^ (int)flip, __double2loint(v.x));
          v.y = __hiloint2double(__double2hiint(v.y) ^ (int)flip, __double2loint(v.y));
          *reinterpret_cast<double2 *>(pb + red_idx<W8>(r, c)) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar(3, EPI_THREADS);
        if (t == 0) {
          const int4 rc = p.coords[(tg.row_start + (int64_t)ti * BM + RED_ROWS * pc) >> 3];
          int32_t c5[5];
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            const int src = p.tm_src[2][d];
            c5[d] = src < 4 ? coord_of(rc, src) : coord_of(cc, src - 4);
          }
          tma_reduce_add(tmC, p.tm_rank[2], c5, pb);
        }
        nb ^= 1;
      }
      if (t == 0) {  // this target's adds performed: hand the tile to the next term
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (p.use_tickets) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          st_release_gpu(p.tickets + tg.ticket_base + pos, tg.order + 1);
        }
      }
    }
    named_bar(3, EPI_THREADS);  // every warp is done with this M buffer
    if (lane == 0) mbar_arrive(&epi_empty[eb]);
    if (++eb == EPI_BUFS) {
      eb = 0;
      ephase ^= 1;
    }
  }
}

// One side of one k-chunk, summed in place by the summing warpgroup: view v0
// becomes s0 * V_v0 +/- V_v0+1 ... in view order (sign flip of the first view,
// one DADD / DSUB per later view: the roundings of the consumers' fragment-load
// sums and of the reference's packing, _jit.py:43-65).  All views share the
// swizzled layout, so thread t owns the double2 elements t, t + 128, ... of
// every view of the side.
template <int VD>
__device__ __forceinline__ void sum_side(double2 *__restrict__ st, int v0, int n, uint32_t negmask, int t) {
  constexpr int VD2 = VD / 2;
  // at most 4 double2 per thread at a time (the summing warps' 56 registers)
  constexpr int PER = VD2 / (32 * SUM_WARPS) < 4 ? VD2 / (32 * SUM_WARPS) : 4;
  constexpr int STEP = 32 * SUM_WARPS * PER;
  const int fl = static_cast<int>(((negmask >> v0) & 1u) << 31);
#pragma unroll 1
  for (int base = 0; base < VD2; base += STEP) {
    double2 a[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const double2 v = st[v0 * VD2 + base + t + 32 * SUM_WARPS * i];
      a[i].x = __hiloint2double(__double2hiint(v.x) ^ fl, __double2loint(v.x));
      a[i].y = __hiloint2double(__double2hiint(v.y) ^ fl, __double2loint(v.y));
    }
    for (int v = v0 + 1; v < v0 + n; ++v) {
      double2 b[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) b[i] = st[v * VD2 + base + t + 32 * SUM_WARPS * i];
      if ((negmask >> v) & 1u) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          a[i].x = __dsub_rn(a[i].x, b[i].x);
          a[i].y = __dsub_rn(a[i].y, b[i].y);
        }
      } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          a[i].x = __dadd_rn(a[i].x, b[i].x);
          a[i].y = __dadd_rn(a[i].y, b[i].y);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) st[v0 * VD2 + base + t + 32 * SUM_WARPS * i] = a[i];
  }
}

// Summing warpgroup: per chunk stage (after the TMA loads land), sum the A side
// (and with psum bit 1 the B side) in place, then release the stage to the
// consumers (summed[stage]).  Each element is summed once per CTA -- the
// consumers' fragment-load sums repeat A 4x and B 2x across the warps sharing
// the fragments -- and the summers' waits for the FP64 unit, which the DMMAs
// occupy, never hold up a DMMA issue.
template <int TS>
__device__ __forceinline__ void summer_warps(const GemmArgs &p, double *stages, int sstride, int S, uint64_t *full,
                                             uint64_t *summed, const int *stage_item, int t) {
  using SH = Shape<TS>;
  const int lane = t & 31;
  const bool sum_b = (p.psum & 2) != 0;
  int rs = 0;
  uint32_t rph = 0;
  int cur = -1, na = 0, nb = 0;
  uint32_t negmask = 0;
  bool do_a = false, do_b = false;
  for (;;) {
    mbar_wait(&full[rs], rph);
    const int item = stage_item[rs];
    if (item >= 0) {
      if (item != cur) {
        cur = item;
        int slot, ti, tj;
        tile_of(p, item, slot, ti, tj);
        const TermDesc td = p.terms[slot];
        na = td.a_count;
        nb = td.b_count;
        bool neg = false;
        if (lane < na + nb)
          neg = __double_as_longlong(p.ops[lane < na ? td.a_first + lane : td.b_first + lane - na].sign) < 0;
        negmask = __ballot_sync(0xffffffffu, neg);
        do_a = na > 1 || (negmask & 1u);
        do_b = sum_b && (nb > 1 || ((negmask >> na) & 1u));
      }
      double *st = stages + (size_t)rs * sstride;
      if (do_a) sum_side<SH::AV>(reinterpret_cast<double2 *>(st), 0, na, negmask, t);
      if constexpr (TS == 0)  // shapes 1, 2 run with psum = 1
        if (do_b) sum_side<SH::BV>(reinterpret_cast<double2 *>(st + na * SH::AV), 0, nb, negmask >> na, t);
      // generic writes before the async proxy (TMA) refills this stage
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&summed[rs]);
    if (item < 0) break;
    if (++rs == S) {
      rs = 0;
      rph ^= 1;
    }
  }
}

// A consumer warp whose 64 x 32 tile lies wholly in the quadrant's tile padding
// (rows past p.rows_valid or columns past p.cols_valid: PAD, never stored) keeps
// the stage protocol of consume_item but issues no loads or MMAs, so the other
// warps of its SM sub-partition get the DMMA pipe (m or n = 64 per quadrant:
// half of every tile is padding).
__device__ __forceinline__ void skip_item(int S, uint64_t *full, uint64_t *empty, int &stage, uint32_t &phase,
                                          int kchunks, int lane) {
  for (int c = 0; c < kchunks; ++c) {
    if (c > 0) mbar_wait(&full[stage], phase);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// PS: a summing warpgroup forms (some of) the operand sums in place (p.psum);
// otherwise the consumers form them all in their fragment loads.
// TS: CTA tile shape (Shape<TS>; 1 and 2 only with PS and dense M output).
// ONE: every term has one view per side with sign +1 (pre-summed operand slots,
// Naive's packed sums): the consumers only run consume_item<1, 1> -- without the
// other view-count specialisations in the kernel, the consumers need no spills.
template <int AKF, int BKF, bool PS, int TS, bool ONE = false>
__global__ void __launch_bounds__(PS ? FUSED_THREADS_PS : FUSED_THREADS, 1)
    k_strassen_fused(const GemmArgs p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC) {
  using SH = Shape<TS>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int S = p.stages;
  const int sstride = p.stage_dbl;  // doubles per stage
  const bool red = p.cred != 0;
  double *stages = reinterpret_cast<double *>(smem + FusedLayout::kStages);
  double *redbuf = reinterpret_cast<double *>(smem + FusedLayout::red_off(sstride, S));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + FusedLayout::bar_off(sstride, S, red));
  uint64_t *empty = full + MAX_FUSED_STAGES;
  uint64_t *summed = empty + MAX_FUSED_STAGES;  // PS: the stage's sums are formed (the consumers' full barrier)
  uint64_t *epi_full = summed + MAX_FUSED_STAGES;  // M tile b written by the consumers (ABC: C updates offloaded)
  uint64_t *epi_empty = epi_full + EPI_BUFS;
  int *stage_item = reinterpret_cast<int *>(smem + FusedLayout::meta_off(sstride, S, red));
  int *epi_item = stage_item + MAX_FUSED_STAGES;
  int64_t *epi_rows = reinterpret_cast<int64_t *>(smem + FusedLayout::tab_off(sstride, S, red));
  int64_t *epi_cols = epi_rows + 128;
  const bool offload = p.mscratch != nullptr;  // ABC: epilogue warps update C from the M tiles
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
      mbar_init(&summed[s], SUM_WARPS);
    }
    for (int b = 0; b < EPI_BUFS; ++b) {
      mbar_init(&epi_full[b], CONSUMER_WARPS);
      mbar_init(&epi_empty[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the previous kernel's slots / tables / C complete (PDL launch)
  pdl_launch_dependents();
  const int kchunks = p.kchunks;  // 8-deep chunks

  if (PS && warp >= CONSUMER_WARPS + FUSED_PRODUCER_WARPS) {
    // ===================== summing warpgroup (PS) ======================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PS_SUM_REGS));
    summer_warps<TS>(p, stages, sstride, S, full, summed, stage_item, tid - 32 * (CONSUMER_WARPS + FUSED_PRODUCER_WARPS));
  } else if (warp >= CONSUMER_WARPS) {
    // ===================== producer warp: TMA box loads ================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(FUSED_PRODUCER_REGS));
    if (warp != CONSUMER_WARPS) {
      if (offload && red)
        p.cred8 ? epilogue_warps_red<true>(p, epi_full, epi_empty, epi_item, redbuf, &tmC, tid - 32 * (CONSUMER_WARPS + 1))
                : epilogue_warps_red<false>(p, epi_full, epi_empty, epi_item, redbuf, &tmC, tid - 32 * (CONSUMER_WARPS + 1));
      else if (offload)
        epilogue_warps(p, epi_full, epi_empty, epi_item, epi_rows, epi_cols, tid - 32 * (CONSUMER_WARPS + 1));
      return;
    }
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      int item = 0;
      if (lane == 0) item = atomicAdd(p.counter, 1);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= p.total_items) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          stage_item[stage] = -1;
          mbar_arrive(&full[stage]);
        }
        break;
      }
      int slot, ti, tj;
      tile_of(p, item, slot, ti, tj);
      const TermDesc td = p.terms[slot];
      const int na = td.a_count, U = td.a_count + td.b_count;
      // lane u < U stages view u (A views first, then B views) of every chunk
      int sd = 0;
      int64_t kst = 0;
      int4 xc = make_int4(0, 0, 0, 0);
      if (lane < U) {
        sd = lane < na ? 0 : 1;
        const OpDesc o = p.ops[sd == 0 ? td.a_first + lane : td.b_first + lane - na];
        xc = p.coords[(o.x_start + (int64_t)(sd == 0 ? ti * SH::BMT : tj * SH::BNT)) >> 3];
        kst = o.k_start;
      }
      const CUtensorMap *map = sd == 0 ? &tmA : &tmB;
      const int rank = p.tm_rank[sd];
      int src[5];
#pragma unroll
      for (int d = 0; d < 5; ++d) src[d] = p.tm_src[sd][d];
      const uint32_t bytes = (uint32_t)(na * SH::AV + (U - na) * SH::BV) * 8;
      // stage layout: A view u at u * AV, B view w at na * AV + w * BV
      const size_t vofs = lane < na ? (size_t)lane * SH::AV : (size_t)na * SH::AV + (size_t)(lane - na) * SH::BV;
      for (int c = 0; c < kchunks; ++c) {
        int4 kc = make_int4(0, 0, 0, 0);
        if (lane < U) kc = p.coords[(kst + (int64_t)c * FK) >> 3];
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          stage_item[stage] = item;
          mbar_expect_tx_f(&full[stage], bytes);
        }
        __syncwarp();
        if (lane < U) {
          int32_t cc[5];
#pragma unroll
          for (int d = 0; d < 5; ++d) cc[d] = src[d] < 4 ? coord_of(xc, src[d]) : coord_of(kc, src[d] - 4);
          tma_box_f(stages + (size_t)stage * sstride + vofs, map, rank, cc, &full[stage]);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ===================== consumer warps: sums + DMMA + epilogue =====
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(PS ? PS_CONSUMER_REGS : FUSED_CONSUMER_REGS));
    const int g = lane >> 2, tig = lane & 3;
    // warp -> (wm, wn): the warps of one SM sub-partition (warp % 4) differ in wn by
    // default; with warp_map = 1 in wm, so the warps left when the wm = 1 row half of
    // a tile is padding (skip_item) still cover all four sub-partitions
    // shapes 1 / 2: warp = wn (WM = 1) or wm + 4 wn (WM = 4): all sub-partitions busy either way
    // shape 3: wm = warp / 4, wn = warp % 4: both row halves on every sub-partition
    const int wm = TS == 1 ? 0 : TS == 2 || TS == 4 ? warp & 3 : TS == 3 || p.warp_map ? warp >> 2 : warp & 1;
    const int wn = TS == 1 ? (warp & 7) : TS == 2 || TS == 4 ? warp >> 2 : TS == 3 || p.warp_map ? warp & 3 : warp >> 1;
    const bool idle_warp = warp >= SH::ACTIVE;
    // Fragment offsets inside a view: A (kk, h) + 128 * mt; B (kk, nt & 1) + 128 * (nt >> 1).
    // MMA row (column) g + 8 h of each 16-row block (16-column pair) reads tile row
    // (column) frag_perm(kind, g, h) (stc_common.cuh): with it every half-warp of a
    // fragment load touches 16 distinct 8-byte bank pairs in the swizzled view (the
    // identity would need twice the wavefronts); the epilogue maps rows / columns back.
    int offA[2][2], offB[2][2];
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        offA[kk][h] = view_index(AKF, wm * 16 * SH::MT + frag_perm(AKF + 1, g, h), kk * 4 + tig);
        offB[kk][h] = view_index(BKF, wn * 32 + frag_perm(BKF + 1, g, h), kk * 4 + tig);
      }
    int stage = 0;
    uint32_t phase = 0;
    int eb = 0;  // M scratch buffer (offloaded epilogue)
    uint32_t ephase = 0;
    bool c_seen = false;  // stc_set_c_ready flag observed
    double acc[4][4][4];
    // PS: a stage is ready for the consumers once its sums are formed
    uint64_t *cfull = PS ? summed : full;
    for (;;) {
      mbar_wait(&cfull[stage], phase);
      const int item = stage_item[stage];
      if (item < 0) {
        if (offload) {  // tell the epilogue warps to stop
          mbar_wait(&epi_empty[eb], ephase ^ 1);
          if (tid == 0) epi_item[eb] = -1;
          __syncwarp();
          if (lane == 0) mbar_arrive(&epi_full[eb]);
        }
        break;
      }
      int slot, ti, tj;
      tile_of(p, item, slot, ti, tj);
      const TermDesc td = p.terms[slot];
      const int na = td.a_count, nb = td.b_count;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
      const bool pad_tile = idle_warp || (p.rows_valid > 0 && ti * SH::BMT + wm * 16 * SH::MT >= p.rows_valid) ||
                            (p.cols_valid > 0 && tj * SH::BNT + wn * 32 >= p.cols_valid);
      if (pad_tile) {
        skip_item(S, cfull, empty, stage, phase, kchunks, lane);
      } else if constexpr (PS) {
        // the A sum sits in view slot 0 and the B views from na * AV on
        const int bbase = na * SH::AV;
        if (TS == 0 && (p.psum & 2)) {  // B summed too (first B view)
          consume_item<1, 1, false>(acc, stages, sstride, S, cfull, empty, stage, phase, kchunks, 0u, offA, offB, lane,
                                    bbase);
        } else {  // B views summed in the fragment loads: their signs at bits 1..nb
          bool neg = false;
          if (lane < nb) neg = __double_as_longlong(p.ops[td.b_first + lane].sign) < 0;
          const uint32_t negmask = __ballot_sync(0xffffffffu, neg) << 1;
          switch (nb) {
            case 1: consume_item<1, 1, true, SH::AV, SH::BV, SH::MT>(acc, stages, sstride, S, cfull, empty, stage, phase, kchunks, negmask, offA, offB, lane, bbase); break;
            case 2: consume_item<1, 2, true, SH::AV, SH::BV, SH::MT>(acc, stages, sstride, S, cfull, empty, stage, phase, kchunks, negmask, offA, offB, lane, bbase); break;
            default: consume_item<1, 4, true, SH::AV, SH::BV, SH::MT>(acc, stages, sstride, S, cfull, empty, stage, phase, kchunks, negmask, offA, offB, lane, bbase); break;
          }
        }
      } else if constexpr (ONE) {
        consume_item<1, 1, false, SH::AV, SH::BV, SH::MT, true>(acc, stages, sstride, S, full, empty, stage, phase,
                                                                kchunks, 0u, offA, offB, lane, SH::AV);
      } else {
      // coefficient signs of the item's views: one load per lane, one ballot
      bool neg = false;
      if (lane < na + nb) neg = __double_as_longlong(p.ops[lane < na ? td.a_first + lane : td.b_first + lane - na].sign) < 0;
      const uint32_t negmask = __ballot_sync(0xffffffffu, neg);
      switch (na * 8 + nb) {
        case 9: consume_item<1, 1>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 10: consume_item<1, 2>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 17: consume_item<2, 1>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 18: consume_item<2, 2>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 12: consume_item<1, 4>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 33: consume_item<4, 1>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 20: consume_item<2, 4>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 34: consume_item<4, 2>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        case 36: consume_item<4, 4>(acc, stages, sstride, S, full, empty, stage, phase, kchunks, negmask, offA, offB, lane); break;
        default:  // other view counts (not produced by the Strassen recursion)
          for (int kc = 0; kc < kchunks; ++kc) {
            if (kc > 0) mbar_wait(&full[stage], phase);
            const double *st = stages + (size_t)stage * sstride;
            double a[2][8], b[2][4];
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              int oa[8], ob[4];
#pragma unroll
              for (int mt = 0; mt < 4; ++mt) {
                oa[2 * mt] = offA[kk][0] + 128 * mt;
                oa[2 * mt + 1] = offA[kk][1] + 128 * mt;
              }
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) ob[nt] = offB[kk][nt & 1] + 128 * (nt >> 1);
              side_sum<8>(a[kk], st, 0, na, negmask, oa);
              side_sum<4>(b[kk], st, na, nb, negmask, ob);
            }
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
              for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                  dmma_16x8x4(acc[mt][nt], a[kk][2 * mt], a[kk][2 * mt + 1], b[kk][nt]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA refill
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          break;
      }
      }  // !PS
      if (TS == 0 && offload) {
        // dense M tile into this CTA's scratch buffer; the epilogue warps add it
        // into the C targets while the next item's MMAs run
        mbar_wait(&epi_empty[eb], ephase ^ 1);
        double *Mt = p.mscratch + ((size_t)blockIdx.x * EPI_BUFS + eb) * TILE_DOUBLES;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              *reinterpret_cast<double2 *>(Mt + (size_t)(wm * 64 + epi_row<AKF + 1>(mt, h, g)) * BN + wn * 32 +
                                           epi_col<BKF + 1>(nt, tig)) =
                  make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
        if (tid == 0) epi_item[eb] = item;
        __threadfence_block();
        __syncwarp();
        if (lane == 0) mbar_arrive(&epi_full[eb]);
        if (++eb == EPI_BUFS) {
          eb = 0;
          ephase ^= 1;
        }
        continue;
      }
      if constexpr (TS != 0) {  // shapes 1-3: dense M output only
        if (!idle_warp) epilogue_store<AKF + 1, BKF + 1, 2, SH::BMT, SH::BNT, SH::MT>(p, acc, item, tid, wm, wn, g, tig);
      } else {
        if (!p.dense_out) wait_c_ready(p, tid, c_seen);
        if (red)
          // (8-wide C boxes always go through the epilogue warps: launch_fused)
          epilogue_red<AKF + 1, BKF + 1, false>(p, acc, item, tid, wm, wn, g, tig, redbuf, &tmC);
        else
          epilogue_store<AKF + 1, BKF + 1, 2>(p, acc, item, tid, wm, wn, g, tig);
      }
    }
  }
}

using FusedKernel = void (*)(const GemmArgs, const CUtensorMap, const CUtensorMap, const CUtensorMap);

template <bool PS, int TS, bool ONE = false>
static FusedKernel fused_for_ts(int akf, int bkf) {
  if (akf) return bkf ? k_strassen_fused<1, 1, PS, TS, ONE> : k_strassen_fused<1, 0, PS, TS, ONE>;
  return bkf ? k_strassen_fused<0, 1, PS, TS, ONE> : k_strassen_fused<0, 0, PS, TS, ONE>;
}

static FusedKernel fused_for(int akf, int bkf, bool ps, int ts, bool one) {
  if (ps)
    return ts == 1 ? fused_for_ts<true, 1>(akf, bkf) : ts == 2 ? fused_for_ts<true, 2>(akf, bkf)
           : ts == 3 ? fused_for_ts<true, 3>(akf, bkf) : ts == 4 ? fused_for_ts<true, 4>(akf, bkf)
                                                     : fused_for_ts<true, 0>(akf, bkf);
  if (one)
    return ts == 1 ? fused_for_ts<false, 1, true>(akf, bkf) : ts == 2 ? fused_for_ts<false, 2, true>(akf, bkf)
           : ts == 3 ? fused_for_ts<false, 3, true>(akf, bkf) : ts == 4 ? fused_for_ts<false, 4, true>(akf, bkf)
                                                     : fused_for_ts<false, 0, true>(akf, bkf);
  return fused_for_ts<false, 0>(akf, bkf);
}

cudaError_t launch_fused(const GemmArgs &a, int grid, cudaStream_t s, const void *maps) {
  const bool ps = a.psum != 0;
  // one unsigned view per side (umax 2 with sign-free slots): the spill-free specialisation
  const bool one = !ps && a.umax == 2 && a.one_view;
  // shapes 1 / 2: dense M output, A sums by the summing warpgroup or one view per side
  if (a.tshape != 0 && (!(ps || one) || !a.dense_out || (a.psum & 2))) return cudaErrorInvalidValue;
  if (a.cred && a.cred8 && !a.mscratch) return cudaErrorInvalidValue;  // the consumers' inline TMA-reduce
                                                                      // epilogue has 16-wide boxes only
  const size_t sm = FusedLayout::bytes((size_t)a.stage_dbl, a.stages, a.cred != 0);
  FusedKernel k = fused_for(a.a_kfast, a.b_kfast, ps, a.tshape, one);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  CUtensorMap m[3];
  memcpy(m, maps, (a.cred ? 3 : 2) * sizeof(CUtensorMap));
  if (!a.cred) memset(&m[2], 0, sizeof(CUtensorMap));
  return launch_pdl(k, dim3(grid), dim3(ps ? FUSED_THREADS_PS : FUSED_THREADS), sm, s, a, m[0], m[1], m[2]);
}

// ---- coordinate table --------------------------------------------------------
// coords[i] = tensor-map coordinates (one part: x or k) of pool entry 8 i, for
// the pool ranges of the operand vectors: the producer warp reads one int4 per
// view and chunk instead of dividing.
__global__ void k_pool_coords(const int64_t *__restrict__ pool, int4 *__restrict__ coords, CoordJobs jobs) {
  for (int j = 0; j < jobs.n; ++j) {
    const CoordJob &jb = jobs.job[j];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < jb.count; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e = jb.start / 8 + i;
      const int64_t v = pool[e * 8];
      int32_t c[4] = {0, 0, 0, 0};
      if (v != kPad) {
        int64_t off = v - jb.base;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < jb.np) {
            const int64_t d = off / jb.str[q];
            c[q] = (int32_t)d;
            off -= d * jb.str[q];
          }
      }
      coords[e] = make_int4(c[0], c[1], c[2], c[3]);
    }
  }
}

cudaError_t launch_pool_coords(const int64_t *pool, int4 *coords, const CoordJobs &jobs, cudaStream_t s) {
  int64_t mx = 0;
  for (int j = 0; j < jobs.n; ++j) mx = std::max(mx, jobs.job[j].count);
  if (mx == 0) return cudaSuccess;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((mx + threads - 1) / threads, 148 * 8);
  k_pool_coords<<<blocks, threads, 0, s>>>(pool, coords, jobs);
  return cudaGetLastError();
}

}  // namespace stc
