// stc_gemm.cu -- the gather Strassen DMMA kernel (north-star subsystems 2 + 3):
// the general path (any layout, PAD, L >= 3, force_slow, reference tiling); the
// fused TMA kernel (stc_fused.cu) takes ABC / AB / Naive at L <= 2 otherwise.
//
// One persistent, warp-specialised CTA per SM.  Work items are (term, tile)
// pairs fetched with an atomic counter.  For each 16-deep k-chunk:
//
//   producer warps (8)  stream every view ("unit" = one view of one side for one
//                       chunk, 8 elements per thread) of the term's A and B
//                       sides from HBM/L2 into a ring of raw smem slots with
//                       cp.async (no registers held per load, NRAW-1 units in
//                       flight per thread, zero-fill for PAD) -- or, for
//                       regular views, one TMA box per unit -- then form the
//                       Strassen operand sums (e.g. A0+A3, B1-B3) in registers
//                       in view order and store them into the MMA smem ring --
//                       the work of the reference's pack_a_block /
//                       pack_b_block (_jit.py:27-131).  A k-chunk whose
//                       scatter entries have one constant stride (its
//                       block-scatter entry at GPU-chunk granularity, built on
//                       the device) is addressed as base + k*stride (fast
//                       path); otherwise every element goes through the
//                       scatter vector (slow path).  Same elements either way,
//                       so force_slow is bitwise neutral.
//   consumer warps (8)  mma.sync.m16n8k4.f64 (DMMA) on 64x32 warp tiles with
//                       register accumulators over the whole quadrant k
//                       (replaces microtile / macro_kernel, _jit.py:134-220),
//                       then add +/-M into each C target through the scatter
//                       layout (replaces store_tile, _jit.py:158-186).  Updates
//                       of one C tile by different terms are ordered by
//                       per-tile tickets: deterministic, no atomics on C.
//
// Dense-out mode (AB / Naive) writes M_slot instead of the C targets.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "stc_internal.cuh"
#include "stc_ptx.cuh"
#include "stc_common.cuh"

namespace stc {

constexpr int64_t kIrregular = INT64_MIN;  // chunk has no single stride (or holds PAD)
constexpr int MAX_NRAW = 7;  // raw slots (units in flight + 1); instantiated for 4..7

constexpr int MAX_TMA_RAW = 8;  // TMA raw slots (instantiated for 5..7)

struct SmemLayout {
  static constexpr size_t stage_doubles = (size_t)BK * LDS;
  static constexpr size_t stage_bytes = stage_doubles * 8;
  static constexpr size_t a_off = 0;
  static constexpr size_t b_off = a_off + STAGES * stage_bytes;
  // full[STAGES], empty[STAGES], then (TMA) raw_full[MAX_TMA_RAW], raw_empty[MAX_TMA_RAW]
  static constexpr size_t bar_off = b_off + STAGES * stage_bytes;
  static constexpr size_t meta_off = bar_off + (2 * STAGES + 2 * MAX_TMA_RAW) * 8;  // stage_item[STAGES], s_item
  static constexpr size_t tab_off = (meta_off + (STAGES + 4) * 4 + 127) / 128 * 128;
  // gather mode: xoffA[ops][BM], xoffB[ops][BN], UnitDesc[2 * ops], KInfo[2][2 * ops][kwin],
  //              then raw[nraw][BK * 128] (thread-private, see raw_index)
  // TMA mode:    xcoord[2 * ops] (int4), kcoord[2][2 * ops][kwin] (int4), then raw[nraw][BK * 128] (box order)
  __host__ __device__ static size_t tab_bytes(int ops, int kwin, bool tma) {
    const size_t win = 2 * (2 * (size_t)ops) * (size_t)kwin * 16;
    return tma ? 2 * (size_t)ops * 16 + win : 8 * (size_t)ops * (BM + BN) + 2 * (size_t)ops * 16 + win;
  }
  __host__ __device__ static size_t raw_off(int ops, int kwin, bool tma) {
    const size_t a = tma ? 1024 : 128;  // TMA: the 128-byte swizzle pattern repeats every 1024 bytes
    return (tab_off + tab_bytes(ops, kwin, tma) + a - 1) / a * a;
  }
  static constexpr size_t raw_doubles = (size_t)BK * 128;  // one raw slot (one unit)
  __host__ __device__ static size_t bytes(int ops, int kwin, int nraw, bool tma) {
    return raw_off(ops, kwin, tma) + (size_t)nraw * raw_doubles * 8;
  }
};

constexpr size_t kMaxSmem = 227 * 1024;

// k-info window (chunks): the largest of 32/16/8 that leaves room for 4 raw slots.
int gemm_kwin(int max_ops) {
  int w = 32;
  while (w > 8 && SmemLayout::bytes(max_ops, w, 4, false) > kMaxSmem) w /= 2;
  return w;
}

// TMA mode: k-coordinate window 32 (or 16) and 5..7 raw slots (lookahead nraw - 2 units).
int gemm_tma_config(int max_ops, int &nraw, int &kwin) {
  for (int w = 32; w >= 16; w /= 2)
    for (int n = 7; n >= 5; --n)
      if (SmemLayout::bytes(max_ops, w, n, true) <= kMaxSmem) {
        nraw = n;
        kwin = w;
        return 1;
      }
  return 0;
}

// Raw slots (cp.async units in flight + 1): as many as fit, 4..MAX_NRAW.
int gemm_nraw(int max_ops) {
  const int w = gemm_kwin(max_ops);
  int n = MAX_NRAW;
  if (const char *e = getenv("STC_NRAW")) n = std::max(4, std::min(MAX_NRAW, atoi(e)));
  while (n > 4 && SmemLayout::bytes(max_ops, w, n, false) > kMaxSmem) --n;
  return w < 32 ? 4 : n;  // reduced windows are only instantiated with 4 slots
}

size_t gemm_smem_bytes(int max_ops) { return SmemLayout::bytes(max_ops, gemm_kwin(max_ops), gemm_nraw(max_ops), false); }


// Producer thread mappings (NP = 256 threads, EPT = 8 elements per unit):
//   x-contiguous side (kfast = 0): x = t % 128, k = 8 (t / 128) + e
//   k-contiguous side (kfast = 1): k = (t & 3) + 4 (e & 3), x = (t >> 2) + 64 (e >> 2)
constexpr int NP = 32 * PRODUCER_WARPS;
constexpr int EPT = BK * 128 / NP;
static_assert(NP == 256 && EPT == 8, "producer mapping assumes 256 threads x 8 elements");
static_assert((PRODUCER_WARPS & (PRODUCER_WARPS - 1)) == 0, "issue distribution uses i % PRODUCER_WARPS");

__device__ __forceinline__ int tile_index(int kfast, int t, int e) {
  return kfast ? ((t & 3) + 4 * (e & 3)) * LDS + (t >> 2) + 64 * (e >> 2) : ((t >> 7) * 8 + e) * LDS + (t & 127);
}

// Raw slots are private to each producer thread, independent of the side's
// mapping: element e of thread t lives at e * NP + t (conflict-free).  A slot
// alternately holds A- and B-side units whose tile mappings differ, so a
// tile-position layout would let one thread's cp.async land on data another
// thread has not read yet.
__device__ __forceinline__ int raw_index(int t, int e) { return e * NP + t; }

// Per-unit constants of the current item, staged in smem at item start.  The
// unit's role (side, first/last view, coefficient sign) is derived from its
// index in registers; only the data pointer and k-vector start live here.
struct UnitDesc {
  const double *D;  // side data + the view's data offset
  int64_t kst;      // pool index of the view's k vector
};
static_assert(sizeof(UnitDesc) == 16, "SmemLayout::tab_bytes assumes 16-byte unit slots");

// First k offset and chunk stride (kbs entry) of one unit for one chunk; the
// producer keeps a double-buffered window of KWIN chunks of these in smem so
// that issuing a unit never waits on a global load.
struct KInfo {
  int64_t b0, kstr;
};

// Everything one thread needs to issue one unit, loaded one unit ahead so the
// shared-memory latency of the tables is off the issue path.
struct UnitPre {
  const double *D;
  int64_t kst;
  KInfo ki;
  int64_t x0, x1;  // this thread's x offsets (x1: second row group of a k-contiguous side)
  int kfast;
};

// cp.async one unit of chunk `kc` into a raw slot (zero-fill for PAD).  A
// chunk whose 16 k entries share one stride (its block-scatter entry at GPU
// granularity, kbs) is addressed base + k * stride: the reference's fast path
// (_jit.py:54-65); otherwise every element goes through the scatter vector:
// the slow path (_jit.py:66-78).  PAD rows (x) are handled per row: the whole
// run is zero-filled from a dummy source.
__device__ __forceinline__ void issue_unit(double *__restrict__ dst, const UnitPre &u, const int64_t *__restrict__ pool,
                                           int kc, bool force_slow, int t) {
  const double *D = u.D;
  if (!force_slow && u.ki.kstr != kIrregular) {
    const int64_t kstr = u.ki.kstr;
    if (!u.kfast) {
      const bool ok = u.x0 != kPad;
      const double *src = ok ? D + (u.x0 + u.ki.b0 + (t >> 7) * 8 * kstr) : D;
      const int64_t step = ok ? kstr : 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) cp_async8(dst + raw_index(t, e), src + e * step, ok);
    } else {
      const double *base = D + (u.ki.b0 + (t & 3) * kstr);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t a = j ? u.x1 : u.x0;
        const bool ok = a != kPad;
        const double *src = ok ? base + a : D;
        const int64_t step = ok ? 4 * kstr : 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async8(dst + raw_index(t, 4 * j + i), src + i * step, ok);
      }
    }
  } else {
    const int64_t kst = u.kst + (int64_t)kc * BK;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int k = u.kfast ? (t & 3) + 4 * (e & 3) : (t >> 7) * 8 + e;
      const int64_t a = u.kfast ? ((e >> 2) ? u.x1 : u.x0) : u.x0;
      const int64_t b = __ldg(pool + kst + k);
      const bool ok = a != kPad && b != kPad;
      cp_async8(dst + raw_index(t, e), ok ? D + a + b : D, ok);
    }
  }
}

// s * v for s = +/-1 as a sign flip, then 0.0 + (.) (turns -0.0 into +0.0): exactly the
// reference's first packing step `0.0 + coeff * data` (_jit.py:43-65), on the integer pipe.
__device__ __forceinline__ double first_term(double v, uint64_t signbit) {
  // integer ops only (inline PTX): a zero test written in C++ is turned into a
  // DSETP, which queues behind the consumers' DMMAs on the FP64 pipe
  const uint32_t lo = static_cast<uint32_t>(__double2loint(v));
  const uint32_t hi = static_cast<uint32_t>(__double2hiint(v)) ^ static_cast<uint32_t>(signbit >> 32);
  uint32_t out_hi;
  asm("{\n"
      ".reg .pred pz;\n"
      ".reg .b32 tz;\n"
      "and.b32 tz, %1, 0x7fffffff;\n"
      "or.b32 tz, tz, %2;\n"
      "setp.eq.b32 pz, tz, 0;\n"
      "selp.b32 %0, 0, %1, pz;\n"
      "}\n"
      : "=r"(out_hi)
      : "r"(hi), "r"(lo));
  return __hiloint2double(static_cast<int>(out_hi), static_cast<int>(lo));
}


// ---- TMA box staging (regular views) ---------------------------------------
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// One box (one unit: 128 x 16 doubles) of a rank-2..5 tensor map into smem,
// completing on `bar`.
__device__ __forceinline__ void tma_box(void *dst, const CUtensorMap *map, int rank, const int32_t (&c)[5],
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


// L2 prefetch of one box (no smem, no completion): extends the staging
// lookahead beyond the raw slots.
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map, int rank, const int32_t (&c)[5]) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(m), "r"(c[0]), "r"(c[1])
                   : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(m), "r"(c[0]), "r"(c[1]),
                   "r"(c[2])
                   : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(m), "r"(c[0]),
                   "r"(c[1]), "r"(c[2]), "r"(c[3])
                   : "memory");
      break;
    default:
      asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(m), "r"(c[0]),
                   "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
                   : "memory");
      break;
  }
}

// Coordinates of a pool offset in one part (x or k) of a side's tensor map:
// the part's labels by descending stride (nested strides, checked on the host).
__device__ __forceinline__ int4 part_coords(int64_t off, int np, const int64_t (&str)[4]) {
  int32_t c[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < np) {
      const int64_t q = off / str[i];
      c[i] = (int32_t)q;
      off -= q * str[i];
    }
  return make_int4(c[0], c[1], c[2], c[3]);
}

__device__ __forceinline__ int coord_at(const int4 &v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}


// Producer warps, TMA mode: both sides' views are regular boxes (host-checked,
// stc_tma.cu), so one elected thread stages each unit with a single tensor-map
// box load (cp.async.bulk.tensor, completion on the raw slot's mbarrier) and
// the 256 producer threads only form the Strassen sums, with the gather path's
// thread mapping (same elements per thread, same view order and rounding).
// Raw box layouts: x-contiguous side [k][128]; k-contiguous side [x][16] with
// the 128-byte swizzle (16-byte chunk index ^ x & 7), both read conflict-free.
__device__ __forceinline__ int raw_box_index(int kfast, int t, int e) {
  if (!kfast) return ((t >> 7) * 8 + e) * 128 + (t & 127);
  const int k = (t & 3) + 4 * (e & 3), x = (t >> 2) + 64 * (e >> 2);
  return x * 16 + ((((k >> 1) ^ (x & 7)) << 1) | (k & 1));
}

template <int NRAW, int KWIN>
__device__ __forceinline__ void producer_tma(const GemmArgs &p, const CUtensorMap *tmA, const CUtensorMap *tmB,
                                             unsigned char *smem, double *sA, double *sB, uint64_t *full,
                                             uint64_t *empty, uint64_t *rfull, uint64_t *rempty, int *stage_item,
                                             int *s_item, double *raw, int t) {
  const int mo = p.max_ops;
  int4 *xcoord = reinterpret_cast<int4 *>(smem + SmemLayout::tab_off);  // [2 * mo]
  int4 *kcoord = xcoord + 2 * mo;                                       // [2][2 * mo][KWIN]
  const int lane = t & 31;
  const int akf = p.a_kfast, bkf = p.b_kfast;
  constexpr int D = NRAW - 2;  // units in flight: the slot refilled was released two units ago
  const int PF = p.tma_prefetch;  // further units prefetched into L2 (window refill keeps KWIN/2 chunks ready)
  constexpr uint32_t kUnitBytes = (uint32_t)(SmemLayout::raw_doubles * 8);
  int stage = 0;
  uint32_t phase = 0;
  int rslot = 0, islot = 0;        // consume / issue raw-slot cursors (continue across items)
  uint32_t rphase = 0, iphase = 0;
  for (;;) {
    if (t == 0) *s_item = atomicAdd(p.counter, 1);
    named_bar(1, NP);
    const int item = *s_item;
    if (item >= p.total_items) {
      mbar_wait(&empty[stage], phase ^ 1);
      if (t == 0) stage_item[stage] = -1;
      mbar_arrive(&full[stage]);
      break;
    }
    int slot, ti, tj;
    tile_of(p, item, slot, ti, tj);
    const TermDesc td = p.terms[slot];
    const int na = td.a_count, nb = td.b_count;
    const int U = na + nb;
    uint32_t negmask = 0;
    for (int u = 0; u < U; ++u) {
      const bool is_a = u < na;
      const double sg = p.ops[is_a ? td.a_first + u : td.b_first + u - na].sign;
      negmask |= (__double_as_longlong(sg) < 0 ? 1u : 0u) << u;  // integer test (no DSETP)
    }
    if (t < U) {  // x coordinates of the unit's tile
      const int sd = t < na ? 0 : 1;
      const OpDesc o = p.ops[sd == 0 ? td.a_first + t : td.b_first + t - na];
      const int64_t off = p.pool[o.x_start + (int64_t)(sd == 0 ? ti * BM : tj * BN)] - p.tm_base[sd][0];
      xcoord[t] = part_coords(off, p.tm_np[sd][0], p.tm_pstr[sd][0]);
    }
    const int kchunks = p.kchunks;
    auto fill_kwin = [&](int w) {  // k coordinates of window w into buffer w & 1
      for (int idx = t; idx < U * KWIN; idx += NP) {
        const int u = idx / KWIN, c = idx - u * KWIN;
        const int chunk = w * KWIN + c;
        if (chunk >= kchunks) continue;
        const int sd = u < na ? 0 : 1;
        const int64_t kst = p.ops[sd == 0 ? td.a_first + u : td.b_first + u - na].k_start + (int64_t)chunk * BK;
        const int64_t off = __ldg(p.pool + kst) - p.tm_base[sd][1];
        kcoord[((w & 1) * 2 * mo + u) * KWIN + c] = part_coords(off, p.tm_np[sd][1], p.tm_pstr[sd][1]);
      }
    };
    fill_kwin(0);
    named_bar(1, NP);

    const int G = kchunks * U;
    int ig = 0, ic = 0, iu = 0;  // issue cursor (thread 0)
    int pg = 0, pc = 0, pu = 0;  // L2-prefetch cursor (thread 0), PF units ahead of the issue cursor
    auto coords_of = [&](int c_, int u_, int32_t (&c)[5]) {
      const int sd = u_ < na ? 0 : 1;
      const int4 xc = xcoord[u_];
      const int4 kc = kcoord[(((c_ / KWIN) & 1) * 2 * mo + u_) * KWIN + (c_ & (KWIN - 1))];
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        const int src = p.tm_src[sd][d];
        c[d] = src < 4 ? coord_at(xc, src) : coord_at(kc, src - 4);
      }
      return sd;
    };
    // Issue work is spread over the producer warps: unit i is staged (and
    // prefetched) by lane 0 of warp i % PRODUCER_WARPS; every thread tracks the
    // cursors.
    const int pw = t >> 5;
    auto prefetch_to = [&](int target) {
      for (; pg < target && pg < G; ++pg) {
        if (lane == 0 && (pg & (PRODUCER_WARPS - 1)) == pw) {
          int32_t c[5];
          const int sd = coords_of(pc, pu, c);
          tma_prefetch(sd == 0 ? tmA : tmB, p.tm_rank[sd], c);
        }
        if (++pu == U) {
          pu = 0;
          ++pc;
        }
      }
    };
    auto issue = [&]() {
      if (ig < G) {
        if (PF > 0) prefetch_to(ig + PF);
        if (lane == 0 && (ig & (PRODUCER_WARPS - 1)) == pw) {
          int32_t c[5];
          const int sd = coords_of(ic, iu, c);
          mbar_wait(&rempty[islot], iphase ^ 1);
          mbar_expect_tx(&rfull[islot], kUnitBytes);
          tma_box(raw + islot * SmemLayout::raw_doubles, sd == 0 ? tmA : tmB, p.tm_rank[sd], c, &rfull[islot]);
        }
        if (++iu == U) {
          iu = 0;
          ++ic;
        }
        if (++islot == NRAW) {
          islot = 0;
          iphase ^= 1;
        }
        ++ig;
      }
    };
    for (int d = 0; d < D; ++d) issue();
    double acc[EPT];
    int cu = 0, cc = 0;
    for (int g = 0; g < G; ++g) {
      issue();
      const bool is_a = cu < na;
      const bool first = cu == 0 || cu == na;
      const bool last = cu == na - 1 || cu == U - 1;
      const bool neg = (negmask >> cu) & 1u;
      const double *src = raw + rslot * SmemLayout::raw_doubles;
      mbar_wait(&rfull[rslot], rphase);
      const int kf = is_a ? akf : bkf;
      double v[EPT];
      if (kf) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = src[raw_box_index(1, t, e)];
      } else {
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = src[raw_box_index(0, t, e)];
      }
      if (first) {
        const uint64_t sb = neg ? 0x8000000000000000ull : 0ull;
#pragma unroll
        for (int e = 0; e < EPT; ++e) acc[e] = first_term(v[e], sb);
      } else if (!neg) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) acc[e] = __dadd_rn(acc[e], v[e]);
      } else {
#pragma unroll
        for (int e = 0; e < EPT; ++e) acc[e] = __dsub_rn(acc[e], v[e]);
      }
      // every lane's reads of the slot are done (their values are in acc); order them
      // before the TMA (async proxy) refill of the slot
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&rempty[rslot]);
      if (++rslot == NRAW) {
        rslot = 0;
        rphase ^= 1;
      }
      if (last) {
        if (is_a) mbar_wait(&empty[stage], phase ^ 1);
        double *S = (is_a ? sA : sB) + stage * SmemLayout::stage_doubles;
#pragma unroll
        for (int e = 0; e < EPT; ++e) S[tile_index(kf, t, e)] = acc[e];
      }
      if (++cu == U) {
        cu = 0;
        if (t == 0) stage_item[stage] = item;
        mbar_arrive(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
        ++cc;
        if (cc % KWIN == KWIN / 2 && (cc / KWIN + 1) * KWIN < kchunks) {
          fill_kwin(cc / KWIN + 1);
          named_bar(1, NP);
        }
      }
    }
    named_bar(1, NP);  // tables of this item fully used before the next fill
  }
}

template <int NRAW, int KWIN, bool TMA>
__global__ void __launch_bounds__(THREADS, 1)
    k_strassen_gemm(const GemmArgs p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double *sA = reinterpret_cast<double *>(smem + SmemLayout::a_off);
  double *sB = reinterpret_cast<double *>(smem + SmemLayout::b_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SmemLayout::bar_off);
  uint64_t *empty = full + STAGES;
  int *stage_item = reinterpret_cast<int *>(smem + SmemLayout::meta_off);
  int *s_item = stage_item + STAGES;
  const int mo = p.max_ops;
  double *raw = reinterpret_cast<double *>(smem + SmemLayout::raw_off(mo, KWIN, TMA));
  uint64_t *rfull = empty + STAGES;  // TMA mode: raw slot landed / released
  uint64_t *rempty = rfull + MAX_TMA_RAW;
  int64_t *xoffA = reinterpret_cast<int64_t *>(smem + SmemLayout::tab_off);
  int64_t *xoffB = xoffA + mo * BM;
  UnitDesc *units = reinterpret_cast<UnitDesc *>(xoffB + mo * BN);  // [2 * mo] 
  KInfo *kinfo = reinterpret_cast<KInfo *>(units + 2 * mo);          // [2][2 * mo][KWIN]

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], NP);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    if (TMA)
      for (int r = 0; r < NRAW; ++r) {
        mbar_init(&rfull[r], 1);
        mbar_init(&rempty[r], PRODUCER_WARPS);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= CONSUMER_WARPS) {
    // ===================== producer warps: gather + Strassen sums =====
#ifndef STC_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
#endif
    const int t = tid - 32 * CONSUMER_WARPS;
    if constexpr (TMA) {
      producer_tma<NRAW, KWIN>(p, &tmA, &tmB, smem, sA, sB, full, empty, rfull, rempty, stage_item, s_item, raw, t);
    } else {
    const bool force_slow = p.force_slow != 0;
    const int akf = p.a_kfast, bkf = p.b_kfast;
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      if (t == 0) *s_item = atomicAdd(p.counter, 1);
      named_bar(1, NP);
      const int item = *s_item;
      if (item >= p.total_items) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (t == 0) stage_item[stage] = -1;
        mbar_arrive(&full[stage]);
        break;
      }
      int slot, ti, tj;
      tile_of(p, item, slot, ti, tj);
      const TermDesc td = p.terms[slot];
      const int na = td.a_count, nb = td.b_count;
      const int U = na + nb;  // units per chunk: every view of A, then of B
      uint32_t negmask = 0;   // bit u: unit u's coefficient is negative
      for (int u = 0; u < U; ++u) {
        const bool is_a = u < na;
        const double sg = p.ops[is_a ? td.a_first + u : td.b_first + u - na].sign;
        negmask |= (__double_as_longlong(sg) < 0 ? 1u : 0u) << u;  // integer test (no DSETP)
      }
      if (t < U) {
        const bool is_a = t < na;
        const OpDesc o = p.ops[is_a ? td.a_first + t : td.b_first + t - na];
        UnitDesc u;
        u.D = (is_a ? p.A : p.B) + o.data_off;
        u.kst = o.k_start;
        units[t] = u;
      }
      for (int idx = t; idx < na * BM; idx += NP) {
        const int op = idx / BM, x = idx - op * BM;
        xoffA[idx] = p.pool[p.ops[td.a_first + op].x_start + (int64_t)ti * BM + x];
      }
      for (int idx = t; idx < nb * BN; idx += NP) {
        const int op = idx / BN, x = idx - op * BN;
        xoffB[idx] = p.pool[p.ops[td.b_first + op].x_start + (int64_t)tj * BN + x];
      }
      const int kchunks = p.kchunks;
      // k-info window w (chunks [w*KWIN, (w+1)*KWIN)) into buffer w & 1
      auto fill_kwin = [&](int w) {
        for (int idx = t; idx < U * KWIN; idx += NP) {
          const int u = idx / KWIN, c = idx - u * KWIN;
          const int chunk = w * KWIN + c;
          if (chunk >= kchunks) continue;
          const int64_t kst = p.ops[u < na ? td.a_first + u : td.b_first + u - na].k_start + (int64_t)chunk * BK;
          KInfo ki;
          ki.b0 = __ldg(p.pool + kst);
          ki.kstr = __ldg(p.kbs + (kst >> 4));
          kinfo[((w & 1) * 2 * mo + u) * KWIN + c] = ki;
        }
      };
      fill_kwin(0);  // window 1 follows half-way through window 0
      named_bar(1, NP);

      // descriptor of unit (chunk c, unit u) for this thread
      auto load_pre = [&](int c, int u) {
        UnitPre q;
        const UnitDesc ud = units[u];
        q.D = ud.D;
        q.kst = ud.kst;
        q.ki = kinfo[(((c / KWIN) & 1) * 2 * mo + u) * KWIN + (c & (KWIN - 1))];
        const bool is_a = u < na;
        q.kfast = is_a ? akf : bkf;
        const int64_t *xo = is_a ? xoffA + u * BM : xoffB + (u - na) * BN;
        q.x0 = xo[q.kfast ? (t >> 2) : (t & 127)];
        q.x1 = q.kfast ? xo[(t >> 2) + 64] : 0;
        return q;
      };

      const int G = kchunks * U;
      constexpr int D = NRAW - 1;  // units in flight ahead of the one being summed
      int ig = 0, ic = 0, iu = 0, islot = 0;  // issue cursor
      int cc = 0, cu = 0, cslot = 0;          // consume cursor (chunk, unit, raw slot)
      UnitPre pre = load_pre(0, 0);
      auto issue = [&]() {
        if (ig < G) {
          issue_unit(raw + islot * SmemLayout::raw_doubles, pre, p.pool, ic, force_slow, t);
          if (++iu == U) {
            iu = 0;
            ++ic;
          }
          if (++islot == NRAW) islot = 0;
          if (ig + 1 < G) pre = load_pre(ic, iu);
        }
        cp_async_commit();  // empty groups at the tail keep the wait count uniform
        ++ig;
      };
      for (int d = 0; d < D; ++d) issue();
      double acc[EPT];
      for (int g = 0; g < G; ++g) {
        issue();
        cp_async_wait<D>();  // unit g has landed (this thread's own copies)
        const bool is_a = cu < na;
        const bool first = cu == 0 || cu == na;
        const bool last = cu == na - 1 || cu == U - 1;
        const bool neg = (negmask >> cu) & 1u;
        const double *src = raw + cslot * SmemLayout::raw_doubles;
        if (first) {
          const uint64_t sb = neg ? 0x8000000000000000ull : 0ull;
#pragma unroll
          for (int e = 0; e < EPT; ++e) acc[e] = first_term(src[raw_index(t, e)], sb);
        } else if (!neg) {
          // later views: acc + v or acc - v (a DADD; the sign is exact, so this equals
          // the reference's acc + coeff * v)
#pragma unroll
          for (int e = 0; e < EPT; ++e) acc[e] = __dadd_rn(acc[e], src[raw_index(t, e)]);
        } else {
#pragma unroll
          for (int e = 0; e < EPT; ++e) acc[e] = __dsub_rn(acc[e], src[raw_index(t, e)]);
        }
        if (++cslot == NRAW) cslot = 0;
        if (last) {  // side complete: store its sum into the MMA ring
          if (is_a) mbar_wait(&empty[stage], phase ^ 1);
          const int kf = is_a ? akf : bkf;
          double *S = (is_a ? sA : sB) + stage * SmemLayout::stage_doubles;
#pragma unroll
          for (int e = 0; e < EPT; ++e) S[tile_index(kf, t, e)] = acc[e];
        }
        if (++cu == U) {
          cu = 0;
          if (t == 0) stage_item[stage] = item;
          mbar_arrive(&full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          // half-way through window w, publish window w+1 (its buffer held window
          // w-1, which every producer thread has finished issuing: producers are at
          // most STAGES chunks apart, and the issue cursor is less than KWIN/2
          // chunks ahead)
          ++cc;
          if (cc % KWIN == KWIN / 2 && (cc / KWIN + 1) * KWIN < kchunks) {
            fill_kwin(cc / KWIN + 1);
            named_bar(1, NP);
          }
        }
      }
      cp_async_wait<0>();
      named_bar(1, NP);  // tables of this item fully used before the next fill
    }
    }  // gather producer
  } else {
    // ===================== consumer warps: DMMA + epilogue ============
#ifndef STC_NO_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
#endif
    const int lane = tid & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    int stage = 0;
    uint32_t phase = 0;
    bool c_seen = false;  // stc_set_c_ready flag observed
    double acc[4][4][4];
    for (;;) {
      mbar_wait(&full[stage], phase);
      const int item = stage_item[stage];
      if (item < 0) break;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
      for (int kc = 0; kc < p.kchunks; ++kc) {
        if (kc > 0) mbar_wait(&full[stage], phase);
        const double *as = sA + stage * SmemLayout::stage_doubles + wm * 64 + g;
        const double *bs = sB + stage * SmemLayout::stage_doubles + wn * 32 + g;
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
          const int row = (kk * 4 + tig) * LDS;
          double af[4][2], bf[4];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            af[mt][0] = as[row + mt * 16];
            af[mt][1] = as[row + mt * 16 + 8];
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) bf[nt] = bs[row + nt * 8];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              dmma_16x8x4(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!p.dense_out) wait_c_ready(p, tid, c_seen);
      epilogue_store(p, acc, item, tid, wm, wn, g, tig);
    }
  }
}

using GemmKernel = void (*)(const GemmArgs, const CUtensorMap, const CUtensorMap);

static GemmKernel kernel_for(int nraw, int kwin, bool tma) {
  if (tma) {
    if (kwin == 16) return nraw >= 7 ? k_strassen_gemm<7, 16, true> : nraw == 6 ? k_strassen_gemm<6, 16, true> : k_strassen_gemm<5, 16, true>;
    return nraw >= 7 ? k_strassen_gemm<7, 32, true> : nraw == 6 ? k_strassen_gemm<6, 32, true> : k_strassen_gemm<5, 32, true>;
  }
  if (kwin == 16) return k_strassen_gemm<4, 16, false>;
  if (kwin == 8) return k_strassen_gemm<4, 8, false>;
  switch (nraw) {
    case 4: return k_strassen_gemm<4, 32, false>;
    case 5: return k_strassen_gemm<5, 32, false>;
    case 6: return k_strassen_gemm<6, 32, false>;
    default: return k_strassen_gemm<7, 32, false>;
  }
}

// One persistent CTA per SM: 512 threads x 128 registers fill the register file.
int gemm_max_grid(int max_ops) {
  (void)max_ops;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  static int cached[64] = {};  // SM count per device (queried once; a benign race at worst re-queries)
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (dev >= 0 && dev < 64) cached[dev] = sms;
  return sms;
}

// `maps`: two CUtensorMap (A side, B side) when a.tma, else ignored.
cudaError_t launch_gemm(const GemmArgs &a, int grid, cudaStream_t s, const void *maps) {
  const bool tma = a.tma != 0;
  const size_t sm = SmemLayout::bytes(a.max_ops, a.kwin, a.nraw, tma);
  GemmKernel k = kernel_for(a.nraw, a.kwin, tma);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  CUtensorMap m[2];
  if (tma && maps)
    memcpy(m, maps, sizeof(m));
  else
    memset(m, 0, sizeof(m));
  k<<<grid, THREADS, sm, s>>>(a, m[0], m[1]);
  return cudaGetLastError();
}

}  // namespace stc
