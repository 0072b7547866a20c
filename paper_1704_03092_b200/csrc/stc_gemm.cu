// stc_gemm.cu -- the fused Strassen DMMA kernel (north-star subsystems 2 + 3).
//
// One persistent, warp-specialised CTA per SM.  Work items are (term, tile)
// pairs fetched with an atomic counter.  For each 16-deep k-chunk:
//
//   producer warps (4)  stream every view ("unit" = one view of one side for one
//                       chunk, 16 elements per thread) of the term's A and B
//                       sides from HBM/L2 into a ring of raw smem slots with
//                       cp.async (no registers held per load, NRAW-1 units in
//                       flight per thread, zero-fill for PAD), then form the
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
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "stc_internal.cuh"
#include "stc_ptx.cuh"

namespace stc {

constexpr int64_t kIrregular = INT64_MIN;  // chunk has no single stride (or holds PAD)
constexpr int MAX_NRAW = 7;  // raw slots (units in flight + 1); instantiated for 4..7

struct SmemLayout {
  static constexpr size_t stage_doubles = (size_t)BK * LDS;
  static constexpr size_t stage_bytes = stage_doubles * 8;
  static constexpr size_t a_off = 0;
  static constexpr size_t b_off = a_off + STAGES * stage_bytes;
  static constexpr size_t bar_off = b_off + STAGES * stage_bytes;  // full[STAGES], empty[STAGES]
  static constexpr size_t meta_off = bar_off + 2 * STAGES * 8;    // stage_item[STAGES], s_item
  static constexpr size_t tab_off = (meta_off + (STAGES + 4) * 4 + 127) / 128 * 128;
  // xoffA[ops][BM], xoffB[ops][BN], UnitDesc[2 * ops], then raw[nraw][BK * 128] (thread-private, see raw_index)
  // k-info window: kwin chunks x 2 buffers x (2 * ops) units x 16 bytes
  __host__ __device__ static size_t tab_bytes(int ops, int kwin) {
    return 8 * (size_t)ops * (BM + BN) + 2 * (size_t)ops * 64 + 2 * (2 * (size_t)ops) * (size_t)kwin * 16;
  }
  __host__ __device__ static size_t raw_off(int ops, int kwin) { return (tab_off + tab_bytes(ops, kwin) + 127) / 128 * 128; }
  static constexpr size_t raw_doubles = (size_t)BK * 128;  // one thread-private raw slot
  __host__ __device__ static size_t bytes(int ops, int kwin, int nraw) {
    return raw_off(ops, kwin) + (size_t)nraw * raw_doubles * 8;
  }
};

constexpr size_t kMaxSmem = 227 * 1024;

// k-info window (chunks): the largest of 32/16/8 that leaves room for 4 raw slots.
int gemm_kwin(int max_ops) {
  int w = 32;
  while (w > 8 && SmemLayout::bytes(max_ops, w, 4) > kMaxSmem) w /= 2;
  return w;
}

// Raw slots (cp.async units in flight + 1): as many as fit, 4..MAX_NRAW.
int gemm_nraw(int max_ops) {
  const int w = gemm_kwin(max_ops);
  int n = MAX_NRAW;
  if (const char *e = getenv("STC_NRAW")) n = std::max(4, std::min(MAX_NRAW, atoi(e)));
  while (n > 4 && SmemLayout::bytes(max_ops, w, n) > kMaxSmem) --n;
  return w < 32 ? 4 : n;  // reduced windows are only instantiated with 4 slots
}

size_t gemm_smem_bytes(int max_ops) { return SmemLayout::bytes(max_ops, gemm_kwin(max_ops), gemm_nraw(max_ops)); }

__device__ __forceinline__ void tile_of(const GemmArgs &p, int item, int &slot, int &ti, int &tj) {
  const int P = p.tiles_m * p.tiles_n;
  slot = item / P;
  const int pos = item - slot * P;
  // grouped rasterisation: group_m tile-rows share the B panels in L2
  const int per_group = p.group_m * p.tiles_n;
  const int g = pos / per_group;
  const int first = g * p.group_m;
  const int gsz = min(p.tiles_m - first, p.group_m);
  const int r = pos - g * per_group;
  ti = first + r % gsz;
  tj = r / gsz;
}

// Producer thread mappings (NP = 256 threads, EPT = 8 elements per unit):
//   x-contiguous side (kfast = 0): x = t % 128, k = 8 (t / 128) + e
//   k-contiguous side (kfast = 1): k = (t & 3) + 4 (e & 3), x = (t >> 2) + 64 (e >> 2)
constexpr int NP = 32 * PRODUCER_WARPS;
constexpr int EPT = BK * 128 / NP;
static_assert(NP == 256 && EPT == 8, "producer mapping assumes 256 threads x 8 elements");

__device__ __forceinline__ int tile_index(int kfast, int t, int e) {
  return kfast ? ((t & 3) + 4 * (e & 3)) * LDS + (t >> 2) + 64 * (e >> 2) : ((t >> 7) * 8 + e) * LDS + (t & 127);
}

// Raw slots are private to each producer thread, independent of the side's
// mapping: element e of thread t lives at e * NP + t (conflict-free).  A slot
// alternately holds A- and B-side units whose tile mappings differ, so a
// tile-position layout would let one thread's cp.async land on data another
// thread has not read yet.
__device__ __forceinline__ int raw_index(int t, int e) { return e * NP + t; }

// Everything the producer needs about one unit (one view of one side) of the
// current item, staged in smem at item start.
struct UnitDesc {
  const double *D;     // side data + the view's data offset
  int32_t xo;          // element offset of the view's x offsets in the smem x table
  int32_t _pad;
  int64_t kst;         // pool index of the view's k vector
  uint64_t signbit;    // sign of the coefficient as a bit (first view of a side)
  double sign;         // +/-1 (later views)
  int32_t kfast, is_a, first, last;
};

static_assert(sizeof(UnitDesc) <= 64, "UnitDesc slot");

// First k offset and chunk stride (kbs entry) of one unit for one chunk; the
// producer keeps a double-buffered window of KWIN chunks of these in smem so
// that issuing a unit never waits on a global load.
struct KInfo {
  int64_t b0, kstr;
};

// cp.async one unit of chunk `kc` into a raw slot (zero-fill for PAD).  A
// chunk whose 16 k entries share one stride (its block-scatter entry at GPU
// granularity, kbs) is addressed base + k * stride: the reference's fast path
// (_jit.py:54-65); otherwise every element goes through the scatter vector:
// the slow path (_jit.py:66-78).  PAD rows (x) are handled per row: the whole
// run is zero-filled from a dummy source.
__device__ __forceinline__ void issue_unit(double *__restrict__ dst, const UnitDesc &u, const int64_t *__restrict__ xtab,
                                           const int64_t *__restrict__ pool, KInfo ki, int kc, bool force_slow,
                                           int t) {
  const double *D = u.D;
  const int64_t *xo = xtab + u.xo;
  if (!force_slow && ki.kstr != kIrregular) {
    const int64_t kstr = ki.kstr;
    if (!u.kfast) {
      const int64_t a = xo[t & 127];
      const bool ok = a != kPad;
      const double *src = ok ? D + (a + ki.b0 + (t >> 7) * 8 * kstr) : D;
      const int64_t step = ok ? kstr : 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) cp_async8(dst + raw_index(t, e), src + e * step, ok);
    } else {
      const double *base = D + (ki.b0 + (t & 3) * kstr);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t a = xo[(t >> 2) + 64 * j];
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
      const int x = u.kfast ? (t >> 2) + 64 * (e >> 2) : (t & 127);
      const int k = u.kfast ? (t & 3) + 4 * (e & 3) : (t >> 7) * 8 + e;
      const int64_t a = xo[x], b = __ldg(pool + kst + k);
      const bool ok = a != kPad && b != kPad;
      cp_async8(dst + raw_index(t, e), ok ? D + a + b : D, ok);
    }
  }
}

// s * v for s = +/-1 as a sign flip, then 0.0 + (.) (turns -0.0 into +0.0): exactly the
// reference's first packing step `0.0 + coeff * data` (_jit.py:43-65), on the integer pipe.
__device__ __forceinline__ double first_term(double v, uint64_t signbit) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v)) ^ signbit;
  if ((b << 1) == 0) b = 0;
  return __longlong_as_double(static_cast<long long>(b));
}

template <int NRAW, int KWIN>
__global__ void __launch_bounds__(THREADS, 1) k_strassen_gemm(const GemmArgs p) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *sA = reinterpret_cast<double *>(smem + SmemLayout::a_off);
  double *sB = reinterpret_cast<double *>(smem + SmemLayout::b_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SmemLayout::bar_off);
  uint64_t *empty = full + STAGES;
  int *stage_item = reinterpret_cast<int *>(smem + SmemLayout::meta_off);
  int *s_item = stage_item + STAGES;
  const int mo = p.max_ops;
  double *raw = reinterpret_cast<double *>(smem + SmemLayout::raw_off(mo, KWIN));
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
  }
  __syncthreads();

  if (warp >= CONSUMER_WARPS) {
    // ===================== producer warps: gather + Strassen sums =====
#ifndef STC_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
#endif
    const int t = tid - 32 * CONSUMER_WARPS;
    const bool force_slow = p.force_slow != 0;
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
      if (t < U) {
        const bool is_a = t < na;
        const int op = is_a ? t : t - na;
        const OpDesc o = p.ops[is_a ? td.a_first + op : td.b_first + op];
        UnitDesc u;
        u.D = (is_a ? p.A : p.B) + o.data_off;
        u.xo = is_a ? op * BM : mo * BM + op * BN;
        u.kst = o.k_start;
        u.signbit = o.sign < 0 ? 0x8000000000000000ull : 0ull;
        u.sign = o.sign;
        u.kfast = is_a ? p.a_kfast : p.b_kfast;
        u.is_a = is_a;
        u.first = op == 0;
        u.last = op == (is_a ? na : nb) - 1;
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

      const int G = kchunks * U;
      constexpr int D = NRAW - 1;  // units in flight ahead of the one being summed
      int ig = 0, ic = 0, iu = 0, islot = 0;  // issue cursor
      int cc = 0, cu = 0, cslot = 0;          // consume cursor (chunk, unit, raw slot)
      auto issue = [&]() {
        if (ig < G) {
          issue_unit(raw + islot * SmemLayout::raw_doubles, units[iu], xoffA, p.pool,
                     kinfo[(((ic / KWIN) & 1) * 2 * mo + iu) * KWIN + (ic & (KWIN - 1))], ic, force_slow, t);
          if (++iu == U) {
            iu = 0;
            ++ic;
          }
          if (++islot == NRAW) islot = 0;
        }
        cp_async_commit();  // empty groups at the tail keep the wait count uniform
        ++ig;
      };
      for (int d = 0; d < D; ++d) issue();
      double acc[EPT];
      for (int g = 0; g < G; ++g) {
        issue();
        cp_async_wait<D>();  // unit g has landed (this thread's own copies)
        const UnitDesc &u = units[cu];
        const double *src = raw + cslot * SmemLayout::raw_doubles;
        if (u.first) {
#pragma unroll
          for (int e = 0; e < EPT; ++e) acc[e] = first_term(src[raw_index(t, e)], u.signbit);
        } else {
          // later views: acc + v or acc - v (a DADD; the sign is exact, so this equals
          // the reference's acc + coeff * v)
          if (u.signbit == 0) {
#pragma unroll
            for (int e = 0; e < EPT; ++e) acc[e] = __dadd_rn(acc[e], src[raw_index(t, e)]);
          } else {
#pragma unroll
            for (int e = 0; e < EPT; ++e) acc[e] = __dsub_rn(acc[e], src[raw_index(t, e)]);
          }
        }
        if (++cslot == NRAW) cslot = 0;
        if (u.last) {  // side complete: store its sum into the MMA ring
          if (u.is_a) mbar_wait(&empty[stage], phase ^ 1);
          double *S = (u.is_a ? sA : sB) + stage * SmemLayout::stage_doubles;
#pragma unroll
          for (int e = 0; e < EPT; ++e) S[tile_index(u.kfast, t, e)] = acc[e];
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
          // most STAGES chunks apart)
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
#ifdef STC_EXPERIMENT_NOMMA
              acc[mt][nt][0] += af[mt][0] * bf[nt] * 1e-300;  // timing experiment only
#else
              dmma_16x8x4(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
#endif
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      // ---------------- epilogue -------------------------------------
      int slot, ti, tj;
      tile_of(p, item, slot, ti, tj);
      const TermDesc td = p.terms[slot];
      const int row0 = ti * BM + wm * 64 + g;
      const int col0 = tj * BN + wn * 32 + 2 * tig;
      if (p.dense_out) {
        double *Mt = p.M + (int64_t)td.m_slot * p.m_stride;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double2 v = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
              *reinterpret_cast<double2 *>(Mt + (int64_t)(row0 + mt * 16 + 8 * h) * p.m_ld + col0 + nt * 8) = v;
            }
      } else {
        const int pos = item - slot * p.tiles_m * p.tiles_n;
        for (int j = 0; j < td.c_count; ++j) {
          const TgtDesc tg = p.tgts[td.c_first + j];
          int32_t *ticket = p.tickets + tg.ticket_base + pos;
          if (p.use_tickets) {
            if (tid == 0) {
              while (ld_acquire_gpu(ticket) < tg.order) __nanosleep(128);
            }
            named_bar(2, 32 * CONSUMER_WARPS);
          }
          int64_t co[8];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int b = 0; b < 2; ++b) co[nt * 2 + b] = __ldcg(p.pool + tg.col_start + col0 + nt * 8 + b);
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int64_t ro = __ldcg(p.pool + tg.row_start + row0 + mt * 16 + 8 * h);
              double *Crow = p.C + ro;
              double old[8];
#pragma unroll
              for (int c = 0; c < 8; ++c) old[c] = (ro == kPad || co[c] == kPad) ? 0.0 : __ldcg(Crow + co[c]);
#pragma unroll
              for (int c = 0; c < 8; ++c)
                if (ro != kPad && co[c] != kPad)
                  __stcg(Crow + co[c], old[c] + tg.sign * acc[mt][c >> 1][2 * h + (c & 1)]);
            }
          if (p.use_tickets) {
            __threadfence();
            named_bar(2, 32 * CONSUMER_WARPS);
            if (tid == 0) st_release_gpu(ticket, tg.order + 1);
          }
        }
      }
    }
  }
}

using GemmKernel = void (*)(const GemmArgs);

static GemmKernel kernel_for(int nraw, int kwin) {
  if (kwin == 16) return k_strassen_gemm<4, 16>;
  if (kwin == 8) return k_strassen_gemm<4, 8>;
  switch (nraw) {
    case 4: return k_strassen_gemm<4, 32>;
    case 5: return k_strassen_gemm<5, 32>;
    case 6: return k_strassen_gemm<6, 32>;
    default: return k_strassen_gemm<7, 32>;
  }
}

// One persistent CTA per SM: 512 threads x 128 registers fill the register file.
int gemm_max_grid(int max_ops) {
  (void)max_ops;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sms;
}

cudaError_t launch_gemm(const GemmArgs &a, int grid, cudaStream_t s) {
  const size_t sm = SmemLayout::bytes(a.max_ops, a.kwin, a.nraw);
  GemmKernel k = kernel_for(a.nraw, a.kwin);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<grid, THREADS, sm, s>>>(a);
  return cudaGetLastError();
}

}  // namespace stc
