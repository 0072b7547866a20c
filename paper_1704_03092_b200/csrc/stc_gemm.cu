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
  // xoffA[ops][BM], xoffB[ops][BN], kstA[ops], kstB[ops], doffA[ops], doffB[ops],
  // sgnA[ops], sgnB[ops], then raw[nraw][BK][128] (thread-private, see raw_index)
  __host__ __device__ static size_t tab_bytes(int ops) { return 8 * ((size_t)ops * (BM + BN) + 6 * (size_t)ops); }
  __host__ __device__ static size_t raw_off(int ops) { return (tab_off + tab_bytes(ops) + 127) / 128 * 128; }
  static constexpr size_t raw_doubles = (size_t)BK * 128;  // one thread-private raw slot
  __host__ __device__ static size_t bytes(int ops, int nraw) { return raw_off(ops) + (size_t)nraw * raw_doubles * 8; }
};

constexpr size_t kMaxSmem = 227 * 1024;

int gemm_nraw(int max_ops) {
  int n = MAX_NRAW;
  if (const char *e = getenv("STC_NRAW")) n = std::max(4, std::min(MAX_NRAW, atoi(e)));
  while (n > 4 && SmemLayout::bytes(max_ops, n) > kMaxSmem) --n;
  return n;
}

size_t gemm_smem_bytes(int max_ops) { return SmemLayout::bytes(max_ops, gemm_nraw(max_ops)); }

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

// Element e of a producer thread's 16 in a [BK][LDS] tile:
//   kfast = 0: x = ptid, k = e (x contiguous in memory)
//   kfast = 1: k = (ptid & 3) + 4 (e & 3), x = (ptid >> 2) + 32 (e >> 2) (k contiguous)
__device__ __forceinline__ int tile_index(int kfast, int ptid, int e) {
  return kfast ? ((ptid & 3) + 4 * (e & 3)) * LDS + (ptid >> 2) + 32 * (e >> 2) : e * LDS + ptid;
}

// Raw slots are private to each producer thread, independent of the side's
// mapping: element e of thread ptid lives at e * 128 + ptid (conflict-free).
// (A slot alternately holds A- and B-side units whose tile mappings differ, so
// a tile-position layout would let one thread's cp.async land on data another
// thread has not read yet.)
__device__ __forceinline__ int raw_index(int ptid, int e) { return e * 128 + ptid; }

// cp.async one unit into a raw slot (zero-fill for PAD).
__device__ __forceinline__ void issue_unit(double *__restrict__ dst, const double *__restrict__ D,
                                           const int64_t *__restrict__ xop, const int64_t *__restrict__ kvec,
                                           int64_t kstr, int kfast, bool slow, int ptid) {
  if (!slow && kstr != kIrregular) {
    const int64_t b0 = kvec[0];
    if (!kfast) {
      const int64_t a = xop[ptid];
      const bool ok = a != kPad;
      const double *src = ok ? D + a + b0 : D;
#pragma unroll
      for (int e = 0; e < 16; ++e) cp_async8(dst + raw_index(ptid, e), ok ? src + e * kstr : D, ok);
    } else {
      const double *base = D + b0 + (ptid & 3) * kstr;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t a = xop[(ptid >> 2) + 32 * j];
        const bool ok = a != kPad;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          cp_async8(dst + raw_index(ptid, 4 * j + i), ok ? base + a + 4 * i * kstr : D, ok);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int x = kfast ? (ptid >> 2) + 32 * (e >> 2) : ptid;
      const int k = kfast ? (ptid & 3) + 4 * (e & 3) : e;
      const int64_t a = xop[x], b = __ldg(kvec + k);
      const bool ok = a != kPad && b != kPad;
      cp_async8(dst + raw_index(ptid, e), ok ? D + a + b : D, ok);
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

template <int NRAW>
__global__ void __launch_bounds__(THREADS, 1) k_strassen_gemm(const GemmArgs p) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *sA = reinterpret_cast<double *>(smem + SmemLayout::a_off);
  double *sB = reinterpret_cast<double *>(smem + SmemLayout::b_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SmemLayout::bar_off);
  uint64_t *empty = full + STAGES;
  int *stage_item = reinterpret_cast<int *>(smem + SmemLayout::meta_off);
  int *s_item = stage_item + STAGES;
  const int mo = p.max_ops;
  constexpr int nraw = NRAW;
  double *raw = reinterpret_cast<double *>(smem + SmemLayout::raw_off(mo));
  int64_t *xoffA = reinterpret_cast<int64_t *>(smem + SmemLayout::tab_off);
  int64_t *xoffB = xoffA + mo * BM;
  int64_t *kstA = xoffB + mo * BN;
  int64_t *kstB = kstA + mo;
  int64_t *doffA = kstB + mo;
  int64_t *doffB = doffA + mo;
  double *sgnA = reinterpret_cast<double *>(doffB + mo);
  double *sgnB = sgnA + mo;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 32 * PRODUCER_WARPS);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
  }
  __syncthreads();

  if (warp >= CONSUMER_WARPS) {
    // ===================== producer warps: gather + Strassen sums =====
#ifndef STC_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
#endif
    const int ptid = tid - 32 * CONSUMER_WARPS;
    const int nprod = 32 * PRODUCER_WARPS;
    const bool force_slow = p.force_slow != 0;
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      if (ptid == 0) *s_item = atomicAdd(p.counter, 1);
      named_bar(1, nprod);
      const int item = *s_item;
      if (item >= p.total_items) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (ptid == 0) stage_item[stage] = -1;
        mbar_arrive(&full[stage]);
        break;
      }
      int slot, ti, tj;
      tile_of(p, item, slot, ti, tj);
      const TermDesc td = p.terms[slot];
      const int na = td.a_count, nb = td.b_count;
      const int U = na + nb;  // units per chunk: every view of A, then of B
      for (int i = ptid; i < U; i += nprod) {
        const OpDesc o = p.ops[i < na ? td.a_first + i : td.b_first + i - na];
        if (i < na) {
          kstA[i] = o.k_start;
          doffA[i] = o.data_off;
          sgnA[i] = o.sign;
        } else {
          kstB[i - na] = o.k_start;
          doffB[i - na] = o.data_off;
          sgnB[i - na] = o.sign;
        }
      }
      for (int idx = ptid; idx < na * BM; idx += nprod) {
        const int op = idx / BM, x = idx - op * BM;
        xoffA[idx] = p.pool[p.ops[td.a_first + op].x_start + (int64_t)ti * BM + x];
      }
      for (int idx = ptid; idx < nb * BN; idx += nprod) {
        const int op = idx / BN, x = idx - op * BN;
        xoffB[idx] = p.pool[p.ops[td.b_first + op].x_start + (int64_t)tj * BN + x];
      }
      named_bar(1, nprod);

      const int G = p.kchunks * U;
      constexpr int D = NRAW - 1;  // units in flight ahead of the one being summed
      int ig = 0, ic = 0, iu = 0, islot = 0;  // issue cursor
      int cu = 0, cslot = 0;                  // consume cursor
      auto issue = [&]() {
        if (ig < G) {
          const bool is_a = iu < na;
          const int op = is_a ? iu : iu - na;
          const int64_t kst = (is_a ? kstA : kstB)[op] + (int64_t)ic * BK;
          const int64_t kstr = __ldg(p.kbs + (kst >> 4));
          issue_unit(raw + islot * SmemLayout::raw_doubles, (is_a ? p.A : p.B) + (is_a ? doffA : doffB)[op],
                     is_a ? xoffA + op * BM : xoffB + op * BN, p.pool + kst, kstr, is_a ? p.a_kfast : p.b_kfast,
                     force_slow, ptid);
          if (++iu == U) {
            iu = 0;
            ++ic;
          }
          if (++islot == nraw) islot = 0;
        }
        cp_async_commit();  // empty groups at the tail keep the wait count uniform
        ++ig;
      };
      for (int d = 0; d < D; ++d) issue();
      double acc[16];
      for (int g = 0; g < G; ++g) {
        issue();
        cp_async_wait<D>();  // unit g has landed (this thread's own copies)
        const bool is_a = cu < na;
        const int op = is_a ? cu : cu - na;
        const int kfast = is_a ? p.a_kfast : p.b_kfast;
        const double *src = raw + cslot * SmemLayout::raw_doubles;
        if (op == 0) {
          const uint64_t sb = (is_a ? sgnA : sgnB)[0] < 0 ? 0x8000000000000000ull : 0ull;
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[e] = first_term(src[raw_index(ptid, e)], sb);
        } else {
          const double s = (is_a ? sgnA : sgnB)[op];
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[e] += s * src[raw_index(ptid, e)];
        }
        if (++cslot == nraw) cslot = 0;
        if (op == (is_a ? na : nb) - 1) {  // side complete: store its sum into the MMA ring
          if (is_a) mbar_wait(&empty[stage], phase ^ 1);
          double *S = (is_a ? sA : sB) + stage * SmemLayout::stage_doubles;
#pragma unroll
          for (int e = 0; e < 16; ++e) S[tile_index(kfast, ptid, e)] = acc[e];
        }
        if (++cu == U) {
          cu = 0;
          if (ptid == 0) stage_item[stage] = item;
          mbar_arrive(&full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
#ifdef STC_EXPERIMENT_CHUNKBAR
          named_bar(1, nprod);
#endif
        }
      }
      cp_async_wait<0>();
      named_bar(1, nprod);  // tables of this item fully used before the next fill
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

static GemmKernel kernel_for(int nraw) {
  switch (nraw) {
    case 4: return k_strassen_gemm<4>;
    case 5: return k_strassen_gemm<5>;
    case 6: return k_strassen_gemm<6>;
    default: return k_strassen_gemm<7>;
  }
}

int gemm_max_grid(int max_ops) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nraw = gemm_nraw(max_ops);
  const size_t sm = SmemLayout::bytes(max_ops, nraw);
  GemmKernel k = kernel_for(nraw);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, sm);
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

cudaError_t launch_gemm(const GemmArgs &a, int grid, cudaStream_t s) {
  const size_t sm = SmemLayout::bytes(a.max_ops, a.nraw);
  GemmKernel k = kernel_for(a.nraw);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<grid, THREADS, sm, s>>>(a);
  return cudaGetLastError();
}

}  // namespace stc
