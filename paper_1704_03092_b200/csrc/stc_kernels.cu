// stc_kernels.cu -- sm_100a kernels of the Strassen tensor-contraction path.
//
//   k_build_pool      subsystem (1): scatter vectors built on the device, split
//                     into Strassen quadrants, re-ordered into GPU tiles
//                     (replaces scatter.py:26-165 + strassen.py:101-127)
//   k_block_vector    reference block-scatter vectors (scatter.py:26-40)
//   k_strassen_gemm   subsystems (2)+(3): persistent warp-specialised FP64
//                     tensor-core (DMMA) kernel.  Producer warps gather the
//                     Strassen operand sums (e.g. A0+A3, B1-B3) through the
//                     scatter vectors straight into the MMA smem ring
//                     (replaces _jit.pack_a_block/pack_b_block, _jit.py:27-131);
//                     consumer warps run mma.sync.m16n8k4.f64 with register
//                     accumulators over the whole quadrant k (replaces
//                     _jit.microtile/macro_kernel, _jit.py:134-220) and add
//                     +/-M into 1-4 C quadrants through the scatter layout
//                     (replaces _jit.store_tile, _jit.py:158-186), ordered by
//                     per-tile tickets -- no atomics on C, deterministic.
//   k_accumulate      subsystem (4): C_q += sum_t s_t M_t (AB / Naive;
//                     replaces _jit.accum_dense, _jit.py:223-256)
//   k_unpack          subsystem (4): dense operand sums (Naive; replaces
//                     _jit.unpack_sum, _jit.py:259-309)
#include <algorithm>
#include <cstdio>

#include "stc_internal.cuh"

namespace stc {

// ============================================================ PTX helpers ==
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// D(16x8) += A(16x4, row) * B(4x8, col), FP64 tensor core (DMMA).
__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}
__device__ __forceinline__ double ld_nc(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// ====================================================== subsystem (1) ==
// One output entry of a pool vector.
__device__ __forceinline__ int64_t pool_entry(const VecDesc &d, int64_t o) {
  const int64_t q = o / d.q_len_pad;
  const int64_t ip = o - q * d.q_len_pad;
  if (ip >= d.q_len) return kPad;
  if (d.mode == 1) return ip * d.stride;
  // tile order -> quadrant-local reference index
  int64_t i = ip;
  if (d.nbox > 0) {
    int64_t digit[STC_MAX_LABELS];
    int64_t rem = ip;
    for (int j = 0; j < d.nbox; ++j) {
      const int dim = d.order[j];
      digit[dim] = rem % d.box_ext[dim];
      rem /= d.box_ext[dim];
    }
    i = 0;
    int64_t mult = 1;
    for (int dim = 0; dim < d.nbox; ++dim) {
      i += digit[dim] * mult;
      mult *= d.box_ext[dim];
    }
  }
  const int64_t l = q * d.q_len + i;
  if (l >= d.len) return kPad;  // strassen.py:109-110 padding (pad_view)
  int64_t off = d.base, rem = l;
  for (int j = 0; j < d.nlab; ++j) {  // first label fastest (scatter.py:105-112)
    const int64_t e = d.ext[j];
    off += (rem % e) * d.str[j];
    rem /= e;
  }
  return off;
}

__global__ void k_build_pool(const VecDesc *__restrict__ descs, int ndesc, int64_t total, int64_t *__restrict__ pool) {
  extern __shared__ unsigned char sm_raw[];
  VecDesc *sd = reinterpret_cast<VecDesc *>(sm_raw);
  for (int i = threadIdx.x; i < ndesc * (int)(sizeof(VecDesc) / 8); i += blockDim.x)
    reinterpret_cast<int64_t *>(sd)[i] = reinterpret_cast<const int64_t *>(descs)[i];
  __syncthreads();
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int v = 0;
    while (v + 1 < ndesc && o >= sd[v + 1].out_start) ++v;
    const VecDesc &d = sd[v];
    const int64_t local = o - d.out_start;
    if (local < d.nq * d.q_len_pad) pool[o] = pool_entry(d, local);
  }
}

cudaError_t launch_build_pool(const VecDesc *d_descs, int ndesc, int64_t total, int64_t *pool, cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const size_t sm = sizeof(VecDesc) * (size_t)ndesc;
  k_build_pool<<<(int)blocks, threads, sm, s>>>(d_descs, ndesc, total, pool);
  return cudaGetLastError();
}

// scatter.py:26-40, one thread per block.
__global__ void k_block_vector(const int64_t *__restrict__ scat, int64_t len, int64_t blk, int64_t unit,
                               int64_t *__restrict__ out) {
  const int64_t nb = (len + blk - 1) / blk;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = b * blk, hi = min(lo + blk, len);
    int64_t r = 0;
    bool pad = false;
    for (int64_t i = lo; i < hi; ++i) pad |= scat[i] == kPad;
    if (!pad) {
      if (hi - lo == 1) {
        r = unit > 0 ? unit : 0;
      } else {
        const int64_t d = scat[lo + 1] - scat[lo];
        bool ok = d > 0;
        for (int64_t i = lo + 1; ok && i < hi; ++i) ok = scat[i] - scat[i - 1] == d;
        r = ok ? d : 0;
      }
    }
    out[b] = r;
  }
}

cudaError_t launch_block_vector(const int64_t *scat, int64_t len, int64_t blk, int64_t unit, int64_t *out,
                                cudaStream_t s) {
  const int64_t nb = (len + blk - 1) / blk;
  if (nb <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((nb + 255) / 256, 148 * 8);
  k_block_vector<<<blocks, 256, 0, s>>>(scat, len, blk, unit, out);
  return cudaGetLastError();
}

__global__ void k_copy_pad(const int64_t *__restrict__ in, int64_t len, int64_t len_pad, int64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len_pad; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < len ? in[i] : kPad;
}

cudaError_t launch_copy_pad(const int64_t *in, int64_t len, int64_t len_pad, int64_t *out, cudaStream_t s) {
  if (len_pad <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((len_pad + 255) / 256, 148 * 8);
  k_copy_pad<<<blocks, 256, 0, s>>>(in, len, len_pad, out);
  return cudaGetLastError();
}

// ============================================ subsystems (2)+(3): DMMA ==

// Shared-memory carve-up of k_strassen_gemm (dynamic smem).
struct SmemLayout {
  static constexpr size_t stage_doubles = (size_t)BK * LDS;
  static constexpr size_t a_off = 0;
  static constexpr size_t b_off = a_off + STAGES * stage_doubles * 8;
  static constexpr size_t bar_off = b_off + STAGES * stage_doubles * 8;  // full[STAGES], empty[STAGES]
  static constexpr size_t meta_off = bar_off + 2 * STAGES * 8;          // stage_item[STAGES], s_item
  static constexpr size_t tab_off = (meta_off + (STAGES + 4) * 4 + 15) / 16 * 16;
  // tables (int64 / double), sized by max_ops at run time:
  //   xoffA[ops][BM], xoffB[ops][BN], koffA[2][ops][BK], koffB[2][ops][BK],
  //   kstA[ops], kstB[ops], doffA[ops], doffB[ops], sgnA[ops], sgnB[ops]
  static size_t bytes(int ops) {
    return tab_off + 8 * ((size_t)ops * (BM + BN) + 2 * (size_t)ops * 2 * BK + 6 * (size_t)ops);
  }
};

size_t gemm_smem_bytes(int max_ops) { return SmemLayout::bytes(max_ops); }

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

// Gather + Strassen sum of one operand tile into S[k][x] (LDS stride).
//   KFAST = false: thread owns column x = ptid and walks k (x contiguous in memory)
//   KFAST = true : 4 consecutive k per lane quad, 8 x per warp (k contiguous)
// Sums views in table order starting from 0.0, exactly like the reference
// packing (_jit.py:43-78): out = 0; out += coeff_t * view_t for t in order.
// CHECK = false is the fast path: the tile's scatter entries hold no PAD
// (decided per item / chunk with a barrier reduction), so every load is
// unconditional and 4 views x 8 elements stay in flight per thread.
template <bool KFAST, bool CHECK>
__device__ __forceinline__ void gather_side(double *__restrict__ S, const double *__restrict__ D,
                                            const int64_t *__restrict__ xo, int xstride, const int64_t *__restrict__ ko,
                                            const double *__restrict__ sg, const int64_t *__restrict__ doff, int nops,
                                            int ptid) {
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    double acc[8];
    int xs[8], ks[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ee = h * 8 + e;
      if (KFAST) {
        ks[e] = (ptid & 3) + 4 * (ee & 3);
        xs[e] = (ptid >> 2) + 32 * (ee >> 2);
      } else {
        ks[e] = ee;
        xs[e] = ptid;
      }
      acc[e] = 0.0;
    }
    // views two at a time (16 loads in flight per thread), then a tail view
    int op = 0;
#pragma unroll 1
    for (; op + 1 < nops; op += 2) {
      double v0[8], v1[8];
      const double *D0 = D + doff[op], *D1 = D + doff[op + 1];
      const int64_t *x0 = xo + op * xstride, *x1 = x0 + xstride;
      const int64_t *k0 = ko + op * BK, *k1 = k0 + BK;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int64_t a0 = x0[xs[e]], b0 = k0[ks[e]];
        const int64_t a1 = x1[xs[e]], b1 = k1[ks[e]];
        if (CHECK) {
          v0[e] = (a0 == kPad || b0 == kPad) ? 0.0 : ld_nc(D0 + a0 + b0);
          v1[e] = (a1 == kPad || b1 == kPad) ? 0.0 : ld_nc(D1 + a1 + b1);
        } else {
          v0[e] = ld_nc(D0 + a0 + b0);
          v1[e] = ld_nc(D1 + a1 + b1);
        }
      }
      const double s0 = sg[op], s1 = sg[op + 1];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += s0 * v0[e];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += s1 * v1[e];
    }
    if (op < nops) {
      double v0[8];
      const double *D0 = D + doff[op];
      const int64_t *x0 = xo + op * xstride;
      const int64_t *k0 = ko + op * BK;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int64_t a0 = x0[xs[e]], b0 = k0[ks[e]];
        if (CHECK)
          v0[e] = (a0 == kPad || b0 == kPad) ? 0.0 : ld_nc(D0 + a0 + b0);
        else
          v0[e] = ld_nc(D0 + a0 + b0);
      }
      const double s0 = sg[op];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += s0 * v0[e];
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) S[ks[e] * LDS + xs[e]] = acc[e];
  }
}

template <bool CHECK>
__device__ __forceinline__ void gather_tiles(const GemmArgs &p, double *SA, double *SB, const int64_t *xoffA,
                                             const int64_t *xoffB, const int64_t *kA, const int64_t *kB,
                                             const double *sgnA, const double *sgnB, const int64_t *doffA,
                                             const int64_t *doffB, int na, int nb, int ptid) {
  if (p.a_kfast)
    gather_side<true, CHECK>(SA, p.A, xoffA, BM, kA, sgnA, doffA, na, ptid);
  else
    gather_side<false, CHECK>(SA, p.A, xoffA, BM, kA, sgnA, doffA, na, ptid);
  if (p.b_kfast)
    gather_side<true, CHECK>(SB, p.B, xoffB, BN, kB, sgnB, doffB, nb, ptid);
  else
    gather_side<false, CHECK>(SB, p.B, xoffB, BN, kB, sgnB, doffB, nb, ptid);
}

// bar.sync over the producer threads that also ORs a predicate across them.
__device__ __forceinline__ bool named_bar_or(int id, int nthreads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.u32 p, %1, 0;\n"
      "bar.red.or.pred q, %2, %3, p;\n"
      "selp.u32 %0, 1, 0, q;\n"
      "}\n"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}

__global__ void __launch_bounds__(THREADS, 1) k_strassen_gemm(const GemmArgs p) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *sA = reinterpret_cast<double *>(smem + SmemLayout::a_off);
  double *sB = reinterpret_cast<double *>(smem + SmemLayout::b_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SmemLayout::bar_off);
  uint64_t *empty = full + STAGES;
  int *stage_item = reinterpret_cast<int *>(smem + SmemLayout::meta_off);
  int *s_item = stage_item + STAGES;
  const int mo = p.max_ops;
  int64_t *xoffA = reinterpret_cast<int64_t *>(smem + SmemLayout::tab_off);
  int64_t *xoffB = xoffA + mo * BM;
  int64_t *koffA = xoffB + mo * BN;  // [2][mo][BK]
  int64_t *koffB = koffA + 2 * mo * BK;
  int64_t *kstA = koffB + 2 * mo * BK;
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
      for (int i = ptid; i < na; i += nprod) {
        const OpDesc o = p.ops[td.a_first + i];
        kstA[i] = o.k_start;
        doffA[i] = o.data_off;
        sgnA[i] = o.sign;
      }
      for (int i = ptid; i < nb; i += nprod) {
        const OpDesc o = p.ops[td.b_first + i];
        kstB[i] = o.k_start;
        doffB[i] = o.data_off;
        sgnB[i] = o.sign;
      }
      bool pad = false;  // any PAD among this tile's x entries (item-wide)
      for (int idx = ptid; idx < na * BM; idx += nprod) {
        const int op = idx / BM, x = idx - op * BM;
        const int64_t v = p.pool[p.ops[td.a_first + op].x_start + (int64_t)ti * BM + x];
        pad |= v == kPad;
        xoffA[idx] = v;
      }
      for (int idx = ptid; idx < nb * BN; idx += nprod) {
        const int op = idx / BN, x = idx - op * BN;
        const int64_t v = p.pool[p.ops[td.b_first + op].x_start + (int64_t)tj * BN + x];
        pad |= v == kPad;
        xoffB[idx] = v;
      }
      const bool xpad = named_bar_or(1, nprod, pad);
      // k-offset table of chunk 0
      pad = false;
      for (int idx = ptid; idx < (na + nb) * BK; idx += nprod) {
        const int op = idx / BK, k = idx - op * BK;
        const int64_t v = op < na ? p.pool[kstA[op] + k] : p.pool[kstB[op - na] + k];
        pad |= v == kPad;
        if (op < na)
          koffA[op * BK + k] = v;
        else
          koffB[(op - na) * BK + k] = v;
      }
      bool kpad = named_bar_or(1, nprod, pad);
      for (int kc = 0; kc < p.kchunks; ++kc) {
        const int kb = kc & 1;
        // prefetch the next chunk's k offsets (at most 2*MAX_OPS*BK/128 = 4 per thread)
        int64_t pre[4];
        const bool more = kc + 1 < p.kchunks;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int idx = ptid + r * nprod;
          pre[r] = 0;
          if (more && idx < (na + nb) * BK) {
            const int op = idx / BK, k = idx - op * BK;
            const int64_t base = op < na ? kstA[op] : kstB[op - na];
            pre[r] = p.pool[base + (int64_t)(kc + 1) * BK + k];
          }
        }
        mbar_wait(&empty[stage], phase ^ 1);
        double *SA = sA + stage * SmemLayout::stage_doubles;
        double *SB = sB + stage * SmemLayout::stage_doubles;
        const int64_t *kA = koffA + kb * mo * BK;
        const int64_t *kB = koffB + kb * mo * BK;
        if (xpad || kpad || p.force_slow)
          gather_tiles<true>(p, SA, SB, xoffA, xoffB, kA, kB, sgnA, sgnB, doffA, doffB, na, nb, ptid);
        else
          gather_tiles<false>(p, SA, SB, xoffA, xoffB, kA, kB, sgnA, sgnB, doffA, doffB, na, nb, ptid);
        if (ptid == 0) stage_item[stage] = item;
        mbar_arrive(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
        pad = false;
        if (more) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int idx = ptid + r * nprod;
            if (idx < (na + nb) * BK) {
              const int op = idx / BK, k = idx - op * BK;
              pad |= pre[r] == kPad;
              if (op < na)
                koffA[((kb ^ 1) * mo + op) * BK + k] = pre[r];
              else
                koffB[((kb ^ 1) * mo + op - na) * BK + k] = pre[r];
            }
          }
        }
        kpad = named_bar_or(1, nprod, pad);
      }
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
            for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
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

int gemm_max_grid(int max_ops) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t sm = SmemLayout::bytes(max_ops);
  cudaFuncSetAttribute(k_strassen_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_strassen_gemm, THREADS, sm);
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

cudaError_t launch_gemm(const GemmArgs &a, int grid, cudaStream_t s) {
  const size_t sm = SmemLayout::bytes(a.max_ops);
  cudaError_t e = cudaFuncSetAttribute(k_strassen_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_strassen_gemm<<<grid, THREADS, sm, s>>>(a);
  return cudaGetLastError();
}

// ======================================================= subsystem (4) ==
// C_q(i,j) += s_1 M_1(i,j) + s_2 M_2(i,j) + ... in term order, one RMW per
// element (bitwise the reference's per-term accum_dense sequence).
__global__ void k_accumulate(const AccArgs a) {
  const int q = blockIdx.y;
  const int64_t total = a.mq * a.nq;
  const int64_t rs = a.row_start[q], cs = a.col_start[q];
  const int l0 = a.list_start[q], l1 = a.list_start[q + 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / a.nq, j = e - i * a.nq;
    const int64_t ro = a.pool[rs + i], co = a.pool[cs + j];
    if (ro == kPad || co == kPad) continue;
    double v = a.C[ro + co];
    const double *m = a.M + i * a.m_ld + j;
    for (int l = l0; l < l1; ++l) v += a.list_sign[l] * __ldcs(m + (int64_t)a.list_slot[l] * a.m_stride);
    a.C[ro + co] = v;
  }
}

cudaError_t launch_accumulate(const AccArgs &a, cudaStream_t s) {
  const int64_t total = a.mq * a.nq;
  if (total <= 0 || a.nquads <= 0) return cudaSuccess;
  int bx = (int)std::min<int64_t>((total + 255) / 256, 4096);
  dim3 grid(bx, a.nquads);
  k_accumulate<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// out_slot[k*x_len + x] = sum_op sign * D[x_vec[x] + k_vec[k]]  (view order, PAD -> 0)
__global__ void k_unpack(const UnpackArgs a) {
  const int t = blockIdx.y;
  const TermDesc td = a.terms[t];
  double *out = a.out + (int64_t)td.m_slot * a.slot_stride;
  const int64_t total = a.x_len * a.k_len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / a.x_len, x = e - k * a.x_len;
    double acc = 0.0;
    for (int o = 0; o < td.a_count; ++o) {
      const OpDesc op = a.ops[td.a_first + o];
      const int64_t xo = a.pool[op.x_start + x], ko = a.pool[op.k_start + k];
      if (xo == kPad || ko == kPad) continue;
      acc += op.sign * a.D[op.data_off + xo + ko];
    }
    out[e] = acc;
  }
}

cudaError_t launch_unpack(const UnpackArgs &a, cudaStream_t s) {
  const int64_t total = a.x_len * a.k_len;
  if (total <= 0 || a.nterms <= 0) return cudaSuccess;
  int bx = (int)std::min<int64_t>((total + 255) / 256, 2048);
  dim3 grid(bx, a.nterms);
  k_unpack<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ---- standalone helpers for the kernel-level API --------------------------
__global__ void k_accum_dense_single(const double *__restrict__ M, int64_t ldm, int64_t m, int64_t n,
                                     double *__restrict__ C, const int64_t *__restrict__ rows,
                                     const int64_t *__restrict__ cols, double coeff) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;  // column-major M: coalesced along i
    const int64_t ro = rows[i], co = cols[j];
    if (ro == kPad || co == kPad) continue;
    C[ro + co] += coeff * M[i + j * ldm];
  }
}

cudaError_t launch_accum_dense_single(const double *M, int64_t ldm, int64_t m, int64_t n, double *C,
                                      const int64_t *rows, const int64_t *cols, double coeff, cudaStream_t s) {
  const int64_t total = m * n;
  if (total <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_accum_dense_single<<<blocks, 256, 0, s>>>(M, ldm, m, n, C, rows, cols, coeff);
  return cudaGetLastError();
}

__global__ void k_unpack_views(double *__restrict__ out, int64_t ldo, int64_t m, int64_t n,
                               const double *__restrict__ data, const ViewSet vs) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    double acc = 0.0;
    for (int t = 0; t < vs.n; ++t) {
      const int64_t ro = vs.rows[t][i], co = vs.cols[t][j];
      if (ro == kPad || co == kPad) continue;
      acc += vs.coeff[t] * data[ro + co];
    }
    out[i + j * ldo] = acc;
  }
}

cudaError_t launch_unpack_views(double *out, int64_t ldo, int64_t m, int64_t n, const double *data, const ViewSet &vs,
                                cudaStream_t s) {
  const int64_t total = m * n;
  if (total <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_unpack_views<<<blocks, 256, 0, s>>>(out, ldo, m, n, data, vs);
  return cudaGetLastError();
}

// ---- deterministic squared norms over strided tensors ----------------------
struct NormShape {
  int ndim;
  int64_t ext[STC_MAX_LABELS], xs[STC_MAX_LABELS], rs[STC_MAX_LABELS];
};

__global__ void k_sq_norms(const NormShape sh, int64_t total, const double *__restrict__ x, int64_t xb,
                           const double *__restrict__ r, int64_t rb, double *__restrict__ partials) {
  __shared__ double s0[256], s1[256];
  double a0 = 0.0, a1 = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e, xo = xb, ro = rb;
    for (int d = 0; d < sh.ndim; ++d) {
      const int64_t i = rem % sh.ext[d];
      rem /= sh.ext[d];
      xo += i * sh.xs[d];
      ro += i * sh.rs[d];
    }
    const double rv = r[ro], dv = x[xo] - rv;
    a0 += dv * dv;
    a1 += rv * rv;
  }
  s0[threadIdx.x] = a0;
  s1[threadIdx.x] = a1;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      s0[threadIdx.x] += s0[threadIdx.x + w];
      s1[threadIdx.x] += s1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s0[0];
    partials[2 * blockIdx.x + 1] = s1[0];
  }
}

cudaError_t launch_sq_norms(int ndim, const int64_t *ext, const double *x, const int64_t *xs, int64_t xb,
                            const double *r, const int64_t *rs, int64_t rb, double *partials, int nblocks,
                            cudaStream_t s) {
  NormShape sh{};
  sh.ndim = ndim;
  int64_t total = 1;
  for (int d = 0; d < ndim; ++d) {
    sh.ext[d] = ext[d];
    sh.xs[d] = xs[d];
    sh.rs[d] = rs[d];
    total *= ext[d];
  }
  k_sq_norms<<<nblocks, 256, 0, s>>>(sh, total, x, xb, r, rb, partials);
  return cudaGetLastError();
}

}  // namespace stc
