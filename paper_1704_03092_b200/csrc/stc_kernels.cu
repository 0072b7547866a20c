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
#include "stc_ptx.cuh"

namespace stc {

// ====================================================== subsystem (1) ==
// One output entry of a pool vector.
__device__ __forceinline__ int64_t pool_entry(const VecDesc &d, int64_t o) {
  const int64_t q = o / d.q_len_pad;
  const int64_t ip = o - q * d.q_len_pad;
  if (ip >= d.q_len) return kPad;
  if (d.mode == 1) return ip * d.stride;
  if (d.mode == 2) return q * d.base + ip * d.stride;  // packed quadrant blocks (quadrant stride in `base`)
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

// Block-scatter vector of the whole pool at GPU-chunk granularity (BK entries):
// the constant stride of the chunk, or INT64_MIN if it has none or holds PAD.
// The DMMA producer addresses a regular chunk as base + k * stride.
__global__ void k_chunk_strides(const int64_t *__restrict__ pool, int64_t nchunks, int64_t *__restrict__ kbs) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t *v = pool + c * BK;
    int64_t prev = v[0];
    bool ok = prev != kPad;
    const int64_t d = v[1] - v[0];
    for (int k = 1; ok && k < BK; ++k) {
      const int64_t x = v[k];
      ok = x != kPad && x - prev == d;
      prev = x;
    }
    kbs[c] = ok ? d : kPad;
  }
}

cudaError_t launch_chunk_strides(const int64_t *pool, int64_t nchunks, int64_t *kbs, cudaStream_t s) {
  if (nchunks <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((nchunks + 255) / 256, 148 * 8);
  k_chunk_strides<<<blocks, 256, 0, s>>>(pool, nchunks, kbs);
  return cudaGetLastError();
}

__global__ void k_copy_pad(const int64_t *__restrict__ in, int64_t len, int64_t len_pad, int64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len_pad; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < len ? in[i] : kPad;
}

// Staged upload of a host table: SMs read the page-locked staging buffer over
// PCIe (UVA pointer) and write HBM.  Kept off the copy engines on purpose: a
// cudaMemcpyAsync of a few KB would queue behind any bulk host->device
// transfer in flight (stc_contract_host's operand uploads), stalling the
// launch that needs the table.  Optionally zeroes a second device range.
__global__ void k_stage(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, size_t n, uint8_t *z, size_t zn) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
  size_t done = 0;
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const size_t n16 = n / 16;
    for (size_t i = t; i < n16; i += step) reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    done = n16 * 16;
  }
  for (size_t i = done + t; i < n; i += step) dst[i] = src[i];
  done = 0;
  if (((uintptr_t)z & 15) == 0) {
    const size_t z16 = zn / 16;
    for (size_t i = t; i < z16; i += step) reinterpret_cast<uint4 *>(z)[i] = make_uint4(0, 0, 0, 0);
    done = z16 * 16;
  }
  for (size_t i = done + t; i < zn; i += step) z[i] = 0;
}

cudaError_t launch_stage(const void *host_src, void *dst, size_t bytes, void *zero, size_t zero_bytes,
                         cudaStream_t s) {
  const size_t work = std::max(bytes, zero_bytes) / 16 + 1;
  const int blocks = (int)std::min<size_t>((work + 255) / 256, 64);
  k_stage<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint8_t *>(host_src), reinterpret_cast<uint8_t *>(dst),
                                 bytes, reinterpret_cast<uint8_t *>(zero), zero_bytes);
  return cudaGetLastError();
}

cudaError_t launch_copy_pad(const int64_t *in, int64_t len, int64_t len_pad, int64_t *out, cudaStream_t s) {
  if (len_pad <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((len_pad + 255) / 256, 148 * 8);
  k_copy_pad<<<blocks, 256, 0, s>>>(in, len, len_pad, out);
  return cudaGetLastError();
}

// ======================================================= subsystem (4) ==
// C_q(i,j) += s_1 M_1(i,j) + s_2 M_2(i,j) + ... in term order, one RMW per
// element (bitwise the reference's per-term accum_dense sequence).
__global__ void k_accumulate(const AccArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  if (a.c_ready) {  // stc_set_c_ready: C's upload may still be in flight
    if (threadIdx.x == 0) {
      int v;
      do {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a.c_ready) : "memory");
        if (v == 0) __nanosleep(256);
      } while (v == 0);
    }
    __syncthreads();
  }
  // blockIdx.x = quadrant (fastest): the blocks of one element chunk of every quadrant
  // run together, so an M slot's chunk -- read by each quadrant the term targets (1-4) --
  // comes from DRAM once and from L2 after (cfg2 AB L2: 144 slot reads for 49 slots)
  const int q = blockIdx.x;
  const int64_t total = a.mq * a.nq;
  const int64_t rs = a.row_start[q], cs = a.col_start[q];
  const int l0 = a.list_start[q], l1 = a.list_start[q + 1];
  for (int64_t e = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.y * blockDim.x) {
    const int64_t i = e / a.nq, j = e - i * a.nq;
    const int64_t ro = a.pool[rs + i], co = a.pool[cs + j];
    if (ro == kPad || co == kPad) continue;
    double v = a.C[ro + co];
    const double *m = a.M + i * a.m_ld + j;
#pragma unroll 4
    for (int l = l0; l < l1; ++l) v += a.list_sign[l] * __ldg(m + (int64_t)a.list_slot[l] * a.m_stride);
    a.C[ro + co] = v;
  }
}

cudaError_t launch_accumulate(const AccArgs &a, cudaStream_t s) {
  const int64_t total = a.mq * a.nq;
  if (total <= 0 || a.nquads <= 0) return cudaSuccess;
  const int by = (int)std::min<int64_t>((total + 255) / 256, 65535);
  dim3 grid(a.nquads, by);
  return launch_pdl(k_accumulate, grid, dim3(256), 0, s, a);
}

// out_slot[k*x_len + x] (or [x*k_len + k] when kfast) = sum_op sign * D[x_vec[x] + k_vec[k]]
// (view order, PAD -> 0)
__global__ void k_unpack(const UnpackArgs a) {
  const int t = blockIdx.y;
  const TermDesc td = a.terms[t];
  double *out = a.out + (int64_t)td.m_slot * a.slot_stride;
  const int64_t total = a.x_len * a.k_len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    // the slot layout follows the source's unit stride, so both sides of the copy coalesce
    int64_t k, x;
    if (a.kfast) {
      x = e / a.k_len;
      k = e - x * a.k_len;
    } else {
      k = e / a.x_len;
      x = e - k * a.x_len;
    }
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


// ---- operand repacking for the fused kernel (irregular layouts) -------------
// Block (qa, qb) = (blockIdx.y / Q, blockIdx.y % Q) of one operand side is the
// view of x-quadrant (xfirst ? qa : qb) and k-quadrant (the other) copied into a
// dense [k][x] (kfast = 0) or [x][k] (kfast = 1) block, PAD -> 0.  A pure copy:
// the Strassen sums stay in the fused kernel, in the reference's view order.
#ifndef STC_PACK_ROWS
#define STC_PACK_ROWS 8
#endif
constexpr int UNPACK_ROWS = STC_PACK_ROWS;  // k_pack_views: rows of the slow dimension per block

__global__ void __launch_bounds__(256) k_pack_views(const double *__restrict__ D, const int64_t *__restrict__ pool,
                                                    PackArgs a, double *__restrict__ out) {
  // block: 256 positions along the packed block's contiguous dimension x
  // UNPACK_ROWS of the other (as k_unpack); blockIdx.y = quadrant pair
  const int qa = blockIdx.y / a.Q, qb = blockIdx.y - qa * a.Q;
  const int xq = a.xfirst ? qa : qb, kq = a.xfirst ? qb : qa;
  const int64_t *xv = pool + a.xv + (int64_t)xq * a.xlen;
  const int64_t *kv = pool + a.kv + (int64_t)kq * a.klen;
  double *o = out + (int64_t)blockIdx.y * a.xlen * a.klen;
  const int64_t fast_len = a.kfast ? a.klen : a.xlen, slow_len = a.kfast ? a.xlen : a.klen;
  const int64_t *fv = a.kfast ? kv : xv, *sv = a.kfast ? xv : kv;
  // blockIdx.x = row block * fast blocks + fast block (a long k of a tall-skinny problem
  // exceeds the 65535 blocks of grid.y)
  const int64_t bx = blockIdx.x % a.fast_blocks, by = blockIdx.x / a.fast_blocks;
  const int64_t f = FastMap(a.ustep, a.ugroup, blockDim.x).pos(bx, threadIdx.x, blockDim.x, fast_len);
  if (f < 0) return;
  const int64_t fo = __ldg(fv + f);
  const int64_t s0 = by * UNPACK_ROWS;
  // all of the thread's gathers in flight before the first store
  int64_t so[UNPACK_ROWS];
  double v[UNPACK_ROWS];
#pragma unroll
  for (int r = 0; r < UNPACK_ROWS; ++r) so[r] = s0 + r < slow_len ? __ldg(sv + s0 + r) : kPad;
#pragma unroll
  for (int r = 0; r < UNPACK_ROWS; ++r) v[r] = (fo == kPad || so[r] == kPad) ? 0.0 : __ldg(D + fo + so[r]);
#pragma unroll
  for (int r = 0; r < UNPACK_ROWS; ++r)
    if (s0 + r < slow_len) o[(s0 + r) * fast_len + f] = v[r];
}

cudaError_t launch_pack_views(const double *D, const int64_t *pool, const PackArgs &a0, double *out, cudaStream_t s) {
  PackArgs a = a0;
  const int64_t fast_len = a.kfast ? a.klen : a.xlen, slow_len = a.kfast ? a.xlen : a.klen;
  if (fast_len <= 0 || slow_len <= 0) return cudaSuccess;
  const int64_t gy = (slow_len + UNPACK_ROWS - 1) / UNPACK_ROWS;
  a.fast_blocks = FastMap(a.ustep, a.ugroup, 256).blocks(fast_len, 256);
  if (a.fast_blocks * gy > INT32_MAX || a.Q * a.Q > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)(a.fast_blocks * gy), (unsigned)(a.Q * a.Q));
  k_pack_views<<<grid, 256, 0, s>>>(D, pool, a, out);
  return cudaGetLastError();
}

// ---- pre-summed Strassen operands (k_presum) ---------------------------------
// The level-1 table (strassen.py:56-65; quadrants 0 TL, 1 TR, 2 BL, 3 BR), per
// side: views per term, quadrant and sign of each view.
constexpr int kL1Cnt[2][7] = {{2, 2, 1, 1, 2, 2, 2}, {2, 1, 2, 2, 1, 2, 2}};
constexpr int kL1Q[2][7][2] = {{{0, 3}, {2, 3}, {0, 0}, {3, 0}, {0, 1}, {2, 0}, {1, 3}},
                               {{0, 3}, {0, 0}, {1, 3}, {2, 0}, {3, 0}, {0, 1}, {2, 3}}};
constexpr int kL1S[2][7][2] = {{{1, 1}, {1, 1}, {1, 1}, {1, 1}, {1, 1}, {1, -1}, {1, -1}},
                               {{1, 1}, {1, 1}, {1, -1}, {1, -1}, {1, 1}, {1, 1}, {1, 1}}};

// View O of term T at level L <= 3 (strassen.py:70-94: outer level first -- term
// t1 * 7^(L-1) + ..., view order outer-major, quadrant q1 * 4^(L-1) + ..., sign the
// product), as (x quadrant, k quadrant, sign) of the side.
constexpr int ps_pow7(int l) { return l <= 0 ? 1 : 7 * ps_pow7(l - 1); }
template <int L, int SIDE, int T>
struct PsTerm {
  // base-7 digits of T, outer level first (unused levels: term 2, a single + view of quadrant 0)
  static constexpr int t1 = T / ps_pow7(L - 1);
  static constexpr int t2 = L >= 2 ? (T / ps_pow7(L - 2)) % 7 : 2;
  static constexpr int t3 = L >= 3 ? T % 7 : 2;
  static constexpr int n2 = L >= 2 ? kL1Cnt[SIDE][t2] : 1;
  static constexpr int n3 = L >= 3 ? kL1Cnt[SIDE][t3] : 1;
  static constexpr int count = kL1Cnt[SIDE][t1] * n2 * n3;
};
template <int L, int SIDE, int T, int O>
struct PsOp {
  using TT = PsTerm<L, SIDE, T>;
  static constexpr int o1 = O / (TT::n2 * TT::n3), o2 = (O / TT::n3) % TT::n2, o3 = O % TT::n3;
  static constexpr int q1 = kL1Q[SIDE][TT::t1][o1];
  static constexpr int q2 = L >= 2 ? kL1Q[SIDE][TT::t2][o2] : 0;
  static constexpr int q3 = L >= 3 ? kL1Q[SIDE][TT::t3][o3] : 0;
  static constexpr int sign = kL1S[SIDE][TT::t1][o1] * (L >= 2 ? kL1S[SIDE][TT::t2][o2] : 1) *
                              (L >= 3 ? kL1S[SIDE][TT::t3][o3] : 1);
  // quad_rc: row / column bits of the quadrant path, outer level most significant
  static constexpr int r = L == 3 ? 4 * (q1 >> 1) + 2 * (q2 >> 1) + (q3 >> 1) : L == 2 ? 2 * (q1 >> 1) + (q2 >> 1) : q1 >> 1;
  static constexpr int c = L == 3 ? 4 * (q1 & 1) + 2 * (q2 & 1) + (q3 & 1) : L == 2 ? 2 * (q1 & 1) + (q2 & 1) : q1 & 1;
  static constexpr int xq = SIDE == 0 ? r : c, kq = SIDE == 0 ? c : r;
};

// s (+/-) the remaining views of term T, in view order
template <int L, int SIDE, int T, int O, int Q>
__device__ __forceinline__ double ps_rest(const double (&v)[Q][Q], double s) {
  if constexpr (O < PsTerm<L, SIDE, T>::count) {
    using op = PsOp<L, SIDE, T, O>;
    s = op::sign > 0 ? __dadd_rn(s, v[op::xq][op::kq]) : __dsub_rn(s, v[op::xq][op::kq]);
    return ps_rest<L, SIDE, T, O + 1, Q>(v, s);
  } else {
    return s;
  }
}

// terms [T0, T1) in order (split in halves: 7^3 terms exceed the compiler's linear recursion depth)
template <int L, int SIDE, int T0, int T1, int Q>
__device__ __forceinline__ void ps_terms(const PresumArgs &a, const double (&v)[Q][Q], int64_t pos) {
  if constexpr (T1 - T0 == 1) {
    constexpr int T = T0;
    const int slot = a.slot[T];
    if (slot >= 0) {
      using op0 = PsOp<L, SIDE, T, 0>;
      const double v0 = v[op0::xq][op0::kq];
      // first view: sign applied by flipping the sign bit (the fused kernel's in-SM sums)
      double s = op0::sign > 0 ? v0 : __hiloint2double(__double2hiint(v0) ^ static_cast<int>(0x80000000u),
                                                        __double2loint(v0));
      s = ps_rest<L, SIDE, T, 1, Q>(v, s);
      a.out[(int64_t)slot * a.slot_stride + pos] = s;
    }
  } else {
    constexpr int M = T0 + (T1 - T0) / 2;
    ps_terms<L, SIDE, T0, M, Q>(a, v, pos);
    ps_terms<L, SIDE, M, T1, Q>(a, v, pos);
  }
}

constexpr int PRESUM_ROWS = 2;  // slow-dimension rows per thread

// Block: 256 positions along the slot's contiguous dimension x PRESUM_ROWS rows of
// the other; every thread loads the 4^L quadrant values of its positions, then
// writes the batch's term sums (coalesced along the contiguous dimension).
template <int L, int SIDE>
__device__ __forceinline__ void presum_block(const PresumArgs &a, int64_t bx, int64_t by) {
  constexpr int Q = 1 << L;
  const int64_t fast_len = a.kfast ? a.klen : a.xlen, slow_len = a.kfast ? a.xlen : a.klen;
  const int64_t f = FastMap(a.ustep, a.ugroup, blockDim.x).pos(bx, threadIdx.x, blockDim.x, fast_len);
  if (f < 0) return;
  const int64_t fv = a.kfast ? a.kv : a.xv, sv = a.kfast ? a.xv : a.kv;
  int64_t fo[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) fo[q] = __ldg(a.pool + fv + q * fast_len + f);
#pragma unroll 1
  for (int r = 0; r < PRESUM_ROWS; ++r) {
    const int64_t sl = by * PRESUM_ROWS + r;
    if (sl >= slow_len) break;
    int64_t so[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) so[q] = __ldg(a.pool + sv + q * slow_len + sl);
    double v[Q][Q];
#pragma unroll
    for (int xq = 0; xq < Q; ++xq)
#pragma unroll
      for (int kq = 0; kq < Q; ++kq) {
        const int64_t xo = a.kfast ? so[xq] : fo[xq], ko = a.kfast ? fo[kq] : so[kq];
        v[xq][kq] = (xo == kPad || ko == kPad) ? 0.0 : __ldcs(a.D + xo + ko);
      }
    ps_terms<L, SIDE, 0, ps_pow7(L), Q>(a, v, sl * fast_len + f);
  }
}

// Both sides in one launch: blocks [0, na) cover A's slots, the rest B's.
template <int L>
__global__ void __launch_bounds__(256) k_presum(const PresumArgs pa, const PresumArgs pb, int64_t na_x, int64_t na,
                                                int64_t nb_x) {
  pdl_wait();
  pdl_launch_dependents();
  // the call's tickets and work counters (read by the next kernel, after this grid completes)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pa.zero_words;
       i += (int64_t)gridDim.x * blockDim.x)
    pa.zero[i] = 0;
  const int64_t b = blockIdx.x;
  if (b < na)
    presum_block<L, 0>(pa, b % na_x, b / na_x);
  else
    presum_block<L, 1>(pb, (b - na) % nb_x, (b - na) / nb_x);
}

static void presum_grid(const PresumArgs &a, int64_t &gx, int64_t &gy) {
  const int64_t fast_len = a.kfast ? a.klen : a.xlen, slow_len = a.kfast ? a.xlen : a.klen;
  gx = fast_len > 0 && a.out ? FastMap(a.ustep, a.ugroup, 256).blocks(fast_len, 256) : 0;  // out null: side not pre-summed
  gy = slow_len > 0 ? (slow_len + PRESUM_ROWS - 1) / PRESUM_ROWS : 0;
}

cudaError_t launch_presum2(const PresumArgs &pa, const PresumArgs &pb, cudaStream_t s) {
  if (pa.level != pb.level || pa.side != 0 || pb.side != 1) return cudaErrorInvalidValue;
  int64_t ax, ay, bx, by;
  presum_grid(pa, ax, ay);
  presum_grid(pb, bx, by);
  const int64_t na = ax * ay, total = na + bx * by;
  if (total == 0) return cudaSuccess;
  if (total > INT32_MAX) return cudaErrorInvalidConfiguration;
  const int64_t ax1 = std::max<int64_t>(ax, 1), bx1 = std::max<int64_t>(bx, 1);
  if (pa.level == 1) return launch_pdl(k_presum<1>, dim3((unsigned)total), dim3(256), 0, s, pa, pb, ax1, na, bx1);
  if (pa.level == 2) return launch_pdl(k_presum<2>, dim3((unsigned)total), dim3(256), 0, s, pa, pb, ax1, na, bx1);
  if (pa.level == 3) return launch_pdl(k_presum<3>, dim3((unsigned)total), dim3(256), 0, s, pa, pb, ax1, na, bx1);
  return cudaErrorInvalidValue;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("STC_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ---- plan snapshot restore (stc_capi.cu Resident): a plain device copy ----
__global__ void __launch_bounds__(256) k_restore(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int64_t n) {
  pdl_wait();
  pdl_launch_dependents();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_restore(const void *src, void *dst, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if (bytes % 16 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16)
    return cudaErrorInvalidValue;
  const int64_t n = (int64_t)(bytes / 16);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  return launch_pdl(k_restore, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const uint4 *>(src),
                    reinterpret_cast<uint4 *>(dst), n);
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

// ---- the reference's component kernels as standalone passes ------------------
// pack_a_block / pack_b_block (_jit.py:27-131): out[s, p, i] = sum_t coeff_t * view_t
// element, views added in order from 0.0 (the reference's roundings), PAD and fringe
// positions 0; sliver s = `width` consecutive rows (A) or columns (B), p < kcount.
__global__ void k_pack_panel(const PanelArgs a, const double *__restrict__ data, double *__restrict__ out) {
  const int64_t slivers = (a.xcount + a.width - 1) / a.width;
  const int64_t total = slivers * a.kcount * a.width;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % a.width, p = (e / a.width) % a.kcount, s = e / (a.width * a.kcount);
    const int64_t x = s * a.width + i;
    double acc = 0.0;
    if (x < a.xcount) {
      const int64_t ri = a.side == 0 ? a.x0 + x : a.k0 + p, ci = a.side == 0 ? a.k0 + p : a.x0 + x;
      for (int t = 0; t < a.vs.n; ++t) {
        const int64_t ro = a.vs.rows[t][ri], co = a.vs.cols[t][ci];
        if (ro == kPad || co == kPad) continue;
        acc = __dadd_rn(acc, __dmul_rn(a.vs.coeff[t], data[ro + co]));
      }
    }
    out[(s * a.depth + p) * a.width + i] = acc;
  }
}

// fast / slow sub-blocks as the reference counts them (per sliver x kblock-chunk: fast when
// every view's block vectors are nonzero there): #regular slivers x #regular chunks.
__global__ void k_pack_count(const PanelArgs a, int64_t *__restrict__ counts) {
  __shared__ unsigned long long reg[2];
  if (threadIdx.x < 2) reg[threadIdx.x] = 0;
  __syncthreads();
  const int64_t slivers = (a.xcount + a.width - 1) / a.width, chunks = (a.kcount + a.kblock - 1) / a.kblock;
  for (int64_t e = threadIdx.x; e < slivers + chunks; e += blockDim.x) {
    const bool is_x = e < slivers;
    const int64_t blk = is_x ? (a.x0 + e * a.width) / a.width : (a.k0 + (e - slivers) * a.kblock) / a.kblock;
    bool ok = !a.force_slow;
    for (int t = 0; ok && t < a.vs.n; ++t) ok = (is_x ? a.xbs[t][blk] : a.kbs[t][blk]) != 0;
    if (ok) atomicAdd(&reg[is_x ? 0 : 1], 1ULL);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t fast = (int64_t)(reg[0] * reg[1]);
    counts[0] = fast;
    counts[1] = slivers * chunks - fast;
  }
}

cudaError_t launch_pack_panel(const PanelArgs &a, const double *data, double *out, int64_t *counts, cudaStream_t s) {
  const int64_t slivers = (a.xcount + a.width - 1) / a.width, total = slivers * a.kcount * a.width;
  if (total > 0) {
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_pack_panel<<<blocks, 256, 0, s>>>(a, data, out);
  }
  if (counts) k_pack_count<<<1, 256, 0, s>>>(a, counts);
  return cudaGetLastError();
}

// microtile_mats + store_tile (_jit.py:145-186): element (i, j) of the mr x nr tile
// accumulates a[i, p] * b[p, j] over p in order (a multiply and an add per step, no
// FMA: the reference's roundings), then adds coeff * acc into every target in target
// order (one thread owns an element of all targets: identical targets stay ordered).
__global__ void k_microtile(const double *__restrict__ a, int64_t lda, const double *__restrict__ b, int64_t ldb,
                            int64_t k, int mr, int nr, double *__restrict__ C, const TileTargets t, int force_slow,
                            int64_t *__restrict__ counts) {
  for (int e = threadIdx.x; e < mr * nr; e += blockDim.x) {
    const int i = e / nr, j = e - i * nr;
    double acc = 0.0;
    for (int64_t p = 0; p < k; ++p) acc = __dadd_rn(acc, __dmul_rn(a[i * lda + p], b[p * ldb + j]));
    for (int g = 0; g < t.n_targets; ++g) {
      if (i >= t.m[g] - t.i0[g] || j >= t.n[g] - t.j0[g]) continue;  // fringe tiles are clipped to the view
      const int64_t ro = t.rows[g][t.i0[g] + i], co = t.cols[g][t.j0[g] + j];
      if (ro == kPad || co == kPad) continue;
      C[ro + co] = __dadd_rn(C[ro + co], __dmul_rn(t.coeff[g], acc));
    }
  }
  if (counts && threadIdx.x == 0) {
    int64_t fast = 0;
    for (int g = 0; g < t.n_targets; ++g)
      fast += !force_slow && t.rbs[g][t.i0[g] / mr] != 0 && t.cbs[g][t.j0[g] / nr] != 0;
    counts[0] = fast;
    counts[1] = t.n_targets - fast;
  }
}

cudaError_t launch_microtile(const double *a, int64_t lda, const double *b, int64_t ldb, int64_t k, int mr, int nr,
                             double *C, const TileTargets &t, int force_slow, int64_t *counts, cudaStream_t s) {
  const int threads = std::min(1024, std::max(32, (mr * nr + 31) / 32 * 32));
  k_microtile<<<1, threads, 0, s>>>(a, lda, b, ldb, k, mr, nr, C, t, force_slow, counts);
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

// ---- counter-based synthetic inputs (bench / tests; oracle/synth.py mirror) ----
// value(j) = (mix(key + (j + 1) G) >> 11) * 2^-52 - 1, key = mix(seed + G): depends only
// on the element's flat index j in the FULL tensor, so any shard is generated on its own.
struct FillShape {
  int ndim;
  int64_t ext[STC_MAX_LABELS], str[STC_MAX_LABELS];  // row-major decomposition of the output
};

__device__ __forceinline__ uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) k_fill_uniform(double *__restrict__ out, const FillShape sh, int64_t total,
                                                      int64_t base, uint64_t key) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += stride) {
    int64_t rem = e, j = base;
    for (int d = sh.ndim - 1; d >= 0; --d) {  // last dim fastest (compact row-major output)
      const int64_t i = rem % sh.ext[d];
      rem /= sh.ext[d];
      j += i * sh.str[d];
    }
    const uint64_t z = splitmix_fin(key + ((uint64_t)j + 1ull) * 0x9E3779B97F4A7C15ull);
    out[e] = (double)(z >> 11) * 0x1p-52 - 1.0;
  }
}

cudaError_t launch_fill_uniform(double *out, int ndim, const int64_t *ext, const int64_t *str, int64_t base,
                                uint64_t seed, cudaStream_t s) {
  FillShape sh{};
  int64_t total = 1;
  // merge the trailing dims whose strides are row-major over the output (the common case of
  // a whole tensor or a slab): fewer divisions per element
  sh.ndim = ndim;
  for (int d = 0; d < ndim; ++d) {
    sh.ext[d] = ext[d];
    sh.str[d] = str[d];
    total *= ext[d];
  }
  while (sh.ndim >= 2 && sh.str[sh.ndim - 2] == sh.str[sh.ndim - 1] * sh.ext[sh.ndim - 1]) {
    sh.ext[sh.ndim - 2] *= sh.ext[sh.ndim - 1];
    sh.str[sh.ndim - 2] = sh.str[sh.ndim - 1];
    --sh.ndim;
  }
  if (total == 0) return cudaSuccess;
  uint64_t k = seed + 0x9E3779B97F4A7C15ull;
  k = (k ^ (k >> 30)) * 0xBF58476D1CE4E5B9ull;
  k = (k ^ (k >> 27)) * 0x94D049BB133111EBull;
  k ^= k >> 31;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_fill_uniform<<<(int)blocks, 256, 0, s>>>(out, sh, total, base, k);
  return cudaGetLastError();
}

}  // namespace stc
