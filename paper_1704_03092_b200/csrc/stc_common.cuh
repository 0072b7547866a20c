// stc_common.cuh -- pieces shared by the DMMA kernels: tile rasterisation and
// the epilogue that adds +/-M into the C targets (or writes dense M).
#pragma once

#include "stc_internal.cuh"
#include "stc_ptx.cuh"


namespace stc {

// Work item -> (term slot, tile row ti, tile column tj, tile id pos).  pos numbers
// the quadrant's tiles the same way for every term (per-tile tickets).
__device__ __forceinline__ void tile_of(const GemmArgs &p, int item, int &slot, int &ti, int &tj, int &pos) {
  const int rows = p.tiles_m;
  const int P = rows * p.tiles_n;
  int local;
  if (p.term_inner) {  // dense M: a tile position's terms run together and share its operand panels in L2
    local = item / p.nterms;
    slot = item - local * p.nterms;
  } else {
    slot = item / P;
    local = item - slot * P;
  }
  // grouped rasterisation: group_m tile-rows share the B panels in L2
  const int gm = min(p.group_m, rows);
  const int per_group = gm * p.tiles_n;
  const int g = local / per_group;
  const int first = g * gm;
  const int gsz = min(rows - first, gm);
  const int r = local - g * per_group;
  ti = first + r % gsz;
  tj = r / gsz;
  pos = ti * p.tiles_n + tj;
}
__device__ __forceinline__ void tile_of(const GemmArgs &p, int item, int &slot, int &ti, int &tj) {
  int pos;
  tile_of(p, item, slot, ti, tj, pos);
}

// stc_set_c_ready: block until C has arrived (thread 0 polls, the consumer
// warps meet at named barrier 2).  `seen` keeps it to one poll per CTA.
__device__ __forceinline__ void wait_c_ready(const GemmArgs &p, int tid, bool &seen) {
  if (!p.c_ready || seen) return;
  if (tid == 0)
    while (ld_acquire_gpu(p.c_ready) == 0) __nanosleep(256);
  named_bar(2, 32 * CONSUMER_WARPS);
  seen = true;
}

// Epilogue of one work item (consumer warps 0..7, 64x32 warp tiles of
// m16n8k4 fragments): add sign * M into each C target through the scatter
// layout, C-tile updates ordered across terms by per-tile tickets
// (deterministic, no atomics on C) -- replaces store_tile (_jit.py:158-186);
// or write M densely (AB / Naive).
//
// PA / PB: fragment-to-tile permutation of rows (A side) / columns (B side):
// 0 identity (gather kernel); 1 or 2 the fused kernel's (stc_fused.cu,
// frag_perm) for a side whose unit stride is in x (1) or in k (2).
__host__ __device__ __forceinline__ int frag_perm(int kind, int g, int h) {  // g: 0..7, h: 0..1 -> 0..15
  if (kind == 1) return (g & 1) + 8 * ((g >> 1) & 1) + 2 * (g >> 2) + 4 * h;
  if (kind == 2) return (g & 1) + 2 * h + 4 * (g >> 1);
  return g + 8 * h;
}
template <int PA>
__device__ __forceinline__ int epi_row(int mt, int h, int g) {
  return mt * 16 + frag_perm(PA, g, h);
}
template <int PB>
__device__ __forceinline__ int epi_col(int nt, int tig) {  // first of the pair (b = 0, 1): frag_perm keeps pairs adjacent
  return 16 * (nt >> 1) + frag_perm(PB, 2 * tig, nt & 1);
}

// MT: m16 blocks per warp tile (4: 64 x 32; 2: 32 x 32, dense M output only)
template <int PA = 0, int PB = 0, int RB = 1, int TBM = BM, int TBN = BN, int MT = 4>
__device__ __forceinline__ void epilogue_store(const GemmArgs &p, const double (&acc)[4][4][4], int item, int tid,
                                               int wm, int wn, int g, int tig) {
  int slot, ti, tj, pos;
  tile_of(p, item, slot, ti, tj, pos);
  const TermDesc td = p.terms[slot];
  const int row0 = ti * TBM + wm * 16 * MT;
  const int col0 = tj * TBN + wn * 32;
  if (p.dense_out) {
    double *Mt = p.M + (int64_t)td.m_slot * p.m_stride;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 v = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
          *reinterpret_cast<double2 *>(Mt + (int64_t)(row0 + epi_row<PA>(mt, h, g)) * p.m_ld + col0 +
                                      epi_col<PB>(nt, tig)) = v;
        }
    return;
  }
  if constexpr (MT == 4) {  // (32-row warp tiles run with dense M output only)
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
      for (int b = 0; b < 2; ++b) co[nt * 2 + b] = __ldcg(p.pool + tg.col_start + col0 + epi_col<PB>(nt, tig) + b);
    // batches of RB rows (h = 0, 1 of RB / 2 ... 2 / RB mt blocks): all 8 RB loads of a
    // batch in flight before its stores
#pragma unroll
    for (int bt = 0; bt < 8 / RB; ++bt) {
      int64_t ro[RB];
      double old[RB][8];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int rr = bt * RB + i, mt = rr >> 1, h = rr & 1;
        ro[i] = __ldcg(p.pool + tg.row_start + row0 + epi_row<PA>(mt, h, g));
      }
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) old[i][c] = (ro[i] == kPad || co[c] == kPad) ? 0.0 : __ldcg(p.C + ro[i] + co[c]);
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int rr = bt * RB + i, mt = rr >> 1, h = rr & 1;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (ro[i] != kPad && co[c] != kPad)
            __stcg(p.C + ro[i] + co[c], old[i][c] + tg.sign * acc[mt][c >> 1][2 * h + (c & 1)]);
      }
    }
    if (p.use_tickets) {
      __threadfence();
      named_bar(2, 32 * CONSUMER_WARPS);
      if (tid == 0) st_release_gpu(ticket, tg.order + 1);
    }
  }
  }
}

}  // namespace stc
