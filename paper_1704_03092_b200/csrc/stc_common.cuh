// stc_common.cuh -- pieces shared by the DMMA kernels: tile rasterisation and
// the epilogue that adds +/-M into the C targets (or writes dense M).
#pragma once

#include "stc_internal.cuh"
#include "stc_ptx.cuh"

namespace stc {

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

// Epilogue of one work item (consumer warps 0..7, 64x32 warp tiles of
// m16n8k4 fragments): add sign * M into each C target through the scatter
// layout, C-tile updates ordered across terms by per-tile tickets
// (deterministic, no atomics on C) -- replaces store_tile (_jit.py:158-186);
// or write M densely (AB / Naive).
//
// PERM: the fused kernel's fragment-to-tile permutation (stc_fused.cu): MMA row
// m of a 16-row block holds tile row (m & 1) + 2 ((m >> 3) & 1) + 4 ((m >> 1) & 3),
// and likewise for columns within each 16-column pair of n8 tiles.
template <bool PERM>
__device__ __forceinline__ int epi_row(int mt, int h, int g) {
  return mt * 16 + (PERM ? (g & 1) + 2 * h + 4 * (g >> 1) : g + 8 * h);
}
template <bool PERM>
__device__ __forceinline__ int epi_col(int nt, int tig) {  // first of the pair (b = 0, 1)
  return PERM ? 16 * (nt >> 1) + 2 * (nt & 1) + 4 * tig : nt * 8 + 2 * tig;
}

template <bool PERM = false>
__device__ __forceinline__ void epilogue_store(const GemmArgs &p, const double (&acc)[4][4][4], int item, int tid,
                                               int wm, int wn, int g, int tig) {
  int slot, ti, tj;
  tile_of(p, item, slot, ti, tj);
  const TermDesc td = p.terms[slot];
  const int row0 = ti * BM + wm * 64;
  const int col0 = tj * BN + wn * 32;
  if (p.dense_out) {
    double *Mt = p.M + (int64_t)td.m_slot * p.m_stride;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 v = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
          *reinterpret_cast<double2 *>(Mt + (int64_t)(row0 + epi_row<PERM>(mt, h, g)) * p.m_ld + col0 +
                                      epi_col<PERM>(nt, tig)) = v;
        }
    return;
  }
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
      for (int b = 0; b < 2; ++b) co[nt * 2 + b] = __ldcg(p.pool + tg.col_start + col0 + epi_col<PERM>(nt, tig) + b);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t ro = __ldcg(p.pool + tg.row_start + row0 + epi_row<PERM>(mt, h, g));
        double *Crow = p.C + ro;
        double old[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) old[c] = (ro == kPad || co[c] == kPad) ? 0.0 : __ldcg(Crow + co[c]);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (ro != kPad && co[c] != kPad) __stcg(Crow + co[c], old[c] + tg.sign * acc[mt][c >> 1][2 * h + (c & 1)]);
      }
    if (p.use_tickets) {
      __threadfence();
      named_bar(2, 32 * CONSUMER_WARPS);
      if (tid == 0) st_release_gpu(ticket, tg.order + 1);
    }
  }
}

}  // namespace stc
