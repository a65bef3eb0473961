// kblas_symv_tma.cuh — SYMV / HEMV streaming kernel fed by TMA.
//
// Same tiling and stream-K item split as kblas_symv_kernel (kblas_kernels.cuh):
// a tile is W = NC*CW stored columns with all their stored rows, an item
// is one HS-row chunk of a tile.  What changes is how bytes reach the
// FMAs.  Instead of each warp loading its own columns into registers (the
// paper's register double buffering, which ties bytes in
// flight to the register file and stalls every warp at the per-chunk
// cross-warp reduction), one elected thread streams whole HS x W boxes of A
// into an S-stage shared-memory ring with cp.async.bulk.tensor (TMA), and
// the warps are specialised:
//
//   warps 0..NC-1  consumers: wait full[s], read their CW columns of the
//                  box from shared memory (conflict-free, 8/16 B per lane),
//                  form t1 (row sums, A x_col) and t2 (column sums, op(A)
//                  x_row) exactly as kblas_symv_kernel, drop the t1 partial into
//                  red[s][warp], arrive redfull[s] and empty[s]
//   warp NC        producer: waits empty[s], arms full[s] with the box
//                  byte count and issues the TMA for the next item
//   warp NC+1      reducer: waits redfull[s], sums the NC partials of the
//                  chunk in warp order (deterministic), writes ws1, arrives
//                  empty[s]
//
// So up to S boxes (S*W*256 B, ~160 KB per SM) are in flight while the
// consumers compute and the reducer drains, and no thread ever blocks on
// a CTA-wide barrier inside the main loop.  TMA also does the offset
// realignment for free: a box may start at any row, so chunks start
// exactly at a tile's first stored row, and rows past the operand's end
// are zero-filled by the hardware (out-of-bounds fill).
#pragma once
#include <cuda.h>

#include "kblas_kernels.cuh"

namespace kb {

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// element access in the staged box: a piece is VE consecutive rows (8
// bytes for s/d/c, 16 for z); lane l owns pieces l, l+32, ... (RS of them)
// of every column, so a warp's shared-memory reads are contiguous.
template <class T, int RS> struct Stage {
  static constexpr int VE = sizeof(T) >= 8 ? 1 : 8 / (int)sizeof(T);
  static constexpr int HS = 32 * VE * RS;                // rows per item
  static constexpr int COL_BYTES = HS * (int)sizeof(T);  // 256 B * RS (512 B * RS for z)
};

// The box grid is aligned to HS rows of the tensor (TMA needs 16-byte
// aligned box starts); `lead` is the tensor row of logical row 0, and rows
// outside a tile's stored range are masked in registers.
struct SymTmaParams {
  SymParams sp;      // tiles, ws1/ws2, d, lead, x, stream-K split (A/lda unused)
  int unit_per_elem; // tensor units per element (2 for z)
};

template <class T, int NC, int CW, int RS, int S, bool LOWER, bool HERM>
__global__ void __launch_bounds__((NC + 2) * 32, 1)
    kblas_symv_tma_kernel(const __grid_constant__ CUtensorMap tmap, const SymTmaParams tp) {
  griddep_launch_dependents();
  griddep_wait();  // x staged by a hostvec copy-in grid (no-op otherwise)
  constexpr int VE = Stage<T, RS>::VE;
  constexpr int HS = Stage<T, RS>::HS;
  constexpr int W = NC * CW;
  constexpr int BOX_BYTES = W * Stage<T, RS>::COL_BYTES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T *boxes = reinterpret_cast<T *>(smem_raw);                                  // [S][W][HS]
  T *red = reinterpret_cast<T *>(smem_raw + (size_t)S * BOX_BYTES);           // [S][NC][HS]
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * BOX_BYTES + (size_t)S * NC * HS * sizeof(T));
  uint64_t *full = bars, *empty = bars + S, *redfull = bars + 2 * S;

  const SymParams &p = tp.sp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SymCursor c0;
  if (!c0.init(p)) return;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC + 1);
      mbar_init(&redfull[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  __syncthreads();

  if (warp == NC) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      SymCursor c = c0;
      for (long long qi = 0; !c.done; c.advance(p), ++qi) {
        const SymTile &tl = p.tiles[c.k];
        const int s = (int)(qi % S);
        const uint32_t round = (uint32_t)(qi / S);
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        const int row = (tl.chunk0 + (int)(c.q - tl.prefix)) * HS;  // tensor row (lead included)
        mbar_arrive_expect_tx(&full[s], BOX_BYTES);
        tma_load_2d(boxes + (size_t)s * W * HS, &tmap, row * tp.unit_per_elem, tl.lcol0, &full[s]);
      }
    }
    return;
  }

  T *__restrict__ ws1 = static_cast<T *>(p.ws1);
  if (warp == NC + 1) {
    // ----------------------------------------------------------- reducer
    const uint64_t keep = policy_evict_last();
    SymCursor c = c0;
    for (long long qi = 0; !c.done; c.advance(p), ++qi) {
      const int k = c.k;
      const SymTile &tl = p.tiles[k];
      const int s = (int)(qi % S);
      mbar_wait(&redfull[s], (uint32_t)(qi / S) & 1);
      const T *rs = red + (size_t)s * NC * HS;
      const long long r0 = (long long)(tl.chunk0 + (c.q - tl.prefix)) * HS - p.lead;
#pragma unroll
      for (int t0 = 0; t0 < HS; t0 += 32) {
        const int t = t0 + lane;
        const long long i = r0 + t;
        if (i >= tl.row0 && i < tl.row1) {
          T acc = rs[t];
#pragma unroll
          for (int w = 1; w < NC; ++w) acc = add_(acc, rs[w * HS + t]);
          st_keep(ws1 + (long long)k * p.ws1_ld + i, acc, keep);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *__restrict__ ws2 = static_cast<T *>(p.ws2);
  const int cl = warp * CW;
  SymCursor c = c0;
  long long qi = 0;
  while (!c.done) {
    // one run: consecutive items of one tile within one segment
    const int k = c.k;
    const long long seg = c.s;
    const SymTile tl = p.tiles[k];
    T xc[CW], t2[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      xc[j] = (cl + j < tl.ncols) ? ld_x(x + tl.gcol0 + cl + j) : zero<T>();
      t2[j] = zero<T>();
    }
    for (; !c.done && c.k == k && c.s == seg; c.advance(p), ++qi) {
      const long long q = c.q;
      const int s = (int)(qi % S);
      // logical row of box row 0; piece (r, lane) holds rows r0 + (r*32 + lane)*VE + v
      const long long r0 = (long long)(tl.chunk0 + (q - tl.prefix)) * HS - p.lead;
      T xr[RS][VE];
      bool ok[RS][VE];
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int v = 0; v < VE; ++v) {
          const long long i = r0 + (r * 32 + lane) * VE + v;
          ok[r][v] = i >= tl.row0 && i < tl.row1;
          xr[r][v] = ok[r][v] ? ld_x(x + i) : zero<T>();
        }
      mbar_wait(&full[s], (uint32_t)(qi / S) & 1);
      const T *box = boxes + (size_t)s * W * HS + (size_t)cl * HS + lane * VE;
      T a[CW][RS][VE];
#pragma unroll
      for (int j = 0; j < CW; ++j)
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          if constexpr (VE == 2) {
            const float2 f = *reinterpret_cast<const float2 *>(box + j * HS + r * 32 * VE);
            a[j][r][0] = f.x;
            a[j][r][1] = f.y;
          } else {
            a[j][r][0] = box[j * HS + r * 32];
          }
        }
      T acc[RS][VE];
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int v = 0; v < VE; ++v) acc[r][v] = zero<T>();
      const bool diag = (r0 < (long long)tl.gcol0 + tl.ncols) && (r0 + HS > tl.gcol0);
      const bool inside = r0 >= tl.row0 && r0 + HS <= tl.row1;
      if (!diag && inside) {
#pragma unroll
        for (int j = 0; j < CW; ++j)
#pragma unroll
          for (int r = 0; r < RS; ++r)
#pragma unroll
            for (int v = 0; v < VE; ++v) {
              acc[r][v] = fma_(a[j][r][v], xc[j], acc[r][v]);
              t2[j] = fmax_<HERM>(a[j][r][v], xr[r][v], t2[j]);
            }
      } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const long long c = (long long)tl.gcol0 + cl + j;
#pragma unroll
          for (int r = 0; r < RS; ++r)
#pragma unroll
            for (int v = 0; v < VE; ++v) {
              const long long i = r0 + (r * 32 + lane) * VE + v;
              const bool in1 = ok[r][v] && (LOWER ? i >= c : i <= c);
              const bool in2 = ok[r][v] && (LOWER ? i > c : i < c);
              T e1 = sel(in1, a[j][r][v]);
              if (HERM && i == c) e1 = realify(e1);
              acc[r][v] = fma_(e1, xc[j], acc[r][v]);
              t2[j] = fmax_<HERM>(sel(in2, a[j][r][v]), xr[r][v], t2[j]);
            }
        }
      }
      T *rw = red + (size_t)s * NC * HS + (size_t)warp * HS + lane * VE;
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int v = 0; v < VE; ++v) rw[r * 32 * VE + v] = acc[r][v];
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&redfull[s]);
        mbar_arrive(&empty[s]);
      }
    }
    T *row = ws2 + (long long)(tl.slot0 + (int)(seg - tl.seg0)) * p.ws2_ld;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const T sum = warp_sum(t2[j]);
      if (lane == 0 && cl + j < tl.ncols) row[cl + j] = sum;
    }
  }
}

template <class T, int NC, int CW, int RS, int S>
constexpr size_t symv_tma_smem() {
  return (size_t)S * NC * CW * Stage<T, RS>::COL_BYTES + (size_t)S * NC * Stage<T, RS>::HS * sizeof(T) + 3 * S * 8;
}

}  // namespace kb
