// kblas_kernels.cuh — sm_100a matrix-vector kernels.
//
// Three streaming kernels, one per product shape, each followed by a tiny
// fixed-order epilogue that sums cross-CTA partials and applies alpha/beta:
//
//   kblas_gemv_n_kernel  y = A x        (reference: _gemv_accumulate transposed=False,
//                                  kernels.py:149-201 via run_gemv_n 209-221)
//   kblas_gemv_t_kernel  y = A^T x / A^H x  (run_gemv_t, kernels.py:224-236)
//   kblas_symv_kernel    y = A x from one stored triangle; every element is read
//                  once and used twice: t1 = A_blk x_col -> rows, and
//                  t2 = A_blk^T|H x_row -> columns (_symv_offdiag_accumulate
//                  kernels.py:239-284 and _diag_accumulate 316-359 fused;
//                  diagonal tiles are masked in registers, never mirrored
//                  through memory)
//
// Work distribution is stream-K: the matrix is cut into equal "items"
// (one 32*V*R-row chunk of CW columns per warp, NW warps per CTA) and CTA c
// walks the contiguous item range [c*total/P, (c+1)*total/P).  Every CTA
// streams the same number of bytes, so a grid of P = #SM x occupancy CTAs
// has no wave tail (the paper's TB_R oscillation, PAPER.md:311-332,
// 1259-1292, does not arise).
//
// Lanes read column segments with 256-bit loads (32 contiguous bytes per
// lane, 1 KiB per warp per column); the warp's CW column loads are all
// issued before any FMA so CW x 32 B per lane are in flight.
#pragma once
#include <cooperative_groups.h>

#include "kblas_device.cuh"

#ifndef KBLAS_SYMV_TRACE
#define KBLAS_SYMV_TRACE 0
#endif

namespace kb {

// ---------------------------------------------------------------------------
// Programmatic dependent launch: the epilogue grid is launched while the
// streaming kernel runs (launch latency hidden) and blocks here until the
// streaming grid has completed and its writes are visible.  Every library
// kernel releases its dependents at its start and executes griddep_wait()
// before it touches data an earlier kernel of the stream may still write
// or read; the programmatic dependents are the epilogues, the main kernel
// of a host-vector call (after its copy-in grid) and the copy-in grid
// itself (after the stream's previous kernel).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

struct GemvParams {
  const void *A;    // 32-byte aligned base: physical row 0 of local column 0
  long long lda;
  int m, n;         // logical rows, local columns
  int lead;         // physical row of logical row 0 (offset realignment)
  const void *x;    // N: indexed by global column; T: indexed by logical row
  void *ws;         // partial slots ws[slot * ws_ld + idx]
  long long ws_ld;
  long long total;  // work items
  int P;            // CTAs
  int KS;           // N: column steps per row block; T: row chunks per column block
  ColMap cm;
  // fused epilogue: the last CTA to finish a row (column) block sums its
  // partial slots in slot order and writes y = alpha*sum + beta*y
  void *y;
  unsigned *counters;  // one per row/column block, zero between calls
  double2 alpha, beta; // scalars of the operand type, widened
  int beta_zero;
  long long nglob;     // T: length of y (global columns); N: m
  int pdl = 0;         // launched as the programmatic dependent of a hostvec copy-in grid
                       // (1: prefetch the first A segments before the wait, 2: no prefetch)
};

template <class T> __device__ __forceinline__ T scalar_of(double2 v);
template <> __device__ __forceinline__ float scalar_of<float>(double2 v) { return (float)v.x; }
template <> __device__ __forceinline__ double scalar_of<double>(double2 v) { return v.x; }
template <> __device__ __forceinline__ float2 scalar_of<float2>(double2 v) { return make_float2((float)v.x, (float)v.y); }
template <> __device__ __forceinline__ double2 scalar_of<double2>(double2 v) { return v; }

// y[i] = alpha * s + beta * y[i] (beta == 0: y not read)
template <class T>
__device__ __forceinline__ void axpby_out(T *y, long long i, const GemvParams &p, T s) {
  T r = mul_(scalar_of<T>(p.alpha), s);
  if (!p.beta_zero) r = fma_(scalar_of<T>(p.beta), y[i], r);
  y[i] = r;
}

// Arrival at a block's counter after this CTA wrote its partial slot.
// Returns true (CTA-uniform) for the CTA that completes the block; its
// reads of the other CTAs' slots must then bypass L1 (__ldcg).
__device__ __forceinline__ bool arrive_last(unsigned *counter, int nslots) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == (unsigned)(nslots - 1));
    if (s_last) *counter = 0u;  // self-reset for the next call on this workspace
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Sum of slots [s0, s1) of ws[slot * ld + idx] in slot order; the loads are
// issued eight at a time (independent, so one L2 round trip per batch) and
// added in order, so the result does not depend on timing.
template <class T>
__device__ __forceinline__ T sum_slots(const T *ws, long long ld, long long idx, int s0, int s1) {
  T acc = zero<T>();
  for (int sl = s0; sl < s1; sl += 8) {
    T t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = (sl + u < s1) ? __ldcg(ws + (long long)(sl + u) * ld + idx) : zero<T>();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (sl + u < s1) acc = add_(acc, t[u]);
  }
  return acc;
}

// Whole-CTA fixed-order reduction of nslots partial slots for the nidx
// consecutive workspace indices idx0 .. idx0+nidx-1: the threads split each
// index's slot range into NT/nidx contiguous parts (a function of nidx and
// nslots only), the parts are added in order, and out(k, sum) is called for
// index k by one thread.  Used by the last CTA to arrive at a block.
template <class T, int NT, class F>
__device__ __forceinline__ void cta_slot_sum(const T *ws, long long ld, long long idx0, int nidx, int nslots, F out) {
  __shared__ T sbuf[NT];
  for (int base = 0; base < nidx; base += NT) {
    const int chunk = min(NT, nidx - base);
    const int parts = NT / chunk;
    const int k = threadIdx.x % chunk, part = threadIdx.x / chunk;
    if (part < parts) {
      const int s0 = nslots * part / parts, s1 = nslots * (part + 1) / parts;
      sbuf[part * chunk + k] = sum_slots(ws, ld, idx0 + base + k, s0, s1);
    }
    __syncthreads();
    if ((int)threadIdx.x < chunk) {
      T r = sbuf[threadIdx.x];
      for (int q = 1; q < parts; ++q) r = add_(r, sbuf[q * chunk + threadIdx.x]);
      out(base + (int)threadIdx.x, r);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// GEMV-N.  The NW warps of a CTA are stacked along the rows: a CTA row block
// is RB = NW*32*V*R rows, so every column visit reads RB*sizeof(T) contiguous
// bytes (8 KiB for D) and each warp owns its own rows.  Item = (row block) x
// (CW columns); items are row-block-major, so a CTA sweeps its row block
// across a contiguous column range, keeps the partial row sums in
// registers, and writes them once per row block it touched (no shared
// memory, no barrier).  The next item's loads are issued before the current
// item's FMAs (register double buffering, as the paper's Alg. 1 does with
// its two half-block buffers).
// ---------------------------------------------------------------------------
template <class T, int V, int NW, int CW, int R, int MINB = 2>
__global__ void __launch_bounds__(NW * 32, MINB) kblas_gemv_n_kernel(const GemvParams p) {
  griddep_launch_dependents();
  griddep_wait();  // x / y staged by a hostvec copy-in grid (no-op otherwise)
  constexpr int WR = 32 * V * R;  // rows per warp
  constexpr int RB = NW * WR;     // rows per CTA row block
  const T *__restrict__ A = static_cast<const T *>(p.A);
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *__restrict__ ws = static_cast<T *>(p.ws);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  long long it = sk_start(blockIdx.x, p.total, p.P);
  const long long end = sk_start(blockIdx.x + 1, p.total, p.P);
  const long long plimit = (long long)p.lead + p.m;

  while (it < end) {
    const long long rb = it / p.KS;
    const long long rb_first = rb * p.KS;
    const long long stop = min(end, rb_first + p.KS);
    const long long pw = rb * RB + warp * WR;  // first physical row of this warp
    bool rok[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rok[r] = pw + r * 32 * V + lane * V < plimit;
    T acc[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[r][v] = zero<T>();

    auto load = [&](long long q, Pack<T, V> (&a)[CW][R], T (&xv)[CW]) {
      const int c0 = (int)(q - rb_first) * CW;
      // CW consecutive local columns map to consecutive global columns
      // unless they straddle a distribution block (mgpu only)
      const long long g0 = map_col(p.cm, c0);
      const bool contiguous = p.cm.G == 1 || (c0 % p.cm.nb) + CW <= p.cm.nb;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int col = c0 + j;
        const bool cok = col < p.n;
        const long long gx = contiguous ? g0 + j : map_col(p.cm, col);
        xv[j] = cok ? ld_x(x + gx) : zero<T>();
        const T *colp = A + (long long)col * p.lda + pw + lane * V;
#pragma unroll
        for (int r = 0; r < R; ++r) ld_pack(a[j][r], colp + r * 32 * V, cok && rok[r], pol);
      }
    };
    Pack<T, V> a0[CW][R], a1[CW][R];
    T x0[CW], x1[CW];
    long long q = it;
    load(q, a0, x0);
    while (q < stop) {
      const bool more = q + 1 < stop;
      if (more) load(q + 1, a1, x1);
#pragma unroll
      for (int j = 0; j < CW; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[r][v] = fma_(a0[j][r].v(v), x0[j], acc[r][v]);
      if (!more) break;
      if (q + 2 < stop) load(q + 2, a0, x0);
#pragma unroll
      for (int j = 0; j < CW; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[r][v] = fma_(a1[j][r].v(v), x1[j], acc[r][v]);
      q += 2;
    }

    const int first = sk_owner(rb_first, p.total, p.P);
    const int nslots = sk_owner(rb_first + p.KS - 1, p.total, p.P) - first + 1;
    T *y = static_cast<T *>(p.y);
    if (p.counters == nullptr) {
      // unfused: partial slots only, kblas_gemv_n_epilogue sums them
      const long long slot = (long long)blockIdx.x - first;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const long long i = pw + r * 32 * V + lane * V + v - p.lead;
          if (i >= 0 && i < p.m) ws[slot * p.ws_ld + i] = acc[r][v];
        }
    } else if (nslots == 1) {
      // this CTA owns the whole row block: write y directly
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const long long i = pw + r * 32 * V + lane * V + v - p.lead;
          if (i >= 0 && i < p.m) axpby_out(y, i, p, acc[r][v]);
        }
    } else {
      const long long slot = (long long)blockIdx.x - first;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const long long i = pw + r * 32 * V + lane * V + v - p.lead;
          if (i >= 0 && i < p.m) ws[slot * p.ws_ld + i] = acc[r][v];
        }
      if (arrive_last(p.counters + rb, nslots)) {
        // fixed slot order: the result does not depend on which CTA finishes last
        const long long i0 = max(rb * RB - p.lead, 0LL), i1 = min(rb * RB + RB - p.lead, (long long)p.m);
        cta_slot_sum<T, NW * 32>(ws, p.ws_ld, i0, (int)(i1 - i0), nslots,
                                 [&](int k, T sum) { axpby_out(y, i0 + k, p, sum); });
      }
    }
    it = stop;
  }
}

// ---------------------------------------------------------------------------
// GEMV-N for small and short matrices (the split form).  When the matrix is
// small the stacked-rows kernel above has few row blocks, so many CTAs share
// each one and the partial-slot traffic and its reduction dominate.  Here a
// CTA owns one RB = 32*V-row block (one warp width) and a contiguous range of
// columns; its NW warps take the range's CW-column groups round robin and
// are combined through shared memory, so a row block is shared by only
// KS = #CTAs / #row blocks CTAs.  Those combine through per-CTA slots; the
// last CTA to arrive sums them in slot order and writes y (one kernel,
// deterministic).  Grid: (row block, split) = blockIdx.x / KS, % KS.
// ---------------------------------------------------------------------------
template <class T, int V, int NW, int CW>
__global__ void __launch_bounds__(NW * 32, 2) kblas_gemv_ns_kernel(const GemvParams p) {
  griddep_launch_dependents();
  griddep_wait();  // x / y staged by a hostvec copy-in grid (no-op otherwise)
  constexpr int RB = 32 * V;
  __shared__ T red[NW][RB];
  const T *__restrict__ A = static_cast<const T *>(p.A);
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *__restrict__ ws = static_cast<T *>(p.ws);
  T *y = static_cast<T *>(p.y);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  const long long rb = blockIdx.x / p.KS;
  const int split = (int)(blockIdx.x % p.KS);
  const int c0 = (int)((long long)split * p.n / p.KS), c1 = (int)((long long)(split + 1) * p.n / p.KS);
  const long long pw = rb * RB;  // first physical row of the block
  const bool rok = pw + lane * V < (long long)p.lead + p.m;
  T acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = zero<T>();
  auto load = [&](int g, Pack<T, V> (&a)[CW], T (&xv)[CW]) {
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int col = g + j;
      const bool cok = col < c1;
      xv[j] = cok ? ld_x(x + map_col(p.cm, col)) : zero<T>();
      ld_pack(a[j], A + (long long)col * p.lda + pw + lane * V, cok && rok, pol);
    }
  };
  auto fma_group = [&](const Pack<T, V> (&a)[CW], const T (&xv)[CW]) {
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = fma_(a[j].v(v), xv[j], acc[v]);
  };
  constexpr int STEP = NW * CW;
  Pack<T, V> a0[CW], a1[CW];
  T x0[CW], x1[CW];
  int g = c0 + warp * CW;
  if (g < c1) load(g, a0, x0);
  while (g < c1) {
    const bool more = g + STEP < c1;
    if (more) load(g + STEP, a1, x1);
    fma_group(a0, x0);
    if (!more) break;
    if (g + 2 * STEP < c1) load(g + 2 * STEP, a0, x0);
    fma_group(a1, x1);
    g += 2 * STEP;
  }
#pragma unroll
  for (int v = 0; v < V; ++v) red[warp][lane * V + v] = acc[v];
  __syncthreads();
  const long long i0 = max(pw - p.lead, 0LL), i1 = min(pw + RB - p.lead, (long long)p.m);
  for (int t = threadIdx.x; t < RB; t += NW * 32) {
    const long long i = pw + t - p.lead;
    if (i < i0 || i >= i1) continue;
    T sum = red[0][t];
#pragma unroll
    for (int w = 1; w < NW; ++w) sum = add_(sum, red[w][t]);
    if (p.KS == 1) axpby_out(y, i, p, sum);
    else ws[(long long)split * p.ws_ld + i] = sum;
  }
  if (p.KS > 1 && arrive_last(p.counters + rb, p.KS))
    cta_slot_sum<T, NW * 32>(ws, p.ws_ld, i0, (int)(i1 - i0), p.KS,
                             [&](int k, T sum) { axpby_out(y, i0 + k, p, sum); });
}

// ---------------------------------------------------------------------------
// GEMV-N, row-owning form (small operands).  A CTA owns LR*V rows (LR lanes
// of 32 bytes side by side: a 32*LR-byte segment of every column) and all
// n columns, so no row is shared between CTAs: one kernel, no slots, no
// counters.  Lane = (row lane rl = lane % LR, column lane cl = lane / LR);
// a warp covers CPI = 32/LR columns per step, the NW warps take steps round
// robin, U steps are loaded before any FMA.  At the end the CPI column
// lanes of a row are added with shuffles and the NW warps in shared
// memory, in fixed order.  The GEMV-T column-owning form's transpose; it
// trades segment length (32*LR bytes) for a single pass with every CTA's
// work identical, which wins while the call is latency-bound.
// ---------------------------------------------------------------------------
template <class T, int V, int NW, int LR, int U>
__global__ void __launch_bounds__(NW * 32) kblas_gemv_ro_kernel(const GemvParams p) {
  griddep_launch_dependents();
  constexpr int CPI = 32 / LR, RBo = LR * V, STEP = NW * CPI;
  __shared__ T red[NW][RBo];
  const T *__restrict__ A = static_cast<const T *>(p.A);
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *y = static_cast<T *>(p.y);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rl = lane % LR, cl = lane / LR;
  const uint64_t pol = policy_evict_first();
  const long long pw = (long long)blockIdx.x * RBo + rl * V;  // physical first row of this lane
  const bool rok = pw < (long long)p.lead + p.m;
  T acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = zero<T>();
  // hostvec call: the first two steps' A segments are prefetched into L2
  // before griddepcontrol.wait, so A streams while the copy-in grid is
  // still fetching x (no registers held across the wait)
  if (p.pdl) {
    if (p.pdl == 1) {
#pragma unroll
      for (int u = 0; u < 2 * U; ++u) {
        const int col = warp * CPI + cl + u * STEP;
        if (col < p.n && rok) prefetch_l2(A + (long long)col * p.lda + pw);
      }
    }
    griddep_wait();
  }
  for (int c = warp * CPI + cl; c - cl < p.n; c += U * STEP) {
    Pack<T, V> a[U];
    T xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int col = c + u * STEP;
      const bool cok = col < p.n;
      xv[u] = cok ? ld_x(x + map_col(p.cm, col)) : zero<T>();
      ld_pack(a[u], A + (long long)col * p.lda + pw, cok && rok, pol);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = fma_(a[u].v(v), xv[u], acc[v]);
  }
#pragma unroll
  for (int o = LR; o < 32; o <<= 1)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = add_(acc[v], shfl_xor_(acc[v], o));
  if (cl == 0) {
#pragma unroll
    for (int v = 0; v < V; ++v) red[warp][rl * V + v] = acc[v];
  }
  __syncthreads();
  if ((int)threadIdx.x < RBo) {
    const long long i = (long long)blockIdx.x * RBo + threadIdx.x - p.lead;
    if (i >= 0 && i < p.m) {
      T sum = red[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < NW; ++w) sum = add_(sum, red[w][threadIdx.x]);
      axpby_out(y, i, p, sum);
    }
  }
}

// ---------------------------------------------------------------------------
// GEMV-N split form over a thread-block cluster.  The S CTAs sharing a
// 32*V-row block form one cluster (S = cluster size, up to 16): each CTA
// reduces its warps in shared memory as kblas_gemv_ns_kernel does, then the
// cluster exchanges the S partial row blocks through distributed shared
// memory (CTA rank r sums rows [r*RB/S, (r+1)*RB/S) over ranks 0..S-1 in
// order and writes y).  No global slots, fences or atomics: the cross-CTA
// step is two cluster barriers and on-chip DSMEM reads.
// ---------------------------------------------------------------------------
template <class T, int V, int NW, int CW>
__global__ void __launch_bounds__(NW * 32, 2) kblas_gemv_nc_kernel(const GemvParams p) {
  griddep_launch_dependents();
  griddep_wait();  // x / y staged by a hostvec copy-in grid (no-op otherwise)
  namespace cg = cooperative_groups;
  constexpr int RB = 32 * V;
  __shared__ T red[NW][RB];
  __shared__ T part[RB];
  cg::cluster_group cluster = cg::this_cluster();
  const int S = (int)cluster.num_blocks();
  const int split = (int)cluster.block_rank();
  const T *__restrict__ A = static_cast<const T *>(p.A);
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *y = static_cast<T *>(p.y);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  const long long rb = blockIdx.x / S;
  const int c0 = (int)((long long)split * p.n / S), c1 = (int)((long long)(split + 1) * p.n / S);
  const long long pw = rb * RB;
  const bool rok = pw + lane * V < (long long)p.lead + p.m;
  T acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = zero<T>();
  auto load = [&](int g, Pack<T, V> (&a)[CW], T (&xv)[CW]) {
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int col = g + j;
      const bool cok = col < c1;
      xv[j] = cok ? ld_x(x + map_col(p.cm, col)) : zero<T>();
      ld_pack(a[j], A + (long long)col * p.lda + pw + lane * V, cok && rok, pol);
    }
  };
  auto fma_group = [&](const Pack<T, V> (&a)[CW], const T (&xv)[CW]) {
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = fma_(a[j].v(v), xv[j], acc[v]);
  };
  constexpr int STEP = NW * CW;
  Pack<T, V> a0[CW], a1[CW];
  T x0[CW], x1[CW];
  int g = c0 + warp * CW;
  if (g < c1) load(g, a0, x0);
  while (g < c1) {
    const bool more = g + STEP < c1;
    if (more) load(g + STEP, a1, x1);
    fma_group(a0, x0);
    if (!more) break;
    if (g + 2 * STEP < c1) load(g + 2 * STEP, a0, x0);
    fma_group(a1, x1);
    g += 2 * STEP;
  }
#pragma unroll
  for (int v = 0; v < V; ++v) red[warp][lane * V + v] = acc[v];
  __syncthreads();
  for (int t = threadIdx.x; t < RB; t += NW * 32) {
    T sum = red[0][t];
#pragma unroll
    for (int w = 1; w < NW; ++w) sum = add_(sum, red[w][t]);
    part[t] = sum;
  }
  cluster.sync();  // every CTA's partial row block is in its shared memory
  const int t0 = RB * split / S, t1 = RB * (split + 1) / S;
  for (int t = t0 + (int)threadIdx.x; t < t1; t += NW * 32) {
    const long long i = pw + t - p.lead;
    if (i < 0 || i >= p.m) continue;
    T sum = *cluster.map_shared_rank(part + t, 0);
    for (int q = 1; q < S; ++q) sum = add_(sum, *cluster.map_shared_rank(part + t, q));
    axpby_out(y, i, p, sum);
  }
  cluster.sync();  // keep the partials alive until every rank has read them
}

// ---------------------------------------------------------------------------
// GEMV-T / GEMV-C.  Item = (column block of NW*CW columns) x (row chunk of
// H = 32*V*R rows), column-block-major.  Each lane keeps a partial dot
// product per column in registers across the whole chunk range and reduces
// across the warp once per column block (no shared memory, no barrier).
// Rows outside the logical range are masked with selects, so padding or a
// parent's neighbouring rows (possibly NaN) never enter a sum.
// ---------------------------------------------------------------------------
template <class T, int V, int NW, int CW, int R, bool CONJ, int MINB = 2>
__global__ void __launch_bounds__(NW * 32, MINB) kblas_gemv_t_kernel(const GemvParams p) {
  griddep_launch_dependents();
  griddep_wait();  // x / y staged by a hostvec copy-in grid (no-op otherwise)
  constexpr int H = 32 * V * R;
  constexpr int CBW = NW * CW;
  const T *__restrict__ A = static_cast<const T *>(p.A);
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *__restrict__ ws = static_cast<T *>(p.ws);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  long long it = sk_start(blockIdx.x, p.total, p.P);
  const long long end = sk_start(blockIdx.x + 1, p.total, p.P);
  const long long plimit = (long long)p.lead + p.m;
  // x rows can be fetched as whole vectors when they share A's alignment
  const bool xvec = V > 1 && p.lead == 0 && (reinterpret_cast<uintptr_t>(x) % (V * sizeof(T))) == 0;

  while (it < end) {
    const long long cb = it / p.KS;
    const long long cb_first = cb * p.KS;
    const long long stop = min(end, cb_first + p.KS);
    const int col0 = (int)cb * CBW + warp * CW;
    const T *Aw = A + (long long)col0 * p.lda;
    T t2[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) t2[j] = zero<T>();

    // chunk loads: A (CW columns x R vectors) and the matching x rows;
    // rows outside [0, m) are zeroed in x and masked in A with a select,
    // so padding / a parent's neighbouring rows (possibly NaN) never enter
    auto load = [&](long long q, Pack<T, V> (&a)[CW][R], T (&xr)[R][V]) {
      const long long p0 = (q - cb_first) * H;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long i0 = p0 + r * 32 * V + lane * V - p.lead;
        if (xvec && i0 + V <= p.m) {
          ld_xvec<T, V>(xr[r], x + i0);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const long long i = i0 + v;
            xr[r][v] = (i >= 0 && i < p.m) ? ld_x(x + i) : zero<T>();
          }
        }
      }
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const bool cok = col0 + j < p.n;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const long long ps = p0 + r * 32 * V + lane * V;
          ld_pack(a[j][r], Aw + (long long)j * p.lda + ps, cok && ps < plimit, pol);
        }
      }
    };
    auto fma_chunk = [&](long long q, const Pack<T, V> (&a)[CW][R], const T (&xr)[R][V]) {
      const long long p0 = (q - cb_first) * H;
      const bool interior = p0 >= p.lead && p0 + H <= plimit;
#pragma unroll
      for (int j = 0; j < CW; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const long long i = p0 + r * 32 * V + lane * V + v - p.lead;
            const bool ok = interior || (i >= 0 && i < p.m);
            t2[j] = fmax_<CONJ>(sel(ok, a[j][r].v(v)), xr[r][v], t2[j]);
          }
    };
    Pack<T, V> a0[CW][R], a1[CW][R];
    T x0[R][V], x1[R][V];
    long long q = it;
    load(q, a0, x0);
    while (q < stop) {
      const bool more = q + 1 < stop;
      if (more) load(q + 1, a1, x1);
      fma_chunk(q, a0, x0);
      if (!more) break;
      if (q + 2 < stop) load(q + 2, a0, x0);
      fma_chunk(q + 1, a1, x1);
      q += 2;
    }

    const int first = sk_owner(cb_first, p.total, p.P);
    const int nslots = sk_owner(cb_first + p.KS - 1, p.total, p.P) - first + 1;
    T *y = static_cast<T *>(p.y);
    if (p.counters == nullptr) {
      const long long slot = (long long)blockIdx.x - first;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const T s = warp_sum(t2[j]);
        if (lane == 0 && col0 + j < p.n) ws[slot * p.ws_ld + col0 + j] = s;
      }
    } else if (nslots == 1) {
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const T s = warp_sum(t2[j]);
        if (lane == 0 && col0 + j < p.n) axpby_out(y, map_col(p.cm, col0 + j), p, s);
      }
    } else {
      const long long slot = (long long)blockIdx.x - first;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const T s = warp_sum(t2[j]);
        if (lane == 0 && col0 + j < p.n) ws[slot * p.ws_ld + col0 + j] = s;
      }
      if (arrive_last(p.counters + cb, nslots)) {
        const long long c0 = cb * CBW, c1 = min(c0 + CBW, (long long)p.n);
        cta_slot_sum<T, NW * 32>(ws, p.ws_ld, c0, (int)(c1 - c0), nslots,
                                 [&](int k, T sum) { axpby_out(y, map_col(p.cm, c0 + k), p, sum); });
      }
    }
    it = stop;
  }
}

// ---------------------------------------------------------------------------
// GEMV-T / GEMV-C, column-owning form (small and mid-size operands).  CTA c
// owns CB consecutive columns and ALL their rows: its NW warps take the
// H-row chunks round robin (register double buffered), reduce each column
// across lanes with shuffles and across warps through shared memory in
// fixed order, and write y.  No cross-CTA partials, no fences, no second
// kernel: the split-K reduction tail of kblas_gemv_t_kernel is what bounds a
// small call (ncu: SMs active ~54 % of a 16 us N = 2048 call).
// ---------------------------------------------------------------------------
template <class T, int V, int NW, int CB, bool CONJ>
__global__ void __launch_bounds__(NW * 32, 2) kblas_gemv_tc_kernel(const GemvParams p) {
  griddep_launch_dependents();
  griddep_wait();  // x / y staged by a hostvec copy-in grid (no-op otherwise)
  constexpr int H = 32 * V;
  __shared__ T part[NW][CB];
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *y = static_cast<T *>(p.y);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  const int col0 = blockIdx.x * CB;
  const T *__restrict__ Ac = static_cast<const T *>(p.A) + (long long)col0 * p.lda;
  const long long plimit = (long long)p.lead + p.m;
  const int nch = (int)((plimit + H - 1) / H);
  const bool xvec = V > 1 && p.lead == 0 && (reinterpret_cast<uintptr_t>(x) % (V * sizeof(T))) == 0;
  T t[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) t[j] = zero<T>();
  auto load = [&](int ch, Pack<T, V> (&a)[CB], T (&xr)[V]) {
    const long long ps = (long long)ch * H + lane * V;
    const long long i0 = ps - p.lead;
    if (xvec && i0 + V <= p.m) {
      ld_xvec<T, V>(xr, x + i0);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) xr[v] = (i0 + v >= 0 && i0 + v < p.m) ? ld_x(x + i0 + v) : zero<T>();
    }
#pragma unroll
    for (int j = 0; j < CB; ++j) ld_pack(a[j], Ac + (long long)j * p.lda + ps, col0 + j < p.n && ps < plimit, pol);
  };
  auto fma_chunk = [&](int ch, const Pack<T, V> (&a)[CB], const T (&xr)[V]) {
    const long long p0 = (long long)ch * H;
    const bool interior = p0 >= p.lead && p0 + H <= plimit;
#pragma unroll
    for (int j = 0; j < CB; ++j)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const long long i = p0 + lane * V + v - p.lead;
        const bool ok = interior || (i >= 0 && i < p.m);
        t[j] = fmax_<CONJ>(sel(ok, a[j].v(v)), xr[v], t[j]);
      }
  };
  Pack<T, V> a0[CB], a1[CB];
  T x0[V], x1[V];
  int ch = warp;
  if (ch < nch) load(ch, a0, x0);
  while (ch < nch) {
    const bool more = ch + NW < nch;
    if (more) load(ch + NW, a1, x1);
    fma_chunk(ch, a0, x0);
    if (!more) break;
    if (ch + 2 * NW < nch) load(ch + 2 * NW, a0, x0);
    fma_chunk(ch + NW, a1, x1);
    ch += 2 * NW;
  }
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const T s = warp_sum(t[j]);
    if (lane == 0) part[warp][j] = s;
  }
  __syncthreads();
  if ((int)threadIdx.x < CB && col0 + (int)threadIdx.x < p.n) {
    T s = part[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < NW; ++w) s = add_(s, part[w][threadIdx.x]);
    axpby_out(y, map_col(p.cm, col0 + threadIdx.x), p, s);
  }
}

// ---------------------------------------------------------------------------
// SYMV / HEMV from one stored triangle.
//
// A tile is W = NW*CW consecutive columns [gcol0, gcol0+ncols) together with
// every stored row of those columns: rows [gcol0, d) for 'l', [0, gcol0+ncols)
// for 'u'.  The tile's rows are walked in H-row chunks; each stored element
// a(i,c) is loaded once (256-bit) and used twice:
//   t1[i] += a(i,c) x[c]            for i >= c ('l') / i <= c ('u')
//   t2[c] += op(a(i,c)) x[i]        for i >  c ('l') / i <  c ('u')
// with op = conj for HEMV, identity for SYMV (and complex symmetric), and
// the Hermitian diagonal forced real (kernels.py:353-354).  Only chunks that
// intersect the diagonal band evaluate the triangle masks; elements outside
// the stored triangle are replaced by zero with a select, so the
// unreferenced triangle may hold anything (NaN included).
//
// t1 for a chunk is complete after a shared-memory reduction over the warps
// and is written to ws1[tile][row] (each (tile, row) exactly once).  t2
// stays in registers while a CTA walks consecutive items of one tile and
// is written once per (tile, segment) to its own slot row of ws2.  The
// epilogue sums ws1 over the tiles covering each row and ws2 over the slots
// of the row's own tile, in fixed order.
//
// Schedule ("segments").  The T items are cut into segments of K
// consecutive items dealt round robin to the P CTAs (segment s belongs to
// CTA s mod P) for `rounds` full rounds; the remaining items are split into
// P contiguous tail segments (classic stream-K), so every CTA streams the
// same bytes to within one item.  With K small, the CTAs resident at any
// moment stream NEIGHBOURING row chunks of the same few tiles: the DRAM
// sees 128 columns x (P K / #tiles) KiB runs instead of 148 x 128 scattered
// 1 KiB pages, which removes the column-stride aliasing of ld = N
// operands (profiles/r2_stream_probe*.jsonl: 128 x 1 KiB items at ld =
// 40960 stream at 6.83 TB/s contiguous, 7.05 TB/s interleaved with K = 4,
// the same as with a padded ld).  rounds = 0 is contiguous stream-K.
//
// Tiles come from a host-built table so the same kernel serves the
// single-GPU path, diagonal submatrices (offset API) and the local
// block-column panels of the mgpu layout.
// ---------------------------------------------------------------------------
struct SymTile {
  int gcol0;        // first global column of the tile
  int lcol0;        // first local column (pointer offset in the panel)
  int ncols;        // columns in the tile (<= W)
  int row0, row1;   // stored logical rows [row0, row1)
  int chunk0;       // first physical H-row chunk
  long long prefix; // items before this tile
  int seg0;         // segment holding the tile's first item
  int slot0;        // first ws2 slot row of the tile (one per segment touching it)
  int nseg;         // segments touching the tile
};

struct SymParams {
  const void *A;
  long long lda;
  int d;
  int lead;
  const void *x;
  void *ws1;
  long long ws1_ld;
  void *ws2;
  long long ws2_ld;  // slot row width (= W)
  const SymTile *tiles;
  int ntiles;
  long long total;
  int P;
  int tile_w;  // > 0: tiles are uniform, tile k = columns [k*tile_w, (k+1)*tile_w) (single GPU)
  int K;        // items per interleaved segment
  int rounds;   // full rounds of P interleaved segments
  long long base, rem;  // first tail item (rounds * P * K) and tail length
  long long nseg;       // rounds * P + P
  const int *seg_tile;  // per segment: tile of its first item (host-built)
#if KBLAS_SYMV_TRACE
  unsigned long long *trace = nullptr;  // instrumentation: per-CTA start / end globaltimer, SM id (kblas_set_symv_trace)
#endif
  int pdl = 0;          // launched as the programmatic dependent of a hostvec copy-in grid
                        // (1: prefetch the first A segments before the wait, 2: no prefetch)
  unsigned *tail_ctr = nullptr;  // tail grid of a split call (see run_symv): CTA counter, else nullptr
};

// first item of segment s (s == nseg gives total)
__host__ __device__ __forceinline__ long long sym_seg_lo(long long s, int K, int rounds, int P, long long base,
                                                         long long rem) {
  const long long full = (long long)rounds * P;
  return s < full ? s * K : base + (s - full) * rem / P;
}
// segment holding item q
__host__ __device__ __forceinline__ long long sym_seg_of(long long q, int K, int rounds, int P, long long base,
                                                         long long rem) {
  return q < base ? q / K : (long long)rounds * P + sk_owner(q - base, rem, P);
}

// Walks one CTA's items in order: segments blockIdx.x, +P, +2P, ...; k is
// the tile of item q.  The next segment's start tile is fetched one
// segment ahead so a segment switch does not wait on it.  Item and segment
// indices fit in 32 bits (the host checks total < 2^31).
struct SymCursor {
  int s, q, hi, tnext;
  int k, knext;
  bool done;
  __device__ __forceinline__ int lo_of(const SymParams &p, int seg) const {
    return (int)sym_seg_lo(seg, p.K, p.rounds, p.P, p.base, p.rem);
  }
  __device__ __forceinline__ void set_tile(const SymParams &p, int kk) {
    k = kk;
    tnext = (k + 1 < p.ntiles) ? (int)p.tiles[k + 1].prefix : (int)p.total;
  }
  // first non-empty segment at or after seg (stepping by P)
  __device__ __forceinline__ bool seek(const SymParams &p, int seg) {
    for (; seg < p.nseg; seg += p.P) {
      const int a = lo_of(p, seg), b = lo_of(p, seg + 1);
      if (a < b) {
        s = seg;
        q = a;
        hi = b;
        return true;
      }
    }
    done = true;
    return false;
  }
  __device__ __forceinline__ bool init(const SymParams &p) {
    done = false;
    if (!seek(p, blockIdx.x)) return false;
    set_tile(p, p.seg_tile[s]);
    knext = s + p.P < p.nseg ? p.seg_tile[s + p.P] : 0;
    return true;
  }
  __device__ __forceinline__ void advance(const SymParams &p) {
    if (++q < hi) {
      if (q >= tnext) set_tile(p, k + 1);
      return;
    }
    const int prev = s;
    if (!seek(p, s + p.P)) return;
    set_tile(p, s == prev + p.P ? knext : p.seg_tile[s]);
    knext = s + p.P < p.nseg ? p.seg_tile[s + p.P] : 0;
  }
};

// t1 window record: the tile, first physical row and stored row range of
// an item whose t1 partials wait in shared memory for the window barrier
struct SymT1Meta { int k, p0, clo, chi; };

// XS: keep the tile's x_col values in shared memory (each warp its own CW
// slots, so no extra barrier) instead of CW registers per thread, which
// frees registers for wider per-warp column sets.
// B: items per barrier window.  Each warp drops the t1 partials of B
// consecutive items into shared memory and the CTA meets at one barrier per
// B items, where all NT threads reduce the B x H rows in warp order; warps
// drift freely inside a window, so one late load no longer stalls all 16
// warps at every item (ncu: barrier stalls were ~46 % of warp samples with
// B = 1, profiles/r2a_ncu_summary.md).
//
// Split calls (1-CTA/SM kernels, run_symv): the interleaved rounds run in one
// grid and the last few percent of the items in a second, programmatic-
// dependent grid of small CTAs (tail_ctr != nullptr) that the block
// scheduler hands to SMs as the first grid's CTAs finish, so the SMs that
// finish early take the tail instead of idling.  The tail grid does not
// wait for the first one (it writes other ws1 rows and its own ws2 slots);
// its last CTA does, so the pair completes together for the epilogue.  The
// first grid releases its dependents after its own wait, so the tail grid
// of a host-vector call starts only once x is staged (it never waits at
// its start; p.pdl != 0 would make it wait, the run_symv launch does not
// set it).
template <class T, int V, int NW, int CW, int R, bool LOWER, bool HERM, int MINB = 1, bool XS = false, int B = 1>
__global__ void __launch_bounds__(NW * 32, MINB) kblas_symv_kernel(const SymParams p) {
  if constexpr (MINB != 1) griddep_launch_dependents();
  constexpr int NT = NW * 32;
  constexpr int H = 32 * V * R;
  // t1 partials, double-buffered windows: red[buf][item][warp][row]
  // (dynamic: 2*B*NW*H*sizeof(T)), and the window's item records
  extern __shared__ __align__(16) unsigned char symv_smem[];
  T(*red)[B][NW][H] = reinterpret_cast<T(*)[B][NW][H]>(symv_smem);
  __shared__ SymT1Meta meta[2][B];

  const T *__restrict__ A = static_cast<const T *>(p.A);
  const T *__restrict__ x = static_cast<const T *>(p.x);
  T *__restrict__ ws1 = static_cast<T *>(p.ws1);
  T *__restrict__ ws2 = static_cast<T *>(p.ws2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  const uint64_t keep = policy_evict_last();
  SymCursor c;
#if KBLAS_SYMV_TRACE
  // investigation builds only: the two trace branches cost the 2-CTA/SM
  // variant 5-11 % at d = 4096..8192 (register allocation), so the product
  // build compiles them out
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[3 * blockIdx.x] = globaltimer_ns();
    p.trace[3 * blockIdx.x + 2] = smid;
  }
  if (!c.init(p)) {
    if (p.trace != nullptr && threadIdx.x == 0) p.trace[3 * blockIdx.x + 1] = globaltimer_ns();
    return;
  }
#else
  if (!c.init(p)) {
    if constexpr (MINB == 1) {  // (the host gives every tail CTA work; kept for safety)
      if (p.tail_ctr != nullptr && threadIdx.x == 0 && atomicAdd(p.tail_ctr, 1u) == gridDim.x - 1) {
        griddep_wait();
        *p.tail_ctr = 0u;
      }
    }
    return;
  }
#endif
  const int cl = warp * CW;
  const bool xvec = V > 1 && p.lead == 0 && (reinterpret_cast<uintptr_t>(x) % (V * sizeof(T))) == 0;

  // Software pipeline over the CTA's items: the loads of the next item
  // (possibly in the next tile or segment) are issued right after this
  // item's FMAs, so they are in flight while this item's t1 partial goes
  // through shared memory, the barrier and the fixed-order cross-warp
  // reduction.
  Pack<T, V> a[CW][R];
  T xr[R][V];
  auto load_x = [&](const SymTile &t, long long q) {
    const int p0 = (t.chunk0 + (int)(q - t.prefix)) * H;
    const int vlo = t.row0 + p.lead, vhi = t.row1 + p.lead;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int ps0 = p0 + r * 32 * V + lane * V;
      if (xvec && ps0 >= vlo && ps0 + V <= vhi) {
        ld_xvec<T, V>(xr[r], x + ps0);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int ps = ps0 + v;
          xr[r][v] = (ps >= vlo && ps < vhi) ? ld_x(x + (ps - p.lead)) : zero<T>();
        }
      }
    }
  };
  auto load_a = [&](const SymTile &t, long long q) {
    const int p0 = (t.chunk0 + (int)(q - t.prefix)) * H;
    const int vlo = t.row0 + p.lead, vhi = t.row1 + p.lead;
    const T *Aw = A + (long long)(t.lcol0 + cl) * p.lda;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const bool cok = cl + j < t.ncols;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int vs = p0 + r * 32 * V + lane * V;
        ld_pack(a[j][r], Aw + (long long)j * p.lda + vs, cok && vs < vhi && vs + V > vlo, pol);
      }
    }
  };
  auto load = [&](const SymTile &t, long long q) {
    load_x(t, q);
    load_a(t, q);
  };

  SymTile tl = p.tiles[c.k];
  T t2[CW];
  __shared__ T xs_buf[XS ? NW * CW : 1];
  T xr_c[XS ? 1 : CW];  // x_col in registers (!XS)
  auto set_xc = [&](const SymTile &t) {
    if constexpr (XS) {
      __syncwarp();
      if (lane < CW) xs_buf[cl + lane] = (cl + lane < t.ncols) ? ld_x(x + t.gcol0 + cl + lane) : zero<T>();
      __syncwarp();
    } else {
#pragma unroll
      for (int j = 0; j < CW; ++j) xr_c[j] = (cl + j < t.ncols) ? ld_x(x + t.gcol0 + cl + j) : zero<T>();
    }
  };
  auto xcj = [&](int j) -> T {
    if constexpr (XS) return xs_buf[cl + j]; else return xr_c[j];
  };
  // hostvec call: the first item's A segments are prefetched into L2
  // before griddepcontrol.wait, so A streams while the copy-in grid is
  // still fetching x (no registers held across the wait)
  if (p.pdl == 1) {
    const int p0 = (tl.chunk0 + (int)(c.q - tl.prefix)) * H;
    const int vlo = tl.row0 + p.lead, vhi = tl.row1 + p.lead;
    const T *Aw = A + (long long)(tl.lcol0 + cl) * p.lda;
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int vs = p0 + r * 32 * V + lane * V;
        if (cl + j < tl.ncols && vs < vhi && vs + V > vlo) prefetch_l2(Aw + (long long)j * p.lda + vs);
      }
  }
  if constexpr (MINB == 1) {
    // the tail grid of a split call does not wait for the first grid
    if (p.tail_ctr == nullptr || p.pdl != 0) griddep_wait();
    griddep_launch_dependents();
  } else {
    griddep_wait();
  }
  set_xc(tl);
#pragma unroll
  for (int j = 0; j < CW; ++j) t2[j] = zero<T>();
  load(tl, c.q);
  int buf = 0, wi = 0;  // window buffer, item index inside the window
  for (;;) {
    const int p0 = (tl.chunk0 + (int)(c.q - tl.prefix)) * H;
    const int vlo = tl.row0 + p.lead, vhi = tl.row1 + p.lead;
    const int g0 = p0 - p.lead;  // logical row of the chunk's first physical row
    T acc[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[r][v] = zero<T>();
    const bool diag = (g0 < tl.gcol0 + tl.ncols) && (g0 + H > tl.gcol0);
    const bool inside = p0 >= vlo && p0 + H <= vhi;
    if (!diag && inside) {
#pragma unroll
      for (int j = 0; j < CW; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const T e = a[j][r].v(v);
            acc[r][v] = fma_(e, xcj(j), acc[r][v]);
            t2[j] = fmax_<HERM>(e, xr[r][v], t2[j]);
          }
    } else if (!diag) {
      // first/last chunk of a tile: rows outside the stored range are masked
      // (x is already zero there, so only t1 needs the select)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int ps = p0 + r * 32 * V + lane * V + v;
          const bool ok = ps >= vlo && ps < vhi;
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            const T e = sel(ok, a[j][r].v(v));
            acc[r][v] = fma_(e, xcj(j), acc[r][v]);
            t2[j] = fmax_<HERM>(e, xr[r][v], t2[j]);
          }
        }
    } else {
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int cc = tl.gcol0 + cl + j;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int ps = p0 + r * 32 * V + lane * V + v;
            const int i = ps - p.lead;
            const bool ok = ps >= vlo && ps < vhi;
            const bool in1 = ok && (LOWER ? i >= cc : i <= cc);
            const bool in2 = ok && (LOWER ? i > cc : i < cc);
            T e1 = sel(in1, a[j][r].v(v));
            if (HERM && i == cc) e1 = realify(e1);
            acc[r][v] = fma_(e1, xcj(j), acc[r][v]);
            t2[j] = fmax_<HERM>(sel(in2, a[j][r].v(v)), xr[r][v], t2[j]);
          }
      }
    }

    const int s_cur = c.s, kcur = c.k;
    c.advance(p);
    // end of this CTA's run through the tile (tile, segment or work ends):
    // flush the tile's column sums (t2) into the segment's slot row
    if (c.done || c.k != kcur || c.s != s_cur) {
      T *row = ws2 + (long long)(tl.slot0 + (s_cur - tl.seg0)) * p.ws2_ld;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const T sum = warp_sum(t2[j]);
        if (lane == 0 && cl + j < tl.ncols) row[cl + j] = sum;
        t2[j] = zero<T>();
      }
    }
    const SymTile cur = tl;  // the tile this chunk's t1 belongs to
    if (!c.done) {
      if (c.k != kcur) {
        tl = p.tiles[c.k];
        set_xc(tl);
      }
      load(tl, c.q);  // in flight during the reduction below
    }

#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) red[buf][wi][warp][r * 32 * V + lane * V + v] = acc[r][v];
    if (threadIdx.x == 0) meta[buf][wi] = SymT1Meta{kcur, p0, cur.row0 + p.lead, cur.row1 + p.lead};
    if (++wi == B || c.done) {
      __syncthreads();
      // fixed-order (warp 0..NW-1) sum of every row of the window's items
      for (int t = threadIdx.x; t < wi * H; t += NT) {
        const int it = t / H, row = t - it * H;
        const SymT1Meta m = meta[buf][it];
        const int ps = m.p0 + row;
        if (ps >= m.clo && ps < m.chi) {
          T sm = red[buf][it][0][row];
#pragma unroll
          for (int w = 1; w < NW; ++w) sm = add_(sm, red[buf][it][w][row]);
          st_keep(ws1 + (long long)m.k * p.ws1_ld + (ps - p.lead), sm, keep);
        }
      }
      buf ^= 1;
      wi = 0;
    }
    if (c.done) break;
  }
#if KBLAS_SYMV_TRACE
  if (p.trace != nullptr && threadIdx.x == 0) p.trace[3 * blockIdx.x + 1] = globaltimer_ns();
#endif
  if constexpr (MINB == 1) {
    // tail grid: the last CTA to finish waits for the first grid, so the
    // epilogue (a dependent of this grid) sees both grids' partials
    if (p.tail_ctr != nullptr && threadIdx.x == 0 && atomicAdd(p.tail_ctr, 1u) == gridDim.x - 1) {
      griddep_wait();
      *p.tail_ctr = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// Epilogues: fixed-order sum of partial slots, then y = alpha*sum + beta*y.
// beta_zero: y is written without being read (kernels.py:136-137).
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ void store_axpby(T *y, long long i, T alpha, T s, T beta, int beta_zero) {
  T r = mul_(alpha, s);
  if (!beta_zero) r = fma_(beta, y[i], r);
  y[i] = r;
}

// GEMV epilogues: one CTA per 32 outputs (lane = output), the EW warps split
// the output's slot range into EW fixed contiguous parts (deterministic),
// warp 0 adds the parts in order.
template <class T, int EW>
__device__ __forceinline__ T slot_sum(const T *__restrict__ ws, long long ws_ld, long long idx, int nslots,
                                      bool valid, T (*part)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int len = valid ? nslots : 0;
  const int s0 = (int)((long long)len * warp / EW), s1 = (int)((long long)len * (warp + 1) / EW);
  part[warp][lane] = sum_slots(ws, ws_ld, idx, s0, s1);
  __syncthreads();
  T s = part[0][lane];
#pragma unroll
  for (int w = 1; w < EW; ++w) s = add_(s, part[w][lane]);
  return s;
}

template <class T, int EW>
__global__ void __launch_bounds__(EW * 32) kblas_gemv_n_epilogue(T *y, const T *__restrict__ ws, long long ws_ld, int m,
                                                          int lead, int RB, int KS, long long total, int P,
                                                          T alpha, T beta, int beta_zero) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ T part[EW][32];
  const long long i = (long long)blockIdx.x * 32 + (threadIdx.x & 31);
  const bool valid = i < m;
  int nslots = 0;
  if (valid) {
    const long long rb = (i + lead) / RB;
    nslots = sk_owner(rb * KS + KS - 1, total, P) - sk_owner(rb * KS, total, P) + 1;
  }
  const T s = slot_sum<T, EW>(ws, ws_ld, valid ? i : 0, nslots, valid, part);
  if ((threadIdx.x >> 5) == 0 && valid) store_axpby(y, i, alpha, s, beta, beta_zero);
}

// y indexed by global column c in [0, nglob); columns not owned by this GPU
// (mgpu partial mode) are written as zero.
template <class T, int EW>
__global__ void __launch_bounds__(EW * 32) kblas_gemv_t_epilogue(T *y, const T *__restrict__ ws, long long ws_ld,
                                                          long long nglob, int CBW, int KS, long long total, int P,
                                                          ColMap cm, T alpha, T beta, int beta_zero) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ T part[EW][32];
  const long long c = (long long)blockIdx.x * 32 + (threadIdx.x & 31);
  const long long l = c < nglob ? unmap_col(cm, c) : -1;
  const bool valid = l >= 0;
  int nslots = 0;
  if (valid) {
    const long long cb = l / CBW;
    nslots = sk_owner(cb * KS + KS - 1, total, P) - sk_owner(cb * KS, total, P) + 1;
  }
  const T s = slot_sum<T, EW>(ws, ws_ld, valid ? l : 0, nslots, valid, part);
  if ((threadIdx.x >> 5) == 0 && c < nglob) {
    if (valid) store_axpby(y, c, alpha, s, beta, beta_zero);
    else y[c] = zero<T>();
  }
}

// One CTA per 32 rows (lane = row).  The t1 partials of a row are spread
// over up to d/W tiles and its t2 partials over the CTA slots of the tile
// owning the row's column.  Warp w takes tiles kb+w, kb+w+EW, ... and t2
// slots w, w+EW, ... (a partition that depends only on the row, so the
// summation order is fixed and results are bit-reproducible); the tile
// record is fetched alongside the t1 loads, so a call costs about two L2
// round trips.  Warp 0 then adds the EW parts in order.
// Peer-memory exchange fused into the epilogue of a one-process-per-GPU
// mgpu call (dist.P2PExchange): G == 0 disables it.  A non-root rank's y
// is its slot in the root's HBM; its last CTA publishes flags[rank] = seq.
// The root adds the other ranks' slots to its own partial in rank order,
// then beta*y_in, and its last CTA publishes consumed = seq.
struct Xchg {
  int G, rank;
  const void *slots;  // root's slot array (this rank's mapping of it)
  long long slot_ld;
  unsigned long long *flags, *consumed;
  unsigned *counter;  // local arrival counter, zero between calls
  unsigned long long seq;
  const void *y_in;   // root: the caller's y (beta != 0)
};

template <class T, bool LOWER, int EW>
__global__ void __launch_bounds__(EW * 32) kblas_symv_epilogue(T *y, const SymParams p, T alpha, T beta, int beta_zero,
                                                         const Xchg xg) {
  griddep_launch_dependents();
  griddep_wait();
  if (xg.G > 0 && xg.rank != 0 && xg.seq > 1) {
    // this rank's slot is free once the root consumed the previous call
    if (threadIdx.x == 0) spin_until(xg.consumed, xg.seq - 1);
    __syncthreads();
  }
  __shared__ T part[EW][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long i = min((long long)blockIdx.x * 32 + lane, (long long)p.d - 1);
  const bool valid = (long long)blockIdx.x * 32 + lane < p.d;
  const T *__restrict__ ws1 = static_cast<const T *>(p.ws1);
  const T *__restrict__ ws2 = static_cast<const T *>(p.ws2);
  // nle = number of tiles with gcol0 <= i (tiles sorted by gcol0)
  int nle;
  if (p.tile_w > 0) {
    nle = min(p.ntiles, (int)(i / p.tile_w) + 1);
  } else {
    int lo = 0, hi = p.ntiles;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (p.tiles[mid].gcol0 <= i) lo = mid + 1; else hi = mid;
    }
    nle = lo;
  }
  // the tile owning column i (if any on this GPU)
  SymTile own{};
  if (nle > 0) own = p.tiles[nle - 1];
  int kb, ke;
  if (LOWER) {
    kb = 0;
    ke = nle;
  } else {
    kb = nle;
    if (nle > 0 && (p.tile_w > 0 || own.gcol0 + own.ncols > i)) kb = nle - 1;
    ke = p.ntiles;
  }
  if (!valid) ke = kb;
  T acc = zero<T>();
  for (int k = kb + warp; k < ke; k += 8 * EW) {
    T t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = (k + u * EW < ke) ? ws1[(long long)(k + u * EW) * p.ws1_ld + i] : zero<T>();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k + u * EW < ke) acc = add_(acc, t[u]);
  }
  // t2: the slot rows of the tile owning column i (one per segment)
  if (valid && nle > 0 && i < (long long)own.gcol0 + own.ncols) {
    const T *col = ws2 + (long long)own.slot0 * p.ws2_ld + (i - own.gcol0);
    for (int sl = warp; sl < own.nseg; sl += EW) acc = add_(acc, col[(long long)sl * p.ws2_ld]);
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (xg.G == 0) {
    if (warp != 0 || !valid) return;
    T s = part[0][lane];
#pragma unroll
    for (int w = 1; w < EW; ++w) s = add_(s, part[w][lane]);
    store_axpby(y, i, alpha, s, beta, beta_zero);
    return;
  }
  if (warp == 0) {
    T s = part[0][lane];
#pragma unroll
    for (int w = 1; w < EW; ++w) s = add_(s, part[w][lane]);
    T r = mul_(alpha, s);  // this rank's partial (multidevice.py:224-276)
    if (xg.rank == 0) {
      // the other ranks' slots, in rank order (multidevice.py:276), then
      // beta * y (282-283)
      if (lane == 0)
        for (int g = 1; g < xg.G; ++g) spin_until(xg.flags + g, xg.seq);
      __syncwarp();
      const T *slots = static_cast<const T *>(xg.slots);
      if (valid) {
        for (int g = 1; g < xg.G; ++g) r = add_(r, __ldcv(slots + g * xg.slot_ld + i));
        if (!beta_zero) r = fma_(beta, static_cast<const T *>(xg.y_in)[i], r);
        y[i] = r;
      }
    } else if (valid) {
      y[i] = r;  // a store into the root's HBM
    }
  }
  // the last CTA to finish publishes this rank's arrival (or, on the root,
  // that every slot has been consumed)
  __shared__ bool last;
  if (xg.rank == 0) __threadfence(); else __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(xg.counter, 1u) == gridDim.x - 1;
    if (last) {
      *xg.counter = 0u;
      __threadfence_system();
      st_release_sys(xg.rank == 0 ? xg.consumed : xg.flags + xg.rank, xg.seq);
    }
  }
}

// The same sums as kblas_symv_epilogue, added in the same order (so y is
// bit-identical), for operands whose tiles are 128 columns starting at
// multiples of 128: the wide kernel's tiles on one GPU, or mgpu block
// columns with nb % 128 == 0.  One CTA per 128 rows, which is exactly one
// column block: the block's tile range and owning tile are shared by all
// its rows, and lane l owns rows 32v + l (v = 0..3), so a warp reads a
// tile's t1 partials of the block as one contiguous 128-element run
// (1 KiB for d) instead of 32-element pieces d elements apart.  Measured at
// DSYMV N = 100000 (ws1 of 310 MB, read from HBM): see DESIGN.md §4.
template <class T, bool LOWER, int EW>
__global__ void __launch_bounds__(EW * 32, 2) kblas_symv_epilogue_r128(T *y, const SymParams p, T alpha, T beta,
                                                              int beta_zero, const Xchg xg) {
  griddep_launch_dependents();
  griddep_wait();
  if (xg.G > 0 && xg.rank != 0 && xg.seq > 1) {
    if (threadIdx.x == 0) spin_until(xg.consumed, xg.seq - 1);
    __syncthreads();
  }
  constexpr int RB = 128, VR = RB / 32;
  constexpr int BATCH = sizeof(T) == 16 ? 2 : 4;
  __shared__ T part[EW][RB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long r0 = (long long)blockIdx.x * RB;
  const T *ws1 = static_cast<const T *>(p.ws1);
  const T *ws2 = static_cast<const T *>(p.ws2);
  // local tiles with gcol0 <= r0 (= with gcol0 <= any row of the block)
  int nle;
  if (p.tile_w > 0) {
    nle = min(p.ntiles, (int)(r0 / p.tile_w) + 1);
  } else {
    int lo = 0, hi = p.ntiles;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (p.tiles[mid].gcol0 <= r0) lo = mid + 1; else hi = mid;
    }
    nle = lo;
  }
  SymTile own{};
  if (nle > 0) own = p.tiles[nle - 1];
  const bool owned = nle > 0 && own.gcol0 == r0;  // this GPU holds column block r0 / 128
  int kb, ke;
  if (LOWER) {
    kb = 0;
    ke = nle;
  } else {
    kb = owned ? nle - 1 : nle;
    ke = p.ntiles;
  }
  bool ok[VR];
  long long row[VR];
#pragma unroll
  for (int v = 0; v < VR; ++v) {
    row[v] = r0 + 32 * v + lane;
    ok[v] = row[v] < p.d;
  }
  T acc[VR];
#pragma unroll
  for (int v = 0; v < VR; ++v) acc[v] = zero<T>();
  for (int k = kb + warp; k < ke; k += BATCH * EW) {
    T t[BATCH][VR];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const T *src = ws1 + (long long)(k + u * EW) * p.ws1_ld;
#pragma unroll
      for (int v = 0; v < VR; ++v) t[u][v] = (k + u * EW < ke && ok[v]) ? src[row[v]] : zero<T>();
    }
#pragma unroll
    for (int u = 0; u < BATCH; ++u)
      if (k + u * EW < ke) {
#pragma unroll
        for (int v = 0; v < VR; ++v) acc[v] = add_(acc[v], t[u][v]);
      }
  }
  // t2: the slot rows of the block's own tile (one per segment)
  if (owned) {
    const T *col = ws2 + (long long)own.slot0 * p.ws2_ld;
    for (int sl = warp; sl < own.nseg; sl += EW) {
#pragma unroll
      for (int v = 0; v < VR; ++v)
        if (ok[v] && 32 * v + lane < own.ncols) acc[v] = add_(acc[v], col[(long long)sl * p.ws2_ld + 32 * v + lane]);
    }
  }
#pragma unroll
  for (int v = 0; v < VR; ++v) part[warp][32 * v + lane] = acc[v];
  __syncthreads();
  const int t = threadIdx.x;
  const long long i = r0 + t;
  const bool valid = t < RB && i < p.d;
  T s = zero<T>();
  if (valid) {
    s = part[0][t];
#pragma unroll
    for (int w = 1; w < EW; ++w) s = add_(s, part[w][t]);
  }
  if (xg.G == 0) {
    if (valid) store_axpby(y, i, alpha, s, beta, beta_zero);
    return;
  }
  const T r0v = mul_(alpha, s);  // this rank's partial (multidevice.py:224-276)
  if (xg.rank == 0) {
    // the other ranks' slots, in rank order (multidevice.py:276), then
    // beta * y (282-283)
    if (threadIdx.x == 0)
      for (int g = 1; g < xg.G; ++g) spin_until(xg.flags + g, xg.seq);
    __syncthreads();
    const T *slots = static_cast<const T *>(xg.slots);
    if (valid) {
      T r = r0v;
      for (int g = 1; g < xg.G; ++g) r = add_(r, __ldcv(slots + g * xg.slot_ld + i));
      if (!beta_zero) r = fma_(beta, static_cast<const T *>(xg.y_in)[i], r);
      y[i] = r;
    }
  } else if (valid) {
    y[i] = r0v;  // a store into the root's HBM
  }
  // the last CTA to finish publishes this rank's arrival (or, on the root,
  // that every slot has been consumed)
  __shared__ bool last;
  if (xg.rank == 0) __threadfence(); else __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(xg.counter, 1u) == gridDim.x - 1;
    if (last) {
      *xg.counter = 0u;
      __threadfence_system();
      st_release_sys(xg.rank == 0 ? xg.consumed : xg.flags + xg.rank, xg.seq);
    }
  }
}

// Stages a numpy-vector call's x (and y when beta != 0) from page-locked
// host memory, mapped into the device address space, into the call's
// device staging buffer (replaces two cudaMemcpyAsync H2D copies and their
// copy-engine round trips).  It releases its dependents at once: the main
// kernel, launched with programmatic stream serialization, streams A
// meanwhile and waits in griddepcontrol.wait before it reads x or y.
//
// The grid is itself launched with programmatic stream serialization: on a
// queue of calls it starts while the previous call's last kernel drains.
// Each thread reads its first 16-byte unit of x and y over PCIe first and
// waits in griddepcontrol.wait before its first store, so the staging
// buffer is written only after every earlier kernel of the stream is done
// with it (each library kernel waits on its own primary before it
// completes, so the wait covers the whole stream).
__device__ __forceinline__ void hostvec_copy(char *dst, const char *src, long long bytes, long long tid,
                                             long long nt, bool first_done) {
  if (bytes <= 0) return;
  long long done = 0;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const long long n16 = bytes >> 4;
    for (long long i = tid + (first_done ? nt : 0); i < n16; i += nt)
      reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    done = n16 << 4;
  }
  // element sizes are multiples of 4 bytes
  for (long long i = (done >> 2) + tid; i < (bytes >> 2); i += nt)
    reinterpret_cast<unsigned *>(dst)[i] = reinterpret_cast<const unsigned *>(src)[i];
}

static __global__ void kblas_hostvec_in_kernel(char *dx, const char *hx, long long xbytes, char *dy, const char *hy,
                                        long long ybytes) {
  griddep_launch_dependents();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  auto aligned = [](const char *d, const char *s) {
    return ((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(s)) & 15) == 0;
  };
  const bool px = aligned(dx, hx) && tid < (xbytes >> 4), py = aligned(dy, hy) && tid < (ybytes >> 4);
  uint4 ux = make_uint4(0, 0, 0, 0), uy = make_uint4(0, 0, 0, 0);
  if (px) ux = reinterpret_cast<const uint4 *>(hx)[tid];
  if (py) uy = reinterpret_cast<const uint4 *>(hy)[tid];
  griddep_wait();  // earlier kernels of the stream are done with the staging buffer
  if (px) reinterpret_cast<uint4 *>(dx)[tid] = ux;
  if (py) reinterpret_cast<uint4 *>(dy)[tid] = uy;
  hostvec_copy(dx, hx, xbytes, tid, nt, aligned(dx, hx));
  hostvec_copy(dy, hy, ybytes, tid, nt, aligned(dy, hy));
}

// y <- beta * y (beta == 0: zero fill); run_scal semantics (kernels.py:127-146)
template <class T>
__global__ void kblas_scal_kernel(T *y, long long n, T beta, int beta_zero) {
  griddep_launch_dependents();
  griddep_wait();  // y staged by a hostvec copy-in grid (no-op otherwise)
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  y[i] = beta_zero ? zero<T>() : mul_(beta, y[i]);
}

// mgpu root combine: y = beta*y + sum_g part[g] in device order
// (multidevice.py:161,176,276 then 282-283).  part[g] may be a peer
// pointer on another GPU (NVLink load) or a local copy.
constexpr int kMaxGpus = 16;
template <class T> struct PartList { const T *p[kMaxGpus]; };
template <class T>
__global__ void kblas_mgpu_combine_kernel(T *y, PartList<T> parts, int G, long long n, T beta, int beta_zero) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T s = parts.p[0][i];
  for (int g = 1; g < G; ++g) s = add_(s, parts.p[g][i]);
  y[i] = beta_zero ? s : fma_(beta, y[i], s);
}

// ---------------------------------------------------------------------------
// One-process-per-GPU exchange over peer memory (no NCCL): every rank
// writes its partial y straight into its slot of a root-resident buffer
// (opened with CUDA IPC; NVLink stores when the ranks are on different
// GPUs), then publishes the call's sequence number in flags[rank] with a
// system-scope release.  The root's combine kernel acquires all flags,
// sums the slots in rank order (the reference's device-order sum,
// multidevice.py:276, so results do not depend on arrival order), adds
// beta*y (282-283), and its last CTA publishes `consumed` so ranks may
// reuse their slots.
// ---------------------------------------------------------------------------
// rank side: its partial (written by the preceding kernels on this stream)
// becomes visible system-wide, then flags[rank] = seq
static __global__ void kblas_p2p_signal_kernel(unsigned long long *flag, unsigned long long seq) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(flag, seq);
  }
}

// wait until *flag >= seq (e.g. the root has consumed the previous call)
static __global__ void kblas_p2p_wait_kernel(const unsigned long long *flag, unsigned long long seq) {
  if (threadIdx.x == 0) spin_until(flag, seq);
  __syncthreads();
}

template <class T>
__global__ void kblas_p2p_combine_kernel(const T *__restrict__ slots, long long slot_ld, int G,
                                   const unsigned long long *flags, unsigned long long seq, T *y, long long n,
                                   T beta, int beta_zero, unsigned long long *consumed, unsigned *counter) {
  if (threadIdx.x == 0) {
    for (int g = 0; g < G; ++g) spin_until(flags + g, seq);
  }
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    T s = __ldcv(slots + i);
    for (int g = 1; g < G; ++g) s = add_(s, __ldcv(slots + g * slot_ld + i));
    y[i] = beta_zero ? s : fma_(beta, y[i], s);
  }
  // the last CTA to finish releases the slots for the next call
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
    if (last) {
      *counter = 0u;
      __threadfence_system();
      st_release_sys(consumed, seq);
    }
  }
}

}  // namespace kb
