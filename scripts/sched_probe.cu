// sched_probe.cu — does the SYMV item schedule leave SMs idle at the end?
//
// Streams the lower triangle of an n x n double matrix in the SYMV
// kernel's access pattern (W = 128-column tiles of 128-row chunks, 16 warps
// x 8 columns, one 256-bit load per lane per column, a CTA barrier per
// item, one FMA per element) under three item schedules over 148 CTAs:
//   static  : contiguous stream-K ranges,
//   inter   : segments of K items dealt round robin (the library's
//             schedule, without its even tail split),
//   dynamic : segments of K items taken from a global counter (thread 0
//             takes the next segment one segment ahead; the index reaches
//             the other warps through shared memory at an item barrier).
// Reports the kernel time (events) and the spread of the CTAs' finish times
// (globaltimer), i.e. how long the first finished SMs sit idle.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sched_probe scripts/sched_probe.cu
//   ./scripts/sched_probe N [K]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

struct Tile { int col0, chunk0; long long prefix; };

__device__ __forceinline__ void ld256(uint32_t (&w)[8], const void *p, bool pred) {
  const int pr = pred ? 1 : 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = 0u;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %9, 0;\n\t"
               "@q ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
               : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7])
               : "l"(p), "r"(pr));
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int NW = 16, CW = 8;

__device__ __forceinline__ int tile_of(const Tile *tiles, int ntiles, long long q) {
  int lo = 0, hi = ntiles;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (tiles[mid].prefix <= q) lo = mid; else hi = mid;
  }
  return lo;
}

// MODE 0 static, 1 interleaved, 2 dynamic, 3 hybrid (interleaved for the
// first s_static segments, the rest taken from the counter)
template <int MODE, bool F32>
__global__ void __launch_bounds__(NW * 32, 1) sched(const char *A, long long ld, int n, const Tile *tiles,
                                                    int ntiles, long long total, int P, int K, unsigned *ctr,
                                                    const int *seg_tile, double *out, unsigned long long *tend,
                                                    long long s_static, int part = 0, int KB = 2) {
  constexpr int EB = F32 ? 4 : 8, H = 32 * 32 / EB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 4) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int s_next[2];
  const long long nseg = (total + K - 1) / K;
  // current range [q, hi)
  long long q, hi, seg = 0;
  unsigned grabbed = 0;
  if (MODE == 0) {
    q = (long long)blockIdx.x * total / P;
    hi = (long long)(blockIdx.x + 1) * total / P;
  } else if (MODE == 1) {
    seg = blockIdx.x;
    q = seg * K;
    hi = min(total, q + K);
    if (seg >= nseg) q = hi = total;
  } else if (MODE == 2) {
    seg = blockIdx.x;  // first segment: static
    q = seg * K;
    hi = min(total, q + K);
    if (seg >= nseg) q = hi = total;
    if (threadIdx.x == 0) grabbed = P + atomicAdd(ctr, 1u);  // one segment ahead
  } else if (MODE == 3) {
    seg = blockIdx.x;
    q = seg * K;
    hi = min(total, q + K);
    if (seg >= nseg) q = hi = total;
    if (threadIdx.x == 0)
      grabbed = seg + P < s_static ? (unsigned)(seg + P) : (unsigned)(s_static + atomicAdd(ctr, 1u));
  } else if (part == 0) {  // MODE 4, first kernel: interleaved segments below s_static
    seg = blockIdx.x;
    q = seg * K;
    hi = min(total, q + K);
    if (seg >= s_static) q = hi = total;
  } else {  // MODE 4, second kernel: KB-item CTAs over the rest
    q = s_static * K + (long long)blockIdx.x * KB;
    hi = min(total, q + KB);
    if (q >= total) q = hi = total;
  }
  double acc = 0.0;
  uint32_t a[CW][8];
  int k = q < total ? ((MODE == 0 || (MODE == 4 && part == 1)) ? tile_of(tiles, ntiles, q) : seg_tile[seg]) : 0;
  // dynamic: the next segment and its start tile, fetched a segment ahead
  long long nseg_id = -1;
  int nk = 0;
  Tile t = tiles[k];
  long long tnext = k + 1 < ntiles ? tiles[k + 1].prefix : total;
  auto load = [&](const Tile &tl, long long qq) {
    const long long p0 = (long long)(tl.chunk0 + (qq - tl.prefix)) * H;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const long long row = p0 + lane * (32 / EB);
      ld256(a[j], A + ((long long)(tl.col0 + warp * CW + j) * ld + row) * EB, row < n);
    }
  };
  if (q < hi) load(t, q);
  int par = 0;
  while (q < hi) {
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int v = 0; v < 8; v += 2)
        acc = fma(__hiloint2double((int)a[j][v + 1], (int)a[j][v]), 1.0000001, acc);
    if (MODE >= 2 && threadIdx.x == 0 && q == seg * K) s_next[par] = (int)grabbed;  // after this item's loads
    __syncthreads();
    if (MODE >= 2 && q == seg * K) {
      nseg_id = s_next[par];
      nk = nseg_id < nseg ? seg_tile[nseg_id] : 0;
    }
    long long nq = q + 1;
    if (nq >= hi) {
      // next range
      if (MODE == 0 || (MODE == 4 && part == 1)) {
        nq = hi = total;
      } else if (MODE == 4) {
        seg += P;
        nq = seg * K;
        hi = min(total, nq + K);
        if (seg >= s_static) nq = hi = total;
        if (nq < hi) k = seg_tile[seg];
      } else if (MODE == 1) {
        seg += P;
        nq = seg * K;
        hi = min(total, nq + K);
        if (seg >= nseg) nq = hi = total;
        if (nq < hi) k = seg_tile[seg];
      } else {
        seg = nseg_id;
        par ^= 1;
        nq = seg * K;
        hi = min(total, nq + K);
        if (seg >= nseg) nq = hi = total;
        if (threadIdx.x == 0 && seg < nseg) {
          if (MODE == 2) grabbed = P + atomicAdd(ctr, 1u);
          else grabbed = seg + P < s_static ? (unsigned)(seg + P) : (unsigned)(s_static + atomicAdd(ctr, 1u));
        }
        k = nk;
      }
      if (nq < hi) {
        t = tiles[k];
        tnext = k + 1 < ntiles ? tiles[k + 1].prefix : total;
      }
    } else if (nq >= tnext) {
      ++k;
      t = tiles[k];
      tnext = k + 1 < ntiles ? tiles[k + 1].prefix : total;
    }
    if (nq < hi) load(t, nq);
    q = nq;
  }
  if (MODE == 4 && part == 1) {
    // the last CTA of the second kernel waits for the first one, so the
    // pair completes together (what an epilogue would wait for)
    if (threadIdx.x == 0 && atomicAdd(ctr, 1u) == gridDim.x - 1) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      *ctr = 0u;
    }
    if (acc == 12345.0) out[0] = acc;
    return;
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) tend[blockIdx.x] = gtimer();
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32768;
  const int K = argc > 2 ? atoi(argv[2]) : 6;
  const bool f32 = argc > 3 && argv[3][0] == 's';
  const double frac = argc > 4 ? atof(argv[4]) : 0.1;  // hybrid: dynamic share of the segments
  const int EB = f32 ? 4 : 8, H = 1024 / EB;
  const long long ld = n;
  const int W = NW * CW;
  std::vector<Tile> tiles;
  long long total = 0;
  for (int c0 = 0; c0 < n; c0 += W) {
    const int chunk0 = c0 / H;
    const int nch = (n + H - 1) / H - chunk0;
    tiles.push_back({c0, chunk0, total});
    total += nch;
  }
  std::vector<int> segt;
  for (long long sg = 0; sg * K < total; ++sg) {
    int kk = 0;
    while (kk + 1 < (int)tiles.size() && tiles[kk + 1].prefix <= sg * K) ++kk;
    segt.push_back(kk);
  }
  int *dseg;
  cudaMalloc(&dseg, sizeof(int) * segt.size());
  cudaMemcpy(dseg, segt.data(), sizeof(int) * segt.size(), cudaMemcpyHostToDevice);
  char *A;
  double *out;
  unsigned *ctr;
  unsigned long long *tend;
  Tile *dt;
  const int P = 148;
  cudaMalloc(&A, (size_t)EB * ld * n);
  cudaMemset(A, 0, (size_t)EB * ld * n);
  cudaMalloc(&out, sizeof(double) * P * NW * 32);
  cudaMalloc(&ctr, sizeof(unsigned));
  cudaMalloc(&tend, sizeof(unsigned long long) * P);
  cudaMalloc(&dt, sizeof(Tile) * tiles.size());
  cudaMemcpy(dt, tiles.data(), sizeof(Tile) * tiles.size(), cudaMemcpyHostToDevice);
  const double bytes = (double)EB * ((double)n * (n + 1) / 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const long long nseg_h = (total + K - 1) / K;
  const long long s_static = (long long)(nseg_h * (1.0 - frac)) / P * P;
  const int KB = argc > 5 ? atoi(argv[5]) : 2;
  const long long s_split = (long long)(nseg_h * (1.0 - frac));  // split: first-kernel segments
  const long long tail_items = std::max<long long>(0, total - s_split * K);
  // split: interleaved segments below s_split in one kernel, the rest as
  // KB-item CTAs in a programmatic dependent that the block scheduler
  // hands to the SMs as the first kernel's CTAs finish
  auto split = [&](bool is32) {
    if (is32) sched<4, true><<<P, NW * 32>>>(A, ld, n, dt, (int)tiles.size(), total, P, K, ctr, dseg, out, tend, s_split, 0, KB);
    else sched<4, false><<<P, NW * 32>>>(A, ld, n, dt, (int)tiles.size(), total, P, K, ctr, dseg, out, tend, s_split, 0, KB);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max<long long>(1, (tail_items + KB - 1) / KB));
    cfg.blockDim = dim3(NW * 32);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const Tile *ct = dt;
    const int nt = (int)tiles.size();
    const int one = 1;
    if (is32) cudaLaunchKernelEx(&cfg, sched<4, true>, (const char *)A, ld, n, ct, nt, total, P, K, ctr, (const int *)dseg, out, tend, s_split, one, KB);
    else cudaLaunchKernelEx(&cfg, sched<4, false>, (const char *)A, ld, n, ct, nt, total, P, K, ctr, (const int *)dseg, out, tend, s_split, one, KB);
  };
  auto run = [&](int mode, int reps, float *ms, double *spread, double *mean_idle) {
    std::vector<unsigned long long> te(P);
    float best = 1e30f;
    double bsp = 0, bidle = 0;
    for (int r = 0; r < reps; ++r) {
      cudaMemset(ctr, 0, sizeof(unsigned));
      cudaEventRecord(e0);
#define SCHED(M, F) sched<M, F><<<P, NW * 32>>>(A, ld, n, dt, (int)tiles.size(), total, P, K, ctr, dseg, out, tend, s_static)
      if (f32) {
        if (mode == 0) SCHED(0, true);
        if (mode == 1) SCHED(1, true);
        if (mode == 2) SCHED(2, true);
        if (mode == 3) SCHED(3, true);
        if (mode == 4) split(true);
      } else {
        if (mode == 0) SCHED(0, false);
        if (mode == 1) SCHED(1, false);
        if (mode == 2) SCHED(2, false);
        if (mode == 3) SCHED(3, false);
        if (mode == 4) split(false);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t;
      cudaEventElapsedTime(&t, e0, e1);
      cudaMemcpy(te.data(), tend, sizeof(unsigned long long) * P, cudaMemcpyDeviceToHost);
      const unsigned long long mx = *std::max_element(te.begin(), te.end());
      const unsigned long long mn = *std::min_element(te.begin(), te.end());
      double idle = 0;
      for (auto v : te) idle += (double)(mx - v);
      if (t < best) {
        best = t;
        bsp = (mx - mn) * 1e-3;
        bidle = idle / P * 1e-3;
      }
    }
    *ms = best;
    *spread = bsp;
    *mean_idle = bidle;
  };
  const char *names[5] = {"static", "interleaved", "dynamic", "hybrid", "split"};
  for (int pass = 0; pass < 2; ++pass)
    for (int mode = 1; mode < 5; mode += (mode == 1 ? 3 : 1)) {
      float ms;
      double sp, idle;
      run(mode, 10, &ms, &sp, &idle);
      if (pass == 1)
        printf("{\"prec\": \"%c\", \"n\": %d, \"K\": %d, \"frac\": %.2f, \"schedule\": \"%s\", \"us\": %.1f, \"gbs\": %.0f, \"finish_spread_us\": %.1f, "
               "\"mean_idle_us\": %.1f, \"items\": %lld, \"KB\": %d}\n",
               f32 ? 's' : 'd', n, K, mode >= 3 ? frac : 0.0, names[mode], ms * 1e3, bytes / (ms * 1e-3) / 1e9, sp, idle, total, KB);
    }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
