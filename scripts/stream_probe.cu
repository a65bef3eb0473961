// stream_probe.cu — DRAM access-pattern probe for the SYMV streaming kernel.
//
// Reads the lower triangle of an n x n double matrix (leading dimension ld)
// in the SYMV kernel's order — W = NW*CW-column tiles, each walked in H =
// 128*R-row chunks ("items"), stream-K over 148 CTAs of NW warps — with no
// arithmetic beyond one FMA per element, so the only variables are the
// access pattern (columns per item, contiguous bytes per column, ld) and
// whether every item ends in a CTA barrier.  Also a plain coalesced read of
// the same bytes (the read-stream ceiling).  Prints one JSON line per case.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe scripts/stream_probe.cu
//   ./stream_probe N [ld ...]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

struct Item { int col0, chunk0; long long prefix; };

__device__ __forceinline__ void ld256(double (&a)[4], const double *p, bool pred) {
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int pr = pred ? 1 : 0;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %9, 0;\n\t"
               "@q ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
               : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7])
               : "l"(p), "r"(pr));
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = __hiloint2double((int)w[2 * k + 1], (int)w[2 * k]);
}

template <int NW, int CW, int R, bool BAR>
__global__ void __launch_bounds__(NW * 32, NW >= 16 ? 1 : 2) tri_probe(const double *A, long long ld, int n, const Item *tiles,
                                                        int ntiles, long long total, int P, double *out) {
  constexpr int H = 128 * R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long it0 = (long long)blockIdx.x * total / P, end = (long long)(blockIdx.x + 1) * total / P;
  int k = 0;
  {
    int lo = 0, hi = ntiles;
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (tiles[mid].prefix <= it0) lo = mid; else hi = mid;
    }
    k = lo;
  }
  double acc = 0.0;
  double a[CW][R][4];
  Item t = tiles[k];
  long long tnext = k + 1 < ntiles ? tiles[k + 1].prefix : total;
  auto load = [&](const Item &tl, long long q) {
    const long long p0 = (long long)(tl.chunk0 + (q - tl.prefix)) * H;
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long row = p0 + r * 128 + lane * 4;
        ld256(a[j][r], A + (long long)(tl.col0 + warp * CW + j) * ld + row, row < n);
      }
  };
  if (it0 < end) load(t, it0);
  for (long long q = it0; q < end; ++q) {
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc = fma(a[j][r][v], 1.0000001, acc);
    if (q + 1 < end) {
      if (q + 1 >= tnext) {
        ++k;
        t = tiles[k];
        tnext = k + 1 < ntiles ? tiles[k + 1].prefix : total;
      }
      load(t, q + 1);
    }
    if (BAR) __syncthreads();
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Same loads, interleaved schedule: CTA c takes blocks of K consecutive
// items, block b of the CTA being global block b * P + c, so at any moment
// the CTAs stream neighbouring row chunks of the same tiles.
__device__ __forceinline__ int find_tile(const Item *tiles, int ntiles, long long it) {
  int lo = 0, hi = ntiles;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (tiles[mid].prefix <= it) lo = mid; else hi = mid;
  }
  return lo;
}

template <int NW, int CW, int R, bool BAR, int K>
__global__ void __launch_bounds__(NW * 32, 1) tri_probe_il(const double *A, long long ld, int n, const Item *tiles,
                                                           int ntiles, long long total, int P, double *out) {
  constexpr int H = 128 * R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  double a[CW][R][4];
  auto item_of = [&](long long j) { return ((j / K) * P + blockIdx.x) * K + (j % K); };
  auto load = [&](long long it) {
    const Item tl = tiles[find_tile(tiles, ntiles, it)];
    const long long p0 = (long long)(tl.chunk0 + (it - tl.prefix)) * H;
#pragma unroll
    for (int j = 0; j < CW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long row = p0 + r * 128 + lane * 4;
        ld256(a[j][r], A + (long long)(tl.col0 + warp * CW + j) * ld + row, row < n);
      }
  };
  long long j = 0;
  if (item_of(0) < total) load(item_of(0));
  for (; item_of(j) < total; ++j) {
#pragma unroll
    for (int jj = 0; jj < CW; ++jj)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc = fma(a[jj][r][v], 1.0000001, acc);
    if (item_of(j + 1) < total) load(item_of(j + 1));
    if (BAR) __syncthreads();
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// plain coalesced read of len doubles (32 B per lane per load, 4 in flight)
__global__ void __launch_bounds__(512) read_probe(const double *A, long long len, double *out) {
  double acc = 0.0;
  const long long step = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < len; i += 4 * step) {
    double a[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ld256(a[u], A + i + u * step, i + u * step + 3 < len);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc = fma(a[u][v], 1.0000001, acc);
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

template <int NW, int CW, int R, bool BAR, int K = 0>
void run_tri(const double *A, long long ld, int n, double *out, int sms, const char *label) {
  constexpr int W = NW * CW, H = 128 * R;
  int occ = 1;
  if (K == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tri_probe<NW, CW, R, BAR>, NW * 32, 0);
  auto launch = [&](const Item *dt, int nt, long long prefix, int P) {
    if constexpr (K == 0)
      tri_probe<NW, CW, R, BAR><<<P, NW * 32>>>(A, ld, n, dt, nt, prefix, P, out);
    else
      tri_probe_il<NW, CW, R, BAR, K><<<P, NW * 32>>>(A, ld, n, dt, nt, prefix, P, out);
  };
  const int P = sms * (occ < 1 ? 1 : occ);
  std::vector<Item> tiles;
  long long prefix = 0;
  for (int c0 = 0; c0 < n; c0 += W) {
    Item t{c0, c0 / H, prefix};
    prefix += (n - (long long)t.chunk0 * H + H - 1) / H;
    tiles.push_back(t);
  }
  Item *dt;
  CK(cudaMalloc(&dt, tiles.size() * sizeof(Item)));
  CK(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(Item), cudaMemcpyHostToDevice));
  long long bytes = 0;  // bytes actually requested (full chunks of the triangle's tiles)
  for (size_t k = 0; k < tiles.size(); ++k) {
    const long long rows = n - (long long)tiles[k].chunk0 * H;
    bytes += rows * W * 8;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) launch(dt, (int)tiles.size(), prefix, P);
  CK(cudaDeviceSynchronize());
  const int reps = 20;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch(dt, (int)tiles.size(), prefix, P);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"case\": \"%s\", \"K\": %d, \"NW\": %d, \"CW\": %d, \"R\": %d, \"bar\": %d, \"cols_per_item\": %d, "
         "\"seg_bytes\": %d, \"n\": %d, \"ld\": %lld, \"ctas\": %d, \"us\": %.1f, \"gbs\": %.0f}\n",
         label, K, NW, CW, R, (int)BAR, W, H * 8, n, ld, P, ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9);
  fflush(stdout);
  cudaFree(dt);
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32768;
  std::vector<long long> lds;
  for (int i = 2; i < argc; ++i) lds.push_back(atoll(argv[i]));
  if (lds.empty()) lds = {n, n + 64};
  long long maxld = 0;
  for (auto l : lds) maxld = l > maxld ? l : maxld;
  double *A, *out;
  CK(cudaMalloc(&A, (size_t)maxld * n * 8));
  CK(cudaMemset(A, 0, (size_t)maxld * n * 8));
  CK(cudaMalloc(&out, 148 * 1024 * 8 * 4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  {
    const long long len = (long long)n * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) read_probe<<<sms * 4, 512>>>(A, len, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) read_probe<<<sms * 4, 512>>>(A, len, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"case\": \"read\", \"bytes\": %lld, \"us\": %.1f, \"gbs\": %.0f}\n", len * 8, ms * 1e3 / 20,
           len * 8 / (ms * 1e-3 / 20) / 1e9);
  }
  for (long long ld : lds) {
    run_tri<16, 8, 1, true>(A, ld, n, out, sms, "symv-like 128col x 1KiB, barrier");
    run_tri<16, 8, 1, true, 1>(A, ld, n, out, sms, "interleaved K=1");
    run_tri<16, 8, 1, true, 2>(A, ld, n, out, sms, "interleaved K=2");
    run_tri<16, 8, 1, true, 4>(A, ld, n, out, sms, "interleaved K=4");
    run_tri<16, 8, 1, true, 8>(A, ld, n, out, sms, "interleaved K=8");
    run_tri<16, 8, 1, true, 16>(A, ld, n, out, sms, "interleaved K=16");
    run_tri<16, 8, 1, true, 64>(A, ld, n, out, sms, "interleaved K=64");
    run_tri<16, 2, 4, true>(A, ld, n, out, sms, "32col x 4KiB, barrier");
    run_tri<16, 2, 4, true, 1>(A, ld, n, out, sms, "32col x 4KiB interleaved K=1");
    run_tri<16, 4, 2, true, 2>(A, ld, n, out, sms, "64col x 2KiB interleaved K=2");
  }
  return 0;
}
