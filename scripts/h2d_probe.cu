// GPU-timeline cost of getting x to the device for a numpy-vector call
// (BASELINE configs[0], DGEMV-N 4096): kernel alone vs cudaMemcpyAsync H2D
// + kernel vs a copy kernel reading mapped pinned memory + kernel, queued
// (wall per call over many calls, GPU-bound) and synchronised per call.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/h2d_probe scripts/h2d_probe.cu \
//        -Lpaper_1410_1726_b200 -lkblas_b200 -Xlinker -rpath=$PWD/paper_1410_1726_b200
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include "../include/kblas_b200.h"

__global__ void copy_mapped(double *dst, const double *src, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

template <class F>
double wall_us(F f, int reps, bool sync, cudaStream_t st) {
  for (int i = 0; i < 50; ++i) { f(i); if (sync) cudaStreamSynchronize(st); }
  cudaStreamSynchronize(st);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) { f(i); if (sync) cudaStreamSynchronize(st); }
  cudaStreamSynchronize(st);
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  const int NC = 4;
  double *A[NC], *dx, *dy, *hx, *hy;
  for (int c = 0; c < NC; ++c) {
    cudaMalloc(&A[c], sizeof(double) * n * n);
    cudaMemset(A[c], 0, sizeof(double) * n * n);
  }
  cudaMalloc(&dx, sizeof(double) * n);
  cudaMalloc(&dy, sizeof(double) * n);
  cudaHostAlloc(&hx, sizeof(double) * n, cudaHostAllocDefault);
  cudaHostAlloc(&hy, sizeof(double) * n, cudaHostAllocDefault);
  for (int i = 0; i < n; ++i) hx[i] = 1.0;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const double one = 1.0, zero = 0.0;
  auto k = [&](int i, double *y) { kblas_dgemv_async('n', n, n, 1.0, A[i % NC], n, dx, 1, 0.0, y, 1, st); };
  auto v_kernel = [&](int i) { k(i, dy); };
  auto v_memcpy = [&](int i) {
    cudaMemcpyAsync(dx, hx, sizeof(double) * n, cudaMemcpyHostToDevice, st);
    k(i, dy);
  };
  auto v_copyk = [&](int i) {
    copy_mapped<<<8, 512, 0, st>>>(dx, hx, n);
    k(i, dy);
  };
  auto v_copyk_yhost = [&](int i) {
    copy_mapped<<<8, 512, 0, st>>>(dx, hx, n);
    k(i, hy);
  };
  auto v_memcpy_both = [&](int i) {
    cudaMemcpyAsync(dx, hx, sizeof(double) * n, cudaMemcpyHostToDevice, st);
    k(i, dy);
    cudaMemcpyAsync(hy, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, st);
  };
  auto v_hostvec = [&](int i) {
    kblas_mv_hostvec_async('d', 'g', 'n', 0, n, n, &one, A[i % NC], n, 0, 0, hx, &zero, nullptr, hy, st);
  };
  struct { const char *name; void (*dummy)(); } x{};
  (void)x;
  const int reps = 2000;
  printf("n=%d  (us per call: queued / synchronised per call)\n", n);
  printf("kernel only                         %7.2f  %7.2f\n", wall_us(v_kernel, reps, false, st), wall_us(v_kernel, reps, true, st));
  printf("memcpy H2D x + kernel               %7.2f  %7.2f\n", wall_us(v_memcpy, reps, false, st), wall_us(v_memcpy, reps, true, st));
  printf("copy kernel (mapped x) + kernel     %7.2f  %7.2f\n", wall_us(v_copyk, reps, false, st), wall_us(v_copyk, reps, true, st));
  printf("copy kernel + kernel (y mapped)     %7.2f  %7.2f\n", wall_us(v_copyk_yhost, reps, false, st), wall_us(v_copyk_yhost, reps, true, st));
  printf("memcpy H2D + kernel + memcpy D2H    %7.2f  %7.2f\n", wall_us(v_memcpy_both, reps, false, st), wall_us(v_memcpy_both, reps, true, st));
  printf("kblas_mv_hostvec_async              %7.2f  %7.2f\n", wall_us(v_hostvec, reps, false, st), wall_us(v_hostvec, reps, true, st));
  return 0;
}
