// CPU-side cost per call of the pieces of a numpy-vector call (timed over
// few enough calls that the launch queue never fills, so the GPU does not
// throttle the host loop).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/cpu_cost_probe scripts/cpu_cost_probe.cu \
//        -Lpaper_1410_1726_b200 -lkblas_b200 -Xlinker -rpath=$PWD/paper_1410_1726_b200
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include "../include/kblas_b200.h"

__global__ void empty_kernel() {}

template <class F>
double cpu_us(F f, cudaStream_t st, int n = 200) {
  for (int i = 0; i < 50; ++i) f();
  cudaStreamSynchronize(st);
  double best = 1e30;
  for (int rep = 0; rep < 20; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
  }
  return best;
}

int main() {
  const int n = 256;
  double *A, *dx, *dy, *hx, *hy;
  cudaMalloc(&A, sizeof(double) * n * n);
  cudaMemset(A, 0, sizeof(double) * n * n);
  cudaMalloc(&dx, sizeof(double) * n);
  cudaMalloc(&dy, sizeof(double) * n);
  cudaHostAlloc(&hx, sizeof(double) * n, cudaHostAllocDefault);
  cudaHostAlloc(&hy, sizeof(double) * n, cudaHostAllocDefault);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const double one = 1.0, zero = 0.0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  printf("CPU us per call (best of 20 x 200 calls)\n");
  printf("empty <<<>>>                      %6.2f\n", cpu_us([&] { empty_kernel<<<8, 256, 0, st>>>(); }, st));
  printf("empty cudaLaunchKernelEx PDL      %6.2f\n", cpu_us([&] {
           cudaLaunchConfig_t cfg = {};
           cfg.gridDim = dim3(8);
           cfg.blockDim = dim3(256);
           cfg.stream = st;
           cfg.attrs = at;
           cfg.numAttrs = 1;
           cudaLaunchKernelEx(&cfg, empty_kernel);
         }, st));
  printf("cudaPointerGetAttributes          %6.2f\n", cpu_us([&] {
           cudaPointerAttributes a{};
           cudaPointerGetAttributes(&a, hx);
         }, st));
  printf("cudaGetDevice                     %6.2f\n", cpu_us([&] { int d; cudaGetDevice(&d); }, st));
  printf("cudaMemcpyAsync H2D 2 KB pinned   %6.2f\n", cpu_us([&] {
           cudaMemcpyAsync(dx, hx, sizeof(double) * n, cudaMemcpyHostToDevice, st);
         }, st));
  printf("kblas_dgemv_async n               %6.2f\n", cpu_us([&] {
           kblas_dgemv_async('n', n, n, 1.0, A, n, dx, 1, 0.0, dy, 1, st);
         }, st));
  printf("kblas_dsymv_async l               %6.2f\n", cpu_us([&] {
           kblas_dsymv_async('l', n, 1.0, A, n, dx, 1, 0.0, dy, 1, st);
         }, st));
  printf("kblas_mv_hostvec_async gemv n     %6.2f\n", cpu_us([&] {
           kblas_mv_hostvec_async('d', 'g', 'n', 0, n, n, &one, A, n, 0, 0, hx, &zero, nullptr, hy, st);
         }, st));
  printf("kblas_mv_hostvec_async symv l     %6.2f\n", cpu_us([&] {
           kblas_mv_hostvec_async('d', 's', 'l', 0, n, n, &one, A, n, 0, 0, hx, &zero, nullptr, hy, st);
         }, st));
  printf("kblas_last_plan                   %6.2f\n", cpu_us([&] { (void)kblas_last_plan(); }, st));
  return 0;
}
