// Host-side cost per call of the C ABI (no Python): kblas_dsymv_async /
// kblas_dgemv_async on tiny operands (kernels negligible) vs an empty
// kernel launch and a PDL launch, so the library's own overhead can be
// separated from the driver's.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/host_overhead \
//        scripts/host_overhead.cu -Lpaper_1410_1726_b200 -lkblas_b200 \
//        -Xlinker -rpath=$PWD/paper_1410_1726_b200
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include "../include/kblas_b200.h"

__global__ void empty_kernel() {}

template <class F>
double per_call_us(F f, int n = 20000) {
  for (int i = 0; i < 200; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
  const int d = 256;
  double *A, *x, *y;
  cudaMalloc(&A, sizeof(double) * d * d);
  cudaMalloc(&x, sizeof(double) * d);
  cudaMalloc(&y, sizeof(double) * d);
  cudaMemset(A, 0, sizeof(double) * d * d);
  cudaMemset(x, 0, sizeof(double) * d);
  cudaStream_t st;
  cudaStreamCreate(&st);
  printf("empty kernel <<<>>>          %.2f us\n", per_call_us([&] { empty_kernel<<<148, 256, 0, st>>>(); }));
  printf("empty kernel x2 (PDL 2nd)    %.2f us\n", per_call_us([&] {
           empty_kernel<<<148, 256, 0, st>>>();
           cudaLaunchConfig_t cfg = {};
           cfg.gridDim = dim3(8);
           cfg.blockDim = dim3(512);
           cfg.stream = st;
           cudaLaunchAttribute at[1];
           at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
           at[0].val.programmaticStreamSerializationAllowed = 1;
           cfg.attrs = at;
           cfg.numAttrs = 1;
           cudaLaunchKernelEx(&cfg, empty_kernel);
         }));
  printf("kblas_dsymv_async d=%d      %.2f us\n", d, per_call_us([&] {
           kblas_dsymv_async('l', d, 1.0, A, d, x, 1, 0.0, y, 1, st);
         }));
  printf("kblas_dgemv_async n d=%d    %.2f us\n", d, per_call_us([&] {
           kblas_dgemv_async('n', d, d, 1.0, A, d, x, 1, 0.0, y, 1, st);
         }));
  printf("kblas_dgemv_async t d=%d    %.2f us\n", d, per_call_us([&] {
           kblas_dgemv_async('t', d, d, 1.0, A, d, x, 1, 0.0, y, 1, st);
         }));
  printf("kblas_last_plan              %.3f us\n", per_call_us([&] { (void)kblas_last_plan(); }));
  return 0;
}
