// kblas_device.cuh — element arithmetic, 256-bit streaming loads and the
// stream-K work split shared by every matrix-vector kernel.
//
// Element types: float (s), double (d), float2 (c), double2 (z).  Complex
// numbers are interleaved (re, im) pairs as in the reference
// (core.py:1-8); cuFloatComplex / cuDoubleComplex are the same layouts.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kb {

// ---------------------------------------------------------------------------
// element arithmetic
// ---------------------------------------------------------------------------
template <class T> struct Elem;
template <> struct Elem<float>   { using R = float;  static constexpr bool cplx = false; };
template <> struct Elem<double>  { using R = double; static constexpr bool cplx = false; };
template <> struct Elem<float2>  { using R = float;  static constexpr bool cplx = true; };
template <> struct Elem<double2> { using R = double; static constexpr bool cplx = true; };

template <class T> __host__ __device__ __forceinline__ T zero();
template <> __host__ __device__ __forceinline__ float zero<float>() { return 0.f; }
template <> __host__ __device__ __forceinline__ double zero<double>() { return 0.0; }
template <> __host__ __device__ __forceinline__ float2 zero<float2>() { return make_float2(0.f, 0.f); }
template <> __host__ __device__ __forceinline__ double2 zero<double2>() { return make_double2(0.0, 0.0); }

// c + a * b
__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float2 fma_(float2 a, float2 b, float2 c) {
  c.x = fmaf(a.x, b.x, c.x); c.x = fmaf(-a.y, b.y, c.x);
  c.y = fmaf(a.x, b.y, c.y); c.y = fmaf(a.y, b.x, c.y);
  return c;
}
__device__ __forceinline__ double2 fma_(double2 a, double2 b, double2 c) {
  c.x = fma(a.x, b.x, c.x); c.x = fma(-a.y, b.y, c.x);
  c.y = fma(a.x, b.y, c.y); c.y = fma(a.y, b.x, c.y);
  return c;
}
// c + conj(a) * b  (identical to fma_ for real types)
__device__ __forceinline__ float fmac_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmac_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float2 fmac_(float2 a, float2 b, float2 c) {
  c.x = fmaf(a.x, b.x, c.x); c.x = fmaf(a.y, b.y, c.x);
  c.y = fmaf(a.x, b.y, c.y); c.y = fmaf(-a.y, b.x, c.y);
  return c;
}
__device__ __forceinline__ double2 fmac_(double2 a, double2 b, double2 c) {
  c.x = fma(a.x, b.x, c.x); c.x = fma(a.y, b.y, c.x);
  c.y = fma(a.x, b.y, c.y); c.y = fma(-a.y, b.x, c.y);
  return c;
}
template <bool CONJ, class T> __device__ __forceinline__ T fmax_(T a, T b, T c) {
  if constexpr (CONJ) return fmac_(a, b, c); else return fma_(a, b, c);
}

__device__ __forceinline__ float add_(float a, float b) { return a + b; }
__device__ __forceinline__ double add_(double a, double b) { return a + b; }
__device__ __forceinline__ float2 add_(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 add_(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ float mul_(float a, float b) { return a * b; }
__device__ __forceinline__ double mul_(double a, double b) { return a * b; }
__device__ __forceinline__ float2 mul_(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 mul_(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// zero the imaginary part (Hermitian diagonal, kernels.py:353-354)
__device__ __forceinline__ float realify(float a) { return a; }
__device__ __forceinline__ double realify(double a) { return a; }
__device__ __forceinline__ float2 realify(float2 a) { a.y = 0.f; return a; }
__device__ __forceinline__ double2 realify(double2 a) { a.y = 0.0; return a; }

template <class T> __device__ __forceinline__ T sel(bool p, T a) { return p ? a : zero<T>(); }

__device__ __forceinline__ float shfl_xor_(float v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ double shfl_xor_(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ float2 shfl_xor_(float2 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m); v.y = __shfl_xor_sync(0xffffffffu, v.y, m); return v;
}
__device__ __forceinline__ double2 shfl_xor_(double2 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m); v.y = __shfl_xor_sync(0xffffffffu, v.y, m); return v;
}
template <class T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = add_(v, shfl_xor_(v, m));
  return v;
}

// ---------------------------------------------------------------------------
// streaming loads.  The matrix is read exactly once, so loads bypass L1
// allocation and are marked evict-first in L2 (the 126 MB L2 is kept for
// the vectors and the partial-sum workspace).  sm_100 has 256-bit global
// loads (SASS LDG.E.ENL2.256): one instruction moves 32 bytes per lane, a
// warp 1 KiB of a column.
// ---------------------------------------------------------------------------
// Partial-sum workspace stores: keep them in L2 (evict-last) so the
// epilogue reads them back from L2 rather than HBM.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep(float *p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(double *p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(float2 *p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_keep(double2 *p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// V consecutive elements starting at p, kept as raw 32-bit words so the
// load writes straight into the registers the FMAs read (a predicated-off
// load leaves the words zero).  V * sizeof(T) == 32 is one 256-bit load
// (p 32-byte aligned); V == 1 loads one element (natural alignment).
template <class T, int V> struct Pack {
  static constexpr int W = V * (int)sizeof(T) / 4;
  uint32_t w[W];
  __device__ __forceinline__ T v(int k) const {
    if constexpr (sizeof(T) == 4) {
      return __uint_as_float(w[k]);
    } else if constexpr (sizeof(T) == 16) {
      return T{__hiloint2double((int)w[4 * k + 1], (int)w[4 * k]), __hiloint2double((int)w[4 * k + 3], (int)w[4 * k + 2])};
    } else if constexpr (Elem<T>::cplx) {
      return T{__uint_as_float(w[2 * k]), __uint_as_float(w[2 * k + 1])};
    } else {
      return __hiloint2double((int)w[2 * k + 1], (int)w[2 * k]);
    }
  }
};

// %globaltimer in ns (instrumentation only)
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// L2 prefetch of the 32-byte segment at p (no register destination)
__device__ __forceinline__ void prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <class T, int V>
__device__ __forceinline__ void ld_pack(Pack<T, V> &a, const T *p, bool pred, uint64_t pol) {
  constexpr int W = Pack<T, V>::W;
#pragma unroll
  for (int k = 0; k < W; ++k) a.w[k] = 0u;
  const int pr = pred ? 1 : 0;
  if constexpr (W == 8) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %9, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]), "+r"(a.w[6]), "+r"(a.w[7])
        : "l"(p), "r"(pr));
  } else if constexpr (W == 4) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %6;\n\t}"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3])
        : "l"(p), "r"(pr), "l"(pol));
  } else if constexpr (W == 2) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %4;\n\t}"
        : "+r"(a.w[0]), "+r"(a.w[1]) : "l"(p), "r"(pr), "l"(pol));
  } else {
    static_assert(W == 1, "unsupported pack width");
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %3;\n\t}"
        : "+r"(a.w[0]) : "l"(p), "r"(pr), "l"(pol));
  }
}

// V consecutive elements of a vector operand (x): cached in L1 (every warp of
// a CTA reads the same rows) and kept in L2 (every CTA of a column range
// does).  One 256-bit load when V * sizeof(T) == 32 (p 32-byte aligned).
// x (and y_in) reads of a streaming kernel: ordinary coherent loads, never
// ld.global.nc.  A main kernel launched as the programmatic dependent of
// the host-vector copy-in grid may read x only after griddepcontrol.wait;
// ptxas treats .nc loads as reads of invariant memory and was seen hoisting
// them above the wait (SASS LDG.E.CONSTANT ahead of ACQBULK, stale x in
// tests/test_gpu_hostvec.py).  The loads are volatile asm, so nvvm keeps
// them after the wait's (volatile) asm; ptxas keeps coherent loads after
// ACQBULK.
__device__ __forceinline__ float ld_x(const float *p) {
  float v;
  asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_x(const double *p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_x(const float2 *p) {
  float2 v;
  asm volatile("ld.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_x(const double2 *p) {
  double2 v;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <class T, int V>
__device__ __forceinline__ void ld_xvec(T (&out)[V], const T *p) {
  if constexpr (V * sizeof(T) == 32) {
    Pack<T, V> a;
    asm volatile("ld.global.L2::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.w[0]), "=r"(a.w[1]), "=r"(a.w[2]), "=r"(a.w[3]), "=r"(a.w[4]), "=r"(a.w[5]),
                   "=r"(a.w[6]), "=r"(a.w[7])
                 : "l"(p));
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = a.v(v);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = ld_x(p + v);
  }
}

// ---------------------------------------------------------------------------
// shared-memory mbarriers (split arrive / wait)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// system-scope acquire/release flags (cross-process peer-memory handshake)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// bounded spin: a peer that never arrives turns into a kernel error
// (~30 s) instead of a hung GPU
__device__ __forceinline__ void spin_until(const unsigned long long *flag, unsigned long long seq) {
  for (unsigned long long it = 0; ld_acquire_sys(flag) < seq; ++it) {
    __nanosleep(256);
    if (it > (1ull << 27)) __trap();
  }
}

// ---------------------------------------------------------------------------
// stream-K split: `total` equal work items over P CTAs; CTA c owns
// [sk_start(c), sk_start(c+1)).  sk_owner(i) is the CTA owning item i.
// Partial sums that straddle CTAs are written to per-CTA workspace slots
// and summed in slot order by the epilogue kernel (deterministic).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ long long sk_start(long long c, long long total, long long P) {
  return c * total / P;
}
__host__ __device__ __forceinline__ int sk_owner(long long i, long long total, long long P) {
  return (int)(((i + 1) * P - 1) / total);
}

// 1D block-column-cyclic column map (multidevice.py:33-35, 72-93): local
// column p of GPU g is global column (g + (p / nb) * G) * nb + p % nb.
struct Xchg;  // peer-memory exchange of a one-process-per-GPU call (kblas_kernels.cuh)
struct ColMap {
  int G, g, nb;
  const Xchg *xg = nullptr;  // host side only: set for a p2p mgpu partial (SYMV/HEMV epilogue)
};
__host__ __device__ __forceinline__ long long map_col(const ColMap &cm, long long p) {
  if (cm.G == 1) return p;
  long long b = p / cm.nb;
  return (cm.g + b * cm.G) * cm.nb + (p - b * cm.nb);
}
// inverse: global column c -> local column, or -1 if not owned by cm.g
__host__ __device__ __forceinline__ long long unmap_col(const ColMap &cm, long long c) {
  if (cm.G == 1) return c;
  long long b = c / cm.nb;
  if (b % cm.G != cm.g) return -1;
  return (b / cm.G) * cm.nb + (c - b * cm.nb);
}

}  // namespace kb
