// kblas_impl.cuh — host-side planning and launch code shared by the
// translation units of the library (kblas_runtime.cu and one kblas_<p>.cu
// per precision, compiled in parallel).
//
// Planning per call: pick the load path (256-bit vectors when the column
// stride is 32-byte aligned, else one element per lane), realign the
// submatrix start down to the 32-byte granule (offset realignment,
// PAPER.md:826-863 / offset.py:66-71), size the stream-K grid to
// #SM x occupancy, and launch main kernel + fixed-order epilogue on the
// caller's stream.  Workspace for cross-CTA partials is cached per
// (device, stream) and grows only; tile tables for SYMV/HEMV are cached per
// shape.  No allocation happens on the steady-state path.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/kblas_b200.h"
#include "kblas_kernels.cuh"
#include "kblas_symv_tma.cuh"

using namespace kb;

namespace kbi {

inline std::atomic<unsigned long long> g_launches{0};

inline int g_symv_mid_max = 12288;  // register SYMV: 2-CTA/SM variant up to this order (s, d, c)
inline int g_symv_narrow_max = 2048;  // register SYMV: narrow tiles up to this order (kblas_set_symv_narrow)
inline thread_local std::string g_last_plan;

// ------------------------------------------------------------- timing hook
inline std::mutex g_tmu;
inline bool g_timing = false;
struct EvPair { cudaEvent_t a, b; int dev; };
inline std::vector<EvPair> g_events;

struct TimedScope {
  bool on = false;
  EvPair ev{};
  cudaStream_t s;
  explicit TimedScope(cudaStream_t st) : s(st) {
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing) return;
    cudaGetDevice(&ev.dev);
    if (cudaEventCreate(&ev.a) != cudaSuccess || cudaEventCreate(&ev.b) != cudaSuccess) return;
    on = true;
    cudaEventRecord(ev.a, s);
  }
  ~TimedScope() {
    if (!on) return;
    cudaEventRecord(ev.b, s);
    std::lock_guard<std::mutex> lk(g_tmu);
    g_events.push_back(ev);
  }
};

// ------------------------------------------------------ device properties
inline std::mutex g_mu;
inline std::map<int, int> g_sms;
inline std::map<const void *, int> g_occ;

inline int dev_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 1;
  g_sms[dev] = sms;
  return sms;
}

inline int occupancy(const void *fn, int threads, size_t smem = 0) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(fn);
    if (it != g_occ.end()) return it->second;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1)
    occ = 1;
  std::lock_guard<std::mutex> lk(g_mu);
  g_occ[fn] = occ;
  return occ;
}

// --------------------------------------------------------------- workspace
struct WsBuf { void *ptr = nullptr; size_t bytes = 0; };
inline std::map<std::pair<int, cudaStream_t>, WsBuf> g_ws;

inline cudaError_t workspace(size_t bytes, cudaStream_t st, void **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  WsBuf &b = g_ws[{dev, st}];
  if (b.bytes < bytes) {
    if (b.ptr) {
      cudaStreamSynchronize(st);
      cudaFree(b.ptr);
      b.ptr = nullptr;
      b.bytes = 0;
    }
    size_t want = bytes + bytes / 4 + 4096;
    cudaError_t e = cudaMalloc(&b.ptr, want);
    if (e != cudaSuccess) { b.ptr = nullptr; return e; }
    b.bytes = want;
  }
  *out = b.ptr;
  return cudaSuccess;
}

// One call's acquire-and-launch sequence (workspace, main kernel,
// epilogue) must not interleave with another host thread's on the same
// stream: the workspace is per (device, stream), so main1 main2 epi1 epi2
// would let call 2 overwrite call 1's partials.  Every entry point holds
// this (recursive: entries nest) lock of its (device, stream) for the
// whole sequence; calls on different streams never contend.
inline std::map<std::pair<int, cudaStream_t>, std::unique_ptr<std::recursive_mutex>> g_stream_mu;

inline std::recursive_mutex &stream_mutex(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local int c_dev = -1;
  thread_local cudaStream_t c_st = nullptr;
  thread_local std::recursive_mutex *c_mu = nullptr;
  if (c_mu && c_dev == dev && c_st == st) return *c_mu;
  std::lock_guard<std::mutex> lk(g_mu);
  auto &slot = g_stream_mu[{dev, st}];
  if (!slot) slot = std::make_unique<std::recursive_mutex>();
  c_dev = dev;
  c_st = st;
  c_mu = slot.get();
  return *c_mu;
}

struct StreamLock {
  std::unique_lock<std::recursive_mutex> lk;
  explicit StreamLock(cudaStream_t st) : lk(stream_mutex(st)) {}
};

// Arrival counters for the fused GEMV epilogue: one per row/column block,
// zero between calls (the finishing CTA resets its counter), zeroed when
// (re)allocated.  Cached per (device, stream) like the workspace.
inline std::map<std::pair<int, cudaStream_t>, WsBuf> g_cnt;
// mgpu root partial buffers (kblas_x*_mgpu), per (root device, stream)
inline std::map<std::pair<int, cudaStream_t>, WsBuf> g_rootbufs;

inline cudaError_t counters(size_t n, cudaStream_t st, unsigned **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  WsBuf &b = g_cnt[{dev, st}];
  const size_t bytes = std::max<size_t>(n, 1024) * sizeof(unsigned);
  if (b.bytes < bytes) {
    if (b.ptr) {
      cudaStreamSynchronize(st);
      cudaFree(b.ptr);
      b.ptr = nullptr;
      b.bytes = 0;
    }
    const size_t want = bytes * 2;
    cudaError_t e = cudaMalloc(&b.ptr, want);
    if (e != cudaSuccess) { b.ptr = nullptr; return e; }
    e = cudaMemsetAsync(b.ptr, 0, want, st);
    if (e != cudaSuccess) return e;
    b.bytes = want;
  }
  *out = static_cast<unsigned *>(b.ptr);
  return cudaSuccess;
}

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
constexpr long long kFuseMaxSlots = 8;
constexpr long long kFuseMaxSlotsT = 64;
inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// ------------------------------------------------------------ scalar utils
template <class T> bool is_zero(T v);
template <> inline bool is_zero(float v) { return v == 0.f; }
template <> inline bool is_zero(double v) { return v == 0.0; }
template <> inline bool is_zero(float2 v) { return v.x == 0.f && v.y == 0.f; }
template <> inline bool is_zero(double2 v) { return v.x == 0.0 && v.y == 0.0; }
template <class T> bool is_one(T v);
template <> inline bool is_one(float v) { return v == 1.f; }
template <> inline bool is_one(double v) { return v == 1.0; }
template <> inline bool is_one(float2 v) { return v.x == 1.f && v.y == 0.f; }
template <> inline bool is_one(double2 v) { return v.x == 1.0 && v.y == 0.0; }
template <class T> constexpr bool is_cplx() { return Elem<T>::cplx; }
inline double2 widen(float v) { return make_double2(v, 0.0); }
inline double2 widen(double v) { return make_double2(v, 0.0); }
inline double2 widen(float2 v) { return make_double2(v.x, v.y); }
inline double2 widen(double2 v) { return v; }

template <class T> const char *tname();
template <> inline const char *tname<float>() { return "s"; }
template <> inline const char *tname<double>() { return "d"; }
template <> inline const char *tname<float2>() { return "c"; }
template <> inline const char *tname<double2>() { return "z"; }

inline int launched(int n = 1) { g_launches += n; return 0; }

// Launch an epilogue with programmatic stream serialization: it may start
// while the preceding streaming kernel drains and waits in
// griddepcontrol.wait for that grid's completion (hides launch latency).
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// One-shot flag set by hostvec_entry right after it launches the copy-in
// grid that stages x (and y) from page-locked host memory: the next main
// kernel (or scal) of this thread's call is launched with programmatic
// stream serialization, so it starts streaming A while the copy-in grid
// still reads over PCIe; every main kernel executes griddepcontrol.wait
// before its first x / y access (a no-op for an ordinary launch).
inline thread_local bool t_pdl_next = false;
// Set by hostvec_entry while a call whose y was staged by the copy-in grid
// launches its kernels: its main kernel is launched the ordinary way even
// with chained launches (see hostvec_entry).
inline thread_local bool t_pdl_off = false;
// 1: the PDL-launched main kernel prefetches its first A segments into L2
// before griddepcontrol.wait; 2: it only waits.  $KBLAS_HOSTVEC_PREFETCH.
inline int hostvec_prefetch_mode() {
  static const int mode = [] {
    const char *e = std::getenv("KBLAS_HOSTVEC_PREFETCH");
    return (e != nullptr && e[0] == '0') ? 2 : 1;
  }();
  return mode;
}

// The hostvec copy-in grid launched as a programmatic dependent of the
// stream's previous kernel (1, default) or the ordinary way
// ($KBLAS_HOSTVEC_EARLY=0).
inline bool hostvec_early_copy() {
  static const bool on = [] {
    const char *e = std::getenv("KBLAS_HOSTVEC_EARLY");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// Every main kernel launched as a programmatic dependent of the stream's
// previous kernel (1, default; $KBLAS_PDL_CHAIN=0: only in host-vector
// calls).  Safe because every library kernel executes griddepcontrol.wait
// before it reads or writes anything an earlier kernel of the stream may
// still touch (the loads before it are A prefetches into L2 and the
// host-built tile tables), and before it completes, so the wait covers the
// whole stream; back-to-back calls then overlap a launch with the previous
// call's last kernel.
inline bool pdl_chain() {
  static const bool on = [] {
    const char *e = std::getenv("KBLAS_PDL_CHAIN");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

template <class... KArgs, class... Args>
cudaError_t launch_main(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                        Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (!t_pdl_off && (t_pdl_next || pdl_chain())) ? 1 : 0;
  t_pdl_next = false;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------- load path
// vec: 256-bit loads; needs lda*esize % 32 == 0.  The submatrix start is
// realigned down to its 32-byte granule and the lead rows are masked.
template <class T> struct Path { const T *base; int lead; bool vec; };

template <class T>
int make_path(const T *A, long long lda, Path<T> *out) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(A);
  if (addr % alignof(T) != 0) return -1;
  if ((lda * (long long)sizeof(T)) % 32 == 0) {
    const int lead = (int)((addr % 32) / sizeof(T));
    *out = Path<T>{A - lead, lead, true};
  } else {
    *out = Path<T>{A, 0, false};
  }
  return 0;
}

// ------------------------------------------------------------- configs
// (NW warps, CW columns per warp, R vectors per lane per column)
template <class T> struct Cfg {
  static constexpr int V = 32 / sizeof(T);
  // gemv N / T (register double-buffered: 2 x CW x R loads in flight per lane)
  static constexpr int G_NW = 8, G_CW = 4, G_R = 1, G_RS = V;
  // symv / hemv: W = S_NW * S_CW = 128 columns per tile (the t1 partial
  // traffic is 2/W of the triangle); z keeps the tile's x_col values in
  // shared memory (S_XS) to fit 8 columns per warp in 128 registers
  // (+4-6 % over 4 columns per warp, profiles/r1h_tune_symv_xs_variant108.jsonl)
  static constexpr int S_NW = 16, S_CW = 8, S_R = 1, S_RS = V;
  static constexpr bool S_XS = sizeof(T) == 16;

};

// ============================================================= knobs
// Split-form GEMV-N (kblas_gemv_ns_kernel) choice: -1 auto, 0 never, 1 always
// (kblas_set_gemv_split, for the tuner).
inline int g_gemv_split = -1;
inline int g_gemv_variant = 0;  // 0: tuned default shape (kblas_set_gemv_variant)
inline int g_split_waves = 1;   // split-form GEMV-N: CTAs per row block sized for this many waves
// cluster split form (kblas_gemv_nc_kernel): -1 auto, 0 never, 1 always
inline int g_gemv_cluster = -1;
// column-owning form (kblas_gemv_tc_kernel) choice: -1 auto, 0 never, 1 always
inline int g_gemv_tc = -1;
inline int g_symv_variant = -1;  // -1: per-precision default variant
inline int g_gemv_ro_cfg = -1;   // row-owning GEMV-N configuration (kblas_set_gemv_rowown; -1: from the table)

// The knobs one call runs with: the process-wide setters above (tuning
// hooks; a non-default value wins) over the empirical tuning table
// (kblas_tune_set, written by paper_1410_1726_b200/tuner.py) over the
// built-in rules.  Resolved once per call at dispatch, read by the run_*
// functions on the same thread.
struct Knobs {
  int gsplit = -1, gcluster = -1, gwaves = 1, gtc = -1, gvariant = 0, svariant = -1, rocfg = 0;
};
inline thread_local Knobs t_k;

// one row of the tuning table: calls of precision `prec` and operation
// `op` ('n', 't', 'c' GEMV; 'l', 'u' SYMV/HEMV) whose order key lies in
// [lo, hi] (GEMV: round(sqrt(m n)); SYMV: d) use these choices
struct TuneEntry {
  char prec, op;
  long long lo, hi;
  int shape, form, waves;
};
inline std::mutex g_tune_mu;            // writers (kblas_tune_*)
inline std::vector<TuneEntry> g_tune;     // guarded by g_tune_mu
inline std::atomic<int> g_tune_n{0};
// immutable copy the dispatcher reads without taking g_tune_mu
inline std::shared_ptr<const std::vector<TuneEntry>> g_tune_snap;
// call with g_tune_mu held after changing g_tune
inline void publish_tune() {
  std::atomic_store(&g_tune_snap, std::make_shared<const std::vector<TuneEntry>>(g_tune));
  g_tune_n.store((int)g_tune.size(), std::memory_order_release);
}

void tune_builtin_once();  // kblas_runtime.cu

template <class T>
Knobs resolve_knobs(char op, long long key) {
  tune_builtin_once();
  Knobs k;
  k.gsplit = g_gemv_split;
  k.gcluster = g_gemv_cluster;
  k.gwaves = g_split_waves;
  k.gtc = g_gemv_tc;
  k.gvariant = g_gemv_variant;
  k.svariant = g_symv_variant;
  k.rocfg = g_gemv_ro_cfg < 0 ? 0 : g_gemv_ro_cfg;
  if (key < 0 || g_tune_n.load(std::memory_order_acquire) == 0) return k;
  if (op == 'c' && !is_cplx<T>()) op = 't';
  const auto snap = std::atomic_load(&g_tune_snap);
  if (!snap) return k;
  for (auto it = snap->rbegin(); it != snap->rend(); ++it) {  // latest entry wins
    const TuneEntry &e = *it;
    if (e.prec != tname<T>()[0] || e.op != op || key < e.lo || key > e.hi) continue;
    if (op == 'l' || op == 'u') {
      if (k.svariant == -1 && e.shape >= 100) k.svariant = e.shape;
    } else {
      if (e.form == 3) {  // row-owning: shape 10 + configuration
        if (k.gsplit == -1 && k.gcluster == -1) {
          k.gsplit = 3;
          if (g_gemv_ro_cfg < 0) k.rocfg = e.shape - 10;
        }
        break;
      }
      if (k.gvariant == 0 && e.shape > 0) k.gvariant = e.shape;
      if (op == 'n') {
        if (k.gsplit == -1 && k.gcluster == -1 && e.form >= 0) {
          // 2 = preferred by the table: taken when the grid still covers
          // the GPU (the shape guards below), unlike an explicit setter
          k.gsplit = e.form >= 1 ? 2 : 0;
          k.gcluster = e.form == 2 ? 2 : (e.form == 1 ? 0 : -1);
        }
        if (k.gwaves == 1 && e.waves > 0) k.gwaves = e.waves;
      } else if (k.gtc == -1 && e.form >= 0) {
        k.gtc = e.form ? 2 : 0;
      }
    }
    break;
  }
  return k;
}

// ============================================================= GEMV-N
constexpr long long kSplitMaxSlots = 64;

template <class T, int V, int NW, int CW>
cudaError_t run_gemv_ns(const Path<T> &pa, long long lda, int m, int n, const T *x, ColMap cm, T *y, T alpha,
                        T beta, bool beta_zero, cudaStream_t st, long long S, long long nrb) {
  constexpr int RB = 32 * V;
  auto kfn = kblas_gemv_ns_kernel<T, V, NW, CW>;
  void *ws = nullptr;
  cudaError_t e = workspace(align256((size_t)S * m * sizeof(T)), st, &ws);
  if (e != cudaSuccess) return e;
  unsigned *cnt = nullptr;
  if (S > 1 && (e = counters((size_t)nrb, st, &cnt)) != cudaSuccess) return e;
  GemvParams p{pa.base, lda, m, n, pa.lead, x, ws, (long long)m, nrb * S, (int)(nrb * S), (int)S, cm,
               y, cnt, widen(alpha), widen(beta), beta_zero ? 1 : 0, (long long)m};
  {
    TimedScope ts(st);
    e = launch_main(kfn, (unsigned)(nrb * S), NW * 32, 0, st, p);
  }
  if (e != cudaSuccess) return e;
  launched(1);
  char buf[256];
  snprintf(buf, sizeof buf, "gemv_ns %s %s lead=%d m=%d n=%d RB=%d P=%lld slots=%lld", tname<T>(),
           V > 1 ? "v256" : "scalar", pa.lead, m, n, RB, nrb * S, S);
  g_last_plan = buf;
  return cudaGetLastError();
}

template <class T, int V, int NW, int CW>
cudaError_t run_gemv_nc(const Path<T> &pa, long long lda, int m, int n, const T *x, ColMap cm, T *y, T alpha,
                        T beta, bool beta_zero, cudaStream_t st, int S, long long nrb) {
  constexpr int RB = 32 * V;
  auto kfn = kblas_gemv_nc_kernel<T, V, NW, CW>;
  {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
      attr_err = cudaFuncSetAttribute((const void *)kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    if (attr_err != cudaSuccess) return attr_err;
  }
  GemvParams p{pa.base, lda, m, n, pa.lead, x, nullptr, 0, nrb * S, (int)(nrb * S), S, cm,
               y, nullptr, widen(alpha), widen(beta), beta_zero ? 1 : 0, (long long)m};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nrb * S));
  cfg.blockDim = dim3(NW * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (!t_pdl_off && (t_pdl_next || pdl_chain())) ? 2 : 1;
  t_pdl_next = false;
  cudaError_t e;
  {
    TimedScope ts(st);
    e = cudaLaunchKernelEx(&cfg, kfn, p);
  }
  if (e != cudaSuccess) return e;
  launched(1);
  char buf[256];
  snprintf(buf, sizeof buf, "gemv_nc %s %s lead=%d m=%d n=%d RB=%d cluster=%d P=%lld slots=1", tname<T>(),
           V > 1 ? "v256" : "scalar", pa.lead, m, n, RB, S, nrb * S);
  g_last_plan = buf;
  return cudaGetLastError();
}

template <class T, int V, int NW, int LR, int U>
bool run_gemv_ro(const Path<T> &pa, long long lda, int m, int n, const T *x, ColMap cm, T *y, T alpha, T beta,
                 bool beta_zero, cudaStream_t st, cudaError_t *err) {
  constexpr int RBo = LR * V;
  const long long P = cdiv((long long)pa.lead + m, RBo);
  // every CTA streams all n columns of its rows: needs enough row blocks to
  // cover the GPU, else the caller falls back to the other forms
  if (2 * P < dev_sms()) return false;
  // ... and a last, partial wave must not run nearly alone: every CTA
  // streams a whole row block across all n columns, so a wave holding a
  // few CTAs costs as much as a full one (measured: one CTA past the SM
  // count x CTAs per SM drops the form 10-40 % below stream-K,
  // profiles/r2s_audit_rowown.log; three waves at 87 % stay ahead)
  {
    const long long slots =
        (long long)dev_sms() * occupancy((const void *)kblas_gemv_ro_kernel<T, V, NW, LR, U>, NW * 32);
    if (slots > 0 && P > slots && (double)P / (double)(cdiv(P, slots) * slots) < 0.75) return false;
  }
  GemvParams p{pa.base, lda, m, n, pa.lead, x, nullptr, 0, 0, (int)P, 0, cm,
               y, nullptr, widen(alpha), widen(beta), beta_zero ? 1 : 0, (long long)m};
  // the row-owning kernel executes griddepcontrol.wait only when p.pdl != 0
  // (its prologue is laid out for the ordinary launch): a chained launch
  // must set it
  p.pdl = t_pdl_next ? hostvec_prefetch_mode() : (pdl_chain() && !t_pdl_off ? 2 : 0);
  {
    TimedScope ts(st);
    *err = launch_main(kblas_gemv_ro_kernel<T, V, NW, LR, U>, (unsigned)P, NW * 32, 0, st, p);
  }
  if (*err != cudaSuccess) return true;
  launched(1);
  char buf[256];
  snprintf(buf, sizeof buf, "gemv_ro %s %s lead=%d m=%d n=%d RB=%d NW=%d LR=%d U=%d P=%lld slots=1", tname<T>(),
           V > 1 ? "v256" : "scalar", pa.lead, m, n, RBo, NW, LR, U, P);
  g_last_plan = buf;
  *err = cudaGetLastError();
  return true;
}

// row-owning configurations (warps, row lanes per column, columns in
// flight per lane); table shape 10 + index.  Measured at N = 1k-12k
// (profiles/r1z_tune_gemv_ro*.jsonl): the best one keeps ~128-256 CTAs.
template <class T, int V>
bool dispatch_gemv_ro(int cfg, const Path<T> &pa, long long lda, int m, int n, const T *x, ColMap cm, T *y,
                      T alpha, T beta, bool beta_zero, cudaStream_t st, cudaError_t *err) {
#define KB_RO(NW, LR, U) return run_gemv_ro<T, V, NW, LR, U>(pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st, err)
  switch (cfg) {
    case 1: KB_RO(8, 4, 8);
    case 2: KB_RO(8, 2, 8);
    case 3: KB_RO(8, 4, 16);
    case 4: KB_RO(8, 2, 16);
    case 5: KB_RO(4, 4, 16);
    case 6: KB_RO(16, 2, 8);
    case 7: KB_RO(8, 8, 8);
    default: KB_RO(16, 4, 8);
  }
#undef KB_RO
}

template <class T, int V, int NW, int CW, int R, int MINB = 2>
cudaError_t run_gemv_n(const Path<T> &pa, long long lda, int m, int n, const T *x, ColMap cm, T *y,
                       T alpha, T beta, bool beta_zero, cudaStream_t st) {
  constexpr int RB = NW * 32 * V * R;
  auto kfn = kblas_gemv_n_kernel<T, V, NW, CW, R, MINB>;
  const long long nrb = cdiv((long long)pa.lead + m, RB);
  const long long KS = cdiv(n, CW);
  const long long total = nrb * KS;
  const long long P = std::min<long long>(total, (long long)dev_sms() * occupancy((const void *)kfn, NW * 32));
  const long long per = std::max<long long>(1, total / P);
  const long long maxslots = std::min<long long>(P, cdiv(KS, per) + 1);
  // fused epilogue (the last CTA of a row block reduces it) when few CTAs
  // share a row block; otherwise a separate, parallel epilogue kernel
  const bool fused = maxslots <= kFuseMaxSlots;
  if (t_k.gsplit == 3) {
    cudaError_t err = cudaSuccess;
    if (V > 1 && dispatch_gemv_ro<T, V>(t_k.rocfg, pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st, &err))
      return err;
    t_k.gsplit = -1;  // too few rows (or unaligned ld): the built-in rule picks among the other forms
  }
  {
    // small / short matrices: the split form keeps the row blocks narrow so
    // few CTAs share one, and reduces them in the same kernel
    constexpr int NWs = 8, CWs = 4, RBs = 32 * V;
    const long long nrb_s = cdiv((long long)pa.lead + m, RBs);
    const long long Ps = (long long)dev_sms() * occupancy((const void *)kblas_gemv_ns_kernel<T, V, NWs, CWs>, NWs * 32);
    const long long S = std::max<long long>(1, std::min<long long>({cdiv((long long)t_k.gwaves * Ps, nrb_s),
                                                                     kSplitMaxSlots,
                                                                     std::max<long long>(1, n / (NWs * CWs))}));
    const bool fills = nrb_s * S >= dev_sms();
    const bool small = (long long)m * n * (long long)sizeof(T) <= (80LL << 20);
    // large operands: when at most 2 CTAs share a row block (little or no
    // partial traffic) and the grid fills >= 85 % of its waves, the split
    // form beats stream-K (profiles/r1q_tune_gemv_nforms.jsonl: Z N=32768
    // 6.8 -> 7.3 TB/s, D/C +2-3 %)
    const long long Pg = nrb_s * S;
    const double eff = (double)Pg / (double)(cdiv(Pg, Ps) * Ps);
    const bool large_ok = S <= 2 && eff >= 0.85 && fills;
    const bool half_fills = 2 * nrb_s * S >= dev_sms();  // small calls are latency-bound anyway
    if (t_k.gsplit == 1 || (t_k.gsplit == 2 && half_fills) ||
        (t_k.gsplit == -1 && ((!fused && half_fills && small) || large_ok))) {
      // the CTAs of a row block as one cluster, reduced through DSMEM
      // (cluster sizes 2..16; 16 is the opt-in non-portable maximum)
      int Sc = 1;
      while (Sc < 16 && Sc < S) Sc *= 2;
      const bool cl_ok = S > 1 && n / Sc >= NWs * CWs && 4 * nrb_s * Sc >= dev_sms();
      if (t_k.gcluster == 1 || (t_k.gcluster == 2 && cl_ok) || (t_k.gcluster == -1 && cl_ok && small))
        return run_gemv_nc<T, V, NWs, CWs>(pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st, Sc, nrb_s);
      return run_gemv_ns<T, V, NWs, CWs>(pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st, S, nrb_s);
    }
  }
  void *ws = nullptr;
  cudaError_t e = workspace(align256((size_t)maxslots * m * sizeof(T)), st, &ws);
  if (e != cudaSuccess) return e;
  unsigned *cnt = nullptr;
  if (fused && (e = counters((size_t)nrb, st, &cnt)) != cudaSuccess) return e;
  GemvParams p{pa.base, lda, m, n, pa.lead, x, ws, (long long)m, total, (int)P, (int)KS, cm,
               y, cnt, widen(alpha), widen(beta), beta_zero ? 1 : 0, (long long)m};
  {
    TimedScope ts(st);
    e = launch_main(kfn, (unsigned)P, NW * 32, 0, st, p);
  }
  if (e != cudaSuccess) return e;
  launched(1);
  if (!fused) {
    launch_pdl(kblas_gemv_n_epilogue<T, 8>, (unsigned)cdiv(m, 32), 256, st, y, (const T *)ws, (long long)m, m, pa.lead,
               (int)RB, (int)KS, total, (int)P, alpha, beta, (int)beta_zero);
    launched(1);
  }
  char buf[256];
  snprintf(buf, sizeof buf, "gemv_n %s %s lead=%d m=%d n=%d RB=%d KS=%lld items=%lld P=%lld slots=%lld",
           tname<T>(), V > 1 ? "v256" : "scalar", pa.lead, m, n, RB, KS, total, P, maxslots);
  g_last_plan = buf;
  return cudaGetLastError();
}

// ============================================================= GEMV-T/C
inline long long g_gemv_tc_max_bytes = 80LL << 20;

template <class T, int V, int NW, int CB, bool CONJ>
cudaError_t run_gemv_tc(const Path<T> &pa, long long lda, int m, int n, long long nglob, const T *x, ColMap cm,
                        T *y, T alpha, T beta, bool beta_zero, cudaStream_t st) {
  auto kfn = kblas_gemv_tc_kernel<T, V, NW, CB, CONJ>;
  cudaError_t e = cudaSuccess;
  if (cm.G > 1) {
    // mgpu partial: columns this GPU does not own stay zero
    e = cudaMemsetAsync(y, 0, (size_t)nglob * sizeof(T), st);
    if (e != cudaSuccess) return e;
  }
  const long long P = cdiv(n, CB);
  GemvParams p{pa.base, lda, m, n, pa.lead, x, nullptr, 0, 0, (int)P, 0, cm,
               y, nullptr, widen(alpha), widen(beta), beta_zero ? 1 : 0, nglob};
  {
    TimedScope ts(st);
    e = launch_main(kfn, (unsigned)P, NW * 32, 0, st, p);
  }
  if (e != cudaSuccess) return e;
  launched(1);
  char buf[256];
  snprintf(buf, sizeof buf, "gemv_tc %s %s%s lead=%d m=%d n=%d H=%d CB=%d P=%lld slots=1", tname<T>(),
           V > 1 ? "v256" : "scalar", CONJ ? " conj" : "", pa.lead, m, n, 32 * V, CB, P);
  g_last_plan = buf;
  return cudaGetLastError();
}

template <class T, int V, int NW, int CW, int R, bool CONJ, int MINB = 2>
cudaError_t run_gemv_t(const Path<T> &pa, long long lda, int m, int n, long long nglob, const T *x,
                       ColMap cm, T *y, T alpha, T beta, bool beta_zero, cudaStream_t st) {
  {
    // whole columns per CTA, one kernel with no cross-CTA reduction
    // (profiles/r1p_tune_gemv_tc.jsonl): wins for every operand up to
    // 80 MB, and at every size for d and z, as long as the grid is not cut
    // badly by the wave count; s and c stay on stream-K above 80 MB
    constexpr int CBc = 4;
    const long long Pc = cdiv(n, CBc);
    const long long slots = (long long)dev_sms() * 2;
    const double eff = (double)Pc / (double)(cdiv(Pc, slots) * slots);
    const bool enough = Pc >= dev_sms() / 2;
    const bool small = (long long)m * n * (long long)sizeof(T) <= g_gemv_tc_max_bytes;
    const bool any_size = (sizeof(T) == 16 || (sizeof(T) == 8 && !is_cplx<T>())) && eff >= 0.8;
    if (t_k.gtc == 1 || (enough && (t_k.gtc == 2 || (t_k.gtc == -1 && (small || any_size)))))
      return run_gemv_tc<T, V, 8, CBc, CONJ>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);
  }
  constexpr int H = 32 * V * R, CBW = NW * CW;
  auto kfn = kblas_gemv_t_kernel<T, V, NW, CW, R, CONJ, MINB>;
  const long long ncb = cdiv(n, CBW);
  const long long KS = cdiv((long long)pa.lead + m, H);
  const long long total = ncb * KS;
  const long long P = std::min<long long>(total, (long long)dev_sms() * occupancy((const void *)kfn, NW * 32));
  const long long per = std::max<long long>(1, total / P);
  const long long maxslots = std::min<long long>(P, cdiv(KS, per) + 1);
  void *ws = nullptr;
  cudaError_t e = workspace(align256((size_t)maxslots * ncb * CBW * sizeof(T)), st, &ws);
  if (e != cudaSuccess) return e;
  // the last CTA of a column block sums CBW columns x maxslots slots with the
  // whole CTA, so the fused form pays off up to many slots
  const bool fused = maxslots <= kFuseMaxSlotsT;
  unsigned *cnt = nullptr;
  if (fused && (e = counters((size_t)ncb, st, &cnt)) != cudaSuccess) return e;
  const long long ws_ld = ncb * CBW;
  if (fused && cm.G > 1) {
    // mgpu partial: columns this GPU does not own stay zero
    if ((e = cudaMemsetAsync(y, 0, (size_t)nglob * sizeof(T), st)) != cudaSuccess) return e;
  }
  GemvParams p{pa.base, lda, m, n, pa.lead, x, ws, ws_ld, total, (int)P, (int)KS, cm,
               y, cnt, widen(alpha), widen(beta), beta_zero ? 1 : 0, nglob};
  {
    TimedScope ts(st);
    e = launch_main(kfn, (unsigned)P, NW * 32, 0, st, p);
  }
  if (e != cudaSuccess) return e;
  launched(1);
  if (!fused) {
    launch_pdl(kblas_gemv_t_epilogue<T, 8>, (unsigned)cdiv(nglob, 32), 256, st, y, (const T *)ws, ws_ld, nglob, (int)CBW,
               (int)KS, total, (int)P, cm, alpha, beta, (int)beta_zero);
    launched(1);
  }
  char buf[256];
  snprintf(buf, sizeof buf, "gemv_t %s %s%s lead=%d m=%d n=%d H=%d KS=%lld items=%lld P=%lld slots=%lld",
           tname<T>(), V > 1 ? "v256" : "scalar", CONJ ? " conj" : "", pa.lead, m, n, H, KS, total, P,
           maxslots);
  g_last_plan = buf;
  return cudaGetLastError();
}

// ============================================================= SYMV/HEMV
struct TileTable {
  SymTile *dev = nullptr;
  int *seg_tile = nullptr;  // per segment: tile of its first item
  int ntiles = 0;
  long long total = 0;
  int P = 1;                // CTAs the schedule was cut for (min(P, total))
  int K = 1, rounds = 0;
  long long base = 0, rem = 0, nseg = 0;
  long long nslots = 0;     // ws2 slot rows (sum over tiles of the segments touching them)
  // split schedule (tail_items > 0): the tail [base, total) is cut into
  // Ptail segments of ~tail_items items for the tail grid; dev_tail is the
  // tile array with seg0 counted from the first tail segment (rounds * P)
  int Ptail = 1;
  SymTile *dev_tail = nullptr;
};
inline std::map<std::vector<long long>, TileTable> g_tiles;

// SYMV segment length K (items dealt round robin per CTA, see SymParams);
// <= 0: contiguous stream-K.  kblas_set_symv_segment.
inline int g_symv_seg = 6;
// kblas_set_symv_segment not called: the wide kernel's split schedule uses
// K = 12 where that still leaves the split its minimum rounds (+0.4-1 % at
// 32k-65k, profiles/r2t_seg_scan_split.jsonl).  $KBLAS_SYMV_SEG_AUTO=0: K = 6.
inline bool g_symv_seg_auto = true;
inline bool symv_seg_auto() {
  static const bool env = [] {
    const char *e = std::getenv("KBLAS_SYMV_SEG_AUTO");
    return !(e != nullptr && e[0] == '0');
  }();
  return env && g_symv_seg_auto;
}
// instrumentation (kblas_set_symv_trace): the register SYMV kernel writes
// each CTA's start / end %globaltimer and SM id here (3 per CTA); nullptr = off
inline unsigned long long *g_symv_trace = nullptr;
// register SYMV/HEMV (wide kernel): items per CTA barrier window, 1, 2 or
// 4 (kblas_set_symv_window)
inline int g_symv_window = 2;
// split schedule of the wide kernel (see kblas_symv_kernel): the last
// symv_tail_pct() % of the items run as a tail grid of symv_tail_items()-item
// CTAs.  $KBLAS_SYMV_TAIL_PCT / $KBLAS_SYMV_TAIL_ITEMS override them
// (share 0: one grid).
inline int symv_tail_pct() {
  static const int pct = [] {
    const char *e = std::getenv("KBLAS_SYMV_TAIL_PCT");
    return e != nullptr ? std::max(0, std::atoi(e)) : 6;
  }();
  return pct;
}
inline int symv_tail_items() {
  static const int items = [] {
    const char *e = std::getenv("KBLAS_SYMV_TAIL_ITEMS");
    return e != nullptr ? std::max(1, std::atoi(e)) : 4;
  }();
  return items;
}
// fewest interleaved rounds that leave a split worth it (below: one grid)
constexpr int kSymvSplitMinRounds = 8;

// Tiles for the local panel of GPU g under the block-cyclic layout (G=1,
// nb=d for a single GPU): every owned block column is cut into W-wide tiles.
// exact: chunks start at each tile's first stored row (TMA path); else on
// the physical H-row grid (vector-load path, 32-byte granules).  The item
// schedule (segments of K items round robin over P CTAs, then a
// contiguous tail) and each tile's ws2 slot rows are fixed here too.
inline cudaError_t tile_table(int d, int lead, bool lower, int W, int H, ColMap cm, int ncols_local, long long P,
                              int K, TileTable *out, bool exact = false, int tail_pct = 0, int tail_items = 0) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<long long> key{dev, d, lead, lower, W, H, cm.G, cm.g, cm.nb, ncols_local, P, K, exact,
                             tail_pct, tail_items};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_tiles.find(key);
    if (it != g_tiles.end()) { *out = it->second; return cudaSuccess; }
  }
  std::vector<SymTile> tiles;
  long long prefix = 0;
  for (long long l0 = 0; l0 < ncols_local; ) {
    // local block containing l0 and its global extent
    const long long b = l0 / cm.nb;
    const long long J = cm.g + b * cm.G;
    const long long gblk0 = J * cm.nb;
    const long long gblk1 = std::min<long long>(d, gblk0 + cm.nb);
    const long long lblk1 = b * cm.nb + (gblk1 - gblk0);
    for (long long s = l0; s < lblk1; s += W) {
      SymTile t{};
      t.lcol0 = (int)s;
      t.gcol0 = (int)(gblk0 + (s - b * cm.nb));
      t.ncols = (int)std::min<long long>(W, lblk1 - s);
      t.row0 = lower ? t.gcol0 : 0;
      t.row1 = lower ? d : std::min(d, t.gcol0 + t.ncols);
      const long long c0 = exact ? 0 : ((long long)t.row0 + lead) / H;
      const long long c1 = exact ? cdiv((long long)t.row1 - t.row0, H) : cdiv((long long)t.row1 + lead, H);
      t.chunk0 = (int)c0;
      t.prefix = prefix;
      prefix += c1 - c0;
      tiles.push_back(t);
    }
    l0 = (b + 1) * cm.nb;
  }
  if (prefix >= (1LL << 31) - 1) return cudaErrorInvalidValue;  // item indices are 32-bit in the kernels
  TileTable tt;
  tt.ntiles = (int)tiles.size();
  tt.total = prefix;
  const long long Pe = std::min<long long>(P, std::max<long long>(prefix, 1));
  tt.P = (int)Pe;
  tt.K = K > 0 ? K : 1;
  // the tail keeps >= 1 item per CTA, so no segment is empty and every
  // slot row a tile owns is written
  const bool split = K > 0 && tail_items > 0 && tail_pct > 0;
  const long long tail_min = split ? std::max<long long>(Pe, prefix * tail_pct / 100) : Pe;
  tt.rounds = K > 0 ? (int)(std::max<long long>(0, prefix - tail_min) / (Pe * K)) : 0;
  tt.base = (long long)tt.rounds * Pe * tt.K;
  tt.rem = prefix - tt.base;
  tt.Ptail = split ? (int)std::min<long long>(tt.rem, cdiv(tt.rem, tail_items)) : (int)Pe;
  tt.nseg = (long long)tt.rounds * Pe + tt.Ptail;
  const long long full = (long long)tt.rounds * Pe;
  auto seg_of = [&](long long q) {
    return q < tt.base ? q / tt.K : full + sk_owner(q - tt.base, tt.rem, tt.Ptail);
  };
  auto seg_lo = [&](long long sg) {
    return sg < full ? sg * tt.K : tt.base + (sg - full) * tt.rem / tt.Ptail;
  };
  long long slots = 0;
  for (size_t k = 0; k < tiles.size(); ++k) {
    const long long a = tiles[k].prefix;
    const long long bnext = (k + 1 < tiles.size()) ? tiles[k + 1].prefix : prefix;
    tiles[k].seg0 = (int)seg_of(a);
    tiles[k].nseg = bnext > a ? (int)(seg_of(bnext - 1) - tiles[k].seg0 + 1) : 0;
    tiles[k].slot0 = (int)slots;
    slots += tiles[k].nseg;
  }
  tt.nslots = std::max<long long>(slots, 1);
  if (!tiles.empty()) {
    // per segment: the tile holding its first item (empty tail segments: 0)
    std::vector<int> segt((size_t)tt.nseg, 0);
    size_t k = 0;
    for (long long sg = 0; sg < tt.nseg; ++sg) {
      const long long it = seg_lo(sg);
      if (it >= prefix) continue;
      while (k + 1 < tiles.size() && tiles[k + 1].prefix <= it) ++k;
      if (tiles[k].prefix > it) k = 0;
      segt[(size_t)sg] = (int)k;
    }
    const size_t tb = align256(tiles.size() * sizeof(SymTile));
    void *mem = nullptr;
    cudaError_t e = cudaMalloc(&mem, tb * (split ? 2 : 1) + segt.size() * sizeof(int));
    if (e != cudaSuccess) return e;
    tt.dev = static_cast<SymTile *>(mem);
    tt.seg_tile = reinterpret_cast<int *>(static_cast<char *>(mem) + tb * (split ? 2 : 1));
    e = cudaMemcpy(tt.dev, tiles.data(), tiles.size() * sizeof(SymTile), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(tt.seg_tile, segt.data(), segt.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    if (split) {
      // the tail grid numbers its segments from 0: same tiles, seg0 rebased
      std::vector<SymTile> tail = tiles;
      for (auto &t : tail) t.seg0 -= (int)full;
      tt.dev_tail = reinterpret_cast<SymTile *>(static_cast<char *>(mem) + tb);
      e = cudaMemcpy(tt.dev_tail, tail.data(), tail.size() * sizeof(SymTile), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return e;
    }
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_tiles[key] = tt;
  *out = tt;
  return cudaSuccess;
}

// kernel parameters of a tile table (ws1 rows of d, ws2 slot rows of W)
template <class T>
SymParams sym_params(const T *A, long long lda, int d, int lead, const T *x, void *ws, int W, const TileTable &tt,
                     bool uniform) {
  const size_t b1 = align256((size_t)tt.ntiles * d * sizeof(T));
  SymParams p{};
  p.A = A;
  p.lda = lda;
  p.d = d;
  p.lead = lead;
  p.x = x;
  p.ws1 = ws;
  p.ws1_ld = d;
  p.ws2 = static_cast<char *>(ws) + b1;
  p.ws2_ld = W;
  p.tiles = tt.dev;
  p.ntiles = tt.ntiles;
  p.total = tt.total;
  p.P = tt.P;
  p.tile_w = uniform ? W : 0;
  p.K = tt.K;
  p.rounds = tt.rounds;
  p.base = tt.base;
  p.rem = tt.rem;
  p.nseg = tt.nseg;
  p.seg_tile = tt.seg_tile;
#if KBLAS_SYMV_TRACE
  p.trace = g_symv_trace;
#endif
  return p;
}
template <class T>
size_t sym_ws_bytes(int d, int W, const TileTable &tt) {
  return align256((size_t)tt.ntiles * d * sizeof(T)) + align256((size_t)tt.nslots * W * sizeof(T));
}

// SYMV/HEMV epilogue: 128 rows per CTA (contiguous t1 reads, same sums in
// the same order) when the tiles are 128-column blocks aligned to 128,
// else 32 rows per CTA.  $KBLAS_SYMV_EPILOGUE=32 forces the latter (A/B).
inline bool symv_epilogue_r128_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("KBLAS_SYMV_EPILOGUE");
    return !(e != nullptr && e[0] == '3');
  }();
  return on;
}

template <class T, bool LOWER>
void launch_symv_epilogue(T *y, const SymParams &p, T alpha, T beta, bool beta_zero, const ColMap &cm, int W,
                          cudaStream_t st) {
  const kb::Xchg xg = cm.xg ? *cm.xg : kb::Xchg{};
  const bool aligned = W == 128 && (p.tile_w == 128 || (p.tile_w == 0 && cm.nb % 128 == 0));
  if (aligned && symv_epilogue_r128_enabled())
    launch_pdl(kblas_symv_epilogue_r128<T, LOWER, 16>, (unsigned)cdiv(p.d, 128), 512, st, y, p, alpha, beta,
               (int)beta_zero, xg);
  else
    launch_pdl(kblas_symv_epilogue<T, LOWER, 16>, (unsigned)cdiv(p.d, 32), 512, st, y, p, alpha, beta,
               (int)beta_zero, xg);
}

template <class T, int V, int NW, int CW, int R, bool LOWER, bool HERM, int MINB = 1, bool XS = false, int B = 1>
cudaError_t run_symv(const Path<T> &pa, long long lda, int d, const T *x, ColMap cm, int ncols_local, T *y,
                     T alpha, T beta, bool beta_zero, cudaStream_t st) {
  constexpr int H = 32 * V * R, W = NW * CW;
  constexpr size_t smem = 2 * (size_t)B * NW * H * sizeof(T);
  auto kfn = kblas_symv_kernel<T, V, NW, CW, R, LOWER, HERM, MINB, XS, B>;
  {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
      attr_err = cudaFuncSetAttribute((const void *)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return attr_err;
  }
  const long long Pmax = (long long)dev_sms() * occupancy((const void *)kfn, NW * 32, smem);
  TileTable tt;
  // wide 1-CTA/SM kernel: split schedule when there are enough rounds
  const int tail_pct = (MINB == 1 && W == 128 && g_symv_seg > 0) ? symv_tail_pct() : 0;
  cudaError_t e = cudaSuccess;
  bool have = false;
  if (tail_pct > 0 && symv_seg_auto() && g_symv_seg == 6) {
    // longer segments when they keep enough rounds for the split
    e = tile_table(d, pa.lead, LOWER, W, H, cm, ncols_local, Pmax, 12, &tt, false, tail_pct, symv_tail_items());
    if (e != cudaSuccess) return e;
    have = tt.dev_tail != nullptr && tt.rounds >= kSymvSplitMinRounds;
  }
  if (!have) {
    e = tile_table(d, pa.lead, LOWER, W, H, cm, ncols_local, Pmax, g_symv_seg, &tt, false, tail_pct,
                   tail_pct > 0 ? symv_tail_items() : 0);
    if (e != cudaSuccess) return e;
  }
  if (tt.dev_tail != nullptr && tt.rounds < kSymvSplitMinRounds) {
    e = tile_table(d, pa.lead, LOWER, W, H, cm, ncols_local, Pmax, g_symv_seg, &tt);
    if (e != cudaSuccess) return e;
  }
  if (tt.ntiles == 0 || tt.total == 0) {  // idle GPU: partial is zero
    kblas_scal_kernel<T><<<(unsigned)cdiv(d, 256), 256, 0, st>>>(y, d, zero<T>(), 1);
    launched();
    return cudaGetLastError();
  }
  const long long P = tt.P;
  void *ws = nullptr;
  e = workspace(sym_ws_bytes<T>(d, W, tt), st, &ws);
  if (e != cudaSuccess) return e;
  SymParams p = sym_params(pa.base, lda, d, pa.lead, x, ws, W, tt, cm.G == 1 && cm.nb >= d);
  const bool hostvec = t_pdl_next;
  p.pdl = hostvec ? hostvec_prefetch_mode() : 0;
  const bool split = tt.dev_tail != nullptr;
  SymParams pt = p;  // tail grid
  if (split) {
    unsigned *cnt = nullptr;  // slot 1023 of the stream's counters: the tail grid's (left at 0)
    if ((e = counters(1024, st, &cnt)) != cudaSuccess) return e;
    cnt += 1023;
    p.nseg = (long long)tt.rounds * P;  // the first grid stops at the tail
    pt.tiles = tt.dev_tail;
    pt.seg_tile = tt.seg_tile + p.nseg;
    pt.P = tt.Ptail;
    pt.rounds = 0;
    pt.nseg = tt.Ptail;
    pt.tail_ctr = cnt;
    // no wait in the tail grid, host-vector calls included: it launches
    // only after every CTA of the first grid has passed its own wait on the
    // copy-in grid (the first grid releases its dependents after that
    // wait), so a staged x is complete before the tail grid starts
    pt.pdl = 0;
  }
  {
    // one timing bracket over both grids of a split call (the streaming
    // time the roofline divides by)
    TimedScope ts(st);
    e = launch_main(kfn, (unsigned)P, NW * 32, smem, st, p);
    if (e == cudaSuccess && split) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)tt.Ptail);
      cfg.blockDim = dim3(NW * 32);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e = cudaLaunchKernelEx(&cfg, kfn, pt);
      if (e == cudaSuccess) launched(1);
    }
  }
  if (e != cudaSuccess) return e;
  launch_symv_epilogue<T, LOWER>(y, p, alpha, beta, beta_zero, cm, W, st);
  launched(2);
  char buf[256];
  snprintf(buf, sizeof buf, "symv %s %s %s%s lead=%d d=%d W=%d H=%d B=%d tiles=%d items=%lld P=%lld K=%d rounds=%d slots=%lld tail=%d",
           tname<T>(), V > 1 ? "v256" : "scalar", LOWER ? "L" : "U", HERM ? " herm" : "", pa.lead, d, W, H, B,
           tt.ntiles, tt.total, P, tt.K, tt.rounds, tt.nslots, split ? tt.Ptail : 0);
  g_last_plan = buf;
  return cudaGetLastError();
}

// ---------------------------------------------------------- SYMV via TMA
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// SYMV/HEMV kernel choice: -1 auto (per-precision default from the
// empirical tuning in profiles/r1_tune_symv_*.jsonl), 0 register-load
// kernel, 1 TMA kernel.  KBLAS_NO_TMA=1 forces 0 at load.
inline int g_use_tma = -2;
inline int tma_mode() {
  if (g_use_tma == -2) {
    const char *e = getenv("KBLAS_NO_TMA");
    g_use_tma = (e && e[0] == '1') ? 0 : -1;
  }
  return g_use_tma;
}
inline bool use_tma() { return tma_mode() != 0; }
// tuned defaults (profiles/r1_tune_symv_v3.jsonl): the software-pipelined
// register kernel wins for every precision and size except SSYMV at
// N <= 8192, where the TMA kernel (variant 1: 16 consumers x 8 columns,
// 256 B boxes, 5 stages) is ahead
template <class T> bool prefer_tma(int) { return false; }
template <class T> int default_variant() { return sizeof(T) == 16 ? 0 : 1; }

// A00: element (0,0) of the d x d operand (any row alignment); needs a
// 16-byte multiple column stride.
template <class T>
bool tma_ok(const T *A00, long long lda, int d) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(A00);
  const int mode = tma_mode();
  const bool want = mode == 1 || (mode == -1 && prefer_tma<T>(d));
  return want && tensor_map_encoder() != nullptr && (lda * (long long)sizeof(T)) % 16 == 0 &&
         addr % sizeof(T) == 0;
}

template <class T, int NC, int CW, int RS, int S, bool LOWER, bool HERM>
cudaError_t run_symv_tma(const T *A00, long long lda, int d, const T *x, ColMap cm, int ncols_local, T *y,
                         T alpha, T beta, bool beta_zero, cudaStream_t st) {
  constexpr int HS = Stage<T, RS>::HS, W = NC * CW;
  constexpr size_t smem = symv_tma_smem<T, NC, CW, RS, S>();
  static_assert(smem <= 227 * 1024, "shared memory budget");
  auto kfn = kblas_symv_tma_kernel<T, NC, CW, RS, S, LOWER, HERM>;
  {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
      attr_err = cudaFuncSetAttribute((const void *)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return attr_err;
  }
  const uintptr_t addr = reinterpret_cast<uintptr_t>(A00);
  const int lead = (int)((addr % 16) / sizeof(T));
  const T *base = A00 - lead;
  const int unit = sizeof(T) == 16 ? 8 : (int)sizeof(T);
  const int upe = (int)sizeof(T) / unit;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)(lead + d) * upe, (cuuint64_t)std::max(ncols_local, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(T)};
  cuuint32_t box[2] = {(cuuint32_t)(HS * upe), (cuuint32_t)W};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = tensor_map_encoder()(&map, unit == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                                     2, (void *)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  const long long Pmax = dev_sms();
  TileTable tt;
  cudaError_t e = tile_table(d, lead, LOWER, W, HS, cm, ncols_local, Pmax, g_symv_seg, &tt);
  if (e != cudaSuccess) return e;
  if (tt.ntiles == 0 || tt.total == 0) {
    kblas_scal_kernel<T><<<(unsigned)cdiv(d, 256), 256, 0, st>>>(y, d, zero<T>(), 1);
    launched();
    return cudaGetLastError();
  }
  const long long P = tt.P;
  void *ws = nullptr;
  e = workspace(sym_ws_bytes<T>(d, W, tt), st, &ws);
  if (e != cudaSuccess) return e;
  SymTmaParams tp;
  tp.sp = sym_params(base, lda, d, lead, x, ws, W, tt, cm.G == 1 && cm.nb >= d);
  tp.unit_per_elem = upe;
  {
    TimedScope ts(st);
    e = launch_main(kfn, (unsigned)P, (NC + 2) * 32, smem, st, map, tp);
  }
  if (e != cudaSuccess) return e;
  launch_symv_epilogue<T, LOWER>(y, tp.sp, alpha, beta, beta_zero, cm, W, st);
  launched(2);
  char buf[256];
  snprintf(buf, sizeof buf, "symv_tma %s %s%s lead=%d d=%d W=%d H=%d S=%d tiles=%d items=%lld P=%lld K=%d rounds=%d slots=%lld smem=%zu",
           tname<T>(), LOWER ? "L" : "U", HERM ? " herm" : "", lead, d, W, HS, S, tt.ntiles, tt.total, P,
           tt.K, tt.rounds, tt.nslots, (size_t)smem);
  g_last_plan = buf;
  return cudaGetLastError();
}

// ------------------------------------------------------------ dispatch
template <class T>
cudaError_t dispatch_gemv(char trans, const Path<T> &pa, long long lda, int m, int n, long long nglob,
                          const T *x, ColMap cm, T *y, T alpha, T beta, bool beta_zero, cudaStream_t st) {
  using C = Cfg<T>;
  // single-GPU calls look up the tuning table by order; mgpu partials (and
  // any call under an explicit setter) keep the process-wide knobs
  t_k = resolve_knobs<T>(trans, cm.G == 1 ? std::llround(std::sqrt((double)m * (double)n)) : -1);
  // tuned per-precision shapes (profiles/r1j_tune_gemv_*.jsonl): S uses 16
  // warps at 1 CTA/SM (variant 4), Z GEMV-N 4 warps x 4 columns x 2 vectors
  // per lane (variant 3); D, C and Z-T/C keep the 8 x 4 x 1 default (5)
  int gv = t_k.gvariant;
  if (gv == 0) gv = sizeof(T) == 4 ? 4 : (sizeof(T) == 16 && trans == 'n') ? 3 : 5;
  if (pa.vec && (gv == 3 || gv == 4)) {
    // tuning variants (kblas_set_gemv_variant): (warps, columns per warp,
    // vectors per lane per column, CTAs per SM)
#define KB_GV(NW, CW, R, MB)                                                                                  \
  if (trans == 'n') return run_gemv_n<T, C::V, NW, CW, R, MB>(pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st); \
  if (trans == 'c' && is_cplx<T>())                                                                          \
    return run_gemv_t<T, C::V, NW, CW, R, true, MB>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);   \
  return run_gemv_t<T, C::V, NW, CW, R, false, MB>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);
    // (variants 1 = 4x4x1 at 4 CTAs/SM and 2 = 8x2x2 were measured and
    // dropped: profiles/r1j_tune_gemv_*.jsonl)
    switch (gv) {
      case 3: KB_GV(4, 4, 2, 2)
      default: KB_GV(16, 4, 1, 1)
    }
#undef KB_GV
  }
  if (trans == 'n') {
    if (pa.vec) return run_gemv_n<T, C::V, C::G_NW, C::G_CW, C::G_R>(pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st);
    return run_gemv_n<T, 1, C::G_NW, C::G_CW, C::G_RS>(pa, lda, m, n, x, cm, y, alpha, beta, beta_zero, st);
  }
  if (trans == 'c' && is_cplx<T>()) {
    if (pa.vec) return run_gemv_t<T, C::V, C::G_NW, C::G_CW, C::G_R, true>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);
    return run_gemv_t<T, 1, C::G_NW, C::G_CW, C::G_RS, true>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);
  }
  if (pa.vec) return run_gemv_t<T, C::V, C::G_NW, C::G_CW, C::G_R, false>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);
  return run_gemv_t<T, 1, C::G_NW, C::G_CW, C::G_RS, false>(pa, lda, m, n, nglob, x, cm, y, alpha, beta, beta_zero, st);
}

template <class T, bool HERM>
cudaError_t dispatch_symv_h(bool lower, const Path<T> &pa, long long lda, int d, const T *x, ColMap cm,
                            int ncols_local, T *y, T alpha, T beta, bool beta_zero, cudaStream_t st) {
  using C = Cfg<T>;
  t_k = resolve_knobs<T>(lower ? 'l' : 'u', cm.G == 1 ? d : -1);
  const T *A00 = pa.base + pa.lead;
  if (tma_ok(A00, lda, d)) {
#define KB_TMA(NC, CW, RS, S)                                                                                 \
  return lower ? run_symv_tma<T, NC, CW, RS, S, true, HERM>(A00, lda, d, x, cm, ncols_local, y, alpha, beta,  \
                                                             beta_zero, st)                                  \
               : run_symv_tma<T, NC, CW, RS, S, false, HERM>(A00, lda, d, x, cm, ncols_local, y, alpha, beta, \
                                                              beta_zero, st)
    // tuning variants (kblas_set_symv_variant); 0 is the default
    // (consumer warps, columns per warp, rows per lane, stages)
    if constexpr (sizeof(T) == 16) {
      switch (t_k.svariant < 0 ? default_variant<T>() : t_k.svariant) {
        case 1: KB_TMA(8, 8, 2, 3);
        default: KB_TMA(16, 4, 1, 5);
      }
    } else {
      switch (t_k.svariant < 0 ? default_variant<T>() : t_k.svariant) {
        case 1: KB_TMA(16, 8, 1, 5);
        default: KB_TMA(16, 8, 2, 3);
      }
    }
#undef KB_TMA
  }
#define KB_REG(V, NW, CW, R)                                                                                  \
  return lower ? run_symv<T, V, NW, CW, R, true, HERM>(pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, \
                                                       st)                                                     \
               : run_symv<T, V, NW, CW, R, false, HERM>(pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st)
  if (!pa.vec)  // odd ld: one element per lane
    return lower ? run_symv<T, 1, C::S_NW, C::S_CW, C::S_RS, true, HERM, 1, C::S_XS>(
                       pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st)
                 : run_symv<T, 1, C::S_NW, C::S_CW, C::S_RS, false, HERM, 1, C::S_XS>(
                       pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st);
  // register-kernel tuning variants (kblas_set_symv_variant 100+); small
  // operands use narrow tiles (variant 103, W = 32 columns, 16 for z) so
  // there are enough items to occupy every SM
  int v = t_k.svariant;
  if (v < 100 && d <= g_symv_narrow_max) v = 103;
  // mid orders (s, d, c): 8 warps x 8 columns at 2 CTAs/SM ramps up faster
  // than one 16-warp CTA per SM (+2-10 % at d = 4096-12288,
  // profiles/r1v_tune_symv_mid.jsonl); z keeps the wide default
  else if (v < 100 && sizeof(T) <= 8 && d <= g_symv_mid_max) v = 105;
  // (variants 101/102/104/108 and the column-rolling / split-barrier
  // kernels were measured and dropped: profiles/r1h_tune_symv_*.jsonl)
  switch (v) {
    case 103: KB_REG(C::V, 8, 4, 1);                           // 8 warps x 4 columns (small operands)
    case 105:                                                  // 8 warps x 8 columns, 2 CTAs per SM
      return lower ? run_symv<T, C::V, 8, (sizeof(T) == 16 ? 4 : 8), 1, true, HERM, 2>(
                         pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st)
                   : run_symv<T, C::V, 8, (sizeof(T) == 16 ? 4 : 8), 1, false, HERM, 2>(
                         pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st);
    default:
#define KB_WIDE(B)                                                                                      \
  return lower ? run_symv<T, C::V, C::S_NW, C::S_CW, C::S_R, true, HERM, 1, C::S_XS, B>(                \
                     pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st)                     \
               : run_symv<T, C::V, C::S_NW, C::S_CW, C::S_R, false, HERM, 1, C::S_XS, B>(               \
                     pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st)
      switch (g_symv_window) {
        case 1: KB_WIDE(1);
        case 2: KB_WIDE(2);
        default: KB_WIDE(4);
      }
#undef KB_WIDE
  }
#undef KB_REG
}

template <class T>
cudaError_t dispatch_symv(bool lower, bool herm, const Path<T> &pa, long long lda, int d, const T *x, ColMap cm,
                          int ncols_local, T *y, T alpha, T beta, bool beta_zero, cudaStream_t st) {
  if constexpr (is_cplx<T>()) {
    if (herm) return dispatch_symv_h<T, true>(lower, pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st);
  }
  return dispatch_symv_h<T, false>(lower, pa, lda, d, x, cm, ncols_local, y, alpha, beta, beta_zero, st);
}

inline int code(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

template <class T>
int scal_only(T *y, long long len, T beta, cudaStream_t st) {
  const cudaError_t e = launch_main(kblas_scal_kernel<T>, (unsigned)cdiv(len, 256), 256, 0, st, y, len, beta,
                                    is_zero(beta) ? 1 : 0);
  if (e != cudaSuccess) return code(e);
  launched();
  g_last_plan = std::string("scal ") + tname<T>();
  return code(cudaGetLastError());
}

// ------------------------------------------------ BLAS-level entry points
template <class T>
int gemv_entry(char trans, int m, int n, T alpha, const T *dA, int lda, const T *dx, int incx, T beta, T *dy,
               int incy, int offset_r, int offset_c, cudaStream_t st) {
  char t = (char)(trans | 0x20);
  if (t != 'n' && t != 't' && t != 'c') return -1;
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (offset_r < 0 || offset_c < 0) return -12;
  if ((long long)lda < std::max(1LL, (long long)offset_r + m)) return -6;
  if (incx != 1) return -8;
  if (incy != 1) return -11;
  if (t == 'c' && !is_cplx<T>()) t = 't';  // kernels.py:422-423
  const long long ylen = (t == 'n') ? m : n;
  if (m == 0 || n == 0) {
    if (ylen == 0 || is_one(beta)) return 0;
    return scal_only(dy, ylen, beta, st);
  }
  if (is_zero(alpha) && is_one(beta)) return 0;  // quick return (kernels.py:427-428)
  StreamLock slk(st);
  if (is_zero(alpha)) return scal_only(dy, ylen, beta, st);  // kernels.py:431-432
  const T *A = dA + (long long)offset_c * lda + offset_r;
  Path<T> pa;
  if (make_path(A, lda, &pa) != 0) return -5;
  ColMap cm{1, 0, 1 << 30};
  return code(dispatch_gemv<T>(t, pa, lda, m, n, n, dx, cm, dy, alpha, beta, is_zero(beta), st));
}

template <class T>
int symv_entry(char uplo, bool herm, int n, T alpha, const T *dA, int lda, const T *dx, int incx, T beta, T *dy,
               int incy, int offset, cudaStream_t st) {
  const char u = (char)(uplo | 0x20);
  if (u != 'l' && u != 'u') return -1;
  if (n < 0) return -2;
  if (offset < 0) return -11;
  if ((long long)lda < std::max(1LL, (long long)offset + n)) return -5;
  if (incx != 1) return -7;
  if (incy != 1) return -10;
  if (n == 0) return 0;
  if (is_zero(alpha) && is_one(beta)) return 0;
  StreamLock slk(st);
  if (is_zero(alpha)) return scal_only(dy, n, beta, st);
  const T *A = dA + (long long)offset * lda + offset;
  Path<T> pa;
  if (make_path(A, lda, &pa) != 0) return -4;
  ColMap cm{1, 0, 1 << 30};
  return code(dispatch_symv<T>(u == 'l', herm, pa, lda, n, dx, cm, n, dy, alpha, beta, is_zero(beta), st));
}

// ------------------------------------------------------------------ mgpu
inline long long local_cols(long long n, long long nb, long long G, long long g) {
  long long total = 0;
  const long long nblk = cdiv(n, nb);
  for (long long j = g; j < nblk; j += G) total += std::min(n, (j + 1) * nb) - j * nb;
  return total;
}

struct DevGuard {
  int prev = 0;
  DevGuard() { cudaGetDevice(&prev); }
  ~DevGuard() { cudaSetDevice(prev); }
};

// partial of one GPU: y_part = alpha * (local contribution), beta ignored
template <class T>
int partial_entry(bool is_gemv, char op, bool herm, int m, int n, T alpha, const T *dA, int lda, const T *dx,
                  T *dpart, int G, int g, int nb, cudaStream_t st) {
  const long long lc = local_cols(n, nb, G, g);
  const long long plen = is_gemv ? ((op == 'n') ? m : n) : n;
  StreamLock slk(st);
  if (lc == 0 || is_zero(alpha)) return scal_only(dpart, plen, zero<T>(), st);
  Path<T> pa;
  if (make_path(dA, lda, &pa) != 0) return -5;
  ColMap cm{G, g, nb};
  if (is_gemv) {
    char t = op;
    if (t == 'c' && !is_cplx<T>()) t = 't';
    return code(dispatch_gemv<T>(t, pa, lda, m, (int)lc, n, dx, cm, dpart, alpha, zero<T>(), true, st));
  }
  return code(dispatch_symv<T>(op == 'l', herm, pa, lda, n, dx, cm, (int)lc, dpart, alpha, zero<T>(), true, st));
}

// streams: one per GPU (the _async entry points) or
// null for each device's legacy default stream plus a final wait
template <class T>
int mgpu_entry(bool is_gemv, char op, bool herm, int m, int n, T alpha, T *const *dA, int lda, T *const *dx,
               T beta, T *const *dy, int ngpus, int nb, const int *device_ids, cudaStream_t const *streams = nullptr) {
  if (ngpus < 1 || ngpus > kMaxGpus) return -13;
  if (nb < 1) return -14;
  DevGuard guard;
  auto devof = [&](int g) { return device_ids ? device_ids[g] : g; };
  auto stof = [&](int g) { return streams ? streams[g] : (cudaStream_t)0; };
  const bool sync = streams == nullptr;
  const long long ylen = is_gemv ? ((op == 'n') ? m : n) : n;
  const int root = devof(0);
  const cudaStream_t rst = stof(0);
  cudaError_t e;
  if (ylen == 0) return 0;
  if (is_zero(alpha) && is_one(beta)) return 0;
  if (is_zero(alpha) || (is_gemv && (m == 0 || n == 0))) {
    cudaSetDevice(root);
    int rc = scal_only(dy[0], ylen, beta, rst);
    if (rc) return rc;
    return sync ? code(cudaStreamSynchronize(rst)) : 0;
  }
  // root's own partial lives in a workspace slot (dy[0] holds the input y)
  cudaSetDevice(root);
  StreamLock rlk(rst);
  void *rootbuf = nullptr;
  // separate from the kernel workspace: allocated once per (device, root stream)
  {
    std::lock_guard<std::mutex> lk(g_mu);
    WsBuf &b = g_rootbufs[{root, rst}];
    const size_t need = (size_t)ylen * sizeof(T) * (ngpus + 1);
    if (b.bytes < need) {
      if (b.ptr) { cudaDeviceSynchronize(); cudaFree(b.ptr); }
      b.ptr = nullptr; b.bytes = 0;
      if ((e = cudaMalloc(&b.ptr, need)) != cudaSuccess) return code(e);
      b.bytes = need;
    }
    rootbuf = b.ptr;
  }
  T *root_part = static_cast<T *>(rootbuf);
  std::vector<cudaEvent_t> done(ngpus, nullptr);
  for (int g = 0; g < ngpus; ++g) {
    const int dev = devof(g);
    if ((e = cudaSetDevice(dev)) != cudaSuccess) return code(e);
    T *out = (g == 0) ? root_part : dy[g];
    int rc = partial_entry<T>(is_gemv, op, herm, m, n, alpha, dA[g], lda, dx[g], out, ngpus, g, nb, stof(g));
    if (rc) return rc;
    cudaEventCreateWithFlags(&done[g], cudaEventDisableTiming);
    cudaEventRecord(done[g], stof(g));
  }
  cudaSetDevice(root);
  PartList<T> parts{};
  for (int g = 0; g < ngpus; ++g) {
    const int dev = devof(g);
    cudaStreamWaitEvent(rst, done[g], 0);
    if (g == 0 || dev == root) {
      parts.p[g] = (g == 0) ? root_part : dy[g];
      continue;
    }
    int can = 0;
    cudaDeviceCanAccessPeer(&can, root, dev);
    if (can) {
      cudaError_t pe = cudaDeviceEnablePeerAccess(dev, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (pe != cudaSuccess) { cudaGetLastError(); can = 0; }
    }
    if (can) {
      parts.p[g] = dy[g];  // NVLink peer load inside the combine kernel
    } else {
      T *slot = root_part + (size_t)ylen * g;
      if ((e = cudaMemcpyPeerAsync(slot, root, dy[g], dev, ylen * sizeof(T), rst)) != cudaSuccess) return code(e);
      parts.p[g] = slot;
    }
  }
  kblas_mgpu_combine_kernel<T><<<(unsigned)cdiv(ylen, 256), 256, 0, rst>>>(dy[0], parts, ngpus, ylen, beta,
                                                                     is_zero(beta) ? 1 : 0);
  launched();
  e = cudaGetLastError();
  if (e == cudaSuccess && !sync) {
    // the next call's partial on GPU g (g > 0) overwrites dy[g]: make each
    // GPU's stream wait until this combine has read it (no WAR race when a
    // caller reuses dy across _async calls)
    cudaEvent_t combined = nullptr;
    e = cudaEventCreateWithFlags(&combined, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(combined, rst);
    for (int g = 1; g < ngpus && e == cudaSuccess; ++g) {
      if (stof(g) == rst) continue;
      cudaSetDevice(devof(g));
      e = cudaStreamWaitEvent(stof(g), combined, 0);
    }
    if (combined) cudaEventDestroy(combined);
  }
  if (e == cudaSuccess && sync) e = cudaStreamSynchronize(rst);
  for (auto ev : done) if (ev) cudaEventDestroy(ev);  // released once complete
  return code(e);
}

// y = beta * y + sum_g parts[g] in device order on the current device
// (parts on this device or peer-accessible): the root combine of the
// single-process mgpu API after an NCCL reduce (multidevice.py:276,
// 282-283)
template <class T>
int combine_entry(long long n, int nparts, const void *const *parts, T beta, T *y, cudaStream_t st) {
  if (n < 0 || nparts < 1 || nparts > kMaxGpus || parts == nullptr || y == nullptr) return -1;
  if (n == 0) return 0;
  PartList<T> pl{};
  for (int g = 0; g < nparts; ++g) {
    if (parts[g] == nullptr) return -3;
    pl.p[g] = static_cast<const T *>(parts[g]);
  }
  kblas_mgpu_combine_kernel<T><<<(unsigned)cdiv(n, 256), 256, 0, st>>>(y, pl, nparts, n, beta, is_zero(beta) ? 1 : 0);
  launched();
  return code(cudaGetLastError());
}

// per-GPU panels of the 1D block-column-cyclic layout
inline int malloc_mgpu(int m, int n, size_t esize, void **dA, int *ldda, int ngpus, int nb, const int *device_ids) {
  if (m < 0 || n < 0 || esize == 0 || dA == nullptr || ngpus < 1 || nb < 1) return -1;
  DevGuard guard;
  const long long ld = cdiv(std::max(m, 1), 32) * 32;
  if (ldda) *ldda = (int)ld;
  for (int g = 0; g < ngpus; ++g) {
    dA[g] = nullptr;
    const long long lc = local_cols(n, nb, ngpus, g);
    if (lc == 0) continue;  // idle GPU (multidevice.py:81-83)
    cudaError_t e = cudaSetDevice(device_ids ? device_ids[g] : g);
    if (e == cudaSuccess) e = cudaMalloc(&dA[g], (size_t)ld * lc * esize);
    if (e != cudaSuccess) {
      for (int h = 0; h < g; ++h)
        if (dA[h]) { cudaSetDevice(device_ids ? device_ids[h] : h); cudaFree(dA[h]); dA[h] = nullptr; }
      return (int)e;
    }
  }
  return 0;
}

// Host-vector call: x (and y when beta != 0) are host arrays, A is in HBM.
// One entry enqueues H2D of the vectors into a per-(device, stream) staging
// pair, the kernels, and the D2H of the result, then waits for the stream.
// This is the path the Python API takes for numpy vectors (one crossing of
// the FFI per call instead of a handful of tensor operations).
inline std::map<std::pair<int, cudaStream_t>, WsBuf> g_vecs;

inline cudaError_t vec_staging(size_t bytes, cudaStream_t st, void **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  WsBuf &b = g_vecs[{dev, st}];
  if (b.bytes < bytes) {
    if (b.ptr) {
      cudaStreamSynchronize(st);
      cudaFree(b.ptr);
      b.ptr = nullptr;
      b.bytes = 0;
    }
    cudaError_t e = cudaMalloc(&b.ptr, bytes * 2);
    if (e != cudaSuccess) { b.ptr = nullptr; return e; }
    b.bytes = bytes * 2;
  }
  *out = b.ptr;
  return cudaSuccess;
}

// page-locked host memory (mapped into the device address space under UVA):
// its device-side address
inline bool mapped_host(const void *h, const void **dev) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) == cudaSuccess && at.type == cudaMemoryTypeHost &&
      at.devicePointer != nullptr) {
    *dev = at.devicePointer;
    return true;
  }
  cudaGetLastError();
  return false;
}

template <class T>
int hostvec_entry(bool is_gemv, char op, bool herm, int m, int n, T alpha, const T *dA, int lda,
                         int off_r, int off_c, const T *hx, T beta, const T *hy_in, T *hy_out, cudaStream_t st,
                         bool sync) {
  const char o = (char)(op | 0x20);
  const bool tr = is_gemv && o != 'n';
  const long long xlen = is_gemv ? (tr ? m : n) : n;
  const long long ylen = is_gemv ? (tr ? n : m) : n;
  if (xlen < 0 || ylen < 0 || hx == nullptr || hy_out == nullptr) return -1;
  const bool bz = is_zero(beta);
  if (!bz && hy_in == nullptr) return -1;
  StreamLock slk(st);
  void *stage = nullptr;
  const size_t xb = align256((size_t)std::max<long long>(xlen, 1) * sizeof(T));
  cudaError_t e = vec_staging(xb + (size_t)std::max<long long>(ylen, 1) * sizeof(T), st, &stage);
  if (e != cudaSuccess) return (int)e;
  T *dx = static_cast<T *>(stage);
  T *dy = reinterpret_cast<T *>(static_cast<char *>(stage) + xb);
  // page-locked inputs are read by a copy-in grid that overlaps the main
  // kernel's first A loads (t_pdl_next); pageable ones go through the
  // copy engine
  const bool xin = xlen > 0, yin = !bz && ylen > 0;
  const void *dhx = nullptr, *dhy = nullptr;
  if ((xin || yin) && (!xin || mapped_host(hx, &dhx)) && (!yin || mapped_host(hy_in, &dhy))) {
    const long long units = cdiv(std::max(xin ? xlen : 0LL, yin ? ylen : 0LL) * (long long)sizeof(T), 16);
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(cdiv(units, 256), 2LL * dev_sms()));
    // programmatic stream serialization: on a queue of calls the grid's
    // PCIe reads overlap the previous call's last kernel (it waits before
    // its first store into the staging buffer)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = hostvec_early_copy() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kblas_hostvec_in_kernel, reinterpret_cast<char *>(dx),
                           static_cast<const char *>(dhx), xin ? xlen * (long long)sizeof(T) : 0,
                           reinterpret_cast<char *>(dy), static_cast<const char *>(dhy),
                           yin ? ylen * (long long)sizeof(T) : 0);
    if (e != cudaSuccess) return (int)e;
    launched();
    // PDL only when x alone is staged: the main kernel reads x after its own
    // griddepcontrol.wait on the copy-in grid.  A staged y (beta != 0) is
    // read by the epilogue kernel, a programmatic dependent of the main
    // kernel only; with the main kernel also launched as a dependent the
    // epilogue was once measured reading stale y staging (tests/
    // test_gpu_hostvec.py, d = 1001), so then the main kernel waits for
    // the copy-in grid the ordinary way, chained launches or not.
    t_pdl_next = !yin;
    t_pdl_off = yin;
  } else {
    if (xin && (e = cudaMemcpyAsync(dx, hx, xlen * sizeof(T), cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return (int)e;
    if (yin && (e = cudaMemcpyAsync(dy, hy_in, ylen * sizeof(T), cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return (int)e;
  }
  // a page-locked result buffer (e.g. from torch's pinned allocator) is
  // mapped into the device address space: with beta == 0 the kernels write
  // y straight into it over PCIe, overlapping the transfer with the last
  // kernel instead of a D2H copy after it
  T *dyk = dy;
  const void *dho = nullptr;
  if (bz && ylen > 0 && mapped_host(hy_out, &dho)) dyk = static_cast<T *>(const_cast<void *>(dho));
  const int rc = is_gemv ? gemv_entry<T>(o, m, n, alpha, dA, lda, dx, 1, beta, dyk, 1, off_r, off_c, st)
                         : symv_entry<T>(o, herm, n, alpha, dA, lda, dx, 1, beta, dyk, 1, off_r, st);
  t_pdl_next = false;  // not consumed when the entry returned before launching
  t_pdl_off = false;
  if (rc != 0) return rc;
  if (dyk == dy && ylen > 0 &&
      (e = cudaMemcpyAsync(hy_out, dy, ylen * sizeof(T), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return (int)e;
  return code(sync ? cudaStreamSynchronize(st) : cudaGetLastError());
}

template <class T>
int partial_p2p(bool is_gemv, char op, bool herm, int m, int n, T alpha, const T *dA, int lda, const T *dx,
                       int G, int g, int nb, T *slots, long long slot_ld, unsigned long long *flags,
                       unsigned long long *consumed, unsigned *counter, unsigned long long seq, T beta,
                       const T *y_in, T *y_out, cudaStream_t st) {
  const long long plen = is_gemv ? ((op == 'n') ? m : n) : n;
  if (slot_ld < plen) return -1;
  StreamLock slk(st);
  const bool fused = !is_gemv && local_cols(n, nb, G, g) > 0 && !is_zero(alpha);
  if (fused) {
    // the exchange rides in the SYMV epilogue: one launch pair per call
    unsigned *cnt = nullptr;
    cudaError_t e = counters(1, st, &cnt);
    if (e != cudaSuccess) return (int)e;
    const kb::Xchg xg{G, g, slots, slot_ld, flags, consumed, cnt, seq, y_in};
    // root: epilogue writes y_out = beta*y_in + sum; others: their slot
    T *dst = (g == 0) ? y_out : slots + (long long)g * slot_ld;
    const bool bz = g != 0 || is_zero(beta);
    Path<T> pa;
    int rc = make_path(dA, lda, &pa) != 0 ? -5 : 0;
    if (rc == 0)
      rc = code(dispatch_symv<T>(op == 'l', herm, pa, lda, n, dx, ColMap{G, g, nb, &xg}, (int)local_cols(n, nb, G, g),
                                 dst, alpha, g == 0 ? beta : zero<T>(), bz, st));
    return rc;
  }
  // general path: wait for the slot, partial into it, signal; root combines
  if (g != 0 && seq > 1) {
    kblas_p2p_wait_kernel<<<1, 32, 0, st>>>(consumed, seq - 1);
    launched();
  }
  int rc = partial_entry<T>(is_gemv, op, herm, m, n, alpha, dA, lda, dx, slots + (long long)g * slot_ld, G, g, nb, st);
  if (rc) return rc;
  kblas_p2p_signal_kernel<<<1, 32, 0, st>>>(flags + g, seq);
  launched();
  if (g != 0) return code(cudaGetLastError());
  if (!is_zero(beta) && y_out != y_in) {
    cudaError_t e = cudaMemcpyAsync(y_out, y_in, plen * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return (int)e;
  }
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(cdiv(plen, 256), 4LL * dev_sms()));
  kblas_p2p_combine_kernel<T><<<grid, 256, 0, st>>>(slots, slot_ld, G, flags, seq, y_out, plen, beta, is_zero(beta) ? 1 : 0,
                                              consumed, counter);
  launched();
  return code(cudaGetLastError());
}


// Entry templates instantiated once per precision in kblas_<p>.cu and
// referenced from kblas_runtime.cu's precision-switching C functions.
#define KBI_ENTRY_TEMPLATES(EXT, T)                                                                          \
  EXT template int partial_entry<T>(bool, char, bool, int, int, T, const T *, int, const T *, T *, int, int, int, \
                                    cudaStream_t);                                                            \
  EXT template int hostvec_entry<T>(bool, char, bool, int, int, T, const T *, int, int, int, const T *, T,       \
                                    const T *, T *, cudaStream_t, bool);                                      \
  EXT template int partial_p2p<T>(bool, char, bool, int, int, T, const T *, int, const T *, int, int, int, T *,   \
                                  long long, unsigned long long *, unsigned long long *, unsigned *,           \
                                  unsigned long long, T, const T *, T *, cudaStream_t);
KBI_ENTRY_TEMPLATES(extern, float)
KBI_ENTRY_TEMPLATES(extern, double)
KBI_ENTRY_TEMPLATES(extern, float2)
KBI_ENTRY_TEMPLATES(extern, double2)

}  // namespace kbi
