// kblas_runtime.cu — the precision-independent part of the C ABI
// (include/kblas_b200.h): precision-switching entry points (mgpu partials,
// host-vector calls, the peer-memory exchange), mgpu allocation and
// layout helpers, panel copies, timing / tuning hooks and the version.
// The per-precision templates are instantiated in kblas_<p>.cu.
#include <map>
#include <cctype>
#include <cstring>
#include "kblas_impl.cuh"

using namespace kb;
using namespace kbi;

namespace {
// The measured B200 table (paper_1410_1726_b200/tuning/b200.json, made by
// scripts/tune_all.py + scripts/merge_tuning.py), installed at load.
const kbi::TuneEntry kBuiltinTuning[] = {
#include "kblas_tuned_b200.inc"
    {0, 0, 0, 0, 0, 0, 0}};

int install_builtin_tuning() {
  std::lock_guard<std::mutex> lk(g_tune_mu);
  g_tune.clear();
  for (const kbi::TuneEntry &e : kBuiltinTuning)
    if (e.prec) g_tune.push_back(e);
  publish_tune();
  return (int)g_tune.size();
}

std::once_flag g_builtin_once;
}  // namespace

namespace kbi {
// first touch of the table installs the built-in entries (lazily: the
// table is an inline variable of the per-precision units, so a static
// initialiser here could run before it is constructed)
void tune_builtin_once() { std::call_once(g_builtin_once, [] { install_builtin_tuning(); }); }
}  // namespace kbi

// ====================================================================
// extern "C" surface
// ====================================================================
extern "C" {

int kblas_mv_mgpu_partial_async(char prec, char kind, char op, int m, int n, const void *alpha,
                                const void *dA_local, int lda, const void *dx, void *dy_partial, int ngpus,
                                int gpu, int nb, int hermitian, cudaStream_t stream) {
  const bool is_gemv = (kind | 0x20) == 'g';
  const char o = (char)(op | 0x20);
  if (ngpus < 1 || gpu < 0 || gpu >= ngpus || nb < 1 || m < 0 || n < 0) return -1;
  switch (prec | 0x20) {
    case 's': return partial_entry<float>(is_gemv, o, false, m, n, *(const float *)alpha, (const float *)dA_local, lda, (const float *)dx, (float *)dy_partial, ngpus, gpu, nb, stream);
    case 'd': return partial_entry<double>(is_gemv, o, false, m, n, *(const double *)alpha, (const double *)dA_local, lda, (const double *)dx, (double *)dy_partial, ngpus, gpu, nb, stream);
    case 'c': return partial_entry<float2>(is_gemv, o, hermitian != 0, m, n, *(const float2 *)alpha, (const float2 *)dA_local, lda, (const float2 *)dx, (float2 *)dy_partial, ngpus, gpu, nb, stream);
    case 'z': return partial_entry<double2>(is_gemv, o, hermitian != 0, m, n, *(const double2 *)alpha, (const double2 *)dA_local, lda, (const double2 *)dx, (double2 *)dy_partial, ngpus, gpu, nb, stream);
  }
  return -1;
}

int kblas_mv_mgpu_combine_async(char prec, long long n, int nparts, const void *const *parts, const void *beta,
                                void *y, cudaStream_t stream) {
  if (beta == nullptr) return -5;
  switch (prec | 0x20) {
    case 's': return combine_entry<float>(n, nparts, parts, *(const float *)beta, (float *)y, stream);
    case 'd': return combine_entry<double>(n, nparts, parts, *(const double *)beta, (double *)y, stream);
    case 'c': return combine_entry<float2>(n, nparts, parts, *(const float2 *)beta, (float2 *)y, stream);
    case 'z': return combine_entry<double2>(n, nparts, parts, *(const double2 *)beta, (double2 *)y, stream);
  }
  return -1;
}

int kblas_mgpu_local_cols(int n, int nb, int ngpus, int gpu) {
  if (n < 0 || nb < 1 || ngpus < 1 || gpu < 0 || gpu >= ngpus) return -1;
  return (int)local_cols(n, nb, ngpus, gpu);
}

int kblas_mgpu_local_ld(int m) { return (int)(cdiv(std::max(m, 1), 32) * 32); }

int kblas_malloc_mgpu_1d(int m, int n, size_t esize, void **dA, int *ldda, int ngpus, int nb,
                         const int *device_ids) {
  return malloc_mgpu(m, n, esize, dA, ldda, ngpus, nb, device_ids);
}

int kblas_free_mgpu(void **dA, int ngpus, const int *device_ids) {
  if (dA == nullptr || ngpus < 1) return -1;
  DevGuard guard;
  for (int g = 0; g < ngpus; ++g) {
    if (!dA[g]) continue;
    cudaSetDevice(device_ids ? device_ids[g] : g);
    cudaError_t e = cudaFree(dA[g]);
    if (e != cudaSuccess) return (int)e;
    dA[g] = nullptr;
  }
  return 0;
}

// the SYMV/HEMV tile width: a distribution block of this width (or a
// multiple) keeps every tile inside one block, so no tile is cut short
int kblas_mgpu_block_size(char prec, char kind) {
  const char p = (char)(prec | 0x20), k = (char)(kind | 0x20);
  if (p != 's' && p != 'd' && p != 'c' && p != 'z') return -1;
  if (k != 'g' && k != 's') return -2;
  return 128;
}

static int copy_mgpu(bool to_dev, int m, int n, size_t esize, const void *hA_c, void *hA, int ldha,
                     void *const *dA, int ldda, int ngpus, int nb, const int *device_ids) {
  if (m < 0 || n < 0 || ngpus < 1 || nb < 1 || ldha < std::max(1, m) || ldda < std::max(1, m)) return -1;
  DevGuard guard;
  const long long nblk = cdiv(n, nb);
  for (long long j = 0; j < nblk; ++j) {
    const int g = (int)(j % ngpus);
    const long long b = j / ngpus;
    const long long c0 = j * nb, w = std::min<long long>(n, c0 + nb) - c0;
    cudaSetDevice(device_ids ? device_ids[g] : g);
    char *dp = static_cast<char *>(dA[g]) + (size_t)(b * nb) * ldda * esize;
    cudaError_t e;
    if (to_dev)
      e = cudaMemcpy2D(dp, (size_t)ldda * esize, static_cast<const char *>(hA_c) + (size_t)c0 * ldha * esize,
                       (size_t)ldha * esize, (size_t)m * esize, (size_t)w, cudaMemcpyHostToDevice);
    else
      e = cudaMemcpy2D(static_cast<char *>(hA) + (size_t)c0 * ldha * esize, (size_t)ldha * esize, dp,
                       (size_t)ldda * esize, (size_t)m * esize, (size_t)w, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

int kblas_setmatrix_mgpu_1d(int m, int n, size_t esize, const void *hA, int ldha, void *const *dA, int ldda,
                            int ngpus, int nb, const int *device_ids) {
  return copy_mgpu(true, m, n, esize, hA, nullptr, ldha, dA, ldda, ngpus, nb, device_ids);
}

int kblas_getmatrix_mgpu_1d(int m, int n, size_t esize, void *const *dA, int ldda, void *hA, int ldha, int ngpus,
                            int nb, const int *device_ids) {
  return copy_mgpu(false, m, n, esize, nullptr, hA, ldha, dA, ldda, ngpus, nb, device_ids);
}

int kblas_setmatrix_async(int rows, int cols, size_t esize, const void *hA, int ldha, void *dA, int ldda,
                          cudaStream_t stream) {
  if (rows < 0 || cols < 0 || ldha < std::max(1, rows) || ldda < std::max(1, rows)) return -1;
  if (rows == 0 || cols == 0) return 0;
  return code(cudaMemcpy2DAsync(dA, (size_t)ldda * esize, hA, (size_t)ldha * esize, (size_t)rows * esize,
                                (size_t)cols, cudaMemcpyHostToDevice, stream));
}

int kblas_getmatrix_async(int rows, int cols, size_t esize, const void *dA, int ldda, void *hA, int ldha,
                          cudaStream_t stream) {
  if (rows < 0 || cols < 0 || ldha < std::max(1, rows) || ldda < std::max(1, rows)) return -1;
  if (rows == 0 || cols == 0) return 0;
  return code(cudaMemcpy2DAsync(hA, (size_t)ldha * esize, dA, (size_t)ldda * esize, (size_t)rows * esize,
                                (size_t)cols, cudaMemcpyDeviceToHost, stream));
}

namespace {
int mv_hostvec(char prec, char kind, char op, int hermitian, int m, int n, const void *alpha, const void *dA,
               int lda, int offset_r, int offset_c, const void *hx, const void *beta, const void *hy_in,
               void *hy_out, cudaStream_t stream, bool sync) {
  const bool g = (kind | 0x20) == 'g';
  if (!g && (kind | 0x20) != 's') return -2;
  if (!g && offset_r != offset_c) return -11;
  switch (prec | 0x20) {
    case 's': return hostvec_entry<float>(g, op, false, m, n, *(const float *)alpha, (const float *)dA, lda, offset_r, offset_c, (const float *)hx, *(const float *)beta, (const float *)hy_in, (float *)hy_out, stream, sync);
    case 'd': return hostvec_entry<double>(g, op, false, m, n, *(const double *)alpha, (const double *)dA, lda, offset_r, offset_c, (const double *)hx, *(const double *)beta, (const double *)hy_in, (double *)hy_out, stream, sync);
    case 'c': return hostvec_entry<float2>(g, op, hermitian != 0, m, n, *(const float2 *)alpha, (const float2 *)dA, lda, offset_r, offset_c, (const float2 *)hx, *(const float2 *)beta, (const float2 *)hy_in, (float2 *)hy_out, stream, sync);
    case 'z': return hostvec_entry<double2>(g, op, hermitian != 0, m, n, *(const double2 *)alpha, (const double2 *)dA, lda, offset_r, offset_c, (const double2 *)hx, *(const double2 *)beta, (const double2 *)hy_in, (double2 *)hy_out, stream, sync);
  }
  return -1;
}
}  // namespace

int kblas_mv_hostvec(char prec, char kind, char op, int hermitian, int m, int n, const void *alpha,
                     const void *dA, int lda, int offset_r, int offset_c, const void *hx, const void *beta,
                     const void *hy_in, void *hy_out, cudaStream_t stream) {
  return mv_hostvec(prec, kind, op, hermitian, m, n, alpha, dA, lda, offset_r, offset_c, hx, beta, hy_in, hy_out,
                    stream, true);
}

int kblas_mv_hostvec_async(char prec, char kind, char op, int hermitian, int m, int n, const void *alpha,
                           const void *dA, int lda, int offset_r, int offset_c, const void *hx, const void *beta,
                           const void *hy_in, void *hy_out, cudaStream_t stream) {
  return mv_hostvec(prec, kind, op, hermitian, m, n, alpha, dA, lda, offset_r, offset_c, hx, beta, hy_in, hy_out,
                    stream, false);
}

int kblas_stream_sync(cudaStream_t stream) { return code(cudaStreamSynchronize(stream)); }

int kblas_stream_order(cudaStream_t waiter, cudaStream_t signaler) {
  if (waiter == signaler) return 0;
  // one reusable event per (thread, device): a wait captures the event's
  // state when it is enqueued, so re-recording it later is safe
  thread_local std::map<int, cudaEvent_t> evs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  cudaEvent_t &ev = evs[dev];
  if (ev == nullptr && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) {
    ev = nullptr;
    return (int)e;
  }
  if ((e = cudaEventRecord(ev, signaler)) != cudaSuccess) return (int)e;
  return code(cudaStreamWaitEvent(waiter, ev, 0));
}

// ------------------------------------------------ peer-memory exchange
int kblas_ipc_get_handle(const void *dptr, void *handle_out) {
  if (dptr == nullptr || handle_out == nullptr) return -1;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(dptr));
  if (e != cudaSuccess) return (int)e;
  memcpy(handle_out, &h, sizeof h);
  return 0;
}

int kblas_ipc_open_handle(const void *handle, void **dptr_out) {
  if (handle == nullptr || dptr_out == nullptr) return -1;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  return code(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
}

int kblas_ipc_close(void *dptr) { return code(cudaIpcCloseMemHandle(dptr)); }

int kblas_p2p_signal_async(unsigned long long *flag, unsigned long long seq, cudaStream_t stream) {
  if (flag == nullptr) return -1;
  kblas_p2p_signal_kernel<<<1, 32, 0, stream>>>(flag, seq);
  launched();
  return code(cudaGetLastError());
}

int kblas_p2p_wait_async(const unsigned long long *flag, unsigned long long seq, cudaStream_t stream) {
  if (flag == nullptr) return -1;
  kblas_p2p_wait_kernel<<<1, 32, 0, stream>>>(flag, seq);
  launched();
  return code(cudaGetLastError());
}

int kblas_mv_mgpu_partial_p2p_async(char prec, char kind, char op, int m, int n, const void *alpha,
                                    const void *dA_local, int lda, const void *dx, int ngpus, int gpu, int nb,
                                    int hermitian, void *slots, long long slot_ld, unsigned long long *flags,
                                    unsigned long long *consumed, unsigned *counter, unsigned long long seq,
                                    const void *beta, const void *y_in, void *y_out, cudaStream_t stream) {
  const bool is_gemv = (kind | 0x20) == 'g';
  const char o = (char)(op | 0x20);
  if (ngpus < 1 || ngpus > kMaxGpus || gpu < 0 || gpu >= ngpus || nb < 1 || m < 0 || n < 0) return -1;
  if (slots == nullptr || flags == nullptr || consumed == nullptr || seq < 1) return -1;
  if (gpu == 0 && (y_out == nullptr || counter == nullptr)) return -1;
  switch (prec | 0x20) {
#define KB_PP(CH, T, H)                                                                                         \
  case CH:                                                                                                      \
    return partial_p2p<T>(is_gemv, o, H, m, n, *(const T *)alpha, (const T *)dA_local, lda, (const T *)dx,        \
                          ngpus, gpu, nb, (T *)slots, slot_ld, flags, consumed, counter, seq, *(const T *)beta,   \
                          (const T *)y_in, (T *)y_out, stream);
    KB_PP('s', float, false)
    KB_PP('d', double, false)
    KB_PP('c', float2, hermitian != 0)
    KB_PP('z', double2, hermitian != 0)
#undef KB_PP
  }
  return -1;
}

int kblas_p2p_combine_async(char prec, int nranks, const void *slots, long long slot_ld,
                            const unsigned long long *flags, unsigned long long seq, const void *beta, void *y,
                            long long n, unsigned long long *consumed, unsigned *counter, cudaStream_t stream) {
  if (nranks < 1 || slots == nullptr || flags == nullptr || y == nullptr || consumed == nullptr ||
      counter == nullptr || n < 0 || slot_ld < n)
    return -1;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(cdiv(n, 256), 4LL * dev_sms()));
  switch (prec | 0x20) {
#define KB_P2P(CH, T)                                                                                         \
  case CH: {                                                                                                  \
    const T b = *static_cast<const T *>(beta);                                                                \
    kblas_p2p_combine_kernel<T><<<grid, 256, 0, stream>>>(static_cast<const T *>(slots), slot_ld, nranks, flags, seq, \
                                                    static_cast<T *>(y), n, b, is_zero(b) ? 1 : 0, consumed,      \
                                                    counter);                                                 \
    break;                                                                                                    \
  }
    KB_P2P('s', float)
    KB_P2P('d', double)
    KB_P2P('c', float2)
    KB_P2P('z', double2)
#undef KB_P2P
    default: return -1;
  }
  launched();
  return code(cudaGetLastError());
}

int kblas_clear_cache(void) {
  // every cached buffer (workspaces, counters, staging, mgpu root buffers,
  // tile tables); waits for the devices that own them first
  std::lock_guard<std::mutex> lk(g_mu);
  DevGuard guard;
  int rc = 0;
  auto release = [&](std::map<std::pair<int, cudaStream_t>, WsBuf> &m) {
    for (auto &kv : m) {
      if (!kv.second.ptr) continue;
      cudaSetDevice(kv.first.first);
      cudaDeviceSynchronize();
      if (cudaFree(kv.second.ptr) != cudaSuccess) rc = 1;
    }
    m.clear();
  };
  release(g_ws);
  release(g_cnt);
  release(g_vecs);
  release(g_rootbufs);
  for (auto &kv : g_tiles) {
    if (!kv.second.dev) continue;
    cudaSetDevice((int)kv.first[0]);
    cudaDeviceSynchronize();
    if (cudaFree(kv.second.dev) != cudaSuccess) rc = 1;
  }
  g_tiles.clear();
  return rc;
}

unsigned long long kblas_launch_count(void) { return g_launches.load(); }

int kblas_timing_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = enable != 0;
  return 0;
}

int kblas_timing_read(double *total_ms, int *launches) {
  std::vector<EvPair> evs;
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    evs.swap(g_events);
  }
  DevGuard guard;
  double tot = 0.0;
  int rc = 0;
  for (auto &ev : evs) {
    cudaSetDevice(ev.dev);
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(ev.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev.a, ev.b);
    if (e != cudaSuccess) rc = (int)e;
    tot += ms;
    cudaEventDestroy(ev.a);
    cudaEventDestroy(ev.b);
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (int)evs.size();
  return rc;
}

const char *kblas_last_plan(void) { return g_last_plan.c_str(); }

int kblas_set_symv_variant(int v) {
  const int prev = g_symv_variant;
  g_symv_variant = v;
  return prev;
}

int kblas_set_symv_mid(int max_order) {
  const int prev = g_symv_mid_max;
  g_symv_mid_max = max_order;
  return prev;
}

int kblas_set_symv_window(int items) {
  const int prev = g_symv_window;
  g_symv_window = items;
  return prev;
}

int kblas_set_symv_trace(void *dev_buf) {
#if KBLAS_SYMV_TRACE
  g_symv_trace = static_cast<unsigned long long *>(dev_buf);
  return 0;
#else
  (void)dev_buf;
  return -1;  // product build: the trace branches are compiled out
#endif
}

int kblas_set_symv_segment(int items) {
  const int prev = g_symv_seg;
  g_symv_seg = items;
  g_symv_seg_auto = false;  // an explicit K is used as given
  return prev;
}

int kblas_set_symv_narrow(int max_order) {
  const int prev = g_symv_narrow_max;
  g_symv_narrow_max = max_order;
  return prev;
}

int kblas_set_gemv_variant(int v) {
  const int prev = g_gemv_variant;
  g_gemv_variant = v;
  return prev;
}

int kblas_set_gemv_cluster(int mode) {
  const int prev = g_gemv_cluster;
  g_gemv_cluster = mode < 0 ? -1 : (mode ? 1 : 0);
  return prev;
}

int kblas_set_gemv_split_waves(int waves) {
  const int prev = g_split_waves;
  if (waves >= 1) g_split_waves = waves;
  return prev;
}

int kblas_set_gemv_tc(int mode, long long max_bytes) {
  const int prev = g_gemv_tc;
  g_gemv_tc = mode < 0 ? -1 : (mode ? 1 : 0);
  if (max_bytes > 0) g_gemv_tc_max_bytes = max_bytes;
  return prev;
}

int kblas_set_gemv_split(int mode) {
  const int prev = g_gemv_split;
  g_gemv_split = mode < 0 ? -1 : (mode == 3 ? 3 : mode ? 1 : 0);
  return prev;
}

int kblas_set_gemv_rowown(int cfg) {
  const int prev = g_gemv_ro_cfg;
  g_gemv_ro_cfg = cfg < 0 ? -1 : cfg;
  return prev;
}

int kblas_tune_set(char prec, char op, long long n_lo, long long n_hi, int shape, int form, int waves) {
  tune_builtin_once();
  prec = (char)std::tolower((unsigned char)prec);
  op = (char)std::tolower((unsigned char)op);
  if (!std::strchr("sdcz", prec) || prec == 0) return -1;
  const bool gemv = op == 'n' || op == 't' || op == 'c';
  if (!gemv && op != 'l' && op != 'u') return -2;
  if (n_lo < 0) return -3;
  if (n_hi < n_lo) return -4;
  const bool rowown = op == 'n' && form == 3;
  if (rowown ? !(shape >= 10 && shape <= 17)
             : gemv ? !(shape == 0 || shape == 3 || shape == 4 || shape == 5)
                    : !(shape == -1 || shape == 100 || shape == 103 || shape == 105))
    return -5;
  if (form < -1 || form > (op == 'n' ? 3 : gemv ? 1 : -1)) return -6;
  if (waves < 0 || waves > 64 || (waves && op != 'n')) return -7;
  std::lock_guard<std::mutex> lk(g_tune_mu);
  for (TuneEntry &e : g_tune)
    if (e.prec == prec && e.op == op && e.lo == n_lo && e.hi == n_hi) {
      e.shape = shape;
      e.form = form;
      e.waves = waves;
      publish_tune();
      return 0;
    }
  g_tune.push_back(TuneEntry{prec, op, n_lo, n_hi, shape, form, waves});
  publish_tune();
  return 0;
}


int kblas_tune_defaults(void) {
  tune_builtin_once();
  return install_builtin_tuning();
}

int kblas_tune_clear(void) {
  tune_builtin_once();
  std::lock_guard<std::mutex> lk(g_tune_mu);
  g_tune.clear();
  publish_tune();
  return 0;
}

int kblas_tune_count(void) {
  tune_builtin_once();
  return g_tune_n.load(std::memory_order_acquire);
}

int kblas_tune_get(int i, char *prec, char *op, long long *n_lo, long long *n_hi, int *shape, int *form,
                   int *waves) {
  tune_builtin_once();
  std::lock_guard<std::mutex> lk(g_tune_mu);
  if (i < 0 || i >= (int)g_tune.size()) return -1;
  const TuneEntry &e = g_tune[i];
  if (prec) *prec = e.prec;
  if (op) *op = e.op;
  if (n_lo) *n_lo = e.lo;
  if (n_hi) *n_hi = e.hi;
  if (shape) *shape = e.shape;
  if (form) *form = e.form;
  if (waves) *waves = e.waves;
  return 0;
}

int kblas_set_tma(int mode) {
  const int prev = tma_mode();
  g_use_tma = mode < 0 ? -1 : (mode ? 1 : 0);
  return prev;
}

const char *kblas_version(void) { return "kblas-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
