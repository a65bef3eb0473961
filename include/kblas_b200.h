/*
 * kblas_b200.h — C ABI of the B200-native KBLAS matrix-vector library.
 *
 * Drop-in boundary for the reference's GEMV / SYMV / HEMV hot path.  The
 * reference (`blockmv`, /root/reference/pkg/src/blockmv) exposes these
 * operations as Python functions; the paper it simulates
 * names the C routines kblas_x{gemv,symv,hemv}[_offset|_mgpu][_async].
 * Each entry point below cites the reference function whose behaviour it
 * replaces.
 *
 * Conventions (all entry points)
 *   - Column-major storage, BLAS argument order, device pointers.
 *   - Element (i, j) of A lives at dA[j * lda + i].
 *   - incx / incy must be 1 (the reference's scope).
 *   - y is updated in place: y <- alpha * op(A) x + beta * y.
 *   - beta == 0 writes y without reading it (NaN/Inf in y never propagate,
 *     kernels.py:136-137, 382-383).
 *   - alpha == 0 and beta == 1: quick return, nothing launched
 *     (kernels.py:427-428).  alpha == 0 otherwise: y <- beta * y and A is
 *     not read (BLAS semantics).
 *   - Results are bit-deterministic: every cross-CTA reduction is a
 *     fixed-order two-pass sum (no floating-point atomics).
 *   - Synchronous variants launch on the legacy default stream (0);
 *     `_async` variants take an explicit stream.
 *   - Kernels are launched as programmatic dependents of the stream's
 *     previous kernel and release their own dependents early; each waits
 *     (griddepcontrol.wait) before touching data an earlier kernel may
 *     still use.  A caller's kernel launched with the programmatic-
 *     serialization attribute after a call must do the same before it
 *     reads the call's output ($KBLAS_PDL_CHAIN=0: ordinary launches).
 *
 * Return codes
 *   0   success
 *   -k  argument k (1-based, BLAS xerbla numbering) is invalid
 *   >0  CUDA error code (cudaError_t) from a launch or allocation
 */
#ifndef KBLAS_B200_H
#define KBLAS_B200_H

#include <cuComplex.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ */
/* GEMV: y = alpha * op(A) x + beta * y, op in {N, T, C}.              */
/* Replaces blockmv.kernels.gemv (kernels.py:402-440); 'c' on a real   */
/* precision behaves as 't' (kernels.py:422-423).                      */
/* ------------------------------------------------------------------ */
int kblas_sgemv(char trans, int m, int n, float alpha, const float *dA, int lda,
                const float *dx, int incx, float beta, float *dy, int incy);
int kblas_dgemv(char trans, int m, int n, double alpha, const double *dA, int lda,
                const double *dx, int incx, double beta, double *dy, int incy);
int kblas_cgemv(char trans, int m, int n, cuFloatComplex alpha, const cuFloatComplex *dA,
                int lda, const cuFloatComplex *dx, int incx, cuFloatComplex beta,
                cuFloatComplex *dy, int incy);
int kblas_zgemv(char trans, int m, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA,
                int lda, const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                cuDoubleComplex *dy, int incy);

int kblas_sgemv_async(char trans, int m, int n, float alpha, const float *dA, int lda,
                      const float *dx, int incx, float beta, float *dy, int incy,
                      cudaStream_t stream);
int kblas_dgemv_async(char trans, int m, int n, double alpha, const double *dA, int lda,
                      const double *dx, int incx, double beta, double *dy, int incy,
                      cudaStream_t stream);
int kblas_cgemv_async(char trans, int m, int n, cuFloatComplex alpha,
                      const cuFloatComplex *dA, int lda, const cuFloatComplex *dx, int incx,
                      cuFloatComplex beta, cuFloatComplex *dy, int incy, cudaStream_t stream);
int kblas_zgemv_async(char trans, int m, int n, cuDoubleComplex alpha,
                      const cuDoubleComplex *dA, int lda, const cuDoubleComplex *dx,
                      int incx, cuDoubleComplex beta, cuDoubleComplex *dy, int incy,
                      cudaStream_t stream);

/* ------------------------------------------------------------------ */
/* SYMV (s, d; and complex-symmetric c, z) / HEMV (c, z):              */
/* y = alpha * A x + beta * y with A stored in one triangle (uplo).    */
/* Replaces blockmv.kernels.symv / hemv / symv_hemv                    */
/* (kernels.py:443-500).  The unreferenced triangle is never read      */
/* except inside diagonal tiles, where it is masked (never used).      */
/* HEMV ignores the imaginary part of the stored diagonal              */
/* (kernels.py:353-354).                                               */
/* ------------------------------------------------------------------ */
int kblas_ssymv(char uplo, int n, float alpha, const float *dA, int lda, const float *dx,
                int incx, float beta, float *dy, int incy);
int kblas_dsymv(char uplo, int n, double alpha, const double *dA, int lda, const double *dx,
                int incx, double beta, double *dy, int incy);
int kblas_chemv(char uplo, int n, cuFloatComplex alpha, const cuFloatComplex *dA, int lda,
                const cuFloatComplex *dx, int incx, cuFloatComplex beta, cuFloatComplex *dy,
                int incy);
int kblas_zhemv(char uplo, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA, int lda,
                const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                cuDoubleComplex *dy, int incy);
/* complex symmetric (non-Hermitian): symv_hemv(..., hermitian=False)   */
/* on a complex precision (kernels.py:466-469).                        */
int kblas_csymv(char uplo, int n, cuFloatComplex alpha, const cuFloatComplex *dA, int lda,
                const cuFloatComplex *dx, int incx, cuFloatComplex beta, cuFloatComplex *dy,
                int incy);
int kblas_zsymv(char uplo, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA, int lda,
                const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                cuDoubleComplex *dy, int incy);

int kblas_ssymv_async(char uplo, int n, float alpha, const float *dA, int lda,
                      const float *dx, int incx, float beta, float *dy, int incy,
                      cudaStream_t stream);
int kblas_dsymv_async(char uplo, int n, double alpha, const double *dA, int lda,
                      const double *dx, int incx, double beta, double *dy, int incy,
                      cudaStream_t stream);
int kblas_chemv_async(char uplo, int n, cuFloatComplex alpha, const cuFloatComplex *dA,
                      int lda, const cuFloatComplex *dx, int incx, cuFloatComplex beta,
                      cuFloatComplex *dy, int incy, cudaStream_t stream);
int kblas_zhemv_async(char uplo, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA,
                      int lda, const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                      cuDoubleComplex *dy, int incy, cudaStream_t stream);
int kblas_csymv_async(char uplo, int n, cuFloatComplex alpha, const cuFloatComplex *dA,
                      int lda, const cuFloatComplex *dx, int incx, cuFloatComplex beta,
                      cuFloatComplex *dy, int incy, cudaStream_t stream);
int kblas_zsymv_async(char uplo, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA,
                      int lda, const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                      cuDoubleComplex *dy, int incy, cudaStream_t stream);

/* ------------------------------------------------------------------ */
/* Submatrix ("new interface").  dA points at the    */
/* ORIGINAL matrix; (offset_r, offset_c) locate the m x n submatrix.   */
/* Replaces blockmv.offset.gemv_offset (offset.py:83-143) with         */
/* OffsetRequest(parent, row_off, col_off, sub_m, sub_n)               */
/* (offset.py:37-51).  Loads realign to the 16-byte granule at or      */
/* below the submatrix start and mask the lead rows.                   */
/* ------------------------------------------------------------------ */
int kblas_sgemv_offset(char trans, int m, int n, float alpha, const float *dA, int lda,
                       const float *dx, int incx, float beta, float *dy, int incy,
                       int offset_r, int offset_c);
int kblas_dgemv_offset(char trans, int m, int n, double alpha, const double *dA, int lda,
                       const double *dx, int incx, double beta, double *dy, int incy,
                       int offset_r, int offset_c);
int kblas_cgemv_offset(char trans, int m, int n, cuFloatComplex alpha,
                       const cuFloatComplex *dA, int lda, const cuFloatComplex *dx, int incx,
                       cuFloatComplex beta, cuFloatComplex *dy, int incy, int offset_r,
                       int offset_c);
int kblas_zgemv_offset(char trans, int m, int n, cuDoubleComplex alpha,
                       const cuDoubleComplex *dA, int lda, const cuDoubleComplex *dx,
                       int incx, cuDoubleComplex beta, cuDoubleComplex *dy, int incy,
                       int offset_r, int offset_c);
int kblas_sgemv_offset_async(char trans, int m, int n, float alpha, const float *dA, int lda,
                             const float *dx, int incx, float beta, float *dy, int incy,
                             int offset_r, int offset_c, cudaStream_t stream);
int kblas_dgemv_offset_async(char trans, int m, int n, double alpha, const double *dA,
                             int lda, const double *dx, int incx, double beta, double *dy,
                             int incy, int offset_r, int offset_c, cudaStream_t stream);
int kblas_cgemv_offset_async(char trans, int m, int n, cuFloatComplex alpha,
                             const cuFloatComplex *dA, int lda, const cuFloatComplex *dx,
                             int incx, cuFloatComplex beta, cuFloatComplex *dy, int incy,
                             int offset_r, int offset_c, cudaStream_t stream);
int kblas_zgemv_offset_async(char trans, int m, int n, cuDoubleComplex alpha,
                             const cuDoubleComplex *dA, int lda, const cuDoubleComplex *dx,
                             int incx, cuDoubleComplex beta, cuDoubleComplex *dy, int incy,
                             int offset_r, int offset_c, cudaStream_t stream);

/* Diagonal submatrix of a triangle-stored matrix: n x n block at      */
/* (offset, offset).  Replaces blockmv.offset.symv_hemv_offset         */
/* (offset.py:146-208).                                                */
int kblas_ssymv_offset(char uplo, int n, float alpha, const float *dA, int lda,
                       const float *dx, int incx, float beta, float *dy, int incy,
                       int offset);
int kblas_dsymv_offset(char uplo, int n, double alpha, const double *dA, int lda,
                       const double *dx, int incx, double beta, double *dy, int incy,
                       int offset);
int kblas_chemv_offset(char uplo, int n, cuFloatComplex alpha, const cuFloatComplex *dA,
                       int lda, const cuFloatComplex *dx, int incx, cuFloatComplex beta,
                       cuFloatComplex *dy, int incy, int offset);
int kblas_zhemv_offset(char uplo, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA,
                       int lda, const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                       cuDoubleComplex *dy, int incy, int offset);
int kblas_csymv_offset(char uplo, int n, cuFloatComplex alpha, const cuFloatComplex *dA,
                       int lda, const cuFloatComplex *dx, int incx, cuFloatComplex beta,
                       cuFloatComplex *dy, int incy, int offset);
int kblas_zsymv_offset(char uplo, int n, cuDoubleComplex alpha, const cuDoubleComplex *dA,
                       int lda, const cuDoubleComplex *dx, int incx, cuDoubleComplex beta,
                       cuDoubleComplex *dy, int incy, int offset);
int kblas_ssymv_offset_async(char uplo, int n, float alpha, const float *dA, int lda,
                             const float *dx, int incx, float beta, float *dy, int incy,
                             int offset, cudaStream_t stream);
int kblas_dsymv_offset_async(char uplo, int n, double alpha, const double *dA, int lda,
                             const double *dx, int incx, double beta, double *dy, int incy,
                             int offset, cudaStream_t stream);
int kblas_chemv_offset_async(char uplo, int n, cuFloatComplex alpha,
                             const cuFloatComplex *dA, int lda, const cuFloatComplex *dx,
                             int incx, cuFloatComplex beta, cuFloatComplex *dy, int incy,
                             int offset, cudaStream_t stream);
int kblas_zhemv_offset_async(char uplo, int n, cuDoubleComplex alpha,
                             const cuDoubleComplex *dA, int lda, const cuDoubleComplex *dx,
                             int incx, cuDoubleComplex beta, cuDoubleComplex *dy, int incy,
                             int offset, cudaStream_t stream);
int kblas_csymv_offset_async(char uplo, int n, cuFloatComplex alpha,
                             const cuFloatComplex *dA, int lda, const cuFloatComplex *dx,
                             int incx, cuFloatComplex beta, cuFloatComplex *dy, int incy,
                             int offset, cudaStream_t stream);
int kblas_zsymv_offset_async(char uplo, int n, cuDoubleComplex alpha,
                             const cuDoubleComplex *dA, int lda, const cuDoubleComplex *dx,
                             int incx, cuDoubleComplex beta, cuDoubleComplex *dy, int incy,
                             int offset, cudaStream_t stream);

/* ------------------------------------------------------------------ */
/* Multi-GPU, 1D block-column-cyclic layout (PAPER.md:458-476;          */
/* blockmv.multidevice, multidevice.py:72-284).  Block column j (width */
/* nb) of the global m x n matrix lives on GPU j mod ngpus, packed      */
/* contiguously into that GPU's local panel dA[g] (ld = lda, common).  */
/* dx[g] holds a full replica of x on GPU g.  dy[0] is the root: it    */
/* holds y on input and the result on output; dy[g] for g > 0 must be  */
/* full-length device buffers on GPU g and receive that GPU's partial. */
/* device_ids may be NULL (GPU g = CUDA device g); several logical     */
/* GPUs may share one device.                                          */
/* The sum of partials is done by a root kernel that reads each        */
/* partial in device order over NVLink peer memory (or after a peer     */
/* copy when peer access is unavailable), fused with beta * y:         */
/* deterministic, matching multidevice.py:161,176,276,282-283.          */
/* Replaces gemv_mgpu (multidevice.py:119-180) and symv_hemv_mgpu      */
/* (multidevice.py:183-284); for SYMV/HEMV nb is the distribution      */
/* block width (must equal the kernel block size in the reference,     */
/* multidevice.py:205-208; here any nb >= 1 is accepted).              */
/* ------------------------------------------------------------------ */
int kblas_sgemv_mgpu(char trans, int m, int n, float alpha, float *const *dA, int lda,
                     float *const *dx, int incx, float beta, float *const *dy, int incy,
                     int ngpus, int nb, const int *device_ids);
int kblas_dgemv_mgpu(char trans, int m, int n, double alpha, double *const *dA, int lda,
                     double *const *dx, int incx, double beta, double *const *dy, int incy,
                     int ngpus, int nb, const int *device_ids);
int kblas_cgemv_mgpu(char trans, int m, int n, cuFloatComplex alpha,
                     cuFloatComplex *const *dA, int lda, cuFloatComplex *const *dx, int incx,
                     cuFloatComplex beta, cuFloatComplex *const *dy, int incy, int ngpus,
                     int nb, const int *device_ids);
int kblas_zgemv_mgpu(char trans, int m, int n, cuDoubleComplex alpha,
                     cuDoubleComplex *const *dA, int lda, cuDoubleComplex *const *dx,
                     int incx, cuDoubleComplex beta, cuDoubleComplex *const *dy, int incy,
                     int ngpus, int nb, const int *device_ids);
int kblas_ssymv_mgpu(char uplo, int n, float alpha, float *const *dA, int lda,
                     float *const *dx, int incx, float beta, float *const *dy, int incy,
                     int ngpus, int nb, const int *device_ids);
int kblas_dsymv_mgpu(char uplo, int n, double alpha, double *const *dA, int lda,
                     double *const *dx, int incx, double beta, double *const *dy, int incy,
                     int ngpus, int nb, const int *device_ids);
int kblas_chemv_mgpu(char uplo, int n, cuFloatComplex alpha, cuFloatComplex *const *dA,
                     int lda, cuFloatComplex *const *dx, int incx, cuFloatComplex beta,
                     cuFloatComplex *const *dy, int incy, int ngpus, int nb,
                     const int *device_ids);
int kblas_zhemv_mgpu(char uplo, int n, cuDoubleComplex alpha, cuDoubleComplex *const *dA,
                     int lda, cuDoubleComplex *const *dx, int incx, cuDoubleComplex beta,
                     cuDoubleComplex *const *dy, int incy, int ngpus, int nb,
                     const int *device_ids);
int kblas_csymv_mgpu(char uplo, int n, cuFloatComplex alpha, cuFloatComplex *const *dA,
                     int lda, cuFloatComplex *const *dx, int incx, cuFloatComplex beta,
                     cuFloatComplex *const *dy, int incy, int ngpus, int nb,
                     const int *device_ids);
int kblas_zsymv_mgpu(char uplo, int n, cuDoubleComplex alpha, cuDoubleComplex *const *dA,
                     int lda, cuDoubleComplex *const *dx, int incx, cuDoubleComplex beta,
                     cuDoubleComplex *const *dy, int incy, int ngpus, int nb,
                     const int *device_ids);
/* _async forms (every routine has one): streams[g] is */
/* the stream on GPU g; the root's combine runs on streams[0] after     */
/* events from the others, and every streams[g] then waits for the      */
/* combine, so dy[g] may be reused by the next call at once; nothing is */
/* waited for on the host.  A non-NULL streams array is required (last  */
/* argument index).                                                     */
int kblas_sgemv_mgpu_async(char trans, int m, int n, float alpha, float *const *dA, int lda,
                           float *const *dx, int incx, float beta, float *const *dy, int incy,
                           int ngpus, int nb, const int *device_ids, cudaStream_t const *streams);
int kblas_dgemv_mgpu_async(char trans, int m, int n, double alpha, double *const *dA, int lda,
                           double *const *dx, int incx, double beta, double *const *dy, int incy,
                           int ngpus, int nb, const int *device_ids, cudaStream_t const *streams);
int kblas_cgemv_mgpu_async(char trans, int m, int n, cuFloatComplex alpha,
                           cuFloatComplex *const *dA, int lda, cuFloatComplex *const *dx, int incx,
                           cuFloatComplex beta, cuFloatComplex *const *dy, int incy, int ngpus,
                           int nb, const int *device_ids, cudaStream_t const *streams);
int kblas_zgemv_mgpu_async(char trans, int m, int n, cuDoubleComplex alpha,
                           cuDoubleComplex *const *dA, int lda, cuDoubleComplex *const *dx,
                           int incx, cuDoubleComplex beta, cuDoubleComplex *const *dy, int incy,
                           int ngpus, int nb, const int *device_ids, cudaStream_t const *streams);
int kblas_ssymv_mgpu_async(char uplo, int n, float alpha, float *const *dA, int lda,
                           float *const *dx, int incx, float beta, float *const *dy, int incy,
                           int ngpus, int nb, const int *device_ids, cudaStream_t const *streams);
int kblas_dsymv_mgpu_async(char uplo, int n, double alpha, double *const *dA, int lda,
                           double *const *dx, int incx, double beta, double *const *dy, int incy,
                           int ngpus, int nb, const int *device_ids, cudaStream_t const *streams);
int kblas_chemv_mgpu_async(char uplo, int n, cuFloatComplex alpha, cuFloatComplex *const *dA,
                           int lda, cuFloatComplex *const *dx, int incx, cuFloatComplex beta,
                           cuFloatComplex *const *dy, int incy, int ngpus, int nb,
                           const int *device_ids, cudaStream_t const *streams);
int kblas_zhemv_mgpu_async(char uplo, int n, cuDoubleComplex alpha, cuDoubleComplex *const *dA,
                           int lda, cuDoubleComplex *const *dx, int incx, cuDoubleComplex beta,
                           cuDoubleComplex *const *dy, int incy, int ngpus, int nb,
                           const int *device_ids, cudaStream_t const *streams);
int kblas_csymv_mgpu_async(char uplo, int n, cuFloatComplex alpha, cuFloatComplex *const *dA,
                           int lda, cuFloatComplex *const *dx, int incx, cuFloatComplex beta,
                           cuFloatComplex *const *dy, int incy, int ngpus, int nb,
                           const int *device_ids, cudaStream_t const *streams);
int kblas_zsymv_mgpu_async(char uplo, int n, cuDoubleComplex alpha, cuDoubleComplex *const *dA,
                           int lda, cuDoubleComplex *const *dx, int incx, cuDoubleComplex beta,
                           cuDoubleComplex *const *dy, int incy, int ngpus, int nb,
                           const int *device_ids, cudaStream_t const *streams);

/* Per-device partial only (no cross-device reduction, no beta): the    */
/* building block for one-process-per-GPU deployments, where the       */
/* caller combines partials with an NCCL reduce.  Computes on the      */
/* current device: dy_partial = alpha * (local contribution of GPU g). */
/* prec: 's','d','c','z'; op: 'n','t','c' (gemv) or 'l','u' (symv,     */
/* hemv when hermitian != 0).  alpha points to a host scalar of the    */
/* precision's type.                                                   */
int kblas_mv_mgpu_partial_async(char prec, char kind, char op, int m, int n,
                                const void *alpha, const void *dA_local, int lda,
                                const void *dx, void *dy_partial, int ngpus, int gpu,
                                int nb, int hermitian, cudaStream_t stream);

/* Root combine of per-GPU partials: y = beta * y + sum_g parts[g],     */
/* summed in g order (the reference's device-order sum,                */
/* multidevice.py:176,276, then beta, 282-283) by one kernel on the    */
/* current device; parts[g] are length-n device vectors on this device  */
/* or peer-accessible.  beta points to a host scalar of the precision's */
/* type (beta == 0: y is written, not read).  For callers that reduce   */
/* partials themselves (e.g. NCCL) and fuse beta here.                 */
int kblas_mv_mgpu_combine_async(char prec, long long n, int nparts, const void *const *parts,
                                const void *beta, void *y, cudaStream_t stream);

/* One-process-per-GPU exchange over peer memory, replacing the host-  */
/* side device-order sum of the partials (multidevice.py:276, 282-283)  */
/* without NCCL.  The root owns `slots` (nranks x slot_ld elements),    */
/* `flags` (nranks u64), `consumed` (u64) and `counter` (u32, zero),    */
/* shares them with CUDA IPC handles (64 bytes), and every rank writes  */
/* its partial into its slot through kblas_mv_mgpu_partial_async, then */
/* kblas_p2p_signal_async(&flags[rank], seq).  Before reusing its slot */
/* for call seq a rank waits for consumed >= seq-1                     */
/* (kblas_p2p_wait_async).  kblas_p2p_combine_async (root) waits for    */
/* all flags >= seq, writes y = beta*y + sum_g slots[g] in rank order   */
/* and publishes consumed = seq.  All calls are stream-ordered.         */
int kblas_ipc_get_handle(const void *dptr, void *handle_out);
int kblas_ipc_open_handle(const void *handle, void **dptr_out);
int kblas_ipc_close(void *dptr);
int kblas_p2p_signal_async(unsigned long long *flag, unsigned long long seq,
                           cudaStream_t stream);
int kblas_p2p_wait_async(const unsigned long long *flag, unsigned long long seq,
                         cudaStream_t stream);
/* The whole per-rank step of a one-process-per-GPU mgpu call with the  */
/* peer-memory exchange: this rank's partial (as                        */
/* kblas_mv_mgpu_partial_async) into its slot, the handshake, and on    */
/* rank 0 the rank-order combine with beta (y_out = beta*y_in + sum).   */
/* For SYMV/HEMV the exchange is fused into the partial's epilogue      */
/* kernel (waits, peer stores, flags); GEMV uses the separate kernels   */
/* above.  slots/flags/consumed are this rank's mappings of rank 0's    */
/* buffers; counter (rank 0) is a zeroed u32 in rank 0's HBM; seq      */
/* counts calls from 1.                                                 */
int kblas_mv_mgpu_partial_p2p_async(char prec, char kind, char op, int m, int n,
                                    const void *alpha, const void *dA_local, int lda,
                                    const void *dx, int ngpus, int gpu, int nb, int hermitian,
                                    void *slots, long long slot_ld, unsigned long long *flags,
                                    unsigned long long *consumed, unsigned *counter,
                                    unsigned long long seq, const void *beta,
                                    const void *y_in, void *y_out, cudaStream_t stream);
int kblas_p2p_combine_async(char prec, int nranks, const void *slots, long long slot_ld,
                            const unsigned long long *flags, unsigned long long seq,
                            const void *beta, void *y, long long n,
                            unsigned long long *consumed, unsigned *counter,
                            cudaStream_t stream);

/* ------------------------------------------------------------------ */
/* mgpu helpers: column count held by one GPU under */
/* the cyclic layout (multidevice.py:38-43), and the local ld (rows    */
/* padded to 32 elements, multidevice.py:46-52,85).                    */
/* ------------------------------------------------------------------ */
int kblas_mgpu_local_cols(int n, int nb, int ngpus, int gpu);
int kblas_mgpu_local_ld(int m);
/* Allocate (free) every GPU's local panel for an m x n matrix in the   */
/* cyclic layout, ld = kblas_mgpu_local_ld(m) returned in *ldda; an     */
/* idle GPU gets NULL (multidevice.py:81-93).  "KBLAS provides          */
/* functions that allocate the necessary memory space on each GPU"      */
/* (PAPER.md:425-427).                                                  */
int kblas_malloc_mgpu_1d(int m, int n, size_t esize, void **dA, int *ldda, int ngpus, int nb,
                         const int *device_ids);
int kblas_free_mgpu(void **dA, int ngpus, const int *device_ids);
/* The distribution block width to use with the mgpu routines for this */
/* precision and kind ('g' gemv, 's' symv/hemv): the SYMV tile width,  */
/* so tiles never straddle a block ("KBLAS exposes   */
/* such values through another set of functions").                     */
int kblas_mgpu_block_size(char prec, char kind);
/* Copy the global host matrix into (pre-allocated) local panels, and   */
/* back (blockmv.distribute / gather, multidevice.py:72-110).  esize is */
/* the element size in bytes.                                          */
int kblas_setmatrix_mgpu_1d(int m, int n, size_t esize, const void *hA, int ldha,
                            void *const *dA, int ldda, int ngpus, int nb,
                            const int *device_ids);
int kblas_getmatrix_mgpu_1d(int m, int n, size_t esize, void *const *dA, int ldda,
                            void *hA, int ldha, int ngpus, int nb, const int *device_ids);

/* Single-GPU host<->device panel copies (cuBLAS-style set/getmatrix):  */
/* rows x cols column-major, element size esize, pitched by ldh / ldd.  */
/* Used by the Python API to upload only the referenced part of a host  */
/* operand (e.g. the stored triangle, block column by block column).   */
int kblas_setmatrix_async(int rows, int cols, size_t esize, const void *hA, int ldha, void *dA,
                          int ldda, cudaStream_t stream);
int kblas_getmatrix_async(int rows, int cols, size_t esize, const void *dA, int ldda, void *hA,
                          int ldha, cudaStream_t stream);

/* ------------------------------------------------------------------ */
/* Instrumentation (bench/test harness).                               */
/* ------------------------------------------------------------------ */
/* Host-vector form of every single-GPU entry point (the path the      */
/* Python API takes for numpy vectors): A is in HBM; x, y_in and y_out  */
/* are HOST arrays.  prec in {s,d,c,z}; kind 'g' (gemv: op = trans,    */
/* offsets (offset_r, offset_c) as kblas_xgemv_offset) or 's'           */
/* (symv/hemv: op = uplo, hermitian selects HEMV for c/z, offset_r ==   */
/* offset_c = the diagonal offset).  alpha/beta point to one scalar of  */
/* the precision.  y_in may be NULL when *beta == 0.  Enqueues on      */
/* `stream`: the staging of x (and y_in) -- a copy-in kernel reading    */
/* page-locked host memory through its device mapping (launched as a   */
/* programmatic dependent of the stream's previous kernel; it stores   */
/* only after that kernel has completed), or cudaMemcpyAsync for       */
/* pageable memory --, the kernels, and the result write               */
/* (straight into page-locked y_out when *beta == 0, else a D2H copy),  */
/* then waits.  Same return codes as the entry points it wraps (-1: bad */
/* vector arguments).  Replaces blockmv's numpy-in/numpy-out call shape */
/* (kernels.py:402-440, 443-486; offset.py:83-208).                     */
int kblas_mv_hostvec(char prec, char kind, char op, int hermitian, int m, int n,
                     const void *alpha, const void *dA, int lda, int offset_r,
                     int offset_c, const void *x, const void *beta,
                     const void *y_in, void *y_out, cudaStream_t stream);
/* Same, without the final wait: returns once everything is enqueued.   */
/* x, y_in and y_out must stay valid (and y_out unread) until the       */
/* stream has been synchronised (kblas_stream_sync); lets the caller    */
/* overlap its own bookkeeping with the kernels.                        */
int kblas_mv_hostvec_async(char prec, char kind, char op, int hermitian, int m, int n,
                           const void *alpha, const void *dA, int lda, int offset_r,
                           int offset_c, const void *x, const void *beta,
                           const void *y_in, void *y_out, cudaStream_t stream);
/* cudaStreamSynchronize(stream); 0 or the CUDA error. */
int kblas_stream_sync(cudaStream_t stream);
/* Make `waiter` wait (on the device) for the work enqueued on          */
/* `signaler` so far (event record + stream wait on the current         */
/* device); 0 or the CUDA error.  Used by the Python CommandQueue to    */
/* order a submission after the caller's stream without a host wait.   */
int kblas_stream_order(cudaStream_t waiter, cudaStream_t signaler);
/* Free every cached device buffer (per-stream workspaces, counters,   */
/* vector staging, mgpu root buffers, SYMV tile tables) after waiting   */
/* for the devices that own them.  The next call re-creates what it     */
/* needs.  For long-running processes that used many streams / shapes.  */
int kblas_clear_cache(void);
/* Number of kernels this library has launched since load.             */
unsigned long long kblas_launch_count(void);
/* When enabled, the library brackets every main (matrix-streaming)    */
/* kernel with CUDA events on its launch stream.  kblas_timing_read     */
/* synchronises those events and returns the summed milliseconds and   */
/* the number of timed launches, then clears the record.               */
int kblas_timing_enable(int enable);
int kblas_timing_read(double *total_ms, int *launches);
/* Select the SYMV/HEMV streaming kernel: -1 (default) = per-precision */
/* choice from the empirical tuning, 1 = TMA-fed warp-specialised      */
/* pipeline whenever the operand allows it (column stride a multiple   */
/* of 16 bytes), 0 = register-load kernel.  Returns the previous mode. */
/* (Env KBLAS_NO_TMA=1 selects 0 at load.)                             */
int kblas_set_tma(int mode);
/* Tuning hook for the TMA SYMV/HEMV kernel shape (consumer warps, */
/* columns per warp, rows per lane, pipeline stages); -1 = tuned      */
/* per-precision default.  Used by scripts/tune_symv.py; returns the  */
/* previous variant.                                                  */
int kblas_set_symv_variant(int variant);
/* Select the GEMV-N form: -1 (default) = automatic (the split form,   */
/* narrow row blocks reduced inside one kernel, for small and short    */
/* matrices; the stacked-rows stream-K form otherwise), 1 = always the */
/* split form, 0 = never, 3 = the row-owning form (kblas_gemv_ro_kernel).     */
/* Returns the previous mode.                                          */
int kblas_set_gemv_split(int mode);
/* Row-owning GEMV-N configuration 0..7 (tuning hook; -1 = from the     */
/* tuning table).  Returns the previous value.                          */
int kblas_set_gemv_rowown(int cfg);
/* Tuning hook for the stacked GEMV-N and the GEMV-T/C kernel shapes     */
/* (warps, columns per warp, vectors per lane, CTAs per SM); 0 = tuned   */
/* default.  Returns the previous variant.                               */
int kblas_set_gemv_variant(int variant);
/* Select the GEMV-T/C form: -1 (default) = automatic (column-owning    */
/* CTAs, one kernel, for operands up to max_bytes with >= 2 CTAs per SM; */
/* stream-K otherwise), 1 = always, 0 = never.  max_bytes <= 0 keeps    */
/* the current threshold.  Returns the previous mode.                   */
int kblas_set_gemv_tc(int mode, long long max_bytes);
/* Split-form GEMV-N grid: CTAs per row block sized for this many waves */
/* of the GPU (>= 1).  Returns the previous value.                      */
int kblas_set_gemv_split_waves(int waves);
/* Split-form GEMV-N cross-CTA step: -1 (default) = automatic (thread-  */
/* block clusters reduced through distributed shared memory for small  */
/* operands), 1 = always clusters, 0 = global partial slots.  Returns   */
/* the previous mode.                                                  */
int kblas_set_gemv_cluster(int mode);
/* Empirical tuning table (written by paper_1410_1726_b200/tuner.py,    */
/* the on-device replacement of the reference's analytic tuner,         */
/* tuner.py:168-235).  Calls of precision prec ('s','d','c','z') and    */
/* operation op whose order key lies in [n_lo, n_hi] run with the given  */
/* choices; the key is round(sqrt(m*n)) for GEMV and d for SYMV/HEMV.   */
/* Single-GPU calls only; an explicit kblas_set_* value wins over the    */
/* table, the table over the built-in rules.  A table form is a          */
/* preference: it is skipped (built-in rule) when the call's shape       */
/* gives too few CTAs for it, e.g. a short, wide matrix whose order key  */
/* falls into a row-owning range.  The latest matching entry             */
/* wins; an entry with the same (prec, op, n_lo, n_hi) is replaced.      */
/* The library starts with its built-in measured table (kblas_tune_defaults). */
/*   op 'n': shape 0 auto | 3 (4 warps x 4 cols x 2 vectors, 2 CTAs/SM)  */
/*           | 4 (16 x 4 x 1, 1 CTA/SM) | 5 (8 x 4 x 1, 2 CTAs/SM);       */
/*           form -1 auto | 0 stacked-rows stream-K | 1 split form with   */
/*           global partial slots | 2 split form reduced in a cluster |   */
/*           3 row-owning CTAs (shape 10..17 = its configuration: 16x4x8,  */
/*           8x4x8, 8x2x8, 8x4x16, 8x2x16, 4x4x16, 16x2x8, 8x8x8 as warps x */
/*           row lanes x columns in flight);                              */
/*           waves 0 = default, else split-form grid in waves (1..64).   */
/*   op 't'/'c': shape as for 'n' (stream-K form); form -1 auto |        */
/*           0 stream-K | 1 column-owning; waves must be 0.              */
/*   op 'l'/'u': shape -1 auto | 100 wide tiles (16 warps x 8 columns) | */
/*           103 narrow (8 x 4) | 105 mid (8 x 8, 2 CTAs/SM); form -1,   */
/*           waves 0.                                                    */
/* Returns 0, or -k for an invalid argument k.                          */
int kblas_tune_set(char prec, char op, long long n_lo, long long n_hi, int shape, int form, int waves);
/* Remove every tuning-table entry (built-in rules only). */
int kblas_tune_clear(void);
/* Replace the table by the measured B200 table built into the library  */
/* (installed at load; paper_1410_1726_b200/tuning/b200.json).  Returns  */
/* the number of entries.                                               */
int kblas_tune_defaults(void);
/* Number of tuning-table entries. */
int kblas_tune_count(void);
/* Read entry i (0-based) of the tuning table; -1 if out of range. */
int kblas_tune_get(int i, char *prec, char *op, long long *n_lo, long long *n_hi, int *shape, int *form,
                   int *waves);
/* Register SYMV/HEMV kernel: orders up to max_order use narrow column */
/* tiles (more work items for small operands).  Returns the previous   */
/* threshold (default 2048).                                           */
int kblas_set_symv_narrow(int max_order);
/* Register SYMV/HEMV kernel, s/d/c: orders above the narrow threshold  */
/* and up to max_order use 8-warp CTAs at 2 per SM.  Returns the        */
/* previous threshold (default 12288).                                  */
int kblas_set_symv_mid(int max_order);
/* Register and TMA SYMV/HEMV kernels: work schedule.  items > 0 deals   */
/* segments of `items` consecutive row chunks to the CTAs round robin   */
/* (neighbouring CTAs stream neighbouring chunks of the same tiles);    */
/* items <= 0 gives each CTA one contiguous range (stream-K).  Returns  */
/* the previous value (default 6).                                      */
int kblas_set_symv_segment(int items);
/* Instrumentation: a device buffer of >= 3 * (CTAs) unsigned 64-bit    */
/* words, or NULL to stop.  While set, the register SYMV/HEMV kernel     */
/* writes each CTA's %globaltimer at start and end and its SM id        */
/* (3*cta, 3*cta + 1, 3*cta + 2); scripts/symv_trace.py turns them into */
/* the finish-time spread.  Only in a library built with                */
/* -DKBLAS_SYMV_TRACE=1 (KBLAS_NVCC_EXTRA); the product build returns   */
/* -1 and compiles the trace branches out of the kernel.                */
int kblas_set_symv_trace(void *dev_buf);
/* Register SYMV/HEMV kernel (orders above the mid threshold): row      */
/* chunks per CTA barrier window (1, 2 or 4; the warps' t1 partials of  */
/* a window are reduced together).  Returns the previous value (2).      */
int kblas_set_symv_window(int items);
/* Description of the last plan chosen for a call on this thread      */
/* (kernel family, grid, items, workspace bytes) as a NUL-terminated   */
/* string; for reports and tests.                                      */
const char *kblas_last_plan(void);
/* Library version string. */
const char *kblas_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KBLAS_B200_H */
