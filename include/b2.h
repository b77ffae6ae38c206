/*
 * b2.h — C ABI of the B200 map-execution backend (libb2.so).
 *
 * The reference executor is pure Python (pkg/src/sdfgkit/interp.py); this
 * ABI is what its executor contract binds to through ctypes (see
 * INTEGRATION.md).  Every entry point is `extern "C"`, takes plain pointers,
 * sizes and opaque handles (no torch types), returns 0 on success or a
 * nonzero B2_ERR_* code, and leaves a thread-local message readable through
 * b2_last_error().  Streams are CUDA stream handles passed as void* (NULL =
 * legacy default stream); device pointers are plain device addresses.
 *
 * Reference interfaces each group replaces:
 *   runtime / memory .......... Machine.prepare/outputs, interp.py:180-236
 *   JIT + launch .............. Machine.exec_map / exec_tasklet, interp.py:400-441
 *                               (tasklet bodies: texpr.evaluate, texpr.py:89-133)
 *   copy_view ................. Machine.exec_copy + TRANSPOSE, interp.py:383-398, 474-480
 *   gemm ...................... exec_library MATMUL 2D@2D, interp.py:450-460 (np.matmul)
 *   reduce .................... exec_library REDUCE, interp.py:461-473 (ufunc.reduce)
 *   graph capture ............. Machine.run state loop, interp.py:240-263
 */
#ifndef B2_H
#define B2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define B2_API __attribute__((visibility("default")))
#else
#define B2_API
#endif

#define B2_OK 0
#define B2_ERR_CUDA 1
#define B2_ERR_NVRTC 2
#define B2_ERR_ARG 3
#define B2_ERR_UNSUPPORTED 4

/* dtype codes shared with the Python host side */
#define B2_F64 0
#define B2_I64 1
#define B2_I32 2
#define B2_BOOL 3
#define B2_F32 4

/* write-conflict resolution (ir.py:72-91) */
#define B2_WCR_NONE 0
#define B2_WCR_ADD 1
#define B2_WCR_MUL 2
#define B2_WCR_MIN 3
#define B2_WCR_MAX 4

#define B2_MAX_DIMS 8

typedef struct {
  char name[128];
  int major, minor;
  int sm_count;
  int l2_bytes;
  int max_smem_optin;
  size_t total_mem;
} b2_device_info_t;

/* A strided N-d view of a container: element (i0..i{n-1}) lives at
 * base + elem_size * (offset + sum_d i_d * strides[d]). */
typedef struct {
  void *base;
  int64_t offset;
  int32_t dtype;
  int32_t ndim;
  int64_t shape[B2_MAX_DIMS];
  int64_t strides[B2_MAX_DIMS];
} b2_view_t;

/* ---- runtime ------------------------------------------------------------ */
B2_API int b2_version(void);
B2_API const char *b2_last_error(void);
B2_API int b2_init(int device);
B2_API int b2_device_count(int *n);
B2_API int b2_device_info(int device, b2_device_info_t *out);
B2_API int b2_malloc(void **p, size_t bytes);
B2_API int b2_free(void *p);
B2_API int b2_memcpy_h2d(void *dst, const void *src, size_t bytes, void *stream);
B2_API int b2_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream);
B2_API int b2_memcpy_d2d(void *dst, const void *src, size_t bytes, void *stream);
B2_API int b2_memset(void *dst, int value, size_t bytes, void *stream);
B2_API int b2_stream_create(void **stream);
B2_API int b2_stream_destroy(void *stream);
B2_API int b2_stream_sync(void *stream);
B2_API int b2_device_sync(void);
B2_API int b2_event_create(void **ev);
B2_API int b2_event_destroy(void *ev);
B2_API int b2_event_record(void *ev, void *stream);
/* Inside a stream capture: an event-record node timestamped when the graph
 * replays (per-kernel timing of a captured trace, Machine.profile_launches). */
B2_API int b2_event_record_external(void *ev, void *stream);
B2_API int b2_event_elapsed_ms(void *start, void *end, float *ms);
/* `stream` waits for `ev` (fork/join of side streams, also inside capture). */
B2_API int b2_stream_wait_event(void *stream, void *ev);
B2_API int b2_host_register(void *p, size_t bytes);
B2_API int b2_host_unregister(void *p);
/* CUDA IPC for peer-store halos (dist.PeerHalo): the 64-byte handle of an
 * allocation, its mapping in another process on a peer GPU, unmapping.
 * Replaces the reference's simulated ISEND/IRECV copies
 * (interp.py:443-447, 483-489) when B2_SLAB_PEER=1. */
B2_API int b2_ipc_handle(void *p, void *out64);
B2_API int b2_ipc_open(const void *h64, void **p);
B2_API int b2_ipc_close(void *p);

/* ---- JIT of kernel families with inlined tasklet functors (NVRTC) ------ */
/* Compile CUDA C++ `src` for sm_100a.  On success *cubin_size is the image
 * size; call again with a buffer of that size to fetch it (cubin != NULL).
 * `log` (may be NULL) receives the NVRTC log, truncated to log_len. */
B2_API int b2_jit_compile(const char *src, const char *name, const char *const *opts, int nopts,
                   void *cubin, size_t *cubin_size, char *log, size_t log_len);
B2_API int b2_module_load(const void *image, void **module);
B2_API int b2_module_unload(void *module);
B2_API int b2_module_function(void *module, const char *kernel, void **fn);
B2_API int b2_func_set_max_smem(void *fn, int bytes);
/* Launch `fn` whose single by-value parameter is the byte blob `args`. */
B2_API int b2_launch(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by,
              unsigned bz, unsigned smem, void *stream, const void *args, size_t args_bytes);
/* Same, always with programmatic stream serialization (PDL): the kernel may
 * start before the previous one in the stream finishes and must open with
 * griddepcontrol.wait (used for fold kernels right after their producer). */
B2_API int b2_launch_pdl(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
              unsigned by, unsigned bz, unsigned smem, void *stream, const void *args,
              size_t args_bytes);
/* Same, as a cooperative launch: every CTA co-resident (kernels with grid
 * barriers, e.g. the row pass folding its partials in-kernel) or an error. */
B2_API int b2_launch_coop(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
              unsigned by, unsigned bz, unsigned smem, void *stream, const void *args,
              size_t args_bytes);
/* Number of kernel launches issued through this library so far. */
B2_API int64_t b2_launch_count(void);

/* ---- CUDA-graph capture of a whole state-machine trace ------------------ */
B2_API int b2_capture_begin(void *stream);
B2_API int b2_capture_end(void *stream, void **graph_exec);
B2_API int b2_graph_launch(void *graph_exec, void *stream);
B2_API int b2_graph_destroy(void *graph_exec);
/* Device-side branch in a capture (Machine.eval_cond on a 0-d container,
 * interp.py:265-274, without a host round trip): adds a CUDA conditional
 * IF/ELSE node whose predicate is *flag != 0 at graph run time; the caller
 * captures body_then / body_else on another stream with
 * b2_capture_body_begin/end, then continues after the node with
 * b2_capture_if_end. */
B2_API int b2_capture_if_begin(void *stream, const int *flag, void **node, void **body_then,
                        void **body_else);
B2_API int b2_capture_if_end(void *stream, void *node);
B2_API int b2_capture_body_begin(void *body_stream, void *body_graph);
B2_API int b2_capture_body_end(void *body_stream);
/* dev[0..3] += a0..a3 (interpreter counters accumulated by branch bodies) */
B2_API int b2_counters_add(long long *dev, long long a0, long long a1, long long a2, long long a3,
                    void *stream);

/* TMA descriptor (CUtensorMap, 128 bytes written to out128) for a row-major
 * f64 tensor: dims / box innermost first, no swizzle, zeros outside.  Used by
 * the tma3 stencil sweeps (map scopes of interp.py:420-441 whose inputs are
 * read at constant offsets), passed ahead of the kernel's argument words. */
B2_API int b2_tensor_map_f64(void *out128, const void *base, int rank, const uint64_t *dims,
                             const uint32_t *box);

/* ---- ahead-of-time library kernels ------------------------------------- */
/* dst[flat] (wcr)= convert(src[flat]) over the row-major flattening of both
 * views (equal element counts).  Implements access->access copies with
 * reshape (interp.py:383-398) and TRANSPOSE (interp.py:474-480). */
B2_API int b2_copy_view(const b2_view_t *dst, const b2_view_t *src, int wcr, void *stream);
/* Fill a view with a scalar (given as double). */
B2_API int b2_fill_view(const b2_view_t *dst, double value, void *stream);
/* C[i*rsc + j*csc] (wcr)= sum_k A[i*rsa+k*csa] B[k*rsb+j*csb]  (f64 2D@2D) */
B2_API int b2_gemm_f64(int64_t M, int64_t N, int64_t K, const double *A, int64_t rsa, int64_t csa,
                const double *B, int64_t rsb, int64_t csb, double *C, int64_t rsc,
                int64_t csc, int wcr, void *stream);
/* f32 GEMM with f32 accumulation (SUMMA f32 config). */
B2_API int b2_gemm_f32(int64_t M, int64_t N, int64_t K, const float *A, int64_t rsa, int64_t csa,
                const float *B, int64_t rsb, int64_t csb, float *C, int64_t rsc,
                int64_t csc, int wcr, void *stream);
/* f32 GEMM, f64 products and accumulation (DMMA), one rounding to f32:
 * element-wise within rtol 1e-5 of the f64 product at any K.  Row-major
 * A (M x K, row stride rsa), B (K x N), C (M x N); wcr NONE or ADD. */
B2_API int b2_gemm_f32_f64acc(int64_t M, int64_t N, int64_t K, const float *A, int64_t rsa,
                              const float *B, int64_t rsb, float *C, int64_t rsc, int wcr,
                              void *stream);
/* 3xTF32 operands split once (SUMMA f32): A' (M x Kp) / B'^T (N x Kp) in the
 * CTA-pair kernel's two-segment layout, Kp = b2_tf32_split_cols(K); then
 * C (=|+=) A @ B from the split operands.  A k-panel of a split operand is
 * itself a split operand of the panel's K when panels are 32-aligned. */
B2_API int64_t b2_tf32_split_cols(int64_t K);
B2_API int b2_tf32_split_a(const float *A, int64_t lda, int64_t M, int64_t K, float *Ap,
                           void *stream);
B2_API int b2_tf32_split_bt(const float *B, int64_t ldb, int64_t K, int64_t N, float *Bt,
                            void *stream);
B2_API int b2_gemm_f32_presplit(int64_t M, int64_t N, int64_t K, const float *Ap, const float *Bt,
                                float *C, int64_t ldc, int accumulate, void *stream);
/* out (wcr)= op-reduce of `in` over the dims flagged in axes_mask (bit d),
 * output enumerated row-major over the kept dims (ufunc.reduce semantics). */
B2_API int b2_reduce(const b2_view_t *out, const b2_view_t *in, unsigned axes_mask, int op, int wcr,
              void *stream);

/* ---- multi-GPU: NCCL on the executor stream (graph-capturable) ----------
 * Replaces the simulated ISEND/IRECV/WAITALL/BCAST/DIST_MATMUL events of the
 * reference's rank simulator (interp.py:443-447, 483-489). */
typedef struct {
  void *ptr;
  size_t bytes;
  int peer;
  int send; /* 1 = send, 0 = receive */
} b2_p2p_t;
B2_API int b2_nccl_unique_id(void *out128);
B2_API int b2_nccl_init(int nranks, int rank, const void *id128, void **comm);
B2_API int b2_nccl_destroy(void *comm);
/* One grouped batch of point-to-point transfers (halo exchange). */
B2_API int b2_nccl_group_p2p(void *comm, int n, const b2_p2p_t *ops, void *stream);
B2_API int b2_nccl_bcast(void *comm, void *buf, size_t bytes, int root, void *stream);
/* In-place Allreduce of a WCR-reduced f64 output (op = B2_WCR_*). */
B2_API int b2_nccl_allreduce_f64(void *comm, double *buf, size_t count, int wcr, void *stream);

/* Matrix-vector products (np.matmul 2D@1D / 1D@2D) and their fusions
 * (gemver / atax / bicg) are JIT "rowpass" family kernels: see
 * paper_2107_00555_b200/csrc/families/rowpass.cuh. */

#ifdef __cplusplus
}
#endif
#endif /* B2_H */
