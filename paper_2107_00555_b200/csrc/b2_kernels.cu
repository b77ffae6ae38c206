// b2_kernels.cu — ahead-of-time library kernels of libb2.so (sm_100a).
//
//   b2_copy_view / b2_fill_view : access->access copies with reshape
//       (interp.py:383-398), TRANSPOSE (interp.py:474-480), zero/const fills
//   b2_reduce                   : REDUCE library node (interp.py:461-473)
//   b2_gemm_f64 / b2_gemm_f32   : MATMUL 2D@2D (interp.py:450-460)
//
// Elementwise/stencil/WCR maps and the BLAS-2 passes are JIT families (see
// csrc/families/*.cuh) because their bodies are the program's tasklets.

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "b2.h"
#include "b2_internal.h"

namespace {

constexpr int kMaxDims = B2_MAX_DIMS;

struct ViewDev {
  char *base;
  int64_t offset;
  int32_t esize;
  int32_t ndim;
  int64_t shape[kMaxDims];
  int64_t strides[kMaxDims];
};

int esize_of(int dt) {
  switch (dt) {
    case B2_F64:
    case B2_I64:
      return 8;
    case B2_I32:
    case B2_F32:
      return 4;
    case B2_BOOL:
      return 1;
  }
  return 0;
}

ViewDev to_dev(const b2_view_t *v) {
  ViewDev d;
  d.base = (char *)v->base;
  d.offset = v->offset;
  d.esize = esize_of(v->dtype);
  d.ndim = v->ndim;
  for (int i = 0; i < kMaxDims; ++i) {
    d.shape[i] = i < v->ndim ? v->shape[i] : 1;
    d.strides[i] = i < v->ndim ? v->strides[i] : 0;
  }
  return d;
}

int64_t numel(const b2_view_t *v) {
  int64_t n = 1;
  for (int i = 0; i < v->ndim; ++i) n *= v->shape[i];
  return n;
}

__device__ __forceinline__ int64_t flat_to_offset(const ViewDev &v, int64_t flat) {
  int64_t off = v.offset;
  for (int d = v.ndim - 1; d >= 0; --d) {
    int64_t s = v.shape[d];
    int64_t i = flat % s;
    flat /= s;
    off += i * v.strides[d];
  }
  return off;
}

template <typename T>
__device__ __forceinline__ T load_as(const char *p, int dt);

template <typename T>
__device__ __forceinline__ T load_as(const char *p, int dt) {
  switch (dt) {
    case B2_F64:
      return (T)(*(const double *)p);
    case B2_I64:
      return (T)(*(const long long *)p);
    case B2_I32:
      return (T)(*(const int *)p);
    case B2_F32:
      return (T)(*(const float *)p);
    default:
      return (T)(*(const bool *)p);
  }
}

// numpy.minimum / maximum propagate NaN (ir.py:80-87 uses np.minimum/maximum)
__device__ __forceinline__ double np_min(double a, double b) {
  return (isnan(a) || a < b) ? a : b;
}
__device__ __forceinline__ double np_max(double a, double b) {
  return (isnan(a) || a > b) ? a : b;
}

__device__ __forceinline__ double apply_wcr(int wcr, double old, double v) {
  switch (wcr) {
    case B2_WCR_ADD:
      return old + v;
    case B2_WCR_MUL:
      return old * v;
    case B2_WCR_MIN:
      return np_min(old, v);
    case B2_WCR_MAX:
      return np_max(old, v);
  }
  return v;
}

__device__ __forceinline__ void store_from_double(char *p, int dt, double v, int wcr, bool is_int,
                                                  long long iv) {
  switch (dt) {
    case B2_F64: {
      double *q = (double *)p;
      *q = wcr ? apply_wcr(wcr, *q, v) : v;
      break;
    }
    case B2_F32: {
      float *q = (float *)p;
      *q = wcr ? (float)apply_wcr(wcr, (double)*q, v) : (float)v;
      break;
    }
    case B2_I64: {
      long long *q = (long long *)p;
      long long nv = is_int ? iv : (long long)v;
      if (wcr == B2_WCR_ADD) nv = *q + nv;
      else if (wcr == B2_WCR_MUL) nv = *q * nv;
      else if (wcr == B2_WCR_MIN) nv = nv < *q ? nv : *q;
      else if (wcr == B2_WCR_MAX) nv = nv > *q ? nv : *q;
      *q = nv;
      break;
    }
    case B2_I32: {
      int *q = (int *)p;
      long long nv = is_int ? iv : (long long)v;
      if (wcr == B2_WCR_ADD) nv = *q + nv;
      else if (wcr == B2_WCR_MUL) nv = *q * nv;
      else if (wcr == B2_WCR_MIN) nv = nv < *q ? nv : *q;
      else if (wcr == B2_WCR_MAX) nv = nv > *q ? nv : *q;
      *q = (int)nv;
      break;
    }
    default: {
      bool *q = (bool *)p;
      bool nv = is_int ? (iv != 0) : (v != 0.0);
      if (wcr == B2_WCR_ADD) nv = *q || nv;
      else if (wcr == B2_WCR_MUL) nv = *q && nv;
      *q = nv;
    }
  }
}

__global__ void copy_view_kernel(ViewDev dst, int ddt, ViewDev src, int sdt, int64_t n, int wcr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const char *sp = src.base + flat_to_offset(src, i) * src.esize;
    char *dp = dst.base + flat_to_offset(dst, i) * dst.esize;
    bool sint = (sdt == B2_I64 || sdt == B2_I32 || sdt == B2_BOOL);
    if (sint) {
      long long v = load_as<long long>(sp, sdt);
      store_from_double(dp, ddt, (double)v, wcr, true, v);
    } else {
      double v = load_as<double>(sp, sdt);
      store_from_double(dp, ddt, v, wcr, false, 0);
    }
  }
}

__global__ void fill_view_kernel(ViewDev dst, int ddt, double value, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    char *dp = dst.base + flat_to_offset(dst, i) * dst.esize;
    store_from_double(dp, ddt, value, 0, false, 0);
  }
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

bool contiguous(const b2_view_t *v) {
  int64_t s = 1;
  for (int d = v->ndim - 1; d >= 0; --d) {
    if (v->shape[d] != 1 && v->strides[d] != s) return false;
    s *= v->shape[d];
  }
  return true;
}

// ---------------------------------------------------------------------------
// reduce: one block per output element (grid-stride over outputs).

template <typename T>
__device__ __forceinline__ T red_op(int op, T a, T b);
template <>
__device__ __forceinline__ double red_op<double>(int op, double a, double b) {
  return apply_wcr(op, a, b);
}
template <>
__device__ __forceinline__ long long red_op<long long>(int op, long long a, long long b) {
  switch (op) {
    case B2_WCR_ADD:
      return a + b;
    case B2_WCR_MUL:
      return a * b;
    case B2_WCR_MIN:
      return b < a ? b : a;
    default:
      return b > a ? b : a;
  }
}

template <typename T, bool IsInt>
__global__ void reduce_kernel(ViewDev out, int odt, ViewDev kept, ViewDev red, const char *base,
                              int idt, int64_t nout, int64_t nred, int op, int wcr, T identity) {
  __shared__ T sm[32];
  __shared__ int smh[32];
  const int lane = threadIdx.x & 31;
  for (int64_t o = blockIdx.x; o < nout; o += gridDim.x) {
    int64_t kbase = flat_to_offset(kept, o);
    T acc = identity;
    bool has = false;
    for (int64_t r = threadIdx.x; r < nred; r += blockDim.x) {
      int64_t off = kbase + flat_to_offset(red, r);
      T v = load_as<T>(base + off * red.esize, idt);
      acc = has ? red_op<T>(op, acc, v) : v;
      has = true;
    }
    // warp + block combine in a fixed order (deterministic)
    for (int s = 16; s > 0; s >>= 1) {
      T other = __shfl_down_sync(0xffffffffu, acc, s);
      int oh = __shfl_down_sync(0xffffffffu, (int)has, s);
      if (lane + s < 32 && oh) {
        acc = has ? red_op<T>(op, acc, other) : other;
        has = true;
      }
    }
    int w = threadIdx.x >> 5;
    if (lane == 0) {
      sm[w] = acc;
      smh[w] = has;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int nw = (blockDim.x + 31) >> 5;
      T tot = identity;
      bool th = false;
      for (int i = 0; i < nw; ++i)
        if (smh[i]) {
          tot = th ? red_op<T>(op, tot, sm[i]) : sm[i];
          th = true;
        }
      char *dp = out.base + flat_to_offset(out, o) * out.esize;
      store_from_double(dp, odt, (double)tot, wcr, IsInt, (long long)tot);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// GEMM: register-blocked SIMT kernel (DFMA for f64, FFMA for f32).
// Tile BM x BN x BK, 256 threads, each thread TM x TN outputs.  Operands are
// arbitrary 2-D strided views (np.matmul on squeezed memlet views).

template <typename T, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__(256) gemm_kernel(int64_t M, int64_t N, int64_t K, const T *A,
                                                   int64_t rsa, int64_t csa, const T *B,
                                                   int64_t rsb, int64_t csb, T *C, int64_t rsc,
                                                   int64_t csc, int wcr) {
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN);
  const int ty = tid / (BN / TN);
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    for (int i = tid; i < BM * BK; i += 256) {
      int mm, kk;
      if (csa == 1) {
        kk = i % BK;
        mm = i / BK;
      } else {
        mm = i % BM;
        kk = i / BM;
      }
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[gm * rsa + gk * csa] : T(0);
    }
    for (int i = tid; i < BN * BK; i += 256) {
      int nn, kk;
      if (csb == 1) {
        nn = i % BN;
        kk = i / BN;
      } else {
        kk = i % BK;
        nn = i / BK;
      }
      int64_t gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? B[gk * rsb + gn * csb] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + j * (BN / TN)];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int64_t gn = n0 + tx + j * (BN / TN);
      if (gn >= N) continue;
      T *cp = C + gm * rsc + gn * csc;
      *cp = (wcr == B2_WCR_ADD) ? (*cp + acc[i][j]) : acc[i][j];
    }
  }
}

template <typename T>
int gemm_impl(int64_t M, int64_t N, int64_t K, const T *A, int64_t rsa, int64_t csa, const T *B,
              int64_t rsb, int64_t csb, T *C, int64_t rsc, int64_t csc, int wcr, void *stream) {
  if (wcr != B2_WCR_NONE && wcr != B2_WCR_ADD)
    return b2_fail(B2_ERR_UNSUPPORTED, "gemm: only add WCR is supported");
  if (M <= 0 || N <= 0) return B2_OK;
  constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  B2_CLEAR_ERROR();
  gemm_kernel<T, BM, BN, BK, TM, TN><<<grid, 256, 0, (cudaStream_t)stream>>>(
      M, N, K, A, rsa, csa, B, rsb, csb, C, rsc, csc, wcr);
  B2_LAUNCH_CHECK("gemm launch");
  return B2_OK;
}

}  // namespace

extern "C" int b2_copy_view(const b2_view_t *dst, const b2_view_t *src, int wcr, void *stream) {
  int64_t n = numel(dst);
  if (n != numel(src)) return b2_fail(B2_ERR_ARG, "copy_view: element counts differ");
  if (n == 0) return B2_OK;
  if (!wcr && dst->dtype == src->dtype && contiguous(dst) && contiguous(src)) {
    int es = esize_of(dst->dtype);
    return b2_cuda_check(cudaMemcpyAsync((char *)dst->base + dst->offset * es,
                                         (const char *)src->base + src->offset * es, n * es,
                                         cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
                         "copy_view memcpy");
  }
  B2_CLEAR_ERROR();
  copy_view_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      to_dev(dst), dst->dtype, to_dev(src), src->dtype, n, wcr);
  B2_LAUNCH_CHECK("copy_view launch");
  return B2_OK;
}

extern "C" int b2_fill_view(const b2_view_t *dst, double value, void *stream) {
  int64_t n = numel(dst);
  if (n == 0) return B2_OK;
  B2_CLEAR_ERROR();
  fill_view_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(to_dev(dst), dst->dtype,
                                                                        value, n);
  B2_LAUNCH_CHECK("fill_view launch");
  return B2_OK;
}

extern "C" int b2_reduce(const b2_view_t *out, const b2_view_t *in, unsigned axes_mask, int op,
                         int wcr, void *stream) {
  b2_view_t kept = *in, red = *in;
  kept.ndim = red.ndim = 0;
  kept.offset = red.offset = 0;
  int64_t nout = 1, nred = 1;
  for (int d = 0; d < in->ndim; ++d) {
    if (axes_mask & (1u << d)) {
      red.shape[red.ndim] = in->shape[d];
      red.strides[red.ndim++] = in->strides[d];
      nred *= in->shape[d];
    } else {
      kept.shape[kept.ndim] = in->shape[d];
      kept.strides[kept.ndim++] = in->strides[d];
      nout *= in->shape[d];
    }
  }
  kept.offset = in->offset;
  if (nout != numel(out)) return b2_fail(B2_ERR_ARG, "reduce: output size mismatch");
  if (nout == 0) return B2_OK;
  unsigned grid = (unsigned)(nout < 148 * 16 ? nout : 148 * 16);
  int threads = nred >= 256 ? 256 : 32;
  bool isint = (in->dtype == B2_I64 || in->dtype == B2_I32 || in->dtype == B2_BOOL);
  if (isint) {
    long long ident = op == B2_WCR_MUL ? 1 : (op == B2_WCR_MIN ? INT64_MAX : (op == B2_WCR_MAX ? INT64_MIN : 0));
    B2_CLEAR_ERROR();
    reduce_kernel<long long, true><<<grid, threads, 0, (cudaStream_t)stream>>>(
        to_dev(out), out->dtype, to_dev(&kept), to_dev(&red), (const char *)in->base,
        in->dtype, nout, nred, op, wcr, ident);
  } else {
    double ident = op == B2_WCR_MUL ? 1.0 : (op == B2_WCR_MIN ? INFINITY : (op == B2_WCR_MAX ? -INFINITY : 0.0));
    B2_CLEAR_ERROR();
    reduce_kernel<double, false><<<grid, threads, 0, (cudaStream_t)stream>>>(
        to_dev(out), out->dtype, to_dev(&kept), to_dev(&red), (const char *)in->base,
        in->dtype, nout, nred, op, wcr, ident);
  }
  B2_LAUNCH_CHECK("reduce launch");
  return B2_OK;
}

int b2_dgemm_dmma(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                  int64_t ldb, double *C, int64_t rsc, int64_t csc, int accumulate,
                  void *stream);
int b2_sgemm_128(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                 int64_t ldb, float *C, int64_t ldc, int accumulate, void *stream);
int b2_sgemm_tc(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                int64_t ldb, float *C, int64_t ldc, int accumulate, void *stream);
int b2_sgemm_tc_enabled();

extern "C" int b2_gemm_f64(int64_t M, int64_t N, int64_t K, const double *A, int64_t rsa,
                           int64_t csa, const double *B, int64_t rsb, int64_t csb, double *C,
                           int64_t rsc, int64_t csc, int wcr, void *stream) {
  // FP64 tensor cores (DMMA) for row-major operands of non-trivial size
  if (csa == 1 && csb == 1 && (wcr == B2_WCR_NONE || wcr == B2_WCR_ADD) && M >= 16 &&
      N >= 16 && K >= 4 && M * N * K >= (1LL << 18))
    return b2_dgemm_dmma(M, N, K, A, rsa, B, rsb, C, rsc, csc, wcr == B2_WCR_ADD, stream);
  return gemm_impl<double>(M, N, K, A, rsa, csa, B, rsb, csb, C, rsc, csc, wcr, stream);
}

extern "C" int b2_gemm_f32(int64_t M, int64_t N, int64_t K, const float *A, int64_t rsa,
                           int64_t csa, const float *B, int64_t rsb, int64_t csb, float *C,
                           int64_t rsc, int64_t csc, int wcr, void *stream) {
  // tcgen05 (3xTF32) for large problems: the split pass re-lays both operands
  if (csa == 1 && csb == 1 && csc == 1 && (wcr == B2_WCR_NONE || wcr == B2_WCR_ADD) &&
      M >= 128 && N >= 256 && K >= 32 && M * N * K >= (1LL << 27) && b2_sgemm_tc_enabled())
    return b2_sgemm_tc(M, N, K, A, rsa, B, rsb, C, rsc, wcr == B2_WCR_ADD, stream);
  if (csa == 1 && csb == 1 && csc == 1 && (wcr == B2_WCR_NONE || wcr == B2_WCR_ADD) &&
      rsa % 4 == 0 && rsb % 4 == 0 && (((uintptr_t)A | (uintptr_t)B) & 15) == 0 &&
      M * N * K >= (1LL << 18))
    return b2_sgemm_128(M, N, K, A, rsa, B, rsb, C, rsc, wcr == B2_WCR_ADD, stream);
  return gemm_impl<float>(M, N, K, A, rsa, csa, B, rsb, csb, C, rsc, csc, wcr, stream);
}
