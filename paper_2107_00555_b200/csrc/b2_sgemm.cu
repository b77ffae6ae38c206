// b2_sgemm.cu — FP32 GEMM (FFMA) for the SUMMA f32 configuration.
//
// The reference has no float32 type; the f32 MatMul config
// runs through the C ABI (b2_gemm_f32) with fp32 accumulation (rtol 1e-5).
// CTA tile 128x128x8, 256 threads, 8x8 outputs per thread (two 4-wide
// fragments per dimension so the float4 shared loads stay conflict-free),
// double-buffered shared tiles filled from registers while the previous tile
// is consumed.  Row-major A and B with dimensions that are multiples of 4
// take this path; everything else uses the generic SIMT kernel.

#include <cuda_runtime.h>
#include <stdint.h>

#include "b2.h"
#include "b2_internal.h"

namespace {

constexpr int BM = 128, BN = 128, BK = 8;

__global__ void __launch_bounds__(256, 2)
    sgemm_128(int64_t M, int64_t N, int64_t K, const float *__restrict__ A, int64_t lda,
              const float *__restrict__ B, int64_t ldb, float *__restrict__ C, int64_t ldc,
              int accumulate) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 thread grid
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  // global -> register staging: A tile 128x8 (one float4 of a row per thread),
  // B tile 8x128 (one float4 of a row per thread)
  const int ar = tid >> 1, ac = (tid & 1) * 4;
  const int br = tid >> 5, bc = (tid & 31) * 4;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  auto load_a = [&](int64_t k0) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t gm = m0 + ar, gk = k0 + ac;
    if (gm < M && gk + 3 < K) v = *reinterpret_cast<const float4 *>(A + gm * lda + gk);
    else if (gm < M) {
      float t[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) t[e] = gk + e < K ? A[gm * lda + gk + e] : 0.f;
      v = make_float4(t[0], t[1], t[2], t[3]);
    }
    return v;
  };
  auto load_b = [&](int64_t k0) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t gk = k0 + br, gn = n0 + bc;
    if (gk < K && gn + 3 < N) v = *reinterpret_cast<const float4 *>(B + gk * ldb + gn);
    else if (gk < K) {
      float t[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) t[e] = gn + e < N ? B[gk * ldb + gn + e] : 0.f;
      v = make_float4(t[0], t[1], t[2], t[3]);
    }
    return v;
  };
  auto store = [&](int s, float4 a, float4 b) {
    As[s][ac + 0][ar] = a.x;
    As[s][ac + 1][ar] = a.y;
    As[s][ac + 2][ar] = a.z;
    As[s][ac + 3][ar] = a.w;
    *reinterpret_cast<float4 *>(&Bs[s][br][bc]) = b;
  };

  store(0, load_a(0), load_b(0));
  __syncthreads();
  const int64_t ktiles = (K + BK - 1) / BK;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int s = (int)(kt & 1);
    float4 na, nb;
    const bool more = kt + 1 < ktiles;
    if (more) {
      na = load_a((kt + 1) * BK);
      nb = load_b((kt + 1) * BK);
    }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4 *>(&As[s][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&As[s][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[s][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[s][k][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) store(s ^ 1, na, nb);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gn >= N) continue;
      float *cp = C + gm * ldc + gn;
      *cp = accumulate ? (*cp + acc[i][j]) : acc[i][j];
    }
  }
}

__global__ void widen_f32(const float *__restrict__ src, int64_t rows, int64_t cols, int64_t ld,
                          double *__restrict__ dst) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[i] = (double)src[r * ld + c];
  }
}

__global__ void narrow_f64(const double *__restrict__ src, int64_t rows, int64_t cols,
                           float *__restrict__ dst, int64_t ld, int accumulate) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    float *d = dst + r * ld + c;
    // the f32 += is the caller's WCR add, applied to the rounded product
    *d = accumulate ? *d + (float)src[i] : (float)src[i];
  }
}

double *g_wide = nullptr;
size_t g_wide_bytes = 0;

}  // namespace

int b2_dgemm_dmma(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                  int64_t ldb, double *C, int64_t rsc, int64_t csc, int accumulate,
                  void *stream);

// f32 operands, f64 products and accumulation on the DMMA path, one
// rounding to f32 at the end: the accurate f32 MatMul (element-wise within
// rtol 1e-5 of the f64 product at K = 16384, where any fp32-accumulating
// GEMM — the 3xTF32 kernel, the host's sgemm — is not).  Row-major operands.
extern "C" int b2_gemm_f32_f64acc(int64_t M, int64_t N, int64_t K, const float *A, int64_t rsa,
                                  const float *B, int64_t rsb, float *C, int64_t rsc, int wcr,
                                  void *stream) {
  if (wcr != B2_WCR_NONE && wcr != B2_WCR_ADD)
    return b2_fail(B2_ERR_UNSUPPORTED, "b2_gemm_f32_f64acc: wcr %d", wcr);
  const size_t need = (size_t)(M * K + K * N + M * N) * sizeof(double);
  if (need > g_wide_bytes) {
    if (g_wide) cudaFree(g_wide);
    g_wide = nullptr;
    g_wide_bytes = 0;
    int rc = b2_cuda_check(cudaMalloc(&g_wide, need), "f64 workspace");
    if (rc) return rc;
    g_wide_bytes = need;
  }
  double *a = g_wide, *b = g_wide + M * K, *c = b + K * N;
  cudaStream_t st = (cudaStream_t)stream;
  B2_CLEAR_ERROR();
  widen_f32<<<148 * 8, 256, 0, st>>>(A, M, K, rsa, a);
  widen_f32<<<148 * 8, 256, 0, st>>>(B, K, N, rsb, b);
  B2_LAUNCH_CHECK("widen");
  int rc = b2_dgemm_dmma(M, N, K, a, K, b, N, c, N, 1, 0, stream);
  if (rc) return rc;
  narrow_f64<<<148 * 8, 256, 0, st>>>(c, M, N, C, rsc, wcr == B2_WCR_ADD);
  B2_LAUNCH_CHECK("narrow");
  return B2_OK;
}

int b2_sgemm_128(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                 int64_t ldb, float *C, int64_t ldc, int accumulate, void *stream) {
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  B2_CLEAR_ERROR();
  sgemm_128<<<grid, 256, 0, (cudaStream_t)stream>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate);
  B2_LAUNCH_CHECK("sgemm launch");
  return B2_OK;
}
