// b2_dgemm.cu — FP64 tensor-core GEMM for the MATMUL library node (2D@2D,
// np.matmul semantics, pkg/src/sdfgkit/interp.py:450-460) on sm_100a.
//
// Blackwell has no tcgen05 kind for f64, so the FP64 tensor
// path is DMMA: mma.sync.m16n8k4.f64.  CTA tile 128x128xBK (BK = 32, B2_DGEMM_BK=16 for the 16-deep stages), 8 warps (2 x 4),
// warp tile 64x32 (4 x 4 m16n8 accumulators = 64 doubles per thread), operand
// tiles staged through a 3-stage cp.async shared-memory ring.  Shared layouts
// are padded so every fragment load is exactly two wavefronts (conflict-free):
//   As[m][BK + 4]  (a0 = A[g][t], a1 = A[g + 8][t]; rows 160 B apart)
//   Bs[k][BN + 8]  (b0 = B[t][g];                   rows 1088 B apart)
// Requires row-major A and B (unit column stride); other layouts use the
// SIMT kernel in b2_kernels.cu.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "b2.h"
#include "b2_internal.h"

namespace {

constexpr int BM = 128, BN = 128, STAGES = 3;
constexpr int APAD = 4, BPAD = 8;
constexpr int BS_STRIDE = BN + BPAD;   // 136 doubles
// k depth of one pipeline stage: BK = 16 (113 KB of stages) or 32 (215 KB;
// half the barriers per flop)
template <int BK>
struct Tile {
  static constexpr int AS_STRIDE = BK + APAD;
  static constexpr int AS_TILE = BM * AS_STRIDE;
  static constexpr int BS_TILE = BK * BS_STRIDE;
  static constexpr int SMEM_BYTES = STAGES * (AS_TILE + BS_TILE) * 8;
};

__device__ __forceinline__ void cp8(double *smem, const double *g, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g),
               "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp16(double *smem, const double *g, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

template <bool VEC, int BK>
__device__ __forceinline__ void load_tiles(double *As, double *Bs, const double *A, int64_t lda,
                                           const double *B, int64_t ldb, int64_t M, int64_t N,
                                           int64_t K, int64_t m0, int64_t n0, int64_t k0) {
  constexpr int AS_STRIDE = Tile<BK>::AS_STRIDE;
  const int tid = threadIdx.x;
  if (VEC) {
    // A: 128 rows x BK k in chunks of 2 doubles
#pragma unroll
    for (int i = 0; i < BK / 4; ++i) {
      const int c = tid + i * 256;
      const int r = c / (BK / 2), kk = (c % (BK / 2)) * 2;
      const int64_t gm = m0 + r, gk = k0 + kk;
      int bytes = 0;
      if (gm < M) bytes = gk + 1 < K ? 16 : (gk < K ? 8 : 0);
      cp16(As + r * AS_STRIDE + kk, bytes ? A + gm * lda + gk : A, bytes);
    }
    // B: BK k x 128 cols in chunks of 2 doubles
#pragma unroll
    for (int i = 0; i < BK / 4; ++i) {
      const int c = tid + i * 256;
      const int kk = c >> 6, nn = (c & 63) * 2;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      int bytes = 0;
      if (gk < K) bytes = gn + 1 < N ? 16 : (gn < N ? 8 : 0);
      cp16(Bs + kk * BS_STRIDE + nn, bytes ? B + gk * ldb + gn : B, bytes);
    }
  } else {
#pragma unroll
    for (int i = 0; i < BK / 2; ++i) {
      const int c = tid + i * 256;
      const int r = c / BK, kk = c % BK;
      const int64_t gm = m0 + r, gk = k0 + kk;
      const bool ok = gm < M && gk < K;
      cp8(As + r * AS_STRIDE + kk, ok ? A + gm * lda + gk : A, ok);
    }
#pragma unroll
    for (int i = 0; i < BK / 2; ++i) {
      const int c = tid + i * 256;
      const int kk = c >> 7, nn = c & 127;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      const bool ok = gk < K && gn < N;
      cp8(Bs + kk * BS_STRIDE + nn, ok ? B + gk * ldb + gn : B, ok);
    }
  }
}

template <bool VEC, int BK>
__global__ void __launch_bounds__(256, 1)
    dgemm_dmma(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
               const double *__restrict__ B, int64_t ldb, double *__restrict__ C, int64_t rsc,
               int64_t csc, int accumulate, int num_m, int num_n, int group_m) {
  constexpr int AS_STRIDE = Tile<BK>::AS_STRIDE, AS_TILE = Tile<BK>::AS_TILE,
                BS_TILE = Tile<BK>::BS_TILE;
  extern __shared__ __align__(16) double smem[];
  double *As = smem;
  double *Bs = smem + STAGES * AS_TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
  // grouped rasterisation: resident CTAs cover a group_m-tall band of tiles
  const int pid = blockIdx.x, per_group = group_m * num_n;
  const int first_m = (pid / per_group) * group_m;
  const int gsize = num_m - first_m < group_m ? num_m - first_m : group_m;
  const int64_t m0 = (int64_t)(first_m + (pid % per_group) % gsize) * BM;
  const int64_t n0 = (int64_t)((pid % per_group) / gsize) * BN;
  const int ktiles = (int)((K + BK - 1) / BK);

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      load_tiles<VEC, BK>(As + s * AS_TILE, Bs + s * BS_TILE, A, lda, B, ldb, M, N, K, m0, n0,
                      (int64_t)s * BK);
    commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int pre = kt + STAGES - 1;
    if (pre < ktiles) {
      const int ps = pre % STAGES;
      load_tiles<VEC, BK>(As + ps * AS_TILE, Bs + ps * BS_TILE, A, lda, B, ldb, M, N, K, m0, n0,
                      (int64_t)pre * BK);
    }
    commit();
    wait_group<STAGES - 1>();
    __syncthreads();
    const double *as = As + (kt % STAGES) * AS_TILE;
    const double *bs = Bs + (kt % STAGES) * BS_TILE;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a[4][2], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i][0] = as[(wm + i * 16 + g) * AS_STRIDE + k4 + t];
        a[i][1] = as[(wm + i * 16 + g + 8) * AS_STRIDE + k4 + t];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[(k4 + t) * BS_STRIDE + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncthreads();
  }
  // epilogue: c0,c1 at (g, 2t..2t+1); c2,c3 at (g + 8, 2t..2t+1)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gm = m0 + wm + i * 16 + g + h * 8;
        if (gm >= M) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t gn = n0 + wn + j * 8 + 2 * t + e;
          if (gn >= N) continue;
          double *cp = C + gm * rsc + gn * csc;
          const double v = acc[i][j][h * 2 + e];
          *cp = accumulate ? (*cp + v) : v;
        }
      }
}

}  // namespace

// Called from b2_gemm_f64 for row-major operands; returns B2_ERR_UNSUPPORTED
// when the layout does not qualify so the caller falls back.
int b2_dgemm_dmma(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                  int64_t ldb, double *C, int64_t rsc, int64_t csc, int accumulate,
                  void *stream) {
  static int bk = -1;
  if (bk < 0) {
    const char *e = getenv("B2_DGEMM_BK");
    bk = e && atoi(e) == 16 ? 16 : 32;
    cudaFuncSetAttribute(dgemm_dmma<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tile<16>::SMEM_BYTES);
    cudaFuncSetAttribute(dgemm_dmma<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tile<16>::SMEM_BYTES);
    cudaFuncSetAttribute(dgemm_dmma<true, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tile<32>::SMEM_BYTES);
    cudaFuncSetAttribute(dgemm_dmma<false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tile<32>::SMEM_BYTES);
  }
  const bool vec = (lda % 2 == 0) && (ldb % 2 == 0) && (((uintptr_t)A & 15) == 0) &&
                   (((uintptr_t)B & 15) == 0);
  const int num_m = (int)((M + BM - 1) / BM), num_n = (int)((N + BN - 1) / BN);
  static int group_m = -1;
  if (group_m < 0) {
    const char *e = getenv("B2_DGEMM_GROUP");
    group_m = e ? atoi(e) : 16;
    if (group_m < 1) group_m = 1;
  }
  const unsigned grid = (unsigned)(num_m * num_n);
  cudaStream_t st = (cudaStream_t)stream;
  B2_CLEAR_ERROR();
#define B2_DG(V, K_)                                                                   \
  dgemm_dmma<V, K_><<<grid, 256, Tile<K_>::SMEM_BYTES, st>>>(M, N, K, A, lda, B, ldb, C, rsc, \
                                                            csc, accumulate, num_m, num_n, group_m)
  if (bk == 32) {
    if (vec)
      B2_DG(true, 32);
    else
      B2_DG(false, 32);
  } else {
    if (vec)
      B2_DG(true, 16);
    else
      B2_DG(false, 16);
  }
#undef B2_DG
  B2_LAUNCH_CHECK("dgemm launch");
  return B2_OK;
}
