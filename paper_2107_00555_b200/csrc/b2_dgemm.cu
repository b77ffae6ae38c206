// b2_dgemm.cu — FP64 tensor-core GEMM for the MATMUL library node (2D@2D,
// np.matmul semantics, pkg/src/sdfgkit/interp.py:450-460) on sm_100a.
//
// Blackwell has no tcgen05 kind for f64, so the FP64 tensor
// path is DMMA: mma.sync.m16n8k4.f64.  CTA tile 128x64x16, 4 warps (2 x 2) of
// 64x32 (4 x 4 m16n8 accumulators = 64 doubles per thread), two CTAs per SM,
// operand tiles staged through a 3-stage cp.async shared-memory ring; interior
// tiles load with pointer arithmetic only.  Shared layouts are padded so every
// fragment load is conflict-free per half warp (8-byte accesses):
//   As[m][BK + 4]  (a0 = A[g][t], a1 = A[g + 8][t]; double bank 4g + t)
//   Bs[k][BN + 4]  (b0 = B[t][g];                   double bank 4t + g)
// Requires row-major A and B (unit column stride); other layouts use the
// SIMT kernel in b2_kernels.cu.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "b2.h"
#include "b2_internal.h"

namespace {

constexpr int APAD = 4, BPAD = 4;

// One tile configuration: CTA tile BM x BN x BK, warp tile WM x WN (WM / 16
// m16 fragments x WN / 8 n8 fragments), ST cp.async stages, MINB resident
// CTAs per SM (__launch_bounds__).
template <int BM_, int BN_, int BK_, int WM_, int WN_, int ST_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, ST = ST_, MINB = MINB_;
  static constexpr int NWN = BN / WN, NWARPS = (BM / WM) * (BN / WN), THREADS = NWARPS * 32;
  static constexpr int MI = WM / 16, NJ = WN / 8;
  static constexpr int AS_STRIDE = BK + APAD, BS_STRIDE = BN + BPAD;
  static constexpr int AS_TILE = BM * AS_STRIDE, BS_TILE = BK * BS_STRIDE;
  static constexpr int SMEM_BYTES = ST * (AS_TILE + BS_TILE) * 8;
};
// Default: 128x64x16, 4 warps of 64x32, three stages, two CTAs per SM — a
// CTA's barrier stalls only its own four warps while the other CTA's keep
// the DMMA pipe fed (16384^3: 35.4 TFLOP/s; 64x128 tiles 34.5, 64x64 with
// three CTAs 30.7, 64x128x32 two-stage 33.1).
using CfgTall = Cfg<128, 64, 16, 64, 32, 3, 2>;
// B2_DGEMM_CFG=wide: 128x128x32, 8 warps of 64x32, one CTA per SM (the
// round-1/2 kernel, 32.0 TFLOP/s)
using CfgWide = Cfg<128, 128, 32, 64, 32, 3, 1>;
// B2_DGEMM_CFG=tall32pf: 128x64x32 two stages with the pipelined main loop
// (35.5 TFLOP/s but 255 registers and a small spill)
using CfgTallK32 = Cfg<128, 64, 32, 64, 32, 2, 2>;

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

template <bool VEC, class C>
__device__ __forceinline__ void load_tiles(double *As, double *Bs, const double *A, int64_t lda,
                                           const double *B, int64_t ldb, int64_t M, int64_t N,
                                           int64_t K, int64_t m0, int64_t n0, int64_t k0) {
  constexpr int BK = C::BK, BN = C::BN, T = C::THREADS;
  const int tid = threadIdx.x;
  if (VEC) {
    // A: BM rows x BK k in chunks of 2 doubles
#pragma unroll
    for (int i = 0; i < C::BM * BK / 2 / T; ++i) {
      const int c = tid + i * T;
      const int r = c / (BK / 2), kk = (c % (BK / 2)) * 2;
      const int64_t gm = m0 + r, gk = k0 + kk;
      int bytes = 0;
      if (gm < M) bytes = gk + 1 < K ? 16 : (gk < K ? 8 : 0);
      cp16(As + r * C::AS_STRIDE + kk, bytes ? A + gm * lda + gk : A, bytes);
    }
    // B: BK k x BN cols in chunks of 2 doubles
#pragma unroll
    for (int i = 0; i < BK * BN / 2 / T; ++i) {
      const int c = tid + i * T;
      const int kk = c / (BN / 2), nn = (c % (BN / 2)) * 2;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      int bytes = 0;
      if (gk < K) bytes = gn + 1 < N ? 16 : (gn < N ? 8 : 0);
      cp16(Bs + kk * C::BS_STRIDE + nn, bytes ? B + gk * ldb + gn : B, bytes);
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::BM * BK / T; ++i) {
      const int c = tid + i * T;
      const int r = c / BK, kk = c % BK;
      const int64_t gm = m0 + r, gk = k0 + kk;
      const bool ok = gm < M && gk < K;
      cp8(As + r * C::AS_STRIDE + kk, ok ? A + gm * lda + gk : A, ok);
    }
#pragma unroll
    for (int i = 0; i < BK * BN / T; ++i) {
      const int c = tid + i * T;
      const int kk = c / BN, nn = c % BN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      const bool ok = gk < K && gn < N;
      cp8(Bs + kk * C::BS_STRIDE + nn, ok ? B + gk * ldb + gn : B, ok);
    }
  }
}

// Interior CTA tile with K % BK == 0 and 16-byte aligned rows: every chunk
// is a full 16-byte copy and a thread's chunks sit at fixed row offsets, so
// the loader is pointer arithmetic only (no bounds logic per k tile).
template <class C>
__device__ __forceinline__ void load_tiles_full(double *As, double *Bs, const double *A,
                                                int64_t lda, const double *B, int64_t ldb,
                                                int64_t m0, int64_t n0, int64_t k0) {
  constexpr int BK = C::BK, BN = C::BN, T = C::THREADS;
  constexpr int RA = T / (BK / 2), RB = T / (BN / 2);
  const int tid = threadIdx.x;
  const int ra = tid / (BK / 2), ka = (tid % (BK / 2)) * 2;
  const int kb = tid / (BN / 2), nb = (tid % (BN / 2)) * 2;
  const double *ga = A + (m0 + ra) * lda + k0 + ka;
  const double *gb = B + (k0 + kb) * ldb + n0 + nb;
#pragma unroll
  for (int i = 0; i < C::BM * BK / 2 / T; ++i)
    cp16(As + (ra + i * RA) * C::AS_STRIDE + ka, ga + (int64_t)i * RA * lda, 16);
#pragma unroll
  for (int i = 0; i < BK * BN / 2 / T; ++i)
    cp16(Bs + (kb + i * RB) * C::BS_STRIDE + nb, gb + (int64_t)i * RB * ldb, 16);
}

template <bool VEC, class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    dgemm_dmma(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
               const double *__restrict__ B, int64_t ldb, double *__restrict__ Cm, int64_t rsc,
               int64_t csc, int accumulate, int num_m, int num_n, int group_m) {
  constexpr int BK = C::BK, ST = C::ST, MI = C::MI, NJ = C::NJ;
  extern __shared__ __align__(16) double smem[];
  double *As = smem;
  double *Bs = smem + ST * C::AS_TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / C::NWN) * C::WM, wn = (warp % C::NWN) * C::WN;
  // grouped rasterisation: resident CTAs cover a group_m-tall band of tiles
  const int pid = blockIdx.x, per_group = group_m * num_n;
  const int first_m = (pid / per_group) * group_m;
  const int gsize = num_m - first_m < group_m ? num_m - first_m : group_m;
  const int64_t m0 = (int64_t)(first_m + (pid % per_group) % gsize) * C::BM;
  const int64_t n0 = (int64_t)((pid % per_group) / gsize) * C::BN;
  const int ktiles = (int)((K + BK - 1) / BK);

  double acc[MI][NJ][4];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  const bool full = VEC && m0 + C::BM <= M && n0 + C::BN <= N && K % BK == 0;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < ktiles) {
      if (full)
        load_tiles_full<C>(As + s * C::AS_TILE, Bs + s * C::BS_TILE, A, lda, B, ldb, m0, n0,
                           (int64_t)s * BK);
      else
        load_tiles<VEC, C>(As + s * C::AS_TILE, Bs + s * C::BS_TILE, A, lda, B, ldb, M, N, K,
                           m0, n0, (int64_t)s * BK);
    }
    commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int pre = kt + ST - 1;
    if (pre < ktiles) {
      const int ps = pre % ST;
      if (full)
        load_tiles_full<C>(As + ps * C::AS_TILE, Bs + ps * C::BS_TILE, A, lda, B, ldb, m0, n0,
                           (int64_t)pre * BK);
      else
        load_tiles<VEC, C>(As + ps * C::AS_TILE, Bs + ps * C::BS_TILE, A, lda, B, ldb, M, N, K,
                           m0, n0, (int64_t)pre * BK);
    }
    commit();
    wait_group<ST - 1>();
    __syncthreads();
    const double *as = As + (kt % ST) * C::AS_TILE;
    const double *bs = Bs + (kt % ST) * C::BS_TILE;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a[MI][2], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        a[i][0] = as[(wm + i * 16 + g) * C::AS_STRIDE + k4 + t];
        a[i][1] = as[(wm + i * 16 + g + 8) * C::AS_STRIDE + k4 + t];
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = bs[(k4 + t) * C::BS_STRIDE + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncthreads();
  }
  // epilogue: c0,c1 at (g, 2t..2t+1); c2,c3 at (g + 8, 2t..2t+1)
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gm = m0 + wm + i * 16 + g + h * 8;
        if (gm >= M) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t gn = n0 + wn + j * 8 + 2 * t + e;
          if (gn >= N) continue;
          double *cp = Cm + gm * rsc + gn * csc;
          const double v = acc[i][j][h * 2 + e];
          *cp = accumulate ? (*cp + v) : v;
        }
      }
}

// The same tile with the fragment loads software-pipelined across k steps
// and tiles (CUTLASS-multistage order): one barrier per k tile, placed in
// the tile's last k step after its fragments are in registers, so the slot
// it frees is refilled at once (ST tiles in flight) and the next tile's
// first fragments load under the last step's DMMAs.
template <bool VEC, class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    dgemm_dmma_pf(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
                  const double *__restrict__ B, int64_t ldb, double *__restrict__ Cm,
                  int64_t rsc, int64_t csc, int accumulate, int num_m, int num_n, int group_m) {
  constexpr int BK = C::BK, ST = C::ST, MI = C::MI, NJ = C::NJ, S = BK / 4;
  static_assert(S % 2 == 0, "k steps per tile must be even (fragment double buffer)");
  extern __shared__ __align__(16) double smem[];
  double *As = smem;
  double *Bs = smem + ST * C::AS_TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / C::NWN) * C::WM, wn = (warp % C::NWN) * C::WN;
  const int pid = blockIdx.x, per_group = group_m * num_n;
  const int first_m = (pid / per_group) * group_m;
  const int gsize = num_m - first_m < group_m ? num_m - first_m : group_m;
  const int64_t m0 = (int64_t)(first_m + (pid % per_group) % gsize) * C::BM;
  const int64_t n0 = (int64_t)((pid % per_group) / gsize) * C::BN;
  const int ktiles = (int)((K + BK - 1) / BK);

  double acc[MI][NJ][4];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  const bool full = VEC && m0 + C::BM <= M && n0 + C::BN <= N && K % BK == 0;
#pragma unroll
  for (int s = 0; s < ST; ++s) {
    if (s < ktiles) {
      if (full)
        load_tiles_full<C>(As + s * C::AS_TILE, Bs + s * C::BS_TILE, A, lda, B, ldb, m0, n0,
                           (int64_t)s * BK);
      else
        load_tiles<VEC, C>(As + s * C::AS_TILE, Bs + s * C::BS_TILE, A, lda, B, ldb, M, N, K,
                           m0, n0, (int64_t)s * BK);
    }
    commit();
  }
  wait_group<ST - 1>();
  __syncthreads();
  double a[2][MI][2], b[2][NJ];
  const int arow0 = (wm + g) * C::AS_STRIDE + t, brow0 = t * C::BS_STRIDE + wn + g;
#define B2_FRAG(buf, as, bs, k4)                                                  \
  {                                                                               \
    _Pragma("unroll") for (int i = 0; i < MI; ++i) {                              \
      a[buf][i][0] = (as)[arow0 + i * 16 * C::AS_STRIDE + (k4)];                  \
      a[buf][i][1] = (as)[arow0 + (i * 16 + 8) * C::AS_STRIDE + (k4)];            \
    }                                                                             \
    _Pragma("unroll") for (int j = 0; j < NJ; ++j)                                \
        b[buf][j] = (bs)[brow0 + (k4) * C::BS_STRIDE + j * 8];                    \
  }
  B2_FRAG(0, As, Bs, 0);
  for (int kt = 0; kt < ktiles; ++kt) {
    const int slot = kt % ST, nslot = (kt + 1) % ST;
    const double *as = As + slot * C::AS_TILE, *bs = Bs + slot * C::BS_TILE;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int cur = s & 1, nxt = cur ^ 1;
      if (s == S - 1) {
        // every warp holds this tile's last fragments: tile kt + 1 must have
        // landed, and this tile's slot takes tile kt + ST
        wait_group<ST - 2>();
        __syncthreads();
        if (kt + ST < ktiles) {
          if (full)
            load_tiles_full<C>(As + slot * C::AS_TILE, Bs + slot * C::BS_TILE, A, lda, B, ldb,
                               m0, n0, (int64_t)(kt + ST) * BK);
          else
            load_tiles<VEC, C>(As + slot * C::AS_TILE, Bs + slot * C::BS_TILE, A, lda, B, ldb,
                               M, N, K, m0, n0, (int64_t)(kt + ST) * BK);
        }
        commit();
        B2_FRAG(nxt, As + nslot * C::AS_TILE, Bs + nslot * C::BS_TILE, 0);
      } else {
        B2_FRAG(nxt, as, bs, (s + 1) * 4);
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], a[cur][i][0], a[cur][i][1], b[cur][j]);
    }
  }
#undef B2_FRAG
  wait_group<0>();
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gm = m0 + wm + i * 16 + g + h * 8;
        if (gm >= M) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t gn = n0 + wn + j * 8 + 2 * t + e;
          if (gn >= N) continue;
          double *cp = Cm + gm * rsc + gn * csc;
          const double v = acc[i][j][h * 2 + e];
          *cp = accumulate ? (*cp + v) : v;
        }
      }
}

template <class C>
void set_smem() {
  cudaFuncSetAttribute(dgemm_dmma<true, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::SMEM_BYTES);
  cudaFuncSetAttribute(dgemm_dmma<false, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::SMEM_BYTES);
  cudaFuncSetAttribute(dgemm_dmma_pf<true, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::SMEM_BYTES);
  cudaFuncSetAttribute(dgemm_dmma_pf<false, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::SMEM_BYTES);
}

template <class C, bool PF = false>
void launch(bool vec, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda,
            const double *B, int64_t ldb, double *Cm, int64_t rsc, int64_t csc, int accumulate,
            int group_m, cudaStream_t st) {
  const int num_m = (int)((M + C::BM - 1) / C::BM), num_n = (int)((N + C::BN - 1) / C::BN);
  const unsigned grid = (unsigned)(num_m * num_n);
  auto k = PF ? (vec ? dgemm_dmma_pf<true, C> : dgemm_dmma_pf<false, C>)
               : (vec ? dgemm_dmma<true, C> : dgemm_dmma<false, C>);
  k<<<grid, C::THREADS, C::SMEM_BYTES, st>>>(M, N, K, A, lda, B, ldb, Cm, rsc, csc, accumulate,
                                              num_m, num_n, group_m);
}

}  // namespace

// Called from b2_gemm_f64 for row-major operands; returns B2_ERR_UNSUPPORTED
// when the layout does not qualify so the caller falls back.
int b2_dgemm_dmma(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                  int64_t ldb, double *C, int64_t rsc, int64_t csc, int accumulate,
                  void *stream) {
  static int cfg = -1, group_m = -1;
  if (cfg < 0) {
    const char *e = getenv("B2_DGEMM_CFG");
    cfg = e && !strcmp(e, "wide") ? 1 : e && !strcmp(e, "tall32pf") ? 2 : 0;
    set_smem<CfgTall>();
    set_smem<CfgWide>();
    set_smem<CfgTallK32>();
    const char *gm = getenv("B2_DGEMM_GROUP");
    group_m = gm ? atoi(gm) : 16;
    if (group_m < 1) group_m = 1;
  }
  const bool vec = (lda % 2 == 0) && (ldb % 2 == 0) && (((uintptr_t)A & 15) == 0) &&
                   (((uintptr_t)B & 15) == 0);
  cudaStream_t st = (cudaStream_t)stream;
  B2_CLEAR_ERROR();
  if (cfg == 1)
    launch<CfgWide>(vec, M, N, K, A, lda, B, ldb, C, rsc, csc, accumulate, group_m, st);
  else if (cfg == 2)
    launch<CfgTallK32, true>(vec, M, N, K, A, lda, B, ldb, C, rsc, csc, accumulate, group_m, st);
  else
    launch<CfgTall>(vec, M, N, K, A, lda, B, ldb, C, rsc, csc, accumulate, group_m, st);
  B2_LAUNCH_CHECK("dgemm launch");
  return B2_OK;
}
