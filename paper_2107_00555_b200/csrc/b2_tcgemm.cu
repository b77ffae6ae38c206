// b2_tcgemm.cu — FP32 GEMM on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with the 3xTF32 split, for the SUMMA f32 configuration.
//
// The reference has no float32 type; the f32 MatMul config
// is defined against an f64 product of the f32 inputs at rtol 1e-5.  One TF32
// product keeps only 10 mantissa bits, so each operand is split into
// hi = rna_tf32(x) and lo = x - hi (exact in fp32) and
//   A B ~= lo(A) hi(B) + hi(A) lo(B) + hi(A) hi(B)
// which is a single TF32 GEMM over a K dimension three times as long:
//   A' = [lo(A) | hi(A) | hi(A)]   (M x 3K, K-major; interleaved per 32-wide
//   B' = [hi(B) | lo(B) | hi(B)]^T (N x 3K, K-major)  k block, see split_a)
// A' and B' are produced by two HBM-bound split kernels into a workspace;
// the GEMM then runs entirely on the tensor cores:
//   * CTA tile 128 x 256, K step 32 (one 128-byte swizzle atom of fp32),
//     4-stage TMA -> shared memory ring (48 KB per stage, SWIZZLE_128B),
//   * warp 0 lane 0 issues the TMA loads (mbarrier complete_tx),
//   * warp 1 lane 0 issues tcgen05.mma (M=128, N=256, K=8) x 4 per stage into
//     a 128 x 256 fp32 accumulator in TMEM and releases each stage with
//     tcgen05.commit,
//   * default: CTA pairs (tc_sgemm_pair, cta_group::2, 256 x 256 tiles,
//     two-segment operands A' = [lo|hi], B' = [hi|lo] per 32-wide k block so
//     the three products lo.hi, hi.lo, hi.hi come from one stage; 3 stages of
//     64 KB per CTA); B2_TC_PAIR=0 selects the single-CTA kernel,
//   * long in-TMEM accumulations lose accuracy (the error grows with the
//     accumulation length), so the MMA warp accumulates chunks of 128 k into
//     two alternating 256-column TMEM buffers and eight epilogue warps drain
//     each finished chunk with tcgen05.ld into an fp32 register accumulator
//     (IEEE adds) while the next chunk accumulates; the WCR (C = / += result)
//     is applied once at the end.

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "b2.h"
#include "b2_internal.h"

namespace {

constexpr int TM = 128, TN = 256, TK = 32, STAGES = 4;
constexpr int A_BYTES = TM * TK * 4;  // 16 KB
constexpr int B_BYTES = TN * TK * 4;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 128;
constexpr uint32_t TMEM_COLS = 512;  // two 256-column chunk accumulators
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + 32 * EPI_WARPS;
// instruction descriptor: D f32 (bit 4), A/B tf32 (bits 7, 10), K-major
// operands, N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) |
                           ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "B2_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra B2_DONE;\n\t"
      "bra B2_WAIT;\n\t"
      "B2_DONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row core-matrix
// groups 1024 bytes apart (SBO), sm100 descriptor version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *out) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) out[j] = __uint_as_float(v[j]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    tc_sgemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
             int64_t M, int64_t N, int nk, int chunk, float *__restrict__ C, int64_t ldc,
             int accumulate, int num_m, int num_n, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sa = smem;
  uint8_t *sb = smem + STAGES * A_BYTES;
  uint64_t *full = (uint64_t *)(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;  // [2] chunk accumulated in TMEM buffer b
  uint64_t *tempty = tfull + 2;      // [2] TMEM buffer b drained by the epilogue
  uint32_t *tmem_slot = (uint32_t *)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation: concurrently resident CTAs cover a group_m-tall
  // band of tiles, so their A and B k-slabs are shared through L2
  const int pid = blockIdx.x, per_group = group_m * num_n;
  const int first_m = (pid / per_group) * group_m;
  const int gsize = num_m - first_m < group_m ? num_m - first_m : group_m;
  const int m0 = (first_m + (pid % per_group) % gsize) * TM;
  const int n0 = ((pid % per_group) / gsize) * TN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tb) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) + 1) & 1);
        mbar_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(sa + s * A_BYTES, &ta, &full[s], kb * TK, m0);
        tma_load_2d(sb + s * B_BYTES, &tb, &full[s], kb * TK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // MMA issuer: chunk j accumulates in TMEM buffer j & 1 (256 columns)
      for (int kb = 0; kb < nk; ++kb) {
        const int j = kb / chunk, b = j & 1;
        const bool first = kb - j * chunk == 0;
        if (first && j >= 2) {
          mbar_wait(&tempty[b], ((j >> 1) + 1) & 1);
          fence_after();
        }
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        fence_after();
        const uint64_t da = sw128_desc(smem_u32(sa + s * A_BYTES));
        const uint64_t db = sw128_desc(smem_u32(sb + s * B_BYTES));
#pragma unroll
        for (int k = 0; k < TK / 8; ++k)  // 8 tf32 = 32 bytes = 2 descriptor units
          mma_tf32(tmem + (uint32_t)(b * TN), da + 2 * k, db + 2 * k, !(first && k == 0));
        mma_commit(&empty[s]);
        if (kb - j * chunk == chunk - 1 || kb == nk - 1) mma_commit(&tfull[b]);
      }
    }
  } else {
    // epilogue warps: warp w may read TMEM lanes 32 * (w % 4) ..; the eight
    // warps split the 256 columns in two halves.  Chunk partial sums are added
    // into an fp32 register accumulator (IEEE adds) as they complete.
    const int q = warp & 3, half = (warp - 2) >> 2;
    float acc[TN / 2];
#pragma unroll
    for (int i = 0; i < TN / 2; ++i) acc[i] = 0.f;
    const int nchunks = (nk + chunk - 1) / chunk;
    for (int j = 0; j < nchunks; ++j) {
      const int b = j & 1;
      mbar_wait(&tfull[b], (j >> 1) & 1);
      fence_after();
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * TN + half * (TN / 2));
#pragma unroll
      for (int c = 0; c < TN / 2; c += 16) {
        float v[16];
        tmem_ld16(base + (uint32_t)c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[c + i] += v[i];
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    const int64_t row = m0 + q * 32 + lane;
    if (row < M) {
      float *crow = C + row * ldc + n0 + half * (TN / 2);
      const int64_t ncol = N - (n0 + half * (TN / 2));
#pragma unroll
      for (int i = 0; i < TN / 2; ++i)
        if (i < ncol) crow[i] = accumulate ? crow[i] + acc[i] : acc[i];
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ---- CTA-pair variant (cta_group::2) ---------------------------------------
// A cluster of two CTAs computes a 256 x 256 tile: CTA r loads rows
// m0 + 128 r of A' and rows n0 + 128 r of B' (32 KB per stage, 6 stages), the
// leader issues tcgen05.mma.cta_group::2 (M=256, N=256, K=8) reading both
// CTAs' shared tiles, and each CTA's TMEM holds its 128 accumulator rows.
// Both CTAs' TMA bytes complete on the leader's full barrier; MMA commits are
// multicast to both CTAs' empty / chunk-full barriers; the peer's epilogue
// warps release a TMEM buffer by arriving on the leader's barrier.
// The pair kernel reads two-segment operands (A' = [lo | hi], B' = [hi | lo]
// per 32-wide k block): each stage holds one raw k block and the leader
// issues the three products lo·hi, hi·lo, hi·hi from it — hi is loaded once,
// not twice, so the split writes 2x (not 3x) and TMA moves 2/3 of the bytes.
constexpr int P_SEG = 128 * TK * 4;      // one 128-row x 32-k fp32 segment: 16 KB
constexpr int P_STAGES = 3;
constexpr int P_A_BYTES = 2 * P_SEG;     // A lo, A hi
constexpr int P_B_BYTES = 2 * P_SEG;     // B hi, B lo (this CTA's half of N = 256)
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE_BYTES + 1024 + 256;
constexpr uint32_t P_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// arrive on the same-offset mbarrier of cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *b, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(b)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint64_t *bar,
                                                 int x, int y) {
  // completes on the leader CTA's barrier (peer bit cleared)
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(P_IDESC), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Persistent: the grid holds one CTA pair per two SMs and each pair walks the
// tiles pid, pid + pairs, ... (grouped rasterisation).  Stage and chunk
// counters run on across tiles, so the TMA producer and the MMA warp start
// the next tile while the epilogue warps still store the previous one (the
// two TMEM chunk buffers decouple them); per tile the arithmetic is unchanged.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    tc_sgemm_pair(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                  int64_t M, int64_t N, int nk, int chunk, float *__restrict__ C, int64_t ldc,
                  int accumulate, int num_m, int num_n, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sa = smem;
  uint8_t *sb = smem + P_STAGES * P_A_BYTES;
  uint64_t *full = (uint64_t *)(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t *empty = full + P_STAGES;
  uint64_t *tfull = empty + P_STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = (uint32_t *)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int num_tiles = num_m * num_n, pairs = (int)(gridDim.x >> 1);
  const int per_group = group_m * num_n;
  const int nchunks = (nk + chunk - 1) / chunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tb) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  int tiles_done = 0;
  for (int tile = (int)(blockIdx.x >> 1); tile < num_tiles; tile += pairs, ++tiles_done) {
    const int first_m = (tile / per_group) * group_m;
    const int gsize = num_m - first_m < group_m ? num_m - first_m : group_m;
    const int m0 = (first_m + (tile % per_group) % gsize) * 256;
    const int n0 = ((tile % per_group) / gsize) * 256;
    const int g0 = tiles_done * nk;       // stage counter at this tile's first k block
    const int j0 = tiles_done * nchunks;  // chunk counter at this tile's first chunk
    if (warp == 0) {
      if (lane == 0) {
        // TMA producer (both CTAs): this CTA's halves of A' and B'
        for (int kb = 0; kb < nk; ++kb) {
          const int g = g0 + kb, s = g % P_STAGES;
          if (g >= P_STAGES) mbar_wait(&empty[s], ((g / P_STAGES) + 1) & 1);
          if (leader) mbar_expect_tx(&full[s], 2 * P_STAGE_BYTES);
          const int ma = m0 + (int)rank * 128, nb = n0 + (int)rank * 128;
          tma_load_2d_pair(sa + s * P_A_BYTES, &ta, &full[s], kb * 2 * TK, ma);
          tma_load_2d_pair(sa + s * P_A_BYTES + P_SEG, &ta, &full[s], kb * 2 * TK + TK, ma);
          tma_load_2d_pair(sb + s * P_B_BYTES, &tb, &full[s], kb * 2 * TK, nb);
          tma_load_2d_pair(sb + s * P_B_BYTES + P_SEG, &tb, &full[s], kb * 2 * TK + TK, nb);
        }
      }
    } else if (warp == 1) {
      if (lane == 0 && leader) {
        for (int kb = 0; kb < nk; ++kb) {
          const int jl = kb / chunk, J = j0 + jl, b = J & 1;
          const bool first = kb - jl * chunk == 0;
          if (first && J >= 2) {
            mbar_wait(&tempty[b], ((J >> 1) + 1) & 1);
            fence_after();
          }
          const int g = g0 + kb, s = g % P_STAGES;
          mbar_wait(&full[s], (g / P_STAGES) & 1);
          fence_after();
          const uint64_t a_lo = sw128_desc(smem_u32(sa + s * P_A_BYTES));
          const uint64_t a_hi = sw128_desc(smem_u32(sa + s * P_A_BYTES + P_SEG));
          const uint64_t b_hi = sw128_desc(smem_u32(sb + s * P_B_BYTES));
          const uint64_t b_lo = sw128_desc(smem_u32(sb + s * P_B_BYTES + P_SEG));
          const uint32_t d = tmem + (uint32_t)(b * 256);
#pragma unroll
          for (int k = 0; k < TK / 8; ++k) {  // small products first
            mma_tf32_pair(d, a_lo + 2 * k, b_hi + 2 * k, !(first && k == 0));
            mma_tf32_pair(d, a_hi + 2 * k, b_lo + 2 * k, 1);
            mma_tf32_pair(d, a_hi + 2 * k, b_hi + 2 * k, 1);
          }
          mma_commit_pair(&empty[s]);
          if (kb - jl * chunk == chunk - 1 || kb == nk - 1) mma_commit_pair(&tfull[b]);
        }
      }
    } else {
      const int q = warp & 3, half = (warp - 2) >> 2;
      float acc[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) acc[i] = 0.f;
      for (int jl = 0; jl < nchunks; ++jl) {
        const int J = j0 + jl, b = J & 1;
        mbar_wait(&tfull[b], (J >> 1) & 1);
        fence_after();
        const uint32_t base =
            tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * 256 + half * 128);
#pragma unroll
        for (int c = 0; c < 128; c += 16) {
          float v[16];
          tmem_ld16(base + (uint32_t)c, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c + i] += v[i];
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&tempty[b], 0);  // the leader's barrier
      }
      // the TMEM buffers are released: the next tile's MMAs run during the stores
      const int64_t row = m0 + (int64_t)rank * 128 + q * 32 + lane;
      if (row < M) {
        float *crow = C + row * ldc + n0 + half * 128;
        const int64_t ncol = N - (n0 + half * 128);
        if (ncol >= 128 && (((uintptr_t)crow) & 15) == 0) {
          float4 *c4 = (float4 *)crow;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float4 o;
            if (accumulate) {
              const float4 x = c4[i];
              o = make_float4(x.x + acc[4 * i], x.y + acc[4 * i + 1], x.z + acc[4 * i + 2],
                              x.w + acc[4 * i + 3]);
            } else {
              o = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
            }
            c4[i] = o;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i < ncol) crow[i] = accumulate ? crow[i] + acc[i] : acc[i];
        }
      }
    }
  }
  fence_before();
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// A (M x K, row stride lda) -> A' (M x Kp): per 32-wide k block b the 96
// columns [lo | hi | hi] of A[:, 32b : 32b + 32] (zero past K), so any range
// of k blocks is a contiguous range of A' columns.  Block (32, 8): lane =
// column in the k block (coalesced read, three coalesced writes), rows 8
// per CTA; grid (k blocks, row groups) — no per-element division.
__global__ void split_a(const float *__restrict__ A, int64_t lda, int64_t M, int64_t K,
                        int64_t Kp, int segs, float *__restrict__ Ap) {
  const int64_t kb = blockIdx.x;
  const int64_t k = kb * TK + threadIdx.x;
  for (int64_t i = (int64_t)blockIdx.y * 8 + threadIdx.y; i < M; i += (int64_t)gridDim.y * 8) {
    float lo = 0.f, hi = 0.f;
    if (k < K) {
      const float a = A[i * lda + k];
      hi = tf32_rna(a);
      lo = a - hi;
    }
    float *dst = Ap + i * Kp + kb * segs * TK + threadIdx.x;
    dst[0] = lo;
    dst[TK] = hi;
    if (segs == 3) dst[2 * TK] = hi;
  }
}

// B (K x N, row stride ldb) -> B'^T (N x Kp): per k block [hi | lo | hi],
// through a 32 x 32 shared tile so both the read and the write are coalesced
__global__ void split_bt(const float *__restrict__ B, int64_t ldb, int64_t K, int64_t N,
                         int64_t Kp, int segs, float *__restrict__ Bt) {
  __shared__ float t[32][33];
  const int64_t kb = blockIdx.y, k0 = kb * 32, n0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t k = k0 + ty + 8 * r, n = n0 + tx;
    t[ty + 8 * r][tx] = (k < K && n < N) ? B[k * ldb + n] : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t n = n0 + ty + 8 * r;
    if (n < N) {
      const float b = t[tx][ty + 8 * r];
      const float hi = tf32_rna(b);
      float *dst = Bt + n * Kp + kb * segs * TK + tx;
      dst[0] = hi;
      dst[TK] = b - hi;
      if (segs == 3) dst[2 * TK] = hi;
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        p)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

int make_map(CUtensorMap *map, const float *base, uint64_t inner, uint64_t outer,
             uint32_t box_outer) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return b2_fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {(cuuint32_t)TK, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return b2_fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return B2_OK;
}

int64_t tc_chunk_kblocks() {
  static int64_t c = -1;
  if (c < 0) {
    const char *e = getenv("B2_TC_CHUNK");  // k elements per accumulation chunk
    const int64_t k = e ? atoll(e) : 128;
    c = k > 0 ? (k + TK - 1) / TK : ((int64_t)1 << 28);
  }
  return c;
}

// Grid of the pair kernel.  Persistent (one pair per two SMs walking the
// tiles) pays off for short K: the per-tile prologue and epilogue are then a
// large share of a tile, and the persistent kernel overlaps them with the
// next tile's MMAs (SUMMA panels, K <= 8192: measured 5-11 % faster).  For
// long K one tile per pair is better: a wave of pairs starting together
// walks the same k blocks of A' and B' at the same time, so they are shared
// in L2 (16384^3 measured 6 % slower persistent, sustained).
// B2_TC_PERSIST=0 / 1 forces either.
int tc_pairs(int tiles, int nk) {
  static int pairs = -1, mode = -1;
  if (pairs < 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    pairs = sms / 2 > 0 ? sms / 2 : 1;
    const char *e = getenv("B2_TC_PERSIST");
    mode = e ? atoi(e) : 2;
  }
  const bool persist = mode == 1 || (mode == 2 && nk <= 256);
  return persist && tiles > pairs ? pairs : tiles;
}

// split-operand workspace, grown on demand (one process drives one GPU)
float *g_ws = nullptr;
size_t g_ws_bytes = 0;

}  // namespace

// C (row stride ldc, unit column stride) (=|+=) A @ B, A row-major M x K
// (row stride lda), B row-major K x N (row stride ldb).
int b2_sgemm_tc(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                int64_t ldb, float *C, int64_t ldc, int accumulate, void *stream) {
  static int group_m = -1, pair = -1;
  if (group_m < 0) {
    const char *e = getenv("B2_TC_GROUP");
    group_m = e ? atoi(e) : 4;  // measured: 4-tile bands of 256-row pair tiles
    if (group_m < 1) group_m = 1;
    const char *p2 = getenv("B2_TC_PAIR");
    pair = !(p2 && p2[0] == '0');
  }
  // the CTA-pair kernel reads two-segment operands, the single-CTA one three
  const int segs = pair ? 2 : 3;
  const int64_t nkb = (K + TK - 1) / TK, Kp = nkb * segs * TK;
  const size_t need = (size_t)(M + N) * (size_t)Kp * sizeof(float);
  cudaStream_t s = (cudaStream_t)stream;
  B2_CLEAR_ERROR();
  if (need > g_ws_bytes) {
    if (g_ws) {
      cudaStreamSynchronize(s);
      cudaFree(g_ws);
      g_ws = nullptr;
      g_ws_bytes = 0;
    }
    if (cudaMalloc(&g_ws, need) != cudaSuccess) {
      g_ws = nullptr;
      return b2_fail(B2_ERR_CUDA, "tc sgemm workspace (%zu bytes)", need);
    }
    g_ws_bytes = need;
  }
  float *Ap = g_ws, *Bt = g_ws + (size_t)M * Kp;
  {
    const unsigned ry = (unsigned)((M + 7) / 8 < 2048 ? (M + 7) / 8 : 2048);
    split_a<<<dim3((unsigned)nkb, ry), dim3(32, 8), 0, s>>>(A, lda, M, K, Kp, segs, Ap);
  }
  B2_LAUNCH_CHECK("split_a");
  dim3 tb(32, 8), gb((unsigned)((N + 31) / 32), (unsigned)nkb);
  split_bt<<<gb, tb, 0, s>>>(B, ldb, K, N, Kp, segs, Bt);
  B2_LAUNCH_CHECK("split_bt");
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc_sgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(tc_sgemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             P_SMEM_BYTES) != cudaSuccess)
      return b2_fail(B2_ERR_CUDA, "tc sgemm smem attribute");
    attr = true;
  }
  int rc;
  if (pair) {
    CUtensorMap pa, pb;
    rc = make_map(&pa, Ap, (uint64_t)Kp, (uint64_t)M, 128);
    if (rc) return rc;
    rc = make_map(&pb, Bt, (uint64_t)Kp, (uint64_t)N, 128);
    if (rc) return rc;
    const int pm = (int)((M + 255) / 256), pn = (int)((N + 255) / 256);
    // one pipeline stage = one raw 32-wide k block (both segments)
    tc_sgemm_pair<<<2 * tc_pairs(pm * pn, (int)nkb), THREADS, P_SMEM_BYTES, s>>>(
        pa, pb, M, N, (int)nkb, (int)tc_chunk_kblocks(), C, ldc, accumulate, pm, pn, group_m);
    B2_LAUNCH_CHECK("tc sgemm pair");
    return B2_OK;
  }
  CUtensorMap ma, mb;
  rc = make_map(&ma, Ap, (uint64_t)Kp, (uint64_t)M, TM);
  if (rc) return rc;
  rc = make_map(&mb, Bt, (uint64_t)Kp, (uint64_t)N, TN);
  if (rc) return rc;
  const int num_m = (int)((M + TM - 1) / TM), num_n = (int)((N + TN - 1) / TN);
  tc_sgemm<<<num_m * num_n, THREADS, SMEM_BYTES, s>>>(
      ma, mb, M, N, (int)(3 * nkb), (int)(3 * tc_chunk_kblocks()), C, ldc, accumulate, num_m,
      num_n, group_m);
  B2_LAUNCH_CHECK("tc sgemm");
  return B2_OK;
}

// ---------------------------------------------------------------------------
// Pre-split operands (SUMMA f32: split each local block ONCE per call, then
// broadcast and multiply the split panels).  Layouts are those the CTA-pair
// kernel reads: A' = M x Kp, B'^T = N x Kp, Kp = ceil(K / 32) * 2 * 32,
// per 32-wide k block [lo | hi] (A) and [hi | lo] (B).

extern "C" int64_t b2_tf32_split_cols(int64_t K) { return (K + TK - 1) / TK * 2 * TK; }

extern "C" int b2_tf32_split_a(const float *A, int64_t lda, int64_t M, int64_t K, float *Ap,
                               void *stream) {
  const int64_t nkb = (K + TK - 1) / TK, Kp = nkb * 2 * TK;
  const unsigned ry = (unsigned)((M + 7) / 8 < 2048 ? (M + 7) / 8 : 2048);
  B2_CLEAR_ERROR();
  split_a<<<dim3((unsigned)nkb, ry), dim3(32, 8), 0, (cudaStream_t)stream>>>(A, lda, M, K, Kp, 2,
                                                                             Ap);
  B2_LAUNCH_CHECK("split_a");
  return B2_OK;
}

extern "C" int b2_tf32_split_bt(const float *B, int64_t ldb, int64_t K, int64_t N, float *Bt,
                                void *stream) {
  const int64_t nkb = (K + TK - 1) / TK, Kp = nkb * 2 * TK;
  B2_CLEAR_ERROR();
  split_bt<<<dim3((unsigned)((N + 31) / 32), (unsigned)nkb), dim3(32, 8), 0,
             (cudaStream_t)stream>>>(B, ldb, K, N, Kp, 2, Bt);
  B2_LAUNCH_CHECK("split_bt");
  return B2_OK;
}

// C (row stride ldc) (=|+=) A @ B from split operands (tcgen05 CTA pairs)
extern "C" int b2_gemm_f32_presplit(int64_t M, int64_t N, int64_t K, const float *Ap,
                                    const float *Bt, float *C, int64_t ldc, int accumulate,
                                    void *stream) {
  static int group_m = -1;
  if (group_m < 0) {
    const char *e = getenv("B2_TC_GROUP");
    group_m = e ? atoi(e) : 4;
    if (group_m < 1) group_m = 1;
  }
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc_sgemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             P_SMEM_BYTES) != cudaSuccess)
      return b2_fail(B2_ERR_CUDA, "tc sgemm smem attribute");
    attr = true;
  }
  const int64_t nkb = (K + TK - 1) / TK, Kp = nkb * 2 * TK;
  CUtensorMap pa, pb;
  int rc = make_map(&pa, Ap, (uint64_t)Kp, (uint64_t)M, 128);
  if (rc) return rc;
  rc = make_map(&pb, Bt, (uint64_t)Kp, (uint64_t)N, 128);
  if (rc) return rc;
  const int pm = (int)((M + 255) / 256), pn = (int)((N + 255) / 256);
  B2_CLEAR_ERROR();
  tc_sgemm_pair<<<2 * tc_pairs(pm * pn, (int)nkb), THREADS, P_SMEM_BYTES, (cudaStream_t)stream>>>(
      pa, pb, M, N, (int)nkb, (int)tc_chunk_kblocks(), C, ldc, accumulate, pm, pn, group_m);
  B2_LAUNCH_CHECK("tc sgemm pair (presplit)");
  return B2_OK;
}

int b2_sgemm_tc_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("B2_TC_SGEMM");
    on = !(e && e[0] == '0');
  }
  return on;
}
