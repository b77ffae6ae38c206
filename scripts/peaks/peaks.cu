// peaks.cu — compute / on-chip bandwidth ceilings measured on the box
// ("measure DMMA-f64, FFMA-f64, FFMA-f32 and tcgen05-tf32
// peaks on the box first").  Prints one JSON object.
//
//   dmma_f64   mma.sync.m16n8k4 f64 (the DGEMM's tensor path), register
//              operands, 8 independent accumulators per warp
//   dfma_f64   FP64 FMA on CUDA cores, 8 independent chains per thread
//   ffma_f32   FP32 FMA, 8 independent chains per thread
//   l2_read    GB/s reading a 48 MB buffer (L2-resident) with 16-B loads
//   hbm_read   GB/s reading a 4 GB buffer with 16-B loads
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peaks peaks.cu

#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                  \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int ITERS = 4096;

__global__ void k_dmma(double *out, double seed) {
  double a0 = seed + threadIdx.x, a1 = seed * 0.5, b0 = seed * 0.25;
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
          "{%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <typename T>
__global__ void k_fma(T *out, T seed) {
  T a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + (T)(threadIdx.x + i);
  const T m = (T)0.999999, b = (T)1e-7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, b);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == (T)1.2345) out[threadIdx.x] = s;
}

__global__ void k_read(const int4 *__restrict__ p, size_t n16, int reps, int *out) {
  int acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
         i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(p + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678) out[0] = acc;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double *dout;
  CK(cudaMalloc(&dout, 1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best;

  // DMMA: each mma is 16*8*4 = 512 FMA = 1024 flop per warp
  const int dmma_blocks = sms * 4, dmma_tpb = 256;
  k_dmma<<<dmma_blocks, dmma_tpb>>>(dout, 1.0);
  CK(cudaDeviceSynchronize());
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dmma<<<dmma_blocks, dmma_tpb>>>(dout, 1.0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = time_ms(e0, e1);
    if (ms < best) best = ms;
  }
  double warps = (double)dmma_blocks * dmma_tpb / 32;
  double dmma = warps * ITERS * 8 * 1024.0 / (best * 1e-3) / 1e12;

  const int fblocks = sms * 8, ftpb = 256;
  k_fma<double><<<fblocks, ftpb>>>(dout, 1.0);
  CK(cudaDeviceSynchronize());
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fma<double><<<fblocks, ftpb>>>(dout, 1.0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = time_ms(e0, e1);
    if (ms < best) best = ms;
  }
  double dfma = (double)fblocks * ftpb * ITERS * 8 * 2.0 / (best * 1e-3) / 1e12;

  k_fma<float><<<fblocks, ftpb>>>((float *)dout, 1.0f);
  CK(cudaDeviceSynchronize());
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fma<float><<<fblocks, ftpb>>>((float *)dout, 1.0f);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = time_ms(e0, e1);
    if (ms < best) best = ms;
  }
  double ffma = (double)fblocks * ftpb * ITERS * 8 * 2.0 / (best * 1e-3) / 1e12;

  // L2-resident read: 48 MB, 20 passes per launch
  size_t l2b = 48ull << 20, hbmb = 4ull << 30;
  int4 *buf;
  CK(cudaMalloc(&buf, hbmb));
  CK(cudaMemset(buf, 1, hbmb));
  const int rblocks = sms * 8, rtpb = 512;
  k_read<<<rblocks, rtpb>>>(buf, l2b / 16, 20, (int *)dout);
  CK(cudaDeviceSynchronize());
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_read<<<rblocks, rtpb>>>(buf, l2b / 16, 20, (int *)dout);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = time_ms(e0, e1);
    if (ms < best) best = ms;
  }
  double l2 = 20.0 * l2b / (best * 1e-3) / 1e9;
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_read<<<rblocks, rtpb>>>(buf, hbmb / 16, 1, (int *)dout);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = time_ms(e0, e1);
    if (ms < best) best = ms;
  }
  double hbm = (double)hbmb / (best * 1e-3) / 1e9;
  printf("{\"dmma_f64_tflops\": %.2f, \"dfma_f64_tflops\": %.2f, \"ffma_f32_tflops\": %.2f, "
         "\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"sms\": %d, \"clock_khz\": %d}\n",
         dmma, dfma, ffma, l2, hbm, sms, prop.clockRate);
  return 0;
}
