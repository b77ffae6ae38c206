// dmma_shapes.cu — FP64 tensor throughput per mma.sync shape (m16n8k4 /
// m16n8k8 / m16n8k16), register operands, 8 independent accumulators per
// warp, and a fragment-layout check of k8 / k16 against k4 (one warp).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_shapes dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ void mma4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
}
__device__ __forceinline__ void mma8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int K>
__global__ void rate(double *out, double seed) {
  double c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
  for (int i = 0; i < 4; ++i) b[i] = seed * 0.5 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 4) mma4(c[i], a[0], a[1], b[0]);
      if (K == 8) mma8(c[i], *(const double(*)[4])a, *(const double(*)[2])b);
      if (K == 16) mma16(c[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[threadIdx.x] = s;
}

// one warp: C(16x8) = A(16xK) B(Kx8) via the shape's fragments, A, B in global
template <int K>
__global__ void check(const double *A, const double *B, double *C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double d[4] = {0, 0, 0, 0};
  if (K == 4) {
    mma4(d, A[g * K + t], A[(g + 8) * K + t], B[t * 8 + g]);
  } else if (K == 8) {
    double a[4] = {A[g * K + t], A[(g + 8) * K + t], A[g * K + t + 4], A[(g + 8) * K + t + 4]};
    double b[2] = {B[t * 8 + g], B[(t + 4) * 8 + g]};
    mma8(d, a, b);
  } else {
    double a[8], b[4];
    for (int q = 0; q < 4; ++q) {
      a[2 * q] = A[g * K + t + 4 * q];
      a[2 * q + 1] = A[(g + 8) * K + t + 4 * q];
      b[q] = B[(t + 4 * q) * 8 + g];
    }
    mma16(d, a, b);
  }
  C[g * 8 + 2 * t] = d[0];
  C[g * 8 + 2 * t + 1] = d[1];
  C[(g + 8) * 8 + 2 * t] = d[2];
  C[(g + 8) * 8 + 2 * t + 1] = d[3];
}

template <int K>
void run_rate(int sms, double *dout) {
  const int blocks = sms * 4, tpb = 256;
  rate<K><<<blocks, tpb>>>(dout, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    rate<K><<<blocks, tpb>>>(dout, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double warps = (double)blocks * tpb / 32;
  printf("{\"shape\": \"m16n8k%d\", \"tflops\": %.2f}\n", K,
         warps * ITERS * 8 * (16.0 * 8 * K * 2) / (best * 1e-3) / 1e12);
}

template <int K>
void run_check() {
  double hA[16 * 16], hB[16 * 8], hC[128], ref[128];
  for (int i = 0; i < 16 * K; ++i) hA[i] = (double)((i * 7919) % 97) / 13.0 - 3.0;
  for (int i = 0; i < K * 8; ++i) hB[i] = (double)((i * 104729) % 89) / 11.0 - 4.0;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += hA[m * K + k] * hB[k * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dC, sizeof hC);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  check<K><<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) {
    const double e = hC[i] - ref[i];
    err = e * e > err ? e * e : err;
  }
  printf("{\"shape\": \"m16n8k%d\", \"layout_max_sq_err\": %.3e, \"err\": \"%s\"}\n", K, err,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *dout;
  cudaMalloc(&dout, 4096 * 8);
  run_check<4>();
  run_check<8>();
  run_check<16>();
  run_rate<4>(sms, dout);
  run_rate<8>(sms, dout);
  run_rate<16>(sms, dout);
  return 0;
}
