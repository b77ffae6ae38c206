// jaclab.cu — jacobi_2d N=2000 sweep variants (B = 0.2 * (c + w + e + s + n)
// in the generated op order), timed back to back A -> B, B -> A with PDL,
// checked bitwise against the generated tile2 kernel after 4 sweeps.
// Build: nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a -o jaclab jaclab.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define B2_NO_PDL
#include "../../paper_2107_00555_b200/csrc/families/prelude.cuh"
#include "gen_jac.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
constexpr int N = 2000, I = N - 2;
constexpr double SWEEP_BYTES = 8.0 * N * N + 8.0 * I * I;

__device__ __forceinline__ double jpt(double c, double w, double e, double s, double n) {
  return 0.2 * ((((c + w) + e) + s) + n);
}

// rows marched per thread (register reuse of the north / centre rows)
template <int BX, int BY, int V>
__global__ void __launch_bounds__(BX *BY) march2(const double *__restrict__ A, double *__restrict__ B) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int tiles_x = (I + BX - 1) / BX, tiles_y = (I + BY * V - 1) / (BY * V);
  for (int vb = blockIdx.x; vb < tiles_x * tiles_y; vb += gridDim.x) {
    const int tx = vb % tiles_x, ty = vb / tiles_x;
    const int j = tx * BX + threadIdx.x + 1;
    const int i0 = (ty * BY + threadIdx.y) * V + 1;
    if (j > N - 2 || i0 > N - 2) continue;
    const double *a = A + (long)i0 * N + j;
    double n_ = a[-N], c = a[0];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (i0 + v > N - 2) break;
      const double s = a[(long)(v + 1) * N];
      B[(long)(i0 + v) * N + j] = jpt(c, a[(long)v * N - 1], a[(long)v * N + 1], s, n_);
      n_ = c;
      c = s;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


// two sweeps per launch on a TX x TY tile: A (tile + 2 halo) -> shared,
// B (tile + 1 halo) evaluated in shared memory (stored to global only when
// SB: B is dead until the last pass), A' (tile) -> the other A buffer
template <int TX, int TY, int NTH, bool SB>
__global__ void __launch_bounds__(NTH) pair2d(const double *__restrict__ A, double *__restrict__ B,
                                              double *__restrict__ An) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int AX = TX + 4, AY = TY + 4, BXW = TX + 2, BYW = TY + 2;
  __shared__ double sa[AY * AX];
  __shared__ double sb[BYW * BXW];
  constexpr int tiles_x = (I + TX - 1) / TX, tiles_y = (I + TY - 1) / TY;
  const int tid = threadIdx.x;
  for (int vb = blockIdx.x; vb < tiles_x * tiles_y; vb += gridDim.x) {
    const int tx = vb % tiles_x, ty = vb / tiles_x;
    const int x0 = 1 + tx * TX, y0 = 1 + ty * TY;
    for (int r = tid; r < AX * AY; r += NTH) {
      const int row = r / AX, col = r - row * AX;
      const int gy = y0 - 2 + row, gx = x0 - 2 + col;
      if (gy >= 0 && gy < N && gx >= 0 && gx < N) sa[r] = A[(long)gy * N + gx];
    }
    __syncthreads();
    for (int r = tid; r < BXW * BYW; r += NTH) {
      const int row = r / BXW, col = r - row * BXW;
      const int gy = y0 - 1 + row, gx = x0 - 1 + col;
      if (gy < 0 || gy > N - 1 || gx < 0 || gx > N - 1) continue;
      double v;
      if (gy >= 1 && gy <= N - 2 && gx >= 1 && gx <= N - 2) {
        const int c = (row + 1) * AX + col + 1;
        v = jpt(sa[c], sa[c - 1], sa[c + 1], sa[c + AX], sa[c - AX]);
        if (SB && row >= 1 && row <= TY && col >= 1 && col <= TX) B[(long)gy * N + gx] = v;
      } else {
        v = B[(long)gy * N + gx];
      }
      sb[r] = v;
    }
    __syncthreads();
    for (int r = tid; r < TX * TY; r += NTH) {
      const int row = r / TX, col = r - row * TX;
      const int gy = y0 + row, gx = x0 + col;
      if (gy > N - 2 || gx > N - 2) continue;
      const int c = (row + 1) * BXW + col + 1;
      An[(long)gy * N + gx] = jpt(sb[c], sb[c - 1], sb[c + 1], sb[c + BXW], sb[c - BXW]);
    }
    __syncthreads();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


// two sweeps per launch in registers: warp w owns B columns 30 w .. 30 w + 31
// (lanes) and A' columns 30 w + 1 .. 30 w + 30 (lanes 1..30); each thread
// marches V output rows keeping A rows i-1, i, i+1 and B rows i-2, i-1, i
// in registers, x neighbours by shuffle (edge lanes load theirs).  Same op
// order as two sweeps, so bitwise.  SB: store B's owned points (needed only
// after the last pass).
template <int WARPS, int V, bool SB>
__global__ void __launch_bounds__(32 * WARPS) jac2reg(const double *__restrict__ A,
                                                     double *__restrict__ B,
                                                     double *__restrict__ An) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int strips = (I + 29) / 30, chunks = (I + V - 1) / V;
  for (int vb = blockIdx.x; vb < ((strips + WARPS - 1) / WARPS) * chunks; vb += gridDim.x) {
    const int st = (vb % ((strips + WARPS - 1) / WARPS)) * WARPS + w;
    const int ch = vb / ((strips + WARPS - 1) / WARPS);
    if (st >= strips) continue;
    const int cb = 30 * st + lane;          // this lane's B column (global)
    const bool live = cb <= N - 1;
    const bool bint = cb >= 1 && cb <= N - 2;  // B evaluated here (else boundary value)
    const bool aout = lane >= 1 && lane <= 30 && cb >= 1 && cb <= N - 2;
    const int i0 = 1 + ch * V;               // first A' row of this chunk
    const int i1 = min(i0 + V, N - 1);       // one past the last
    // A rows i0-2 .. i0 (to evaluate B row i0-1 we need A rows i0-2, i0-1, i0)
    auto ld = [&](int r, int c) -> double { return (live && r >= 0 && r <= N - 1 && c >= 0 && c <= N - 1) ? A[(long)r * N + c] : 0.0; };
    double am = ld(i0 - 2, cb), ac = ld(i0 - 1, cb), ap;
    double bm2 = 0.0, bm1 = 0.0;  // B rows (i - 2), (i - 1) at cb
    for (int i = i0 - 1; i <= i1; ++i) {  // B row i
      ap = ld(i + 1, cb);
      // x neighbours of A row i
      double aw = __shfl_up_sync(0xffffffffu, ac, 1), ae = __shfl_down_sync(0xffffffffu, ac, 1);
      if (lane == 0) aw = ld(i, cb - 1);
      if (lane == 31) ae = ld(i, cb + 1);
      double b;
      if (i >= 1 && i <= N - 2 && bint) {
        b = 0.2 * ((((ac + aw) + ae) + ap) + am);
        if (SB && i >= i0 && i < i1 && aout) B[(long)i * N + cb] = b;
      } else {
        b = live && i >= 0 && i <= N - 1 ? B[(long)i * N + cb] : 0.0;
      }
      // A' row i - 1 from B rows i - 2, i - 1, i
      if (i - 1 >= i0) {
        double bw = __shfl_up_sync(0xffffffffu, bm1, 1), be = __shfl_down_sync(0xffffffffu, bm1, 1);
        if (aout) An[(long)(i - 1) * N + cb] = 0.2 * ((((bm1 + bw) + be) + b) + bm2);
      }
      bm2 = bm1;
      bm1 = b;
      am = ac;
      ac = ap;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


// jac2reg with every A row of the chunk loaded up front (registers, fully
// unrolled) so the loads overlap; full chunks only take this path
template <int WARPS, int V, bool SB>
__global__ void __launch_bounds__(32 * WARPS) jac2u(const double *__restrict__ A,
                                                   double *__restrict__ B,
                                                   double *__restrict__ An) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int strips = (I + 29) / 30, chunks = (I + V - 1) / V, sw = (strips + WARPS - 1) / WARPS;
  for (int vb = blockIdx.x; vb < sw * chunks; vb += gridDim.x) {
    const int st = (vb % sw) * WARPS + w, ch = vb / sw;
    if (st >= strips) continue;
    const int cb = 30 * st + lane;
    const bool live = cb <= N - 1;
    const bool bint = cb >= 1 && cb <= N - 2;
    const bool aout = lane >= 1 && lane <= 30 && bint;
    const int i0 = 1 + ch * V, i1 = min(i0 + V, N - 1);
    auto ld = [&](int r, int c) -> double {
      return (live && r >= 0 && r <= N - 1 && c >= 0 && c <= N - 1) ? A[(long)r * N + c] : 0.0;
    };
    double a[V + 3], ax[V + 1];  // A rows i0-2 .. i0+V at cb; edge lanes' outer neighbour
#pragma unroll
    for (int k = 0; k < V + 3; ++k) a[k] = ld(i0 - 2 + k, cb);
#pragma unroll
    for (int k = 0; k < V + 1; ++k)  // rows i0-1 .. i0+V-1 (B rows): lane 0 west, lane 31 east
      ax[k] = lane == 0 ? ld(i0 - 1 + k, cb - 1) : (lane == 31 ? ld(i0 - 1 + k, cb + 1) : 0.0);
    double bm2 = 0.0, bm1 = 0.0;
#pragma unroll
    for (int k = 0; k < V + 2; ++k) {  // B row i = i0 - 1 + k
      const int i = i0 - 1 + k;
      double b = 0.0;
      if (k <= V) {
        const double ac = a[k + 1];
        double aw = __shfl_up_sync(0xffffffffu, ac, 1), ae = __shfl_down_sync(0xffffffffu, ac, 1);
        if (lane == 0) aw = ax[k];
        if (lane == 31) ae = ax[k];
        if (i >= 1 && i <= N - 2 && i <= i1 && bint) {
          b = 0.2 * ((((ac + aw) + ae) + a[k + 2]) + a[k]);
          if (SB && i >= i0 && i < i1 && aout) B[(long)i * N + cb] = b;
        } else if (live && i >= 0 && i <= N - 1) {
          b = B[(long)i * N + cb];
        }
      }
      if (k >= 2 && i - 1 < i1) {  // A' row i - 1 from B rows i - 2 .. i
        double bw = __shfl_up_sync(0xffffffffu, bm1, 1), be = __shfl_down_sync(0xffffffffu, bm1, 1);
        if (aout) An[(long)(i - 1) * N + cb] = 0.2 * ((((bm1 + bw) + be) + b) + bm2);
      }
      bm2 = bm1;
      bm1 = b;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void init(double *a, double *b) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (long)N * N; i += (long)gridDim.x * blockDim.x) {
    unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    a[i] = (double)(h & 0xFFFFFF) / 16777216.0;
    b[i] = a[i];
  }
}
__global__ void ndiff(const double *a, const double *b, unsigned long long *cnt) {
  unsigned long long c = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (long)N * N; i += (long)gridDim.x * blockDim.x)
    c += (__double_as_longlong(a[i]) != __double_as_longlong(b[i]));
  atomicAdd(cnt, c);
}

struct V { const char *name; void (*f)(const double *, double *); dim3 blk; int grid; bool gen; };
static int *g_flag;
static void launch(const V &v, const double *a, double *b, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.grid); cfg.blockDim = v.blk; cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  if (v.gen) { B2Args ar; ar.w[0] = (long long)a; ar.w[1] = (long long)b; ar.w[2] = (long long)g_flag; CK(cudaLaunchKernelEx(&cfg, gen_jac, ar)); }
  else CK(cudaLaunchKernelEx(&cfg, v.f, a, b));
}
template <int BX, int BY, int VV>
V mk(const char *name) {
  constexpr int g = ((I + BX - 1) / BX) * ((I + BY * VV - 1) / (BY * VV));
  return V{name, march2<BX, BY, VV>, dim3(BX, BY), g, false};
}

int main(int argc, char **argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 200;
  const size_t bytes = (size_t)N * N * 8;
  double *A, *B, *RA, *RB; unsigned long long *cnt;
  CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&RA, bytes)); CK(cudaMalloc(&RB, bytes));
  CK(cudaMalloc(&cnt, 8)); CK(cudaMalloc(&g_flag, 8));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  if (getenv("PAIR")) {
    double *An; CK(cudaMalloc(&An, bytes));
    init<<<592, 256, 0, s>>>(RA, RB);
    V gv0{"generated_tile2", nullptr, dim3(32, 8), 8000, true};
    for (int t = 0; t < 4; ++t) { launch(gv0, RA, RB, s); launch(gv0, RB, RA, s); }
    struct PV { const char *name; void (*f)(const double *, double *, double *); void (*fsb)(const double *, double *, double *); int nth; int grid; };
#define PVM(TX, TY, NT) PV{"pair2d_" #TX "x" #TY "_t" #NT, pair2d<TX, TY, NT, false>, pair2d<TX, TY, NT, true>, NT, ((I + TX - 1) / TX) * ((I + TY - 1) / TY)}
#define JRM(WW, VV) PV{"jac2reg_w" #WW "_v" #VV, jac2reg<WW, VV, false>, jac2reg<WW, VV, true>, 32 * WW, (((I + 29) / 30 + WW - 1) / WW) * ((I + VV - 1) / VV)}
#define JUM(WW, VV) PV{"jac2u_w" #WW "_v" #VV, jac2u<WW, VV, false>, jac2u<WW, VV, true>, 32 * WW, (((I + 29) / 30 + WW - 1) / WW) * ((I + VV - 1) / VV)}
    PV pvs[] = {JRM(8, 8), JUM(4, 8), JUM(8, 8), JUM(4, 16), JUM(8, 16), JUM(2, 16), JUM(4, 12), JUM(8, 4)};
    auto pl = [&](void (*f)(const double *, double *, double *), int nth, int grid, const double *a, double *b, double *an) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid); cfg.blockDim = dim3(nth); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, f, a, b, an));
    };
    for (const PV &v : pvs) {
      init<<<592, 256, 0, s>>>(A, B);
      CK(cudaMemcpyAsync(An, A, bytes, cudaMemcpyDeviceToDevice, s));
      for (int t = 0; t < 4; ++t) {
        auto f = t == 3 ? v.fsb : v.f;
        if (t & 1) pl(f, v.nth, v.grid, An, B, A); else pl(f, v.nth, v.grid, A, B, An);
      }
      CK(cudaMemsetAsync(cnt, 0, 8, s));
      ndiff<<<592, 256, 0, s>>>(A, RA, cnt); ndiff<<<592, 256, 0, s>>>(B, RB, cnt);
      unsigned long long h = 0; CK(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s)); CK(cudaStreamSynchronize(s));
      for (int w = 0; w < 10; ++w) pl(v.f, v.nth, v.grid, w & 1 ? An : A, B, w & 1 ? A : An);
      CK(cudaEventRecord(e0, s));
      for (int r = 0; r < reps; ++r) pl(v.f, v.nth, v.grid, r & 1 ? An : A, B, r & 1 ? A : An);
      CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = ms * 1e3 / reps;
      printf("{\"variant\": \"%s\", \"grid\": %d, \"us_per_pass\": %.3f, \"us_per_sweep\": %.3f, \"algo_GBps\": %.1f, \"mismatches\": %llu}\n", v.name, v.grid, us, us / 2, 2 * SWEEP_BYTES / (us * 1e-6) / 1e9, h);
    }
    return 0;
  }
  V gv{"generated_tile2", nullptr, dim3(32, 8), 8000, true};
  V vars[] = {gv,
              mk<32, 8, 4>("march2_32x8_v4"), mk<32, 8, 8>("march2_32x8_v8"), mk<32, 8, 16>("march2_32x8_v16"),
              mk<64, 4, 8>("march2_64x4_v8"), mk<64, 4, 16>("march2_64x4_v16"), mk<128, 2, 8>("march2_128x2_v8"),
              mk<32, 16, 8>("march2_32x16_v8"), mk<64, 8, 4>("march2_64x8_v4"), mk<64, 8, 8>("march2_64x8_v8")};
  init<<<592, 256, 0, s>>>(RA, RB);
  for (int t = 0; t < 2; ++t) { launch(gv, RA, RB, s); launch(gv, RB, RA, s); }
  for (const V &v : vars) {
    init<<<592, 256, 0, s>>>(A, B);
    for (int t = 0; t < 2; ++t) { launch(v, A, B, s); launch(v, B, A, s); }
    CK(cudaMemsetAsync(cnt, 0, 8, s));
    ndiff<<<592, 256, 0, s>>>(A, RA, cnt); ndiff<<<592, 256, 0, s>>>(B, RB, cnt);
    unsigned long long h = 0; CK(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s)); CK(cudaStreamSynchronize(s));
    for (int w = 0; w < 10; ++w) launch(v, w & 1 ? B : A, w & 1 ? A : B, s);
    CK(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) launch(v, r & 1 ? B : A, r & 1 ? A : B, s);
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = ms * 1e3 / reps;
    printf("{\"variant\": \"%s\", \"grid\": %d, \"us\": %.3f, \"GBps\": %.1f, \"mismatches\": %llu}\n", v.name, v.grid, us, SWEEP_BYTES / (us * 1e-6) / 1e9, h);
  }
  return 0;
}
