// rowpass.cuh — one-HBM-pass BLAS-2 family (f64) for the MATMUL library
// node in its matrix-vector forms (np.matmul 2D@1D / 1D@2D, interp.py:
// 450-460) and their fusions in gemver / atax / bicg.
//
// R is an M x N row-contiguous matrix view (row stride RP_RS).  One pass over
// R computes, per row m,
//     x'[m,n] = PROLOGUE(x[m,n])        (optional elementwise map, written back)
//     dot[m]  = sum_n x'[m,n] * v[n]    (optional;  A @ v)
//     acc[n] += coef(m) * x'[m,n]       (optional;  u @ A, coef = u[m] or dot[m])
// Blocks own interleaved rows (m = blockIdx.x + i * gridDim.x) so concurrently
// running CTAs stream neighbouring rows; grid.y tiles columns in RP_CW chunks
// whose v / acc slices live in shared memory; the next row is prefetched into
// registers while the current row's dot is block-reduced.  Column partials go
// to a workspace reduced by rp_finalize in a fixed order (deterministic).
//
// The including translation unit defines RP_* constants, struct RpArgs and
// the hooks rp_row_setup / rp_elem / rp_dot_vec / rp_coef / rp_store_dot.

#ifndef RP_KPT
#error "rowpass.cuh needs RP_KPT"
#endif

// RP_COMP (opt-in, B2_RP_COMP=1): compensated accumulation.  Every product enters its sum
// error-free (TwoProd via fma) and every addition is a TwoSum whose error
// term is carried (Ogita-Rump-Oishi Dot2), per thread, across the warp /
// block reductions (double-double), in the column partials (hi + lo
// workspaces) and in the fold; results are rounded to double once.  The
// device sums are then near correctly rounded whatever their association,
// i.e. at least as accurate as the reference's BLAS (interp.py:450-460) —
// the exact-sum criterion of tests/test_gpu_config.py.  RP_COMP 0 (the
// default; already within 1e-12 of the exact value at N=8000) = plain sums
// (mul + add, no contraction).
#ifndef RP_COMP
#define RP_COMP 0
#endif
#define RP_RED (RP_COMP ? 128 : 64)  // reduction scratch (doubles)
#ifndef RP_VSMEM
#define RP_VSMEM 0
#endif

__device__ __forceinline__ void rp_two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// (s, c) += a * b
__device__ __forceinline__ void rp_acc(double &s, double &c, double a, double b) {
#if RP_COMP
  const double p = a * b;
  const double ep = fma(a, b, -p);
  double t, et;
  rp_two_sum(s, p, t, et);
  s = t;
  c += et + ep;
#else
  s += a * b;
  (void)c;
#endif
}

// (h, l) += (h2, l2), renormalised
__device__ __forceinline__ void rp_dd_add(double &h, double &l, double h2, double l2) {
#if RP_COMP
  double s, e;
  rp_two_sum(h, h2, s, e);
  e += l + l2;
  h = s + e;
  l = e - (h - s);
#else
  h += h2;
  (void)l;
  (void)l2;
#endif
}

__device__ __forceinline__ double rp_block_sum(double v, double vl, double *red, int parity) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const double h2 = __shfl_xor_sync(0xffffffffu, v, s);
    const double l2 = RP_COMP ? __shfl_xor_sync(0xffffffffu, vl, s) : 0.0;
    rp_dd_add(v, vl, h2, l2);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[parity * 32 + w] = v;
    if (RP_COMP) red[64 + parity * 32 + w] = vl;
  }
  __syncthreads();
  double t = 0.0, tl = 0.0;
#pragma unroll
  for (int i = 0; i < RP_TPB / 32; ++i)
    rp_dd_add(t, tl, red[parity * 32 + i], RP_COMP ? red[64 + parity * 32 + i] : 0.0);
  return RP_COMP ? t + tl : t;
}

#ifndef RP_REV
#define RP_REV 0
#endif
// row of step index mi (bottom-up for RP_REV passes; see blas2.RP_REV_DOT)
#define RP_ROW(mi) (RP_REV ? (RP_M - 1 - (mi)) : (mi))

#if RP_TMA
// TMA variant: rows stream through an RP_S-deep ring of shared-memory row
// buffers filled by 1-D bulk copies (cp.async.bulk + mbarrier), so up to
// RP_S rows per SM are in flight without register staging; the dot vector
// slice and the column accumulators live in registers.  Shared layout:
// [staged column vectors (RP_NSTAGED x RP_CW)] [reduction scratch 64] [ring].
extern "C" __global__ void __launch_bounds__(RP_TPB) RP_NAME(const __grid_constant__ RpArgs a) {
  B2_PDL_ENTRY();
  extern __shared__ __align__(16) double rp_smem[];
  __shared__ __align__(8) unsigned long long rp_bar[RP_S];
  double *red = rp_smem + RP_NSTAGED * RP_CW;
  // RP_VSMEM: the dot vector slice lives in shared memory instead of
  // registers (compensated dot + axpy would otherwise exceed 128 registers)
  double *vsm = red + RP_RED;
  double *ring = vsm + (RP_VSMEM ? RP_CW : 0);
  const int tid = threadIdx.x;
  const b2_ll c0 = (b2_ll)blockIdx.y * RP_CW;
  const int cw = (int)((RP_N - c0) < RP_CW ? (RP_N - c0) : RP_CW);
  const unsigned bytes = (unsigned)cw * 8u;
  const double *__restrict__ R = (const double *)a.w[0];
  rp_stage_cols(a, c0, cw, tid);
#if RP_VSMEM
  for (int j = tid; j < cw; j += RP_TPB) vsm[j] = rp_dot_vec(a, c0 + j);
#define RP_V(k) ((tid + (k) * RP_TPB) < cw ? vsm[tid + (k) * RP_TPB] : 0.0)
  double acc[RP_KPT], accl[RP_KPT];
#else
#define RP_V(k) vreg[k]
  double vreg[RP_KPT], acc[RP_KPT], accl[RP_KPT];
#endif
#pragma unroll
  for (int k = 0; k < RP_KPT; ++k) {
#if !RP_VSMEM
    const int j = tid + k * RP_TPB;
    vreg[k] = (RP_DOT && j < cw) ? rp_dot_vec(a, c0 + j) : 0.0;
#endif
    acc[k] = 0.0;
    accl[k] = 0.0;
  }
  if (tid == 0) {
    for (int s = 0; s < RP_S; ++s) b2_mbar_init(&rp_bar[s], 1);
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < RP_S; ++s) {
      const b2_ll m = blockIdx.x + (b2_ll)s * gridDim.x;
      if (m < RP_M) b2_bulk_load(ring + s * RP_CW, R + RP_ROW(m) * RP_RS + c0, bytes, &rp_bar[s]);
    }
  }
  int parity = 0;
  int it = 0;
  for (b2_ll mi = blockIdx.x; mi < RP_M; mi += gridDim.x, ++it) {
    const b2_ll m = RP_ROW(mi);  // the row this step processes
    const int s = it % RP_S;
    b2_mbar_wait(&rp_bar[s], (unsigned)((it / RP_S) & 1));
    double x[RP_KPT];
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) {
      const int j = tid + k * RP_TPB;
      x[k] = (j < cw) ? ring[s * RP_CW + j] : 0.0;
    }
#if RP_PROLOGUE
    {
      RpRow rr;
      rp_row_setup(a, m, rr);
#pragma unroll
      for (int k = 0; k < RP_KPT; ++k) {
        const int j = tid + k * RP_TPB;
        if (j < cw) {
          x[k] = rp_elem(a, rr, m, c0 + j, x[k], j);
#if RP_WRITEBACK
          ((double *)a.w[0])[m * RP_RS + c0 + j] = x[k];
#endif
        }
      }
    }
#endif
#if RP_DOT
    double p = 0.0, pl = 0.0;
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) rp_acc(p, pl, x[k], RP_V(k));
    const double d = rp_block_sum(p, pl, red, parity);  // its barrier also retires slot s
    parity ^= 1;
    if (tid == 0) rp_store_dot(a, m, d, blockIdx.y);
#else
    const double d = 0.0;
    __syncthreads();  // every thread has read slot s
#endif
    if (tid == 0) {
      const b2_ll mn = mi + (b2_ll)RP_S * gridDim.x;
      if (mn < RP_M) b2_bulk_load(ring + s * RP_CW, R + RP_ROW(mn) * RP_RS + c0, bytes, &rp_bar[s]);
    }
#if RP_AXPY
    const double c = rp_coef(a, m, d);
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) rp_acc(acc[k], accl[k], c, x[k]);
#endif
    (void)d;
  }
#if RP_AXPY
  double *ws = (double *)a.w[1];
#pragma unroll
  for (int k = 0; k < RP_KPT; ++k) {
    const int j = tid + k * RP_TPB;
    if (j < cw) {
      ws[(b2_ll)blockIdx.x * RP_N + c0 + j] = acc[k];
      if (RP_COMP) ws[(b2_ll)(RP_G + blockIdx.x) * RP_N + c0 + j] = accl[k];
    }
  }
#endif
}
#else
extern "C" __global__ void __launch_bounds__(RP_TPB) RP_NAME(const __grid_constant__ RpArgs a) {
  B2_PDL_ENTRY();
  extern __shared__ double rp_smem[];
  double *acc_s = rp_smem;                     // [RP_CW] column accumulators (hi)
  double *accl_s = acc_s + (RP_AXPY ? RP_CW : 0);  // [RP_CW] (lo, RP_COMP)
  double *v_s = accl_s + (RP_AXPY && RP_COMP ? RP_CW : 0);  // [RP_CW] dot vector slice
  double *red = v_s + (RP_DOT ? RP_CW : 0);     // reduction scratch
  const int tid = threadIdx.x;
  const b2_ll c0 = (b2_ll)blockIdx.y * RP_CW;
  const int cw = (int)((RP_N - c0) < RP_CW ? (RP_N - c0) : RP_CW);
  for (int j = tid; j < cw; j += RP_TPB) {
    if (RP_AXPY) acc_s[j] = 0.0;
    if (RP_AXPY && RP_COMP) accl_s[j] = 0.0;
    if (RP_DOT) v_s[j] = rp_dot_vec(a, c0 + j);
  }
  rp_stage_cols(a, c0, cw, tid);
  __syncthreads();
  const double *__restrict__ R = (const double *)a.w[0];
  double x[RP_KPT], xn[RP_KPT];
  b2_ll m = blockIdx.x;
  if (m < RP_M) {
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) {
      const int j = tid + k * RP_TPB;
      x[k] = (j < cw) ? R[m * RP_RS + c0 + j] : 0.0;
    }
  }
  int parity = 0;
  for (; m < RP_M; m += gridDim.x) {
    const b2_ll mn = m + gridDim.x;
    if (mn < RP_M) {
#pragma unroll
      for (int k = 0; k < RP_KPT; ++k) {
        const int j = tid + k * RP_TPB;
        xn[k] = (j < cw) ? R[mn * RP_RS + c0 + j] : 0.0;
      }
    }
#if RP_PROLOGUE
    {
      RpRow rr;
      rp_row_setup(a, m, rr);
#pragma unroll
      for (int k = 0; k < RP_KPT; ++k) {
        const int j = tid + k * RP_TPB;
        if (j < cw) {
          x[k] = rp_elem(a, rr, m, c0 + j, x[k], j);
#if RP_WRITEBACK
          ((double *)a.w[0])[m * RP_RS + c0 + j] = x[k];
#endif
        }
      }
    }
#endif
#if RP_DOT
    double p = 0.0, pl = 0.0;
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) {
      const int j = tid + k * RP_TPB;
      if (j < cw) rp_acc(p, pl, x[k], v_s[j]);
    }
    const double d = rp_block_sum(p, pl, red, parity);
    parity ^= 1;
    if (tid == 0) rp_store_dot(a, m, d, blockIdx.y);
#else
    const double d = 0.0;
#endif
#if RP_AXPY
    const double c = rp_coef(a, m, d);
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) {
      const int j = tid + k * RP_TPB;
      if (j < cw) {
#if RP_COMP
        rp_acc(acc_s[j], accl_s[j], c, x[k]);
#else
        acc_s[j] += c * x[k];
#endif
      }
    }
#endif
    (void)d;
#pragma unroll
    for (int k = 0; k < RP_KPT; ++k) x[k] = xn[k];
  }
#if RP_AXPY
  double *ws = (double *)a.w[1];
  for (int j = tid; j < cw; j += RP_TPB) {
    ws[(b2_ll)blockIdx.x * RP_N + c0 + j] = acc_s[j];
    if (RP_COMP) ws[(b2_ll)(RP_G + blockIdx.x) * RP_N + c0 + j] = accl_s[j];
  }
#endif
}
#endif  // RP_TMA

// out[n] (wcr)= sum over G row-groups of ws[g][n]  (+ per-tile dot partials).
// Block 32 x RP_FY: 32 columns per block, the RP_FY thread rows split the G
// partials (strided, independent loads in flight), then thread row 0 adds
// the RP_FY sums in a fixed order (deterministic).
#ifndef RP_FY
#define RP_FY 32
#endif
extern "C" __global__ void __launch_bounds__(32 * RP_FY) RP_FIN_NAME(const __grid_constant__ RpArgs a) {
  B2_PDL_ENTRY();
  __shared__ double part[RP_FY][33];
  __shared__ double partl[RP_COMP ? RP_FY : 1][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const b2_ll i = (b2_ll)blockIdx.x * 32 + tx;
#if RP_AXPY
  {
    const double *ws = (const double *)a.w[1];
    double s = 0.0, sl = 0.0;
    if (i < RP_N)
      for (int g = ty; g < RP_G; g += RP_FY)
        rp_dd_add(s, sl, ws[(b2_ll)g * RP_N + i],
                  RP_COMP ? ws[(b2_ll)(RP_G + g) * RP_N + i] : 0.0);
    part[ty][tx] = s;
    if (RP_COMP) partl[ty][tx] = sl;
    __syncthreads();
    if (ty == 0 && i < RP_N) {
      double t = part[0][tx], tl = RP_COMP ? partl[0][tx] : 0.0;
#pragma unroll
      for (int k = 1; k < RP_FY; ++k) rp_dd_add(t, tl, part[k][tx], RP_COMP ? partl[k][tx] : 0.0);
      rp_store_axpy(a, i, RP_COMP ? t + tl : t);
    }
  }
#endif
  if (ty != 0) return;
#if RP_DOT && RP_CTILES > 1
  if (i < RP_M) {
    const double *wd = (const double *)a.w[2];
    double s = 0.0, sl = 0.0;
    for (int t = 0; t < RP_CTILES; ++t) rp_dd_add(s, sl, wd[(b2_ll)t * RP_M + i], 0.0);
    rp_store_dot_final(a, i, RP_COMP ? s + sl : s);
  }
#endif
}
