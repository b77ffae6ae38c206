// prelude.cuh — device helpers shared by every JIT kernel family.
//
// Scalar semantics follow the reference tasklet language (texpr.evaluate,
// pkg/src/sdfgkit/texpr.py:89-133) and numpy scalar arithmetic; see
// SURVEY.md Appendix A.  Compiled by NVRTC with --fmad=false.

typedef long long b2_ll;
typedef unsigned long long b2_ull;

__device__ __forceinline__ double b2_nan() { return __longlong_as_double(0x7ff8000000000000LL); }
__device__ __forceinline__ double b2_inf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Python int floor division (symbolic.py:196-199, texpr '//')
__device__ __forceinline__ b2_ll b2_floordiv_ll(b2_ll a, b2_ll b) {
  b2_ll q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return q;
}
__device__ __forceinline__ b2_ll b2_min_ll(b2_ll a, b2_ll b) { return a < b ? a : b; }
__device__ __forceinline__ b2_ll b2_max_ll(b2_ll a, b2_ll b) { return a > b ? a : b; }
// bulk L2 prefetch of [p, p + bytes) (16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void b2_prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// ... with an L2 evict_last policy on the prefetched lines
__device__ __forceinline__ void b2_prefetch_l2_last(const void *p, unsigned bytes) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p),
               "r"(bytes), "l"(pol) : "memory");
}
__device__ __forceinline__ b2_ll b2_abs_ll(b2_ll a) { return a < 0 ? -a : a; }
__device__ __forceinline__ b2_ll b2_ipow(b2_ll a, b2_ll e) {
  b2_ll r = 1;
  while (e > 0) {
    if (e & 1) r *= a;
    a *= a;
    e >>= 1;
  }
  return r;
}

// CPython float_floor_div / numpy npy_divmod
__device__ __forceinline__ double b2_floordiv_d(double a, double b) {
  if (b == 0.0) return a / b;
  double mod = fmod(a, b);
  double div = (a - mod) / b;
  if (mod != 0.0) {
    if ((b < 0.0) != (mod < 0.0)) div -= 1.0;
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (div - fl > 0.5) fl += 1.0;
  } else {
    fl = copysign(0.0, a / b);
  }
  return fl;
}

// Python builtins min/max: min(a, b) returns b only if b < a
template <typename T>
__device__ __forceinline__ T b2_pymin(T a, T b) { return (b < a) ? b : a; }
template <typename T>
__device__ __forceinline__ T b2_pymax(T a, T b) { return (b > a) ? b : a; }

// numpy.minimum / maximum (WCR min/max, ir.py:80-87): NaN propagates
__device__ __forceinline__ double b2_npmin(double a, double b) { return (isnan(a) || a < b) ? a : b; }
__device__ __forceinline__ double b2_npmax(double a, double b) { return (isnan(a) || a > b) ? a : b; }
__device__ __forceinline__ b2_ll b2_npmin(b2_ll a, b2_ll b) { return a < b ? a : b; }
__device__ __forceinline__ b2_ll b2_npmax(b2_ll a, b2_ll b) { return a > b ? a : b; }
__device__ __forceinline__ int b2_npmin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int b2_npmax(int a, int b) { return a > b ? a : b; }

// ---- write-conflict resolution on values (register accumulators) ----------
// Value form: taking the address of a register accumulator inside a
// data-dependent branch made nvcc 12.9 emit a non-terminating loop for sm_100a.
template <typename T>
__device__ __forceinline__ T b2_op_add(T a, T v) { return a + v; }
template <typename T>
__device__ __forceinline__ T b2_op_mul(T a, T v) { return a * v; }
template <typename T>
__device__ __forceinline__ T b2_op_min(T a, T v) { return b2_npmin(a, v); }
template <typename T>
__device__ __forceinline__ T b2_op_max(T a, T v) { return b2_npmax(a, v); }
__device__ __forceinline__ bool b2_op_add(bool a, bool v) { return a || v; }
__device__ __forceinline__ bool b2_op_mul(bool a, bool v) { return a && v; }
__device__ __forceinline__ bool b2_op_min(bool a, bool v) { return a && v; }
__device__ __forceinline__ bool b2_op_max(bool a, bool v) { return a || v; }

// ---- write-conflict resolution commits -----------------------------------
// Plain read-modify-write (the location is private to the thread).
template <typename T>
__device__ __forceinline__ void b2_wcr_add(T *p, T v) { *p = *p + v; }
template <typename T>
__device__ __forceinline__ void b2_wcr_mul(T *p, T v) { *p = *p * v; }
template <typename T>
__device__ __forceinline__ void b2_wcr_min(T *p, T v) { *p = b2_npmin(*p, v); }
template <typename T>
__device__ __forceinline__ void b2_wcr_max(T *p, T v) { *p = b2_npmax(*p, v); }
__device__ __forceinline__ void b2_wcr_add(bool *p, bool v) { *p = *p || v; }
__device__ __forceinline__ void b2_wcr_mul(bool *p, bool v) { *p = *p && v; }
__device__ __forceinline__ void b2_wcr_min(bool *p, bool v) { *p = *p && v; }
__device__ __forceinline__ void b2_wcr_max(bool *p, bool v) { *p = *p || v; }

// Atomic commits (the location is shared by concurrent map points).
__device__ __forceinline__ void b2_atomic_add(double *p, double v) { atomicAdd(p, v); }
__device__ __forceinline__ void b2_atomic_add(b2_ll *p, b2_ll v) {
  atomicAdd((b2_ull *)p, (b2_ull)v);
}
__device__ __forceinline__ void b2_atomic_add(int *p, int v) { atomicAdd(p, v); }

template <typename F>
__device__ __forceinline__ void b2_cas_double(double *p, F f) {
  b2_ull *a = (b2_ull *)p;
  b2_ull old = *a, assumed;
  do {
    assumed = old;
    double nv = f(__longlong_as_double((b2_ll)assumed));
    old = atomicCAS(a, assumed, (b2_ull)__double_as_longlong(nv));
  } while (assumed != old);
}
template <typename F>
__device__ __forceinline__ void b2_cas_ll(b2_ll *p, F f) {
  b2_ull *a = (b2_ull *)p;
  b2_ull old = *a, assumed;
  do {
    assumed = old;
    old = atomicCAS(a, assumed, (b2_ull)f((b2_ll)assumed));
  } while (assumed != old);
}
template <typename F>
__device__ __forceinline__ void b2_cas_int(int *p, F f) {
  unsigned *a = (unsigned *)p;
  unsigned old = *a, assumed;
  do {
    assumed = old;
    old = atomicCAS(a, assumed, (unsigned)f((int)assumed));
  } while (assumed != old);
}
__device__ __forceinline__ void b2_atomic_mul(double *p, double v) {
  b2_cas_double(p, [v](double o) { return o * v; });
}
__device__ __forceinline__ void b2_atomic_min(double *p, double v) {
  b2_cas_double(p, [v](double o) { return b2_npmin(o, v); });
}
__device__ __forceinline__ void b2_atomic_max(double *p, double v) {
  b2_cas_double(p, [v](double o) { return b2_npmax(o, v); });
}
__device__ __forceinline__ void b2_atomic_mul(b2_ll *p, b2_ll v) {
  b2_cas_ll(p, [v](b2_ll o) { return o * v; });
}
__device__ __forceinline__ void b2_atomic_min(b2_ll *p, b2_ll v) { atomicMin(p, v); }
__device__ __forceinline__ void b2_atomic_max(b2_ll *p, b2_ll v) { atomicMax(p, v); }
__device__ __forceinline__ void b2_atomic_mul(int *p, int v) {
  b2_cas_int(p, [v](int o) { return o * v; });
}
__device__ __forceinline__ void b2_atomic_min(int *p, int v) { atomicMin(p, v); }
__device__ __forceinline__ void b2_atomic_max(int *p, int v) { atomicMax(p, v); }
// bool containers: byte-wide; emulate with a 32-bit CAS on the aligned word
template <typename F>
__device__ __forceinline__ void b2_cas_bool(bool *p, F f) {
  size_t addr = (size_t)p;
  unsigned *w = (unsigned *)(addr & ~(size_t)3);
  unsigned sh = (unsigned)(addr & 3) * 8u;
  unsigned old = *w, assumed;
  do {
    assumed = old;
    bool cur = ((assumed >> sh) & 0xffu) != 0;
    unsigned nb = f(cur) ? 1u : 0u;
    unsigned nw = (assumed & ~(0xffu << sh)) | (nb << sh);
    old = atomicCAS(w, assumed, nw);
  } while (assumed != old);
}
__device__ __forceinline__ void b2_atomic_add(bool *p, bool v) { b2_cas_bool(p, [v](bool o) { return o || v; }); }
__device__ __forceinline__ void b2_atomic_mul(bool *p, bool v) { b2_cas_bool(p, [v](bool o) { return o && v; }); }
__device__ __forceinline__ void b2_atomic_min(bool *p, bool v) { b2_cas_bool(p, [v](bool o) { return o && v; }); }
__device__ __forceinline__ void b2_atomic_max(bool *p, bool v) { b2_cas_bool(p, [v](bool o) { return o || v; }); }

// Warp-aggregated atomic add for a target shared by the whole warp (WCR
// reductions: one commit per warp instead of per map point).
__device__ __forceinline__ double b2_warp_sum(double v) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  return v;
}

// ---- asynchronous global -> shared copies (LDGSTS), zero-fill when !valid ----
template <int BYTES>
__device__ __forceinline__ void b2_cp_async(void *smem, const void *gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? BYTES : 0;
  if (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem),
                 "n"(BYTES), "r"(n));
}
__device__ __forceinline__ void b2_cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void b2_cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- programmatic dependent launch -----------------------------------------
// Every JIT kernel starts with this: wait until the previous kernel in the
// stream has completed (its writes visible), then let the next one launch.
#ifdef B2_NO_PDL
#define B2_PDL_ENTRY() \
  do {                 \
  } while (0)
#else
#define B2_PDL_ENTRY()                                          \
  do {                                                          \
    asm volatile("griddepcontrol.wait;" ::: "memory");          \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)
#endif

// ---- TMA bulk copies (cp.async.bulk, 1-D) completed on an mbarrier ----------
__device__ __forceinline__ void b2_mbar_init(unsigned long long *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(b)),
               "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void b2_mbar_wait(unsigned long long *b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "B2_MW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra B2_MD;\n\t"
      "bra B2_MW;\n\t"
      "B2_MD:\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
// dst, src 16-byte aligned; bytes a multiple of 16
__device__ __forceinline__ void b2_bulk_load(void *dst, const void *src, unsigned bytes,
                                             unsigned long long *bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

// Device-side bounds guard for accesses the host cannot check statically
// (memlets inside nested scopes): records the first violation.
__device__ __forceinline__ bool b2_oob(b2_ll off, b2_ll size, int site, int *flag) {
  if (off < 0 || off >= size) {
    atomicCAS(flag, 0, site + 1);
    return true;
  }
  return false;
}
