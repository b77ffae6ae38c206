// b2_runtime.cu — runtime half of libb2.so: error handling, device/memory/
// stream/event management, NVRTC JIT of the kernel families, driver-level
// launches and CUDA-graph capture.  See include/b2.h for the contract.
//
// The driver API is reached through cudaGetDriverEntryPoint so the library
// links only cudart_static + nvrtc and loads on GPU-less hosts (the CPU
// test tier checks the exported symbols there).

#include <cuda.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "b2.h"
#include "b2_internal.h"

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

int b2_fail(int code, const char *fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int b2_cuda_check(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return B2_OK;
  return b2_fail(B2_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

void b2_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" int b2_version(void) { return 1; }
extern "C" const char *b2_last_error(void) { return g_err.c_str(); }
extern "C" int64_t b2_launch_count(void) { return g_launches.load(); }

// ---------------------------------------------------------------------------
// driver entry points

typedef CUresult (*PFN_ModuleLoadData)(CUmodule *, const void *);
typedef CUresult (*PFN_ModuleUnload)(CUmodule);
typedef CUresult (*PFN_ModuleGetFunction)(CUfunction *, CUmodule, const char *);
typedef CUresult (*PFN_LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned,
                                     unsigned, unsigned, unsigned, CUstream, void **, void **);
typedef CUresult (*PFN_FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
typedef CUresult (*PFN_LaunchKernelEx)(const CUlaunchConfig *, CUfunction, void **, void **);
typedef CUresult (*PFN_GetErrorString)(CUresult, const char **);

static struct {
  std::once_flag once;
  int status = -1;
  PFN_ModuleLoadData moduleLoadData = nullptr;
  PFN_ModuleUnload moduleUnload = nullptr;
  PFN_ModuleGetFunction moduleGetFunction = nullptr;
  PFN_LaunchKernel launchKernel = nullptr;
  PFN_LaunchKernelEx launchKernelEx = nullptr;  // programmatic dependent launch
  PFN_FuncSetAttribute funcSetAttribute = nullptr;
  PFN_GetErrorString getErrorString = nullptr;
} drv;

static int load_driver() {
  std::call_once(drv.once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
#define B2_GET(sym, field, T)                                                         \
  p = nullptr;                                                                        \
  if (cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q) != cudaSuccess || !p) { \
    drv.status = 1;                                                                   \
    return;                                                                           \
  }                                                                                   \
  drv.field = (T)p;
    B2_GET("cuModuleLoadData", moduleLoadData, PFN_ModuleLoadData);
    B2_GET("cuModuleUnload", moduleUnload, PFN_ModuleUnload);
    B2_GET("cuModuleGetFunction", moduleGetFunction, PFN_ModuleGetFunction);
    B2_GET("cuLaunchKernel", launchKernel, PFN_LaunchKernel);
    B2_GET("cuLaunchKernelEx", launchKernelEx, PFN_LaunchKernelEx);
    B2_GET("cuFuncSetAttribute", funcSetAttribute, PFN_FuncSetAttribute);
    B2_GET("cuGetErrorString", getErrorString, PFN_GetErrorString);
#undef B2_GET
    drv.status = 0;
  });
  if (drv.status != 0) {
    cudaGetLastError();
    return b2_fail(B2_ERR_CUDA, "CUDA driver entry points unavailable (no GPU/driver?)");
  }
  return B2_OK;
}

static int cu_check(CUresult r, const char *what) {
  if (r == CUDA_SUCCESS) return B2_OK;
  const char *s = "?";
  if (drv.getErrorString) drv.getErrorString(r, &s);
  return b2_fail(B2_ERR_CUDA, "%s: %s (CUresult %d)", what, s, (int)r);
}

// ---------------------------------------------------------------------------
// device, memory, streams, events

extern "C" int b2_device_count(int *n) {
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *n = 0;
  }
  return B2_OK;
}

extern "C" int b2_init(int device) {
  int rc = b2_cuda_check(cudaSetDevice(device), "cudaSetDevice");
  if (rc) return rc;
  rc = b2_cuda_check(cudaFree(nullptr), "context init");
  if (rc) return rc;
  return load_driver();
}

extern "C" int b2_device_info(int device, b2_device_info_t *out) {
  cudaDeviceProp p;
  int rc = b2_cuda_check(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
  if (rc) return rc;
  memset(out, 0, sizeof *out);
  strncpy(out->name, p.name, sizeof(out->name) - 1);
  out->major = p.major;
  out->minor = p.minor;
  out->sm_count = p.multiProcessorCount;
  out->l2_bytes = p.l2CacheSize;
  out->max_smem_optin = (int)p.sharedMemPerBlockOptin;
  out->total_mem = p.totalGlobalMem;
  return B2_OK;
}

extern "C" int b2_malloc(void **p, size_t bytes) {
  return b2_cuda_check(cudaMalloc(p, bytes ? bytes : 1), "cudaMalloc");
}
extern "C" int b2_free(void *p) { return b2_cuda_check(cudaFree(p), "cudaFree"); }
extern "C" int b2_memcpy_h2d(void *dst, const void *src, size_t n, void *s) {
  return b2_cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, (cudaStream_t)s),
                       "memcpy h2d");
}
extern "C" int b2_memcpy_d2h(void *dst, const void *src, size_t n, void *s) {
  return b2_cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, (cudaStream_t)s),
                       "memcpy d2h");
}
extern "C" int b2_memcpy_d2d(void *dst, const void *src, size_t n, void *s) {
  return b2_cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, (cudaStream_t)s),
                       "memcpy d2d");
}
extern "C" int b2_memset(void *dst, int v, size_t n, void *s) {
  return b2_cuda_check(cudaMemsetAsync(dst, v, n, (cudaStream_t)s), "memset");
}
extern "C" int b2_stream_create(void **s) {
  return b2_cuda_check(cudaStreamCreateWithFlags((cudaStream_t *)s, cudaStreamNonBlocking),
                       "stream create");
}
extern "C" int b2_stream_destroy(void *s) {
  return b2_cuda_check(cudaStreamDestroy((cudaStream_t)s), "stream destroy");
}
extern "C" int b2_stream_sync(void *s) {
  return b2_cuda_check(cudaStreamSynchronize((cudaStream_t)s), "stream sync");
}
extern "C" int b2_device_sync(void) {
  return b2_cuda_check(cudaDeviceSynchronize(), "device sync");
}
extern "C" int b2_event_create(void **ev) {
  return b2_cuda_check(cudaEventCreate((cudaEvent_t *)ev), "event create");
}
extern "C" int b2_event_destroy(void *ev) {
  return b2_cuda_check(cudaEventDestroy((cudaEvent_t)ev), "event destroy");
}
extern "C" int b2_event_record(void *ev, void *s) {
  return b2_cuda_check(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)s), "event record");
}
// inside a stream capture: an event record NODE (timestamped at replay), not
// a capture-internal dependency
extern "C" int b2_event_record_external(void *ev, void *s) {
  return b2_cuda_check(
      cudaEventRecordWithFlags((cudaEvent_t)ev, (cudaStream_t)s, cudaEventRecordExternal),
      "event record external");
}
extern "C" int b2_event_elapsed_ms(void *a, void *b, float *ms) {
  int rc = b2_cuda_check(cudaEventSynchronize((cudaEvent_t)b), "event sync");
  if (rc) return rc;
  return b2_cuda_check(cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b), "elapsed");
}
extern "C" int b2_stream_wait_event(void *s, void *ev) {
  return b2_cuda_check(cudaStreamWaitEvent((cudaStream_t)s, (cudaEvent_t)ev, 0),
                       "stream wait event");
}
extern "C" int b2_host_register(void *p, size_t n) {
  return b2_cuda_check(cudaHostRegister(p, n, cudaHostRegisterDefault), "host register");
}
extern "C" int b2_host_unregister(void *p) {
  return b2_cuda_check(cudaHostUnregister(p), "host unregister");
}
// CUDA IPC: a peer process maps this allocation (peer-store halos)
extern "C" int b2_ipc_handle(void *p, void *out64) {
  cudaIpcMemHandle_t h;
  int rc = b2_cuda_check(cudaIpcGetMemHandle(&h, p), "ipc get handle");
  if (rc) return rc;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(out64, &h, sizeof(h));
  return B2_OK;
}
extern "C" int b2_ipc_open(const void *h64, void **p) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h64, sizeof(h));
  return b2_cuda_check(cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess),
                       "ipc open handle");
}
extern "C" int b2_ipc_close(void *p) {
  return b2_cuda_check(cudaIpcCloseMemHandle(p), "ipc close handle");
}

// ---------------------------------------------------------------------------
// NVRTC JIT

extern "C" int b2_jit_compile(const char *src, const char *name, const char *const *opts,
                              int nopts, void *cubin, size_t *cubin_size, char *log,
                              size_t log_len) {
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src, name, 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return b2_fail(B2_ERR_NVRTC, "nvrtcCreateProgram: %s", nvrtcGetErrorString(r));
  r = nvrtcCompileProgram(prog, nopts, opts);
  size_t lsz = 0;
  nvrtcGetProgramLogSize(prog, &lsz);
  std::string lg(lsz, '\0');
  if (lsz) nvrtcGetProgramLog(prog, &lg[0]);
  if (log && log_len) {
    size_t n = lg.size() < log_len - 1 ? lg.size() : log_len - 1;
    memcpy(log, lg.data(), n);
    log[n] = 0;
  }
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return b2_fail(B2_ERR_NVRTC, "nvrtc compile of %s failed: %s\n%s", name,
                   nvrtcGetErrorString(r), lg.c_str());
  }
  size_t sz = 0;
  r = nvrtcGetCUBINSize(prog, &sz);
  if (r != NVRTC_SUCCESS || sz == 0) {
    nvrtcDestroyProgram(&prog);
    return b2_fail(B2_ERR_NVRTC, "no CUBIN produced for %s (pass --gpu-architecture=sm_100a)",
                   name);
  }
  if (cubin) {
    if (*cubin_size < sz) {
      nvrtcDestroyProgram(&prog);
      return b2_fail(B2_ERR_ARG, "cubin buffer too small (%zu < %zu)", *cubin_size, sz);
    }
    nvrtcGetCUBIN(prog, (char *)cubin);
  }
  *cubin_size = sz;
  nvrtcDestroyProgram(&prog);
  return B2_OK;
}

extern "C" int b2_module_load(const void *image, void **module) {
  int rc = load_driver();
  if (rc) return rc;
  return cu_check(drv.moduleLoadData((CUmodule *)module, image), "cuModuleLoadData");
}
extern "C" int b2_module_unload(void *module) {
  int rc = load_driver();
  if (rc) return rc;
  return cu_check(drv.moduleUnload((CUmodule)module), "cuModuleUnload");
}
extern "C" int b2_module_function(void *module, const char *kernel, void **fn) {
  int rc = load_driver();
  if (rc) return rc;
  return cu_check(drv.moduleGetFunction((CUfunction *)fn, (CUmodule)module, kernel),
                  "cuModuleGetFunction");
}
extern "C" int b2_func_set_max_smem(void *fn, int bytes) {
  int rc = load_driver();
  if (rc) return rc;
  return cu_check(drv.funcSetAttribute((CUfunction)fn,
                                       CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes),
                  "cuFuncSetAttribute");
}

// TMA descriptor for a row-major f64 tensor (tma3 stencil mode): dims and
// box innermost first, no swizzle, no L2 promotion (boxes rows are not
// 256-B aligned: promotion over-fetched 1.8x), zero fill outside the tensor.
typedef CUresult (*PFN_EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int b2_tensor_map_f64(void *out128, const void *base, int rank, const uint64_t *dims,
                                 const uint32_t *box) {
  static PFN_EncodeTiled enc = nullptr;
  if (!enc) {
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) !=
            cudaSuccess || !fp)
      return b2_fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    enc = (PFN_EncodeTiled)fp;
  }
  if (rank < 1 || rank > 5) return b2_fail(B2_ERR_ARG, "tensor map rank %d", rank);
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], es[5];
  uint64_t acc = 8;
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
    if (i > 0) st[i - 1] = acc;
    acc *= dims[i];
  }
  CUtensorMap m;
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void *>(base),
                   d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return b2_fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  memcpy(out128, &m, sizeof(m));
  return B2_OK;
}

static int launch_impl(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                       unsigned by, unsigned bz, unsigned smem, void *stream, const void *args,
                       size_t args_bytes, bool pdl, bool coop = false) {
  if (drv.status != 0) {
    int rc = load_driver();
    if (rc) return rc;
  }
  size_t sz = args_bytes;
  void *cfg[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<void *>(args),
                 CU_LAUNCH_PARAM_BUFFER_SIZE, &sz, CU_LAUNCH_PARAM_END};
  CUresult r;
  if (pdl || coop) {
    CUlaunchAttribute at[1];
    if (coop) {  // all CTAs co-resident (grid barriers), or the launch fails
      at[0].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
      at[0].value.cooperative = 1;
    } else {
      at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      at[0].value.programmaticStreamSerializationAllowed = 1;
    }
    CUlaunchConfig lc = {};
    lc.gridDimX = gx;
    lc.gridDimY = gy;
    lc.gridDimZ = gz;
    lc.blockDimX = bx;
    lc.blockDimY = by;
    lc.blockDimZ = bz;
    lc.sharedMemBytes = smem;
    lc.hStream = (CUstream)stream;
    lc.attrs = at;
    lc.numAttrs = 1;
    // cooperative launches take kernelParams, not the packed-buffer `extra`:
    // every kernel here has one by-value struct parameter, the blob itself
    void *params[] = {const_cast<void *>(args)};
    r = coop ? drv.launchKernelEx(&lc, (CUfunction)fn, params, nullptr)
             : drv.launchKernelEx(&lc, (CUfunction)fn, nullptr, cfg);
  } else {
    r = drv.launchKernel((CUfunction)fn, gx, gy, gz, bx, by, bz, smem, (CUstream)stream,
                         nullptr, cfg);
  }
  if (r != CUDA_SUCCESS) return cu_check(r, "cuLaunchKernel");
  b2_count_launch();
  return B2_OK;
}

extern "C" int b2_launch(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                         unsigned by, unsigned bz, unsigned smem, void *stream, const void *args,
                         size_t args_bytes) {
  // JIT kernels open with griddepcontrol.wait (prelude B2_PDL_ENTRY), so they
  // may be launched programmatically: the launch overlaps the tail of the
  // previous kernel in the stream (also as graph edges under capture)
  static int pdl = -1;
  if (pdl < 0) {  // opt-in, matching runtime.NVRTC_OPTS (-DB2_NO_PDL otherwise)
    const char *e = getenv("B2_PDL");
    pdl = e && e[0] == '1';
  }
  return launch_impl(fn, gx, gy, gz, bx, by, bz, smem, stream, args, args_bytes, pdl != 0);
}

extern "C" int b2_launch_coop(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                              unsigned by, unsigned bz, unsigned smem, void *stream,
                              const void *args, size_t args_bytes) {
  return launch_impl(fn, gx, gy, gz, bx, by, bz, smem, stream, args, args_bytes, false, true);
}

extern "C" int b2_launch_pdl(void *fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                             unsigned by, unsigned bz, unsigned smem, void *stream,
                             const void *args, size_t args_bytes) {
  return launch_impl(fn, gx, gy, gz, bx, by, bz, smem, stream, args, args_bytes, true);
}

// ---------------------------------------------------------------------------
// CUDA graphs: the host state machine is traced once under stream capture
// and replayed as one graph launch per call.

extern "C" int b2_capture_begin(void *stream) {
  return b2_cuda_check(
      cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal),
      "begin capture");
}

extern "C" int b2_capture_end(void *stream, void **graph_exec) {
  cudaGraph_t g = nullptr;
  int rc = b2_cuda_check(cudaStreamEndCapture((cudaStream_t)stream, &g), "end capture");
  if (rc) return rc;
  cudaGraphExec_t ex = nullptr;
  rc = b2_cuda_check(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
  cudaGraphDestroy(g);
  if (rc) return rc;
  *graph_exec = ex;
  return B2_OK;
}

// ---------------------------------------------------------------------------
// Device-side branches inside a capture: a CUDA conditional IF/ELSE node
// whose predicate (*flag != 0) is set on the device when the graph runs, so a
// transition condition that reads device data needs no host round trip.

namespace {
__global__ void b2_cond_set_kernel(cudaGraphConditionalHandle h, const int *flag) {
  cudaGraphSetConditional(h, *flag != 0 ? 1u : 0u);
}
__global__ void b2_counters_add_kernel(long long *c, long long a0, long long a1, long long a2,
                                       long long a3) {
  c[0] += a0;
  c[1] += a1;
  c[2] += a2;
  c[3] += a3;
}
}  // namespace

extern "C" int b2_capture_if_begin(void *stream, const int *flag, void **node, void **body_then,
                                   void **body_else) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaStreamCaptureStatus st;
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t *deps = nullptr;
  size_t nd = 0;
  B2_CLEAR_ERROR();
  int rc = b2_cuda_check(cudaStreamGetCaptureInfo(s, &st, nullptr, &graph, &deps, &nd),
                         "capture info");
  if (rc) return rc;
  if (st != cudaStreamCaptureStatusActive) return b2_fail(B2_ERR_ARG, "stream is not capturing");
  cudaGraphConditionalHandle h;
  rc = b2_cuda_check(cudaGraphConditionalHandleCreate(&h, graph, 0, 0), "conditional handle");
  if (rc) return rc;
  b2_cond_set_kernel<<<1, 1, 0, s>>>(h, flag);
  B2_LAUNCH_CHECK("conditional set");
  rc = b2_cuda_check(cudaStreamGetCaptureInfo(s, &st, nullptr, &graph, &deps, &nd),
                     "capture info");
  if (rc) return rc;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 2;  // body 0 when the value is non-zero, body 1 otherwise
  cudaGraphNode_t n = nullptr;
  rc = b2_cuda_check(cudaGraphAddNode(&n, graph, deps, nd, &p), "conditional node");
  if (rc) return rc;
  *node = n;
  *body_then = p.conditional.phGraph_out[0];
  *body_else = p.conditional.phGraph_out[1];
  return B2_OK;
}

extern "C" int b2_capture_if_end(void *stream, void *node) {
  cudaGraphNode_t n = (cudaGraphNode_t)node;
  return b2_cuda_check(cudaStreamUpdateCaptureDependencies((cudaStream_t)stream, &n, 1,
                                                           cudaStreamSetCaptureDependencies),
                       "capture dependencies");
}

extern "C" int b2_capture_body_begin(void *body_stream, void *body_graph) {
  return b2_cuda_check(cudaStreamBeginCaptureToGraph((cudaStream_t)body_stream,
                                                     (cudaGraph_t)body_graph, nullptr, nullptr,
                                                     0, cudaStreamCaptureModeThreadLocal),
                       "begin body capture");
}

extern "C" int b2_capture_body_end(void *body_stream) {
  cudaGraph_t g = nullptr;
  return b2_cuda_check(cudaStreamEndCapture((cudaStream_t)body_stream, &g), "end body capture");
}

extern "C" int b2_counters_add(long long *dev, long long a0, long long a1, long long a2,
                               long long a3, void *stream) {
  B2_CLEAR_ERROR();
  b2_counters_add_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(dev, a0, a1, a2, a3);
  B2_LAUNCH_CHECK("counters add");
  return B2_OK;
}

extern "C" int b2_graph_launch(void *graph_exec, void *stream) {
  return b2_cuda_check(cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream),
                       "graph launch");
}

extern "C" int b2_graph_destroy(void *graph_exec) {
  return b2_cuda_check(cudaGraphExecDestroy((cudaGraphExec_t)graph_exec), "graph destroy");
}
