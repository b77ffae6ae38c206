"""ctypes binding of libb2.so (include/b2.h) and the NVRTC kernel cache.

This is the only place the host side crosses into native code.  There is no
CPU fallback: if the shared library is missing or no CUDA device is visible,
``lib()``/``device()`` raise ``BackendUnavailable`` and the executor fails
loudly.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import pathlib
import threading

PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG / "libb2.so"
FAMILIES = PKG / "csrc" / "families"
CACHE_DIR = pathlib.Path(os.environ.get("B2_JIT_CACHE", PKG.parent / "build" / "jit_cache"))

B2_F64, B2_I64, B2_I32, B2_BOOL, B2_F32 = 0, 1, 2, 3, 4
DTYPE_CODE = {"f64": B2_F64, "i64": B2_I64, "i32": B2_I32, "bool": B2_BOOL, "f32": B2_F32}
WCR_CODE = {None: 0, "add": 1, "mul": 2, "min": 3, "max": 4}
MAX_DIMS = 8

NVRTC_OPTS = [
    "--gpu-architecture=sm_100a",
    "--std=c++17",
    "--fmad=false",  # Python evaluates op by op: no contraction
    "-default-device",
    "-lineinfo",
]
# programmatic dependent launch is opt-in (B2_PDL=1): measured slower on the
# benchmark programs (heat_3d 41.1 vs 39.9 ms, jacobi_2d 1.92 vs 1.83 ms,
# go_fast 0.435 vs 0.377 ms), faster only on launch-bound nbody (-3 %)
if os.environ.get("B2_PDL", "0") != "1":  # must match b2_launch
    NVRTC_OPTS.append("-DB2_NO_PDL")


class BackendUnavailable(RuntimeError):
    pass


class B2Error(RuntimeError):
    pass


class View(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_void_p),
        ("offset", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("shape", ctypes.c_int64 * MAX_DIMS),
        ("strides", ctypes.c_int64 * MAX_DIMS),
    ]


class DeviceInfo(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 128),
        ("major", ctypes.c_int),
        ("minor", ctypes.c_int),
        ("sm_count", ctypes.c_int),
        ("l2_bytes", ctypes.c_int),
        ("max_smem_optin", ctypes.c_int),
        ("total_mem", ctypes.c_size_t),
    ]


# Every symbol include/b2.h declares (the CPU test tier checks the exports).
EXPORTS = [
    "b2_version", "b2_last_error", "b2_init", "b2_device_count", "b2_device_info",
    "b2_malloc", "b2_free", "b2_memcpy_h2d", "b2_memcpy_d2h", "b2_memcpy_d2d", "b2_memset",
    "b2_stream_create", "b2_stream_destroy", "b2_stream_sync", "b2_device_sync",
    "b2_event_create", "b2_event_destroy", "b2_event_record", "b2_event_record_external",
    "b2_event_elapsed_ms",
    "b2_stream_wait_event", "b2_capture_if_begin", "b2_capture_if_end", "b2_capture_body_begin",
    "b2_capture_body_end", "b2_counters_add",
    "b2_host_register", "b2_host_unregister", "b2_ipc_handle", "b2_ipc_open", "b2_ipc_close",
    "b2_jit_compile", "b2_module_load",
    "b2_module_unload", "b2_module_function", "b2_func_set_max_smem", "b2_launch", "b2_launch_pdl", "b2_launch_coop",
    "b2_launch_count", "b2_capture_begin", "b2_capture_end", "b2_graph_launch",
    "b2_graph_destroy", "b2_copy_view", "b2_fill_view", "b2_gemm_f64", "b2_gemm_f32",
    "b2_reduce", "b2_nccl_unique_id", "b2_nccl_init", "b2_nccl_destroy", "b2_nccl_group_p2p",
    "b2_nccl_bcast", "b2_nccl_allreduce_f64", "b2_tensor_map_f64",
    "b2_gemm_f32_f64acc", "b2_tf32_split_cols", "b2_tf32_split_a", "b2_tf32_split_bt",
    "b2_gemm_f32_presplit",
]


class P2P(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("bytes", ctypes.c_size_t), ("peer", ctypes.c_int),
                ("send", ctypes.c_int)]

_lock = threading.Lock()
_lib = None
_dev_inited: set[int] = set()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_SIGS = {
    "b2_version": ([], ctypes.c_int),
    "b2_last_error": ([], ctypes.c_char_p),
    "b2_init": ([ctypes.c_int], ctypes.c_int),
    "b2_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "b2_device_info": ([ctypes.c_int, ctypes.POINTER(DeviceInfo)], ctypes.c_int),
    "b2_malloc": ([ctypes.POINTER(_vp), ctypes.c_size_t], ctypes.c_int),
    "b2_free": ([_vp], ctypes.c_int),
    "b2_memcpy_h2d": ([_vp, _vp, ctypes.c_size_t, _vp], ctypes.c_int),
    "b2_memcpy_d2h": ([_vp, _vp, ctypes.c_size_t, _vp], ctypes.c_int),
    "b2_memcpy_d2d": ([_vp, _vp, ctypes.c_size_t, _vp], ctypes.c_int),
    "b2_memset": ([_vp, ctypes.c_int, ctypes.c_size_t, _vp], ctypes.c_int),
    "b2_stream_create": ([ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_stream_destroy": ([_vp], ctypes.c_int),
    "b2_stream_sync": ([_vp], ctypes.c_int),
    "b2_device_sync": ([], ctypes.c_int),
    "b2_event_create": ([ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_event_destroy": ([_vp], ctypes.c_int),
    "b2_event_record": ([_vp, _vp], ctypes.c_int),
    "b2_event_record_external": ([_vp, _vp], ctypes.c_int),
    "b2_event_elapsed_ms": ([_vp, _vp, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
    "b2_stream_wait_event": ([_vp, _vp], ctypes.c_int),
    "b2_capture_if_begin": ([_vp, _vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                             ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_capture_if_end": ([_vp, _vp], ctypes.c_int),
    "b2_capture_body_begin": ([_vp, _vp], ctypes.c_int),
    "b2_capture_body_end": ([_vp], ctypes.c_int),
    "b2_counters_add": ([_vp, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong,
                         ctypes.c_longlong, _vp], ctypes.c_int),
    "b2_host_register": ([_vp, ctypes.c_size_t], ctypes.c_int),
    "b2_ipc_handle": ([_vp, _vp], ctypes.c_int),
    "b2_ipc_open": ([_vp, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "b2_ipc_close": ([_vp], ctypes.c_int),
    "b2_host_unregister": ([_vp], ctypes.c_int),
    "b2_jit_compile": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p),
                        ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_size_t), ctypes.c_char_p,
                        ctypes.c_size_t], ctypes.c_int),
    "b2_module_load": ([_vp, ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_module_unload": ([_vp], ctypes.c_int),
    "b2_module_function": ([_vp, ctypes.c_char_p, ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_func_set_max_smem": ([_vp, ctypes.c_int], ctypes.c_int),
    "b2_launch": ([_vp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint,
                   ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _vp, _vp, ctypes.c_size_t],
                  ctypes.c_int),
    "b2_launch_pdl": ([_vp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint,
                       ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _vp, _vp, ctypes.c_size_t],
                      ctypes.c_int),
    "b2_launch_coop": ([_vp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint,
                        ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _vp, _vp, ctypes.c_size_t],
                       ctypes.c_int),
    "b2_launch_count": ([], ctypes.c_int64),
    "b2_capture_begin": ([_vp], ctypes.c_int),
    "b2_capture_end": ([_vp, ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_graph_launch": ([_vp, _vp], ctypes.c_int),
    "b2_graph_destroy": ([_vp], ctypes.c_int),
    "b2_copy_view": ([ctypes.POINTER(View), ctypes.POINTER(View), ctypes.c_int, _vp],
                     ctypes.c_int),
    "b2_fill_view": ([ctypes.POINTER(View), ctypes.c_double, _vp], ctypes.c_int),
    "b2_gemm_f64": ([_i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64,
                     ctypes.c_int, _vp], ctypes.c_int),
    "b2_gemm_f32": ([_i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64,
                     ctypes.c_int, _vp], ctypes.c_int),
    "b2_reduce": ([ctypes.POINTER(View), ctypes.POINTER(View), ctypes.c_uint, ctypes.c_int,
                   ctypes.c_int, _vp], ctypes.c_int),
    "b2_nccl_unique_id": ([_vp], ctypes.c_int),
    "b2_nccl_init": ([ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(_vp)], ctypes.c_int),
    "b2_nccl_destroy": ([_vp], ctypes.c_int),
    "b2_nccl_group_p2p": ([_vp, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "b2_nccl_bcast": ([_vp, _vp, ctypes.c_size_t, ctypes.c_int, _vp], ctypes.c_int),
    "b2_nccl_allreduce_f64": ([_vp, _vp, ctypes.c_size_t, ctypes.c_int, _vp], ctypes.c_int),
    "b2_tf32_split_cols": ([_i64], _i64),
    "b2_tf32_split_a": ([_vp, _i64, _i64, _i64, _vp, _vp], ctypes.c_int),
    "b2_tf32_split_bt": ([_vp, _i64, _i64, _i64, _vp, _vp], ctypes.c_int),
    "b2_gemm_f32_presplit": ([_i64, _i64, _i64, _vp, _vp, _vp, _i64, ctypes.c_int, _vp],
                             ctypes.c_int),
    "b2_gemm_f32_f64acc": ([_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, ctypes.c_int,
                            _vp], ctypes.c_int),
    "b2_tensor_map_f64": ([_vp, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                           ctypes.POINTER(ctypes.c_uint32)], ctypes.c_int),
}


def load_library(path: pathlib.Path | None = None):
    """Load libb2.so and declare signatures (works without a GPU)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path or LIB_PATH)
        if not p.exists():
            raise BackendUnavailable(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if path is None:
            _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().b2_last_error().decode(errors="replace")
        raise B2Error(f"{what}: {msg}" if what else msg)


def device(index: int = 0) -> int:
    """Initialise the CUDA context on ``index`` (fails loudly without a GPU)."""
    L = lib()
    if index in _dev_inited:
        return index
    n = ctypes.c_int(0)
    L.b2_device_count(ctypes.byref(n))
    if n.value <= index:
        raise BackendUnavailable(f"no CUDA device {index} (found {n.value}); the B200 backend "
                                 "has no CPU fallback")
    check(L.b2_init(index), "b2_init")
    _dev_inited.add(index)
    return index


def device_info(index: int = 0) -> DeviceInfo:
    info = DeviceInfo()
    check(lib().b2_device_info(index, ctypes.byref(info)), "device_info")
    return info


# ---------------------------------------------------------------------------
# JIT: NVRTC compile (cached in-process and on disk by source hash).


class Kernel:
    __slots__ = ("module", "fn", "name", "source_hash")

    def __init__(self, module, fn, name, source_hash):
        self.module = module
        self.fn = fn
        self.name = name
        self.source_hash = source_hash


_kcache: dict[tuple[str, str], Kernel] = {}
_prelude_cache: dict[str, str] = {}


def family_source(name: str) -> str:
    s = _prelude_cache.get(name)
    if s is None:
        s = (FAMILIES / name).read_text()
        _prelude_cache[name] = s
    return s


def compile_cubin(src: str, name: str, extra_opts=()) -> bytes:
    """NVRTC compile for sm_100a; pure host work (usable without a GPU)."""
    L = lib()
    opts = [o.encode() for o in list(NVRTC_OPTS) + list(extra_opts)]
    arr = (ctypes.c_char_p * len(opts))(*opts)
    size = ctypes.c_size_t(0)
    log = ctypes.create_string_buffer(1 << 16)
    rc = L.b2_jit_compile(src.encode(), name.encode(), arr, len(opts), None, ctypes.byref(size),
                          log, len(log))
    check(rc, "nvrtc")
    buf = ctypes.create_string_buffer(size.value)
    check(L.b2_jit_compile(src.encode(), name.encode(), arr, len(opts), buf, ctypes.byref(size),
                           None, 0), "nvrtc")
    return buf.raw[: size.value]


def get_cubin(src: str, name: str, extra_opts=()) -> tuple[bytes, str]:
    h = hashlib.sha256((src + "\0" + " ".join(NVRTC_OPTS + list(extra_opts))).encode()).hexdigest()[:32]
    path = CACHE_DIR / f"{name}-{h}.cubin"
    if path.exists():
        return path.read_bytes(), h
    cub = compile_cubin(src, name, extra_opts)
    try:
        CACHE_DIR.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".tmp{os.getpid()}")
        tmp.write_bytes(cub)
        tmp.replace(path)
    except OSError:
        pass
    return cub, h


def get_kernel(src: str, name: str, extra_opts=(), max_smem: int = 0) -> Kernel:
    key = (name, src)
    k = _kcache.get(key)
    if k is not None:
        return k
    # launched with programmatic stream serialization (b2_launch): every JIT
    # kernel must wait on its predecessor before touching memory
    if src.count("__global__") != src.count("B2_PDL_ENTRY();"):
        raise B2Error(f"kernel source for {name} lacks B2_PDL_ENTRY() in a __global__ function")
    cub, h = get_cubin(src, name, extra_opts)
    L = lib()
    mod = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(cub, len(cub))
    check(L.b2_module_load(buf, ctypes.byref(mod)), f"load {name}")
    fn = ctypes.c_void_p()
    check(L.b2_module_function(mod, name.encode(), ctypes.byref(fn)), f"function {name}")
    if max_smem > 48 * 1024:
        check(L.b2_func_set_max_smem(fn, max_smem), "max smem")
    k = Kernel(mod, fn, name, h)
    _kcache[key] = k
    return k


def launch(k: Kernel, grid, block, args_blob: bytes, stream, smem: int = 0,
           pdl: bool = False, coop: bool = False) -> None:
    """pdl: programmatic dependent launch (the kernel must open with
    griddepcontrol.wait, i.e. be compiled with B2_PDL_ENTRY enabled)."""
    gx, gy, gz = (tuple(grid) + (1, 1, 1))[:3]
    bx, by, bz = (tuple(block) + (1, 1, 1))[:3]
    fn = lib().b2_launch_coop if coop else (lib().b2_launch_pdl if pdl else lib().b2_launch)
    check(fn(k.fn, gx, gy, gz, bx, by, bz, smem, stream, args_blob, len(args_blob)),
          f"launch {k.name}")


_tmap_cache: dict = {}


def tensor_map_f64(base: int, shape, box) -> bytes:
    """128-byte TMA descriptor of a row-major f64 tensor (shape outermost
    first, box innermost first), cached per (base, shape, box)."""
    key = (base, tuple(shape), tuple(box))
    hit = _tmap_cache.get(key)
    if hit is None:
        dims = (ctypes.c_uint64 * len(shape))(*reversed([int(x) for x in shape]))
        bx = (ctypes.c_uint32 * len(box))(*[int(x) for x in box])
        out = ctypes.create_string_buffer(128)
        check(lib().b2_tensor_map_f64(out, base, len(shape), dims, bx), "tensor map")
        hit = _tmap_cache[key] = out.raw
    return hit


def make_view(base: int, offset: int, dtype: str, shape, strides) -> View:
    v = View()
    v.base = base
    v.offset = offset
    v.dtype = DTYPE_CODE[dtype]
    v.ndim = len(shape)
    if len(shape) > MAX_DIMS:
        raise B2Error(f"view rank {len(shape)} exceeds {MAX_DIMS}")
    for i, (s, t) in enumerate(zip(shape, strides)):
        v.shape[i] = int(s)
        v.strides[i] = int(t)
    return v
