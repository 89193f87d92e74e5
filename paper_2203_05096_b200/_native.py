"""ctypes binding of libcsrk_cuda.so (the C-ABI declared in include/csrk.h).

There is no fallback: if the library is missing or a CUDA call fails, the
error propagates.  Error codes map to the exception types the reference
raises for the same conditions (ValueError for invalid arguments).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# CSRK_LIB: an alternative build of the same library (A/B experiments, tools/build_variant.sh)
LIB_PATH = os.environ.get("CSRK_LIB") or os.path.join(_PKG, "lib", "libcsrk_cuda.so")

CSRK_OK, CSRK_EINVAL, CSRK_ECUDA, CSRK_ENOMEM, CSRK_ENCCL = 0, 1, 2, 3, 4
CSRK_MG_HALO, CSRK_MG_ALLGATHER, CSRK_MG_ID_BYTES = 0, 1, 128
CSRK_F64, CSRK_F32 = 1, 2
CSRK_SERIAL, CSRK_STRIDED = 0, 1

_lock = threading.Lock()
_lib = None

P = C.c_void_p
I64 = C.c_int64
U32P = C.POINTER(C.c_uint32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)

_SIGNATURES = {
    "csrk_abi_version": ([], C.c_int),
    "csrk_last_error": ([], C.c_char_p),
    "csrk_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "csrk_buffer_alloc": ([C.c_int, I64, C.POINTER(P)], C.c_int),
    "csrk_buffer_free": ([C.c_int, P], C.c_int),
    "csrk_memcpy": ([P, P, I64, C.c_int, P], C.c_int),
    "csrk_memset": ([P, C.c_int, I64, P], C.c_int),
    "csrk_stream_sync": ([P], C.c_int),
    "csrk_device_sync": ([C.c_int], C.c_int),
    "csrk_matrix_upload": ([C.c_int, I64, I64, I64, U32P, U32P, F64P, C.c_int, I64,
                            U32P, I64, U32P, C.c_int, C.POINTER(P)], C.c_int),
    "csrk_matrix_free": ([P], C.c_int),
    "csrk_matrix_shape": ([P, I64P], C.c_int),
    "csrk_matrix_download": ([P, U32P, U32P, F64P, U32P, U32P], C.c_int),
    "csrk_matrix_add_f32": ([P], C.c_int),
    "csrk_matrix_set_plan": ([P, I64, I64, I64], C.c_int),
    "csrk_matrix_plan": ([P, I64P], C.c_int),
    "csrk_matrix_plan_ctas": ([P, C.c_int, I64P], C.c_int),
    "csrk_matrix_set_schedule": ([P, C.c_int, C.c_int], C.c_int),
    "csrk_matrix_set_cut_mode": ([P, C.c_int], C.c_int),
    "csrk_matrix_prepare": ([P, C.c_int, C.c_int, C.c_int], C.c_int),
    "csrk_spmv": ([P, C.c_int, C.c_int, C.c_int, P, P, P], C.c_int),
    "csrk_spmv_tiles": ([P, C.c_int, C.c_int, C.c_int, P, P, I64, I64, P], C.c_int),
    "csrk_matrix_tile_rows": ([P, U32P], C.c_int),
    "csrk_spmv_host": ([P, C.c_int, C.c_int, C.c_int, P, P], C.c_int),
    "csrk_last_kernel_ms": ([P, C.POINTER(C.c_float)], C.c_int),
    "csrk_spmv_listing3": ([P, C.c_int, C.c_int, P, P, P, P], C.c_int),
    "csrk_spmv_listing4": ([P, C.c_int, C.c_int, C.c_int, P, P, P, P], C.c_int),
    "csrk_probe_gather": ([P, C.c_int, P, P, P], C.c_int),
    "csrk_pack": ([C.c_int, I64, I64, U32P, U32P, F64P, I64P, I64P, C.c_int, I64,
                   I64P, I64, I64P, C.POINTER(P)], C.c_int),
    "csrk_gather_f64": ([I64, P, P, P, P], C.c_int),
    "csrk_stats": ([P, I64P], C.c_int),
    "csrk_row_variance": ([P, C.c_double, F64P], C.c_int),
    "csrk_matrix_group_uniform": ([P, I64, I64], C.c_int),
    "csrk_cg": ([P, C.c_int, C.c_int, C.c_int, P, P, P, P, P, C.c_int, F64P, P], C.c_int),
    "csrk_power": ([P, C.c_int, C.c_int, C.c_int, P, P, C.c_int, P], C.c_int),
    "csrk_vec_dot": ([C.c_int, I64, P, P, P, P, P, P], C.c_int),
    "csrk_cg_update": ([C.c_int, I64, P, P, P, P, P, P, P, P], C.c_int),
    "csrk_cg_direction": ([C.c_int, I64, P, P, P, P, P], C.c_int),
    "csrk_dgraph_build": ([P, C.POINTER(P)], C.c_int),
    "csrk_dgraph_relabel": ([P, I64P, C.POINTER(P)], C.c_int),
    "csrk_dgraph_contract": ([P, I64P, I64, C.POINTER(P)], C.c_int),
    "csrk_dgraph_sizes": ([P, I64P], C.c_int),
    "csrk_dgraph_download": ([P, I64P, I64P, I64P, I64P], C.c_int),
    "csrk_dgraph_free": ([P], C.c_int),
    "csrk_dgraph_wbo": ([P, I64P], C.c_int),
    "csrk_dgraph_match": ([P, I64P, C.POINTER(C.c_int)], C.c_int),
    "csrk_dgraph_coarsen": ([P, C.c_double, I64P, C.POINTER(P)], C.c_int),
    "csrk_band_k_device": ([P, C.c_int, F64P, C.POINTER(P)], C.c_int),
    "csrk_sort_pairs": ([C.c_int, I64, P, P, C.c_int, C.c_int, P], C.c_int),
    "csrk_stencil": ([C.c_int, I64, I64, I64, C.c_int, C.POINTER(P)], C.c_int),
    "csrk_coo_to_csr": ([C.c_int, I64, I64, I64, I64P, I64P, F64P, C.POINTER(P)], C.c_int),
    "csrk_mm_parse": ([C.c_char_p, I64, I64, C.c_int, I64, I64, C.c_int, I64P, I64P, F64P],
                      C.c_int),
    "csrk_stencil_slab": ([C.c_int, I64, I64, I64, C.c_int, I64, I64, C.POINTER(P)],
                          C.c_int),
    "csrk_band_k": ([I64, U32P, U32P, C.c_int, F64P, C.POINTER(P)], C.c_int),
    "csrk_bandk_result_sizes": ([P, I64P], C.c_int),
    "csrk_bandk_result_get": ([P, I64P, I64P, I64P], C.c_int),
    "csrk_bandk_result_free": ([P], C.c_int),
    "csrk_heavy_edge_matching": ([I64, I64P, I64P, I64P, I64P], C.c_int),
    "csrk_weighted_bandwidth_order": ([I64, I64P, I64P, I64P, I64P], C.c_int),
    "csrk_build_graph": ([I64, U32P, U32P, C.POINTER(P)], C.c_int),
    "csrk_coarsen": ([I64, I64P, I64P, I64P, I64P, C.c_double, C.POINTER(P)], C.c_int),
    "csrk_graph_sizes": ([P, I64P], C.c_int),
    "csrk_graph_get": ([P, I64P, I64P, I64P, I64P, I64P], C.c_int),
    "csrk_graph_free": ([P], C.c_int),
    "csrk_mg_partition": ([U32P, U32P, U32P, I64, C.c_int, I64P], C.c_int),
    "csrk_mg_footprints": ([U32P, U32P, I64P, C.c_int, I64P], C.c_int),
    "csrk_mg_plan": ([C.c_int, I64P, I64P, I64P, I64, I64P], C.c_int),
    "csrk_mg_unique_id": ([C.c_char_p], C.c_int),
    "csrk_mg_create": ([C.c_int, C.c_int, C.c_char_p, I64P, I64P, P, I64, C.c_int,
                        C.POINTER(P)], C.c_int),
    "csrk_mg_spmv": ([P, C.c_int, C.c_int, C.c_int, P, P, P], C.c_int),
    "csrk_mg_info": ([P, I64P], C.c_int),
    "csrk_mg_destroy": ([P], C.c_int),
}

EXPORTED = tuple(_SIGNATURES)


def lib():
    """The loaded library; raises if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_2203_05096_b200.build` (there is no CPU fallback)")
            handle = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = res
            _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == CSRK_OK:
        return
    msg = lib().csrk_last_error().decode(errors="replace")
    if rc == CSRK_EINVAL:
        raise ValueError(msg)
    if rc == CSRK_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def call_rc(name: str, *args) -> int:
    """Call without raising; returns the CSRK_* code."""
    return int(getattr(lib(), name)(*args))


def u32p(a: np.ndarray):
    return a.ctypes.data_as(U32P)


def i64p(a: np.ndarray):
    return a.ctypes.data_as(I64P)


def f64p(a: np.ndarray):
    return a.ctypes.data_as(F64P)


def vp(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


_device = None


def current_device() -> int:
    """Device ordinal used for new device objects: set_device(), else
    LOCAL_RANK (one process per GPU), else CSRK_DEVICE, else 0."""
    if _device is not None:
        return _device
    for var in ("CSRK_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var, "").strip()
        if v.isdigit():
            return int(v)
    return 0


def set_device(device: int) -> None:
    global _device
    _device = int(device)


def warm_up() -> None:
    """Create the CUDA context of the process's device at package import
    (when the library is built and a GPU is present), so the first call --
    a pack_csrk of a 9 x 9 matrix in the reference's acceptance criterion 1,
    budget 1 s -- does not pay the context creation.  CSRK_LAZY_INIT=1 skips
    it; without a GPU nothing happens (every compute call still raises)."""
    if os.environ.get("CSRK_LAZY_INIT") == "1" or not os.path.exists(LIB_PATH):
        return
    try:
        if device_count() > 0:
            lib().csrk_device_sync(current_device())
    except Exception:  # a broken driver surfaces at the first real call
        pass


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().csrk_device_count(C.byref(n))
    if rc != CSRK_OK:
        return 0
    return int(n.value)


class DeviceBuffer:
    """A raw cudaMalloc allocation owned by Python."""

    __slots__ = ("ptr", "nbytes", "device")

    def __init__(self, nbytes: int, device=None):
        self.device = current_device() if device is None else int(device)
        self.nbytes = int(nbytes)
        out = C.c_void_p()
        call("csrk_buffer_alloc", self.device, self.nbytes, C.byref(out))
        self.ptr = out

    @property
    def address(self) -> int:
        return int(self.ptr.value or 0)

    @classmethod
    def from_array(cls, a: np.ndarray, device=None):
        a = np.ascontiguousarray(a)
        buf = cls(a.nbytes, device)
        call("csrk_memcpy", buf.ptr, vp(a), a.nbytes, 0, None)
        return buf

    def to_array(self, dtype, count) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        call("csrk_memcpy", vp(out), self.ptr, out.nbytes, 1, None)
        return out

    def __del__(self):
        ptr = getattr(self, "ptr", None)
        if ptr and _lib is not None:
            try:
                _lib.csrk_buffer_free(self.device, ptr)
            except Exception:
                pass
            self.ptr = None


class DeviceMatrix:
    """Owner of a csrk_matrix* (device-resident CSR / CSR-k arrays)."""

    __slots__ = ("ptr", "n_rows", "n_cols", "nnz", "k", "n_sr", "n_ssr", "device",
                 "__weakref__")

    def __init__(self, ptr: C.c_void_p):
        self.ptr = ptr
        shape = np.zeros(7, dtype=np.int64)
        call("csrk_matrix_shape", ptr, i64p(shape))
        (self.n_rows, self.n_cols, self.nnz, self.k, self.n_sr, self.n_ssr,
         self.device) = (int(v) for v in shape)

    @classmethod
    def upload(cls, row_ptr, col_idx, vals, n_rows, n_cols, k=1, sr_ptr=None,
               ssr_ptr=None, device=None, f32=False):
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint32)
        ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
        va = np.ascontiguousarray(vals, dtype=np.float64)
        sp = np.ascontiguousarray(sr_ptr if sr_ptr is not None else [0], dtype=np.uint32)
        ssp = np.ascontiguousarray(ssr_ptr if ssr_ptr is not None else [0], dtype=np.uint32)
        out = C.c_void_p()
        call("csrk_matrix_upload", current_device() if device is None else device,
             n_rows, n_cols, len(ci), u32p(rp), u32p(ci), f64p(va), k,
             len(sp) - 1, u32p(sp), len(ssp) - 1, u32p(ssp),
             CSRK_F64 | (CSRK_F32 if f32 else 0), C.byref(out))
        return cls(out)

    def download(self):
        rp = np.empty(self.n_rows + 1, dtype=np.uint32)
        ci = np.empty(self.nnz, dtype=np.uint32)
        va = np.empty(self.nnz, dtype=np.float64)
        sp = np.empty(self.n_sr + 1, dtype=np.uint32) if self.k >= 2 else None
        ssp = np.empty(self.n_ssr + 1, dtype=np.uint32) if self.k == 3 else None
        call("csrk_matrix_download", self.ptr, u32p(rp), u32p(ci), f64p(va),
             u32p(sp) if sp is not None else None,
             u32p(ssp) if ssp is not None else None)
        return rp, ci, va, sp, ssp

    def refresh(self):
        shape = np.zeros(7, dtype=np.int64)
        call("csrk_matrix_shape", self.ptr, i64p(shape))
        (self.n_rows, self.n_cols, self.nnz, self.k, self.n_sr, self.n_ssr,
         self.device) = (int(v) for v in shape)

    def group_uniform(self, srs: int, ssrs: int):
        """Make this handle CSR-k (k = 3) with uniform group sizes."""
        call("csrk_matrix_group_uniform", self.ptr, int(srs), int(ssrs))
        self.refresh()
        return self

    def ensure_f32(self):
        call("csrk_matrix_add_f32", self.ptr)

    def set_plan(self, tile_cost=0, cap=0, stages=0):
        """Streaming-kernel tile plan (0 = defaults); see include/csrk.h."""
        call("csrk_matrix_set_plan", self.ptr, int(tile_cost), int(cap), int(stages))

    def set_schedule(self, gather: int = 0, ctas_per_sm: int = 0):
        """Streaming-kernel schedule (see include/csrk.h): x-gather mode
        (0 inline, 1 gather-first) and resident CTAs per SM (0 = default)."""
        call("csrk_matrix_set_schedule", self.ptr, int(gather), int(ctas_per_sm))

    def set_cut_mode(self, mode: int):
        """Tile cuts: 0 auto, 1 rows, 2 group (SSR) boundaries (include/csrk.h)."""
        call("csrk_matrix_set_cut_mode", self.ptr, int(mode))

    def prepare(self, variant=CSRK_SERIAL, nx=1, f32=False):
        """Build the tile plan a launch of this order would use (no launch)."""
        call("csrk_matrix_prepare", self.ptr, CSRK_F32 if f32 else CSRK_F64, variant, nx)

    def plan(self, f32: bool = False) -> dict:
        """The tile plan; ``ctas_per_sm`` is the figure a launch with the
        given value type uses (fp32 runs more CTAs on regular rows)."""
        out = np.zeros(10, dtype=np.int64)
        call("csrk_matrix_plan", self.ptr, i64p(out))
        keys = ("tile_cost", "cap", "rcap", "stages", "n_tiles", "group_aligned",
                "gather_first", "ctas_per_sm", "cut_mode", "n_long")
        d = {k: int(v) for k, v in zip(keys, out)}
        c = np.zeros(1, dtype=np.int64)
        call("csrk_matrix_plan_ctas", self.ptr, CSRK_F32 if f32 else CSRK_F64, i64p(c))
        d["ctas_per_sm"] = int(c[0])
        return d

    def stats(self):
        out = np.zeros(5, dtype=np.int64)
        call("csrk_stats", self.ptr, i64p(out))
        return out

    def spmv_host(self, x: np.ndarray, variant=CSRK_SERIAL, nx=1, f32=False, out=None):
        dt = np.float32 if f32 else np.float64
        x = np.ascontiguousarray(x, dtype=dt)
        if out is None:
            y = np.empty(self.n_rows, dtype=dt)
        else:
            y = out
            if y.dtype != dt or y.shape != (self.n_rows,) or not y.flags.c_contiguous \
                    or not y.flags.writeable:
                raise ValueError(f"out must be a writable contiguous {np.dtype(dt).name} "
                                 f"array of length {self.n_rows}")
        call("csrk_spmv_host", self.ptr, CSRK_F32 if f32 else CSRK_F64, variant, nx,
             vp(x), vp(y))
        return y

    def spmv_ptr(self, x_ptr: int, y_ptr: int, stream: int = 0, variant=CSRK_SERIAL,
                 nx=1, f32=False):
        call("csrk_spmv", self.ptr, CSRK_F32 if f32 else CSRK_F64, variant, nx,
             C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(stream))

    def spmv_tiles_ptr(self, x_ptr: int, y_ptr: int, t0: int, t1: int, stream: int = 0,
                       variant=CSRK_SERIAL, nx=1, f32=False):
        """csrk_spmv over the plan's tiles [t0, t1) only."""
        call("csrk_spmv_tiles", self.ptr, CSRK_F32 if f32 else CSRK_F64, variant, nx,
             C.c_void_p(x_ptr), C.c_void_p(y_ptr), int(t0), int(t1), C.c_void_p(stream))

    def tile_rows(self) -> np.ndarray:
        """Row bounds of the plan's tiles (n_tiles + 1 entries)."""
        out = np.empty(self.plan()["n_tiles"] + 1, dtype=np.uint32)
        call("csrk_matrix_tile_rows", self.ptr, u32p(out))
        return out

    def last_kernel_ms(self) -> float:
        ms = C.c_float(0.0)
        call("csrk_last_kernel_ms", self.ptr, C.byref(ms))
        return float(ms.value)

    def __del__(self):
        ptr = getattr(self, "ptr", None)
        if ptr and _lib is not None:
            try:
                _lib.csrk_matrix_free(ptr)
            except Exception:  # interpreter shutdown
                pass
            self.ptr = None
