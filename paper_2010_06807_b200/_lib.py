"""ctypes binding of ``libspaqr_b200.so`` (the C-ABI in include/spaqr_b200.h).

There is no fallback: if the shared library is missing or no sm_100a device
is present, loading raises — the B200 path never silently drops to a CPU
implementation.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import (SPQ_ERR_BAD_INPUT, SPQ_ERR_ILL_CONDITIONED, SPQ_ERR_SINGULAR, SPQ_ERR_SPECULATION,
                     IllConditionedInterfaceError, SpeculationError, DeviceError, NestqrError,
                     SingularPivotError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspaqr_b200.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_ctx = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/spaqr_b200.h
SIGNATURES = {
    "spq_version": (C.c_int, []),
    "spq_device_info": (C.c_int, [C.c_char_p, C.c_int]),
    "spq_create": (C.c_int, [C.POINTER(_ctx), C.c_int]),
    "spq_destroy": (None, [_ctx]),
    "spq_last_error": (C.c_int, [_ctx, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_double), C.c_char_p, C.c_int]),
    "spq_set_option": (C.c_int, [_ctx, C.c_char_p, C.c_int64]),
    "spq_load": (C.c_int, [_ctx, C.c_int64, _i64p, _i64p, _f64p, C.c_int, C.c_int, C.c_int,
                           _i32p, _i64p, _i64p, _i64p, _i64p]),
    "spq_factor": (C.c_int, [_ctx, C.c_int, _i32p]),
    "spq_scale": (C.c_int, [_ctx, C.c_int, _i32p, _i32p]),
    "spq_sparsify": (C.c_int, [_ctx, C.c_int, _i32p, C.c_double, _i32p, _i32p, _f64p, _i32p]),
    "spq_sparsify_ex": (C.c_int, [_ctx, C.c_int, _i32p, C.c_double, C.c_int, C.c_int, _i32p,
                                  _i32p, _f64p, _i32p]),
    "spq_merge": (C.c_int, [_ctx, C.c_int, _i32p, _i32p, _i32p]),
    "spq_finish": (C.c_int, [_ctx]),
    "spq_cluster_size": (C.c_int, [_ctx, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "spq_cluster_sizes": (C.c_int, [_ctx, C.c_int, _i32p, _i64p]),
    "spq_total_cols": (C.c_int, [_ctx, C.POINTER(C.c_int64)]),
    "spq_trailing_stats": (C.c_int, [_ctx, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "spq_trailing_stats_async": (C.c_int, [_ctx, C.c_int, C.POINTER(C.c_int64)]),
    "spq_trailing_nnz": (C.c_int, [_ctx, C.c_int, _i64p]),
    "spq_row_of_col": (C.c_int, [_ctx, _i64p]),
    "spq_trailing_keys": (C.c_int, [_ctx, C.c_int64, _i32p, _i32p, C.POINTER(C.c_int64)]),
    "spq_payload_scalars": (C.c_int, [_ctx, C.POINTER(C.c_int64)]),
    "spq_timings": (C.c_int, [_ctx, _f64p, C.c_int]),
    "spq_reset_timings": (C.c_int, [_ctx]),
    "spq_num_records": (C.c_int, [_ctx]),
    "spq_record_info": (C.c_int, [_ctx, C.c_int, _i64p]),
    "spq_record_get": (C.c_int, [_ctx, C.c_int, C.c_int, _vp]),
    "spq_set_matrix": (C.c_int, [_ctx, C.c_int64, _i64p, _i64p, _f64p]),
    "spq_gmres": (C.c_int, [_ctx, _f64p, _vp, C.c_double, C.c_int, C.c_int, _f64p, _f64p,
                            C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "spq_apply_qt_host": (C.c_int, [_ctx, _f64p, _f64p, C.c_int]),
    "spq_solve_w_host": (C.c_int, [_ctx, _f64p, _f64p, C.c_int]),
    "spq_apply_w_host": (C.c_int, [_ctx, _f64p, _f64p, C.c_int]),
    "spq_apply_qt_dev": (C.c_int, [_ctx, _vp, C.c_int]),
    "spq_solve_w_dev": (C.c_int, [_ctx, _vp, C.c_int]),
    "spq_synchronize": (C.c_int, [_ctx]),
    "spq_chain_info": (C.c_int, [_ctx, C.c_int, _i64p]),
    "spq_mark": (C.c_int, [_ctx, C.c_int]),
    "spq_mark_elapsed": (C.c_int, [_ctx, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "spq_qr_house": (C.c_int, [_ctx, C.c_int64, C.c_int64, _f64p, _f64p, _f64p, _f64p, _f64p]),
    "spq_apply_panel": (C.c_int, [_ctx, C.c_int64, C.c_int64, C.c_int64, _f64p, _f64p, _f64p,
                                  C.c_int]),
    "spq_rrqr": (C.c_int, [_ctx, C.c_int64, C.c_int64, _f64p, C.c_double, C.c_int64, _f64p,
                           _f64p, _f64p, _i64p, C.POINTER(C.c_int64)]),
    "spq_tri_solve": (C.c_int, [_ctx, C.c_int64, C.c_int64, _f64p, _f64p, C.c_int, _f64p]),
    "spq_build_t": (C.c_int, [_ctx, C.c_int64, C.c_int64, _f64p, _f64p, _f64p]),
    "spq_bench_gemm": (C.c_int, [_ctx, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "spq_batched_qr": (C.c_int, [_ctx, C.c_int, _i64p, _i64p, _i64p, _f64p, _f64p, _f64p,
                                 C.POINTER(C.c_float)]),
    "spq_batched_rrqr": (C.c_int, [_ctx, C.c_int, C.c_int64, C.c_int64, _f64p, C.c_double, _i64p,
                                   _f64p, C.POINTER(C.c_float)]),
}

TIMING_FAMILIES = ["copy", "qr", "wy", "trsm", "cpqr", "flags", "chain"]

_lib = None


def load_library():
    """Load (building first if sources are newer) the native library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from .build import build
        build()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class Context:
    """Owns one spq_ctx (device block store + transform chains)."""

    def __init__(self, device=0):
        lib = load_library()
        self.lib = lib
        h = _ctx()
        rc = lib.spq_create(C.byref(h), int(device))
        self.h = h
        if rc != 0:
            self.check(rc)

    def check(self, rc):
        if rc == 0:
            return
        code = C.c_int()
        idx = C.c_int64()
        val = C.c_double()
        msg = C.create_string_buffer(1024)
        self.lib.spq_last_error(self.h, C.byref(code), C.byref(idx), C.byref(val), msg, 1024)
        text = msg.value.decode(errors="replace")
        if rc == SPQ_ERR_SINGULAR:
            raise SingularPivotError(int(idx.value), float(val.value), text)
        if rc == SPQ_ERR_BAD_INPUT:
            raise NestqrError(text)
        if rc == SPQ_ERR_SPECULATION:
            raise SpeculationError(text)
        if rc == SPQ_ERR_ILL_CONDITIONED:
            raise IllConditionedInterfaceError(int(idx.value), float(val.value), float(text))
        raise DeviceError(f"native error {rc}: {text}")

    def call(self, name, *args):
        self.check(getattr(self.lib, name)(self.h, *args))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.spq_destroy(self.h)
            self.h = _ctx()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # convenience queries
    def i64(self, name, *args):
        out = C.c_int64()
        self.call(name, *args, C.byref(out))
        return int(out.value)

    def timings(self):
        nf = len(TIMING_FAMILIES)
        buf = np.zeros(4 * nf + 26)
        self.call("spq_timings", buf, int(buf.size))
        out = {f: {"ms": buf[4 * i], "flops": buf[4 * i + 1], "launches": int(buf[4 * i + 2]),
                   "bytes": buf[4 * i + 3]}
               for i, f in enumerate(TIMING_FAMILIES)}
        h = buf[4 * nf:]
        out["host"] = {"alloc_ms": h[0], "sync_ms": h[1], "plan_ms": h[2], "api_ms": h[3],
                       "allocs": int(h[4]), "syncs": int(h[5]), "pool_bytes": int(h[6]),
                       "kernels": int(h[7]),
                       "flags_ms": h[8], "flags_wait_ms": h[9], "front_struct_ms": h[10],
                       "wave_exec_ms": h[11], "sparsify_ms": h[12], "sparsify_wait_ms": h[13],
                       "merge_ms": h[14], "scale_ms": h[15], "pivot_wait_ms": h[16],
                       "stats_ms": h[17], "load_ms": h[18], "finish_ms": h[19],
                       "live_bytes": int(h[20]), "peak_bytes": int(h[21]),
                       "speculate": int(h[22]), "verified_blocks": int(h[23]),
                       "spec_mismatch": int(h[24]), "sparsify_waves": int(h[25])}
        return out


def device_info():
    lib = load_library()
    buf = C.create_string_buffer(256)
    rc = lib.spq_device_info(buf, 256)
    return buf.value.decode() if rc == 0 else None
