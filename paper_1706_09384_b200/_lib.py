"""ctypes binding of libhmx.so (the C-ABI declared in ``include/hmx.h``).

There is no CPU fallback: if the library is missing the import of any
compute entry point raises, and device entry points raise when no CUDA
device is present.
"""

import ctypes as C
import os

import numpy as np

from .errors import STATUS_EXCEPTIONS

LIB_PATH = os.environ.get("HMX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhmx.so")

i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64
P = C.c_void_p
PP = C.POINTER(C.c_void_p)


class HmxKernel(C.Structure):
    _fields_ = [("kind", i32), ("pad", i32), ("kappa", f64), ("kp", f64), ("ks", f64),
                ("lam", f64), ("mu", f64), ("scale", f64)]


class HmxAcaCfg(C.Structure):
    _fields_ = [("eps", f64), ("max_rank", i64), ("sigma3_floor", f64), ("trunc_rule", i32),
                ("aca_kernel", i32), ("mem_budget_gb", f64), ("tc_stages", i32), ("pad", i32),
                ("rsvd_seed", i64), ("eps_recompress", f64)]


class HmxStats(C.Structure):
    _fields_ = [(n, i64) for n in (
        "n_blocks", "n_dense", "n_lowrank", "n_stored", "max_rank_before", "max_rank_after",
        "aca_steps_total", "pairs_evaluated", "n_fallback", "n_unconverged", "n_regularized",
        "aca_passes", "row_elems", "v_elems", "n_levels", "n_tiles", "n_jobs")] + [
        (n, f64) for n in ("t_dense_ms", "t_aca_ms", "t_recompress_ms", "t_form_ms", "t_total_ms",
                           "flops_assembly", "matvec_bytes", "dense_bytes", "lowrank_bytes",
                           "phase1_bytes", "phase2_bytes")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class HmxHluStats(C.Structure):
    _fields_ = [(n, i64) for n in ("n_truncations", "n_truncate_calls", "n_getrf", "max_rank", "dense_image_bytes",
                                   "k_p50", "k_p90", "k_max")] + [(n, f64) for n in ("t_truncate_s", "t_factor_s")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# name -> (restype, argtypes); every symbol include/hmx.h declares
SIGNATURES = {
    "hmx_abi_version": (C.c_int, []),
    "hmx_last_error": (C.c_int, [C.c_char_p, i64]),
    "hmx_ctx_create": (C.c_int, [i32, C.POINTER(P)]),
    "hmx_ctx_set_stream": (C.c_int, [P, u64]),
    "hmx_ctx_sync": (C.c_int, [P]),
    "hmx_ctx_release_cache": (C.c_int, [P]),
    "hmx_ctx_reserve": (C.c_int, [P, C.c_double, C.POINTER(C.c_double)]),
    "hmx_ctx_destroy": (C.c_int, [P]),
    "hmx_tree_build": (C.c_int, [P, i64, i64, C.POINTER(P)]),
    "hmx_tree_num_nodes": (i64, [P]),
    "hmx_tree_export": (C.c_int, [P, P, P, P]),
    "hmx_tree_free": (None, [P]),
    "hmx_blocks_build": (C.c_int, [P, P, f64, C.POINTER(P)]),
    "hmx_blocks_count": (i64, [P]),
    "hmx_blocks_export": (C.c_int, [P, P]),
    "hmx_blocks_free": (None, [P]),
    "hmx_eval_block": (C.c_int, [P, C.POINTER(HmxKernel), P, i64, P, i64, P, i32, f64, P]),
    "hmx_assemble": (C.c_int, [P, C.POINTER(HmxKernel), P, P, i64, P, P, i64,
                               C.POINTER(HmxAcaCfg), f64, C.POINTER(P)]),
    "hmx_hmatrix_load": (C.c_int, [P, i32, i64, P, P, i64, P, PP, PP, C.POINTER(P)]),
    "hmx_hmatrix_stats": (C.c_int, [P, C.POINTER(HmxStats)]),
    "hmx_hmatrix_block_info": (C.c_int, [P, P, P, P, P]),
    "hmx_hmatrix_set_block_info": (C.c_int, [P, P, P, P]),
    "hmx_hmatrix_get_block": (C.c_int, [P, i64, P, P]),
    "hmx_hmatrix_device_layout": (C.c_int, [P, P, P, P, P]),
    "hmx_block_errors": (C.c_int, [P, P, P, P, i64, C.c_double, P, P]),
    "hmx_aca_block": (C.c_int, [P, C.POINTER(HmxKernel), P, i64, P, i64, P, i32, f64, C.POINTER(HmxAcaCfg), i32,
                                i64, P, P, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32)]),
    "hmx_recompress": (C.c_int, [P, i64, i64, i64, P, P, f64, i32, C.POINTER(i64), P, P]),
    "hmx_hmatrix_splice": (C.c_int, [P, P, P, C.POINTER(P)]),
    "hmx_rsvd": (C.c_int, [P, P, i64, i64, f64, i32, i64, i64, P, P, C.POINTER(i64), C.POINTER(i32)]),
    "hmx_truncate_batch": (C.c_int, [P, i64, P, P, P, P, P, P, P, f64, i32, P, P]),
    "hmx_hmatrix_free": (None, [P]),
    "hmx_matvec": (C.c_int, [P, P, P, i32]),
    "hmx_matvec_on": (C.c_int, [P, P, P, i32, u64]),
    "hmx_matvec_profile": (C.c_int, [P, P, P, C.POINTER(C.c_float)]),
    "hmx_profile_begin": (C.c_int, [P]),
    "hmx_profile_end": (C.c_int, [P, C.POINTER(i64), P]),
    "hmx_bench_dfma": (C.c_int, [P, C.POINTER(f64)]),
    "hmx_bench_read_bw": (C.c_int, [P, C.POINTER(f64)]),
    "hmx_gmres": (C.c_int, [P, P, P, f64, i32, i64, i32, C.POINTER(i64), P, i64,
                            C.POINTER(i64), C.POINTER(i32)]),
    "hmx_hlu_build": (C.c_int, [P, i64, P, P, f64, i32, i32, C.POINTER(P)]),
    "hmx_hlu_count": (C.c_int, [P, C.POINTER(i64), C.POINTER(i64)]),
    "hmx_hlu_export": (C.c_int, [P, P, P]),
    "hmx_hlu_factor": (C.c_int, [P, f64, i32, C.POINTER(HmxHluStats)]),
    "hmx_hlu_apply": (C.c_int, [P, i32, P, P, i64, i64]),
    "hmx_hlu_addmul": (C.c_int, [P, P, P, f64, f64, i32]),
    "hmx_hlu_to_dense": (C.c_int, [P, P, i64]),
    "hmx_hlu_truncate": (C.c_int, [P, i64, P, P, P, P, P, P, P, f64, i32, P]),
    "hmx_hlu_release": (C.c_int, [P]),
    "hmx_hlu_free": (None, [P]),
}

_lib = None


def lib():
    """Load libhmx.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -m paper_1706_09384_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error():
    buf = C.create_string_buffer(2048)
    lib().hmx_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status, what=""):
    if status != 0:
        exc = STATUS_EXCEPTIONS.get(status, RuntimeError)
        raise exc(f"{what}: {last_error()} (status {status})")


def ptr(a):
    """Data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags.c_contiguous
    return C.c_void_p(a.ctypes.data)


def f64c(a, shape=None):
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and out.shape != shape:
        raise ValueError(f"expected shape {shape}, got {out.shape}")
    return out


_ctx = {}


_bound = {}


def bind_stream(device, stream_ptr):
    """Make the context launch on ``stream_ptr`` (cudaStream_t); no-op when it
    already does.  Switching synchronises the previous stream once."""
    stream_ptr = int(stream_ptr)
    if _bound.get(device) != stream_ptr:
        check(lib().hmx_ctx_set_stream(context(device), stream_ptr), "hmx_ctx_set_stream")
        _bound[device] = stream_ptr


def bind_torch_stream(device=0):
    """Order the context's launches with torch's current stream on ``device``
    (device-tensor entry points: results are then visible to later torch ops)."""
    import torch

    bind_stream(device, torch.cuda.current_stream(device).cuda_stream)


def release_cached(device=0):
    """Hand the context's cached device blocks back to the driver (before a
    library such as cuSOLVER has to allocate on the same device)."""
    if device in _ctx:
        check(lib().hmx_ctx_release_cache(_ctx[device]), "hmx_ctx_release_cache")


def reserve(device=0, gigabytes=0.0):
    """Opt-in arena (``hmx_ctx_reserve``): one reserved device region (``gigabytes``; 0 = 88% of the
    free memory) serves the context's large requests from then on, so assemblies make no
    cudaMalloc / cudaFree call; ``release_cached`` returns it.  Returns the seconds it took."""
    t = C.c_double(0.0)
    check(lib().hmx_ctx_reserve(context(device), float(gigabytes), C.byref(t)), "hmx_ctx_reserve")
    return t.value


def context(device=0):
    """Process-wide hmx context per device."""
    if device not in _ctx:
        h = C.c_void_p()
        check(lib().hmx_ctx_create(device, C.byref(h)), "hmx_ctx_create")
        _ctx[device] = h
    return _ctx[device]
