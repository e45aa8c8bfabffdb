"""ctypes binding of libmfh.so (the C-ABI declared in include/mfh.h).

The shared library is built in-tree (``paper_1410_2697_b200/libmfh.so``) by
``__graft_entry__.build()`` / ``python -m paper_1410_2697_b200.build``. There is
no fallback: if the library is missing, or a compute entry point is called
without a CUDA device, the call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmfh.so")
# A/B builds only (scripts): another in-tree build of the same library
if os.environ.get("MFH_LIB_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "libmfh_" + os.environ["MFH_LIB_VARIANT"] + ".so")

MFH_OK, MFH_EVALUE, MFH_EPIVOT, MFH_ERUNTIME = 0, 1, 2, 3


class PivotMonotonicityError(RuntimeError):
    """Complete pivoting step bound violated (reference _core.pyx:17)."""


class mfh_params(C.Structure):
    _fields_ = [("n_c", C.c_int64), ("eps", C.c_double), ("d", C.c_int64),
                ("n_leaf", C.c_int64), ("max_rank", C.c_int64)]


# int (*)(void *user, double *d_buf, int64_t count): in-place all-reduce SUM
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)
P2P_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                     C.POINTER(C.c_int32), C.POINTER(C.c_int32))


class mfh_shard_t(C.Structure):
    _fields_ = [("owner", C.POINTER(C.c_int32)), ("rank", C.c_int), ("exchange", EXCHANGE_FN),
                ("user", C.c_void_p), ("p2p", P2P_FN)]


class mfh_stats_t(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "peak_stored_reals", "retained_reals", "structured_fronts", "dense_fronts",
        "full_square_allocs", "n_records", "stored_reals", "device_bytes_peak", "n_blocks",
        "n_dense_fallback")]


class mfh_record_t(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "node_id", "front_size", "n_pivot", "path", "max_offdiag_rank", "stored_reals")]


class mfh_timing_t(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("sample_ms", C.c_double), ("pivot_lu_ms", C.c_double),
                ("skeleton_ms", C.c_double), ("hodlr_factor_ms", C.c_double),
                ("dense_front_ms", C.c_double), ("eliminate_ms", C.c_double),
                ("host_ms", C.c_double), ("host_preamble_ms", C.c_double),
                ("host_select_ms", C.c_double), ("host_sync_wait_ms", C.c_double), ("wall_ms", C.c_double),
                ("apply_build_ms", C.c_double), ("apply_instantiate_ms", C.c_double),
                ("gmres_ms", C.c_double), ("gmres_apply_ms", C.c_double), ("gmres_sync_ms", C.c_double),
                ("kernel_launches", C.c_int64),
                ("pivot_lu_visits", C.c_double), ("sample_entries", C.c_double),
                ("hodlr_flops", C.c_double), ("elim_flops", C.c_double), ("dense_flops", C.c_double),
                ("skeleton_flops", C.c_double), ("sample_lr_flops", C.c_double),
                ("pivot_lu_crit_steps", C.c_double), ("apply_ref_bytes", C.c_double),
                ("exec_flops_skeleton", C.c_double), ("exec_flops_hodlr", C.c_double),
                ("exec_flops_elim", C.c_double), ("exec_flops_dense", C.c_double),
                ("materialize_ms", C.c_double), ("exec_flops_materialize", C.c_double),
                ("idle_gap_ms", C.c_double)]


HOST_OP = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))


class mfh_gmres_ops(C.Structure):
    _fields_ = [("A", C.c_void_p), ("A_cb", HOST_OP), ("A_user", C.c_void_p),
                ("M", C.c_void_p), ("M_cb", HOST_OP), ("M_user", C.c_void_p), ("P", C.c_void_p)]


_lib = None
_lock = threading.RLock()
_finalized = False
_live = []  # weak references to objects owning native handles


def register(obj):
    """Track an object with a ``_release()`` method so it is freed before CUDA tears down."""
    import weakref
    _live.append(weakref.ref(obj))


def _shutdown():
    # Python atexit runs before the CUDA runtime's own exit handlers: release
    # every device object while the context is still alive.
    global _finalized, _ctx
    for r in reversed(_live):
        o = r()
        if o is not None:
            try:
                o._release()
            except Exception:
                pass
    _live.clear()
    if _ctx is not None:
        try:
            _ctx._release()
        except Exception:
            pass
    _finalized = True


import atexit as _atexit  # noqa: E402

_atexit.register(_shutdown)
P = C.c_void_p
I64 = C.c_int64
PP = C.POINTER(C.c_void_p)


def _sig(lib):
    d = C.c_double
    pi = C.POINTER(C.c_int64)
    pd = C.POINTER(C.c_double)
    s = {
        "mfh_last_error": (C.c_char_p, []),
        "mfh_version": (C.c_int, []),
        "mfh_ctx_create": (C.c_int, [C.c_int, PP]),
        "mfh_ctx_destroy": (None, [P]),
        "mfh_ctx_sync": (C.c_int, [P]),
        "mfh_ctx_info": (C.c_int, [P, PP, pi]),
        "mfh_adjacency": (C.c_int, [I64, P, P, P, P, P, pi]),
        "mfh_nd_create": (C.c_int, [I64, P, P, I64, PP]),
        "mfh_nd_sizes": (C.c_int, [P, pi, pi, pi]),
        "mfh_nd_fetch": (C.c_int, [P, P, P, P, P, P, P]),
        "mfh_nd_free": (None, [P]),
        "mfh_etree_create": (C.c_int, [I64, P, P, P, P, PP]),
        "mfh_etree_sizes": (C.c_int, [P, pi, pi, pi, pi]),
        "mfh_etree_fetch": (C.c_int, [P, P, P, P, P, P, P]),
        "mfh_etree_free": (None, [P]),
        "mfh_etree_from_arrays": (C.c_int, [I64, P, I64, I64, P, P, P, I64, P, P, P, P, P, PP]),
        "mfh_factorize": (C.c_int, [P, P, I64, P, P, P, C.c_int, C.POINTER(mfh_params), PP]),
        "mfh_node_op": (C.c_int, [P, I64, C.c_int, P, P]),
        "mfh_factorize_sharded": (C.c_int, [P, P, I64, P, P, P, C.c_int, C.POINTER(mfh_params),
                                            C.POINTER(mfh_shard_t), PP]),
        "mfh_factor_stats": (C.c_int, [P, C.POINTER(mfh_stats_t)]),
        "mfh_factor_records": (C.c_int, [P, P]),
        "mfh_factor_timing": (C.c_int, [P, C.POINTER(mfh_timing_t)]),
        "mfh_factor_blocks": (C.c_int, [P, pi, pi, P, P, P]),
        "mfh_factor_free": (None, [P]),
        "mfh_apply": (C.c_int, [P, P, P, I64, C.c_int]),
        "mfh_apply_bench": (C.c_int, [P, I64, pd, pd]),
        "mfh_csr_create": (C.c_int, [P, I64, I64, P, P, P, PP]),
        "mfh_dense_create": (C.c_int, [P, I64, P, PP]),
        "mfh_spmv": (C.c_int, [P, P, P, C.c_int]),
        "mfh_spmv_bench": (C.c_int, [P, I64, pd]),
        "mfh_precond_diag_create": (C.c_int, [P, I64, P, P, P, PP]),
        "mfh_precond_ilut_create": (C.c_int, [P, I64, P, P, P, I64, d, PP]),
        "mfh_precond_info": (C.c_int, [P, pi, pi, pi, pi]),
        "mfh_precond_ilut_factors": (C.c_int, [P, P, P, P, P, P, P]),
        "mfh_precond_apply": (C.c_int, [P, P, P, C.c_int]),
        "mfh_precond_free": (None, [P]),
        "mfh_ilut_factor": (C.c_int, [I64, P, P, P, I64, d, pi, pi, P, P, P, P, P, P]),
        "mfh_test_gemm_batched": (C.c_int, [P, I64, P, P, P, I64, C.c_int]),
        "mfh_test_gemv_batched": (C.c_int, [P, I64, P, P, P, I64, P, I64, C.c_int]),
        "mfh_gmres_sharded": (C.c_int, [P, I64, P, P, P, P, P, d, I64, I64, P, pi, pi, C.POINTER(C.c_int)]),
        "mfh_csr_free": (None, [P]),
        "mfh_gmres": (C.c_int, [P, C.POINTER(mfh_gmres_ops), I64, P, P, d, I64, I64, P, pi, pi,
                                C.POINTER(C.c_int)]),
        "mfh_gmres_device": (C.c_int, [P, C.POINTER(mfh_gmres_ops), I64, P, P, d, I64, I64, P, pi,
                                       pi, C.POINTER(C.c_int)]),
        "mfh_gmres_batched": (C.c_int, [P, C.POINTER(mfh_gmres_ops), I64, I64, P, P, d, I64, I64, P, I64, P, P,
                                        P]),
        "mfh_gmres_batched_device": (C.c_int, [P, C.POINTER(mfh_gmres_ops), I64, I64, P, P, d, I64, I64, P, I64,
                                               P, P, P]),
        "mfh_full_pivot_lu_batched": (C.c_int, [P, I64, P, P, P, P, I64, d, P, P, P, P, P, P, P]),
        "mfh_test_inverse_batched": (C.c_int, [P, I64, P, P, P, I64, P]),
    }
    for name, (res, args) in s.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return s


EXPORTED = None


def lib():
    """The loaded libmfh.so; raises if it has not been built."""
    global _lib, EXPORTED
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                        "g.build()'` (nvcc, sm_100a)")
                L = C.CDLL(LIB_PATH)
                EXPORTED = sorted(_sig(L))
                _lib = L
    return _lib


def check(rc):
    if rc == MFH_OK:
        return
    msg = lib().mfh_last_error().decode("utf-8", "replace")
    if rc == MFH_EVALUE:
        raise ValueError(msg)
    if rc == MFH_EPIVOT:
        raise PivotMonotonicityError(msg)
    raise RuntimeError(msg)


def ptr(a):
    """Raw data pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One CUDA device + stream + workspaces (mfh_ctx)."""

    def __init__(self, device=0):
        h = C.c_void_p()
        check(lib().mfh_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def sync(self):
        check(lib().mfh_ctx_sync(self.handle))

    def info(self):
        """(cudaStream_t as int, kernels launched so far)."""
        s, n = C.c_void_p(), C.c_int64()
        check(lib().mfh_ctx_info(self.handle, C.byref(s), C.byref(n)))
        return s.value or 0, n.value

    def _release(self):
        if self.handle and not _finalized:
            lib().mfh_ctx_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


_ctx = None


def context():
    """Process-wide default context on ``MFH_DEVICE`` (default: LOCAL_RANK or 0)."""
    global _ctx
    if _ctx is None:
        with _lock:
            if _ctx is None:
                dev = int(os.environ.get("MFH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
                _ctx = Context(dev)
    return _ctx
