"""ctypes binding of libmagnex_b200.so (include/magnex_b200.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, every device-backed call raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MXB_LIB: load another build of the same ABI (variant experiments, tools/build_variant.py)
LIB_PATH = os.environ.get("MXB_LIB") or os.path.join(HERE, "libmagnex_b200.so")

OK, EINVAL, EDEAD, EBLOWUP, ECUDA, ENCCL, EQUILIBRATED = 0, 1, 2, 3, 4, 5, 6
TERM_EXCHANGE, TERM_ANISOTROPY, TERM_DMI, TERM_DEMAG, TERM_BIAS, TERM_CUBIC, TERM_BULK_DMI = (
    1, 2, 4, 8, 16, 32, 64)
GHOST = {"neumann": 0, "dmi": 1, "periodic": 2}
EULER, RK4, MRI_KW3 = 0, 1, 2

_dp = C.POINTER(C.c_double)


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double)]


class Material(C.Structure):
    _fields_ = [("Ms", C.c_double), ("A", C.c_double), ("Ku", C.c_double), ("D", C.c_double),
                ("alpha", C.c_double), ("gamma", C.c_double), ("eK", C.c_double * 3),
                ("Ms_cell", _dp), ("A_cell", _dp), ("Ku_cell", _dp), ("D_cell", _dp),
                ("alpha_cell", _dp), ("eK_cell", _dp),
                ("Kc1", C.c_double), ("c1", C.c_double * 3), ("c2", C.c_double * 3),
                ("Db", C.c_double)]


class Terms(C.Structure):
    _fields_ = [("mask", C.c_uint32), ("ghost_mode", C.c_int32), ("precession", C.c_int32),
                ("damping", C.c_int32)]


class Bias(C.Structure):
    _fields_ = [("vec", C.c_double * 3), ("field", _dp), ("demag_field", _dp)]


class RunArgs(C.Structure):
    _fields_ = [("method", C.c_int32), ("renorm_each_stage", C.c_int32), ("dt", C.c_double),
                ("nsteps", C.c_int64), ("eq_tol", C.c_double), ("stage_bias", _dp),
                ("bias_field", _dp), ("bias_vec", C.c_double * 3), ("fast_mask", C.c_uint32),
                ("pad", C.c_int32), ("theta", C.c_double), ("stage_bias_fields", _dp)]


class StageIO(C.Structure):
    _fields_ = [("ys", C.c_void_p), ("y", C.c_void_p), ("hd", C.c_void_p), ("k1", C.c_void_p),
                ("s", C.c_void_p), ("out", C.c_void_p), ("k1_out", C.c_void_p),
                ("halo_lo", C.c_void_p), ("halo_hi", C.c_void_p), ("hms_lo", C.c_void_p),
                ("hms_hi", C.c_void_p), ("hA_lo", C.c_void_p), ("hA_hi", C.c_void_p),
                ("bias_field", C.c_void_p), ("bias", C.c_double * 3), ("c", C.c_double),
                ("dt6", C.c_double), ("renorm", C.c_int32), ("pad", C.c_int32)]


class RunStats(C.Structure):
    _fields_ = [("steps_done", C.c_int64), ("status", C.c_int32), ("pad", C.c_int32),
                ("mean", C.c_double * 3), ("residual", C.c_double), ("drift", C.c_double),
                ("dead_flat", C.c_int64)]


# every exported entry point with its argtypes (checked by tests/test_abi.py)
SIGNATURES = {
    "mxb_abi_version": ([], C.c_int),
    "mxb_last_error": ([], C.c_char_p),
    "mxb_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "mxb_ctx_create": ([C.POINTER(Grid), C.POINTER(Material), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "mxb_ctx_destroy": ([C.c_void_p], C.c_int),
    "mxb_ctx_set_exact": ([C.c_void_p, C.c_int], C.c_int),
    "mxb_demag_create": ([C.POINTER(Grid), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "mxb_demag_destroy": ([C.c_void_p], C.c_int),
    "mxb_demag_set_packed": ([C.c_void_p, _dp], C.c_int),
    "mxb_demag_build": ([C.c_void_p, C.c_int], C.c_int),
    "mxb_demag_tensor_elements": ([C.c_void_p, _dp], C.c_int),
    "mxb_demag_direct": ([C.c_void_p, _dp, _dp, _dp], C.c_int),
    "mxb_demag_get_spectra": ([C.c_void_p, _dp], C.c_int),
    "mxb_demag_field": ([C.c_void_p, _dp, _dp], C.c_int),
    "mxb_demag_field_dev": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "mxb_demag_bytes": ([C.c_void_p], C.c_size_t),
    "mxb_demag_set_fast": ([C.c_void_p, C.c_int], C.c_int),
    "mxb_demag_kmode": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "mxb_term_field": ([C.c_void_p, C.c_uint32, C.c_int, _dp, _dp], C.c_int),
    "mxb_heff": ([C.c_void_p, C.c_void_p, C.POINTER(Terms), C.POINTER(Bias), _dp, _dp], C.c_int),
    "mxb_llg_rhs": ([C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp], C.c_int),
    "mxb_rhs_total": ([C.c_void_p, C.c_void_p, C.POINTER(Terms), C.POINTER(Bias), _dp, _dp], C.c_int),
    "mxb_renormalize": ([C.c_void_p, _dp, C.POINTER(C.c_int64)], C.c_int),
    "mxb_mean_normalized": ([C.c_void_p, _dp, _dp], C.c_int),
    "mxb_energies": ([C.c_void_p, C.c_void_p, C.POINTER(Terms), C.POINTER(Bias), _dp, _dp], C.c_int),
    "mxb_state_set": ([C.c_void_p, _dp], C.c_int),
    "mxb_state_get": ([C.c_void_p, _dp], C.c_int),
    "mxb_state_mean": ([C.c_void_p, _dp], C.c_int),
    "mxb_run": ([C.c_void_p, C.c_void_p, C.POINTER(Terms), C.POINTER(RunArgs), C.POINTER(RunStats)], C.c_int),
    "mxb_state_energies": ([C.c_void_p, C.c_void_p, C.POINTER(Terms), C.POINTER(Bias), _dp], C.c_int),
    "mxb_demag_create_slab": ([C.POINTER(Grid), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "mxb_demag_slab_info": ([C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "mxb_demag_slab_buffers": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int),
    "mxb_demag_slab_block": ([C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "mxb_demag_x_forward": ([C.c_void_p, C.c_void_p], C.c_int),
    "mxb_demag_yz": ([C.c_void_p], C.c_int),
    "mxb_demag_x_inverse": ([C.c_void_p, C.c_void_p], C.c_int),
    "mxb_demag_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "mxb_ctx_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "mxb_stage_dev": ([C.c_void_p, C.c_int, C.POINTER(Terms), C.POINTER(StageIO)], C.c_int),
    "mxb_pack_halo_planes": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "mxb_step_partials_dev": ([C.c_void_p, C.c_void_p], C.c_int),
    "mxb_step_commit_dev": ([C.c_void_p, C.c_void_p], C.c_int),
    "mxb_ctl_reset": ([C.c_void_p, _dp, C.c_int64, C.c_double], C.c_int),
    "mxb_ctl_get": ([C.c_void_p, C.POINTER(RunStats)], C.c_int),
    "mxb_time_demag": ([C.c_void_p, C.c_void_p, C.c_int, _dp, _dp], C.c_int),
    "mxb_time_steps": ([C.c_void_p, C.c_void_p, C.POINTER(Terms), C.c_double, C.c_int, _dp, _dp, _dp,
                        C.POINTER(C.c_int64)], C.c_int),
    "mxb_time_demag_cufft": ([C.c_void_p, C.c_int, _dp], C.c_int),
    "mxb_host_alloc": ([C.c_size_t, C.POINTER(C.c_void_p)], C.c_int),
    "mxb_host_free": ([C.c_void_p], C.c_int),
    "mxb_fno_create": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp,
                        C.POINTER(C.c_void_p)], C.c_int),
    "mxb_fno_destroy": ([C.c_void_p], None),
    "mxb_fno_infer": ([C.c_void_p, _dp, _dp], C.c_int),
    "mxb_fno_infer_dev": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "mxb_demag_create_fno": ([C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "mxb_fno_spectral_conv": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp],
                              C.c_int),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load the shared library (raising loudly if it is absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_12242_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


class MxbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc: int, what: str = ""):
    if rc == OK:
        return
    msg = load().mxb_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    raise MxbError(rc, f"{what}: {msg}" if what else msg)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need C-contiguous float64"
    return a.ctypes.data_as(_dp)


_device = 0


def set_device(dev: int) -> None:
    """Select the CUDA device for contexts created afterwards."""
    global _device
    _device = int(dev)


def device() -> int:
    return _device


_exact = os.environ.get("MXB_EXACT", "0") == "1"


def set_exact(flag: bool) -> None:
    """Exact mode: reference operation order, no FMA (bit-faithful local terms)."""
    global _exact
    _exact = bool(flag)


def exact() -> bool:
    return _exact
