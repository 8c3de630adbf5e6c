"""ctypes loader for libifgf_b200.so (the sm_100a CUDA library, C ABI in
include/ifgf_b200.h).  There is no fallback: if the library is missing the
import fails loudly, and every compute entry point fails with IFGF_ERUNTIME
when no sm_100 device is visible."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IFGF_B200_LIB") or os.path.join(PKG_DIR, "libifgf_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(PKG_DIR), "include", "ifgf_b200.h")

IFGF_OK, IFGF_EINVAL, IFGF_EDOMAIN, IFGF_ELOGIC, IFGF_ERUNTIME = range(5)
MAX_LEVELS = 22


class CParams(C.Structure):
    _fields_ = [("depth", C.c_int), ("box_lambda", C.c_double), ("points_per_box", C.c_int),
                ("base_s", C.c_int), ("base_theta", C.c_int), ("base_phi", C.c_int),
                ("p_s", C.c_int), ("p_theta", C.c_int), ("p_phi", C.c_int), ("device", C.c_int),
                ("partition", C.c_int)]


class CReport(C.Structure):
    _fields_ = [("setup", C.c_double), ("singular", C.c_double), ("level_d", C.c_double),
                ("interpolation", C.c_double), ("propagation", C.c_double), ("total", C.c_double),
                ("depth", C.c_int), ("n", C.c_size_t), ("h_level_d", C.c_double),
                ("n_levels", C.c_int), ("level_boxes", C.c_size_t * MAX_LEVELS),
                ("level_cones", C.c_size_t * MAX_LEVELS), ("peak_live_blocks", C.c_size_t),
                ("gpu_launches", C.c_size_t)]


class CPlanInfo(C.Structure):
    _fields_ = [("n", C.c_size_t), ("depth", C.c_int), ("cube_origin", C.c_double * 3),
                ("cube_side", C.c_double), ("kappa", C.c_double), ("p_s", C.c_int),
                ("p_theta", C.c_int), ("p_phi", C.c_int), ("P", C.c_int),
                ("boxes", C.c_size_t * MAX_LEVELS), ("cones", C.c_size_t * MAX_LEVELS),
                ("nbr_entries", C.c_size_t * MAX_LEVELS),
                ("cousin_entries", C.c_size_t * MAX_LEVELS), ("h", C.c_double * MAX_LEVELS),
                ("setup_seconds", C.c_double), ("device_bytes", C.c_size_t),
                ("setup_launches", C.c_size_t),
                ("launches", C.c_size_t), ("k4_record_pairs", C.c_size_t),
                ("k4_record_bytes", C.c_size_t)]


class CDistLevel(C.Structure):
    _fields_ = [("owned_cones", C.c_size_t), ("halo_cones", C.c_size_t),
                ("interp_needed", C.c_size_t), ("prop_needed", C.c_size_t),
                ("sent_cones", C.c_size_t)]


class CDistInfo(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("depth", C.c_int),
                ("point_begin", C.c_size_t), ("point_end", C.c_size_t),
                ("levels", CDistLevel * MAX_LEVELS), ("block_bytes", C.c_size_t),
                ("device_bytes", C.c_size_t), ("compute_seconds", C.c_double)]


COMM_ID_BYTES = 128

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_sz = C.c_size_t
_PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); the single source of truth for the binding,
# checked against the header by tests/test_lib_cpu.py.
SIGNATURES = {
    "ifgf_default_params": (None, [C.POINTER(CParams)]),
    "ifgf_last_error": (C.c_char_p, []),
    "ifgf_abi_version": (C.c_int, []),
    "ifgf_device_ok": (C.c_int, []),
    "ifgf_choose_depth": (C.c_int, [_sz, C.c_double, C.c_double, C.POINTER(CParams),
                                    C.POINTER(C.c_int)]),
    "ifgf_plan_create": (C.c_int, [_vp, _vp, _vp, _sz, C.c_int, C.c_double, C.POINTER(CParams),
                                   _PP]),
    "ifgf_plan_create_device": (C.c_int, [_vp, _vp, _vp, _sz, C.c_int, C.c_double,
                                          C.POINTER(CParams), _vp, _PP]),
    "ifgf_plan_destroy": (None, [_vp]),
    "ifgf_plan_set_option": (C.c_int, [_vp, C.c_int, C.c_int]),
    "ifgf_plan_apply": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.POINTER(CReport)]),
    "ifgf_plan_apply_device": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(CReport)]),
    "ifgf_plan_apply_batch": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, C.POINTER(CReport)]),
    "ifgf_plan_apply_batch_device": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp,
                                               C.POINTER(CReport)]),
    "ifgf_apply": (C.c_int, [_sz, _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_double,
                             C.POINTER(CParams), _vp, _vp, C.POINTER(CReport)]),
    "ifgf_plan_get_info": (C.c_int, [_vp, C.POINTER(CPlanInfo)]),
    "ifgf_plan_export_perm": (C.c_int, [_vp, _vp]),
    "ifgf_plan_export_level": (C.c_int, [_vp, C.c_int] + [_vp] * 13),
    "ifgf_plan_set_density": (C.c_int, [_vp, _vp, _vp]),
    "ifgf_plan_zero_result": (C.c_int, [_vp]),
    "ifgf_plan_singular_pass": (C.c_int, [_vp, _sz, _sz]),
    "ifgf_plan_level_d_pass": (C.c_int, [_vp, C.c_uint32, C.c_uint32]),
    "ifgf_plan_propagation_pass": (C.c_int, [_vp, C.c_int, C.c_uint32, C.c_uint32]),
    "ifgf_plan_interpolation_pass": (C.c_int, [_vp, C.c_int, _sz, _sz]),
    "ifgf_plan_read_blocks": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "ifgf_plan_write_blocks": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "ifgf_plan_read_result": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "ifgf_plan_block_stride": (C.c_int, [_vp]),
    "ifgf_plan_pack_blocks": (C.c_int, [_vp, C.c_int, _vp, _sz, _vp, _vp]),
    "ifgf_plan_unpack_blocks": (C.c_int, [_vp, C.c_int, _vp, _sz, _vp, _vp]),
    "ifgf_plan_partition": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    "ifgf_plan_exchange_set": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp,
                                         C.POINTER(C.c_size_t)]),
    "ifgf_comm_unique_id": (C.c_int, [_vp]),
    "ifgf_comm_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _PP]),
    "ifgf_comm_destroy": (None, [_vp]),
    "ifgf_dist_plan_create_device": (C.c_int, [_vp, _vp, _vp, _vp, _sz, C.c_int, C.c_double,
                                               C.POINTER(CParams), _vp, _PP]),
    "ifgf_dist_plan_apply_device": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp,
                                              C.POINTER(CReport)]),
    "ifgf_dist_plan_info": (C.c_int, [_vp, C.POINTER(CDistInfo)]),
    "ifgf_run_distributed": (C.c_int, [_sz, _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_double,
                                       C.POINTER(CParams), C.c_int, _vp, _vp, _vp,
                                       C.POINTER(CReport), _vp]),
    "ifgf_direct_eval": (C.c_int, [_sz, _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_double, _vp, _sz,
                                   C.c_int, _vp, _vp]),
    "ifgf_sample_indices": (C.c_int, [_sz, _sz, C.c_uint64, _vp]),
    "ifgf_error_at_indices": (C.c_int, [_sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int,
                                        C.c_double, _vp, _sz, C.c_int, C.POINTER(C.c_double)]),
    "ifgf_measure_fp64_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
    "ifgf_generate": (C.c_int, [_sz, C.c_int, C.c_double, C.c_int, C.c_uint64, _vp, _vp, _vp,
                                _vp, _vp]),
    "ifgf_generate_surface": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_uint64, _vp, _vp,
                                        _vp, _vp, _vp]),
    "ifgf_checksum_hex": (None, [_vp, _vp, _sz, C.c_char_p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def ptr(a):
    """Raw data pointer of a numpy array (None passes through)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def last_error() -> str:
    return lib.ifgf_last_error().decode()
