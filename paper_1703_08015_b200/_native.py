"""ctypes binding of the native library `libsplbm_b200.so` (include/splbm_b200.h).

The library is built in-tree (`python -m paper_1703_08015_b200.build`, or `__graft_entry__.build()`).
There is no fallback: importing an engine without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPLBM_LIB") or os.path.join(_HERE, "libsplbm_b200.so")
# The tolerance-mode build (same sources, SPLBM_FMA=1: contracted multiply-adds and a reciprocal
# velocity division, ~1e-15 per step instead of the bit-exact default; `arithmetic="fma"`).
FMA_LIB_PATH = os.environ.get("SPLBM_FMA_LIB") or os.path.join(_HERE, "libsplbm_b200_fma.so")

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


class GenerateParams(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("lid_speed", C.c_double), ("inlet_speed", C.c_double),
                ("outlet_density", C.c_double), ("sphere_diameter", C.c_int),
                ("target_porosity", C.c_double), ("seed", C.c_uint64)]


class DevDesc(C.Structure):
    _fields_ = [("d", C.c_int), ("dims", C.c_int * 3), ("types", C.c_void_p),
                ("bc_velocity", C.c_double * 3), ("bc_density", C.c_double), ("tile", C.c_int),
                ("tau", C.c_double), ("incompressible", C.c_int), ("periodic", C.c_int),
                ("device", C.c_int), ("slab_z0", C.c_int), ("slab_z1", C.c_int),
                ("collision", C.c_int), ("mrt_rates", C.c_void_p), ("single_copy", C.c_int),
                ("single_precision", C.c_int)]


class DevInfo(C.Structure):
    _fields_ = [("n_tiles", C.c_uint64), ("n_tiles_stored", C.c_uint64), ("n_tn", C.c_int),
                ("q", C.c_int), ("a", C.c_int), ("d", C.c_int), ("grid_dims", C.c_int * 3),
                ("padded_dims", C.c_int * 3), ("fluid_nodes", C.c_uint64),
                ("device_bytes", C.c_uint64), ("phi_t", C.c_double), ("ratio_tiles", C.c_double),
                ("n_tiles_global", C.c_uint64), ("resident_ctas", C.c_int),
                ("resident_threads", C.c_int), ("mrt_specialised", C.c_int)]


class SlabLayout(C.Structure):
    _fields_ = [("axis", C.c_int), ("z0", C.c_int), ("z1", C.c_int), ("zl", C.c_int),
                ("zh", C.c_int), ("n_low", C.c_uint64), ("n_own", C.c_uint64),
                ("n_high", C.c_uint64), ("g_low0", C.c_uint64), ("g_own0", C.c_uint64),
                ("g_high0", C.c_uint64), ("send_low_tiles", C.c_uint64),
                ("send_high_tiles", C.c_uint64)]


_lib = None

# every symbol include/splbm_b200.h declares (checked by tests/test_native_abi.py)
SIGNATURES = {
    "splbm_last_error": ([], C.c_char_p),
    "splbm_version": ([], C.c_char_p),
    "splbm_dev_info_size": ([], C.c_size_t),
    "splbm_generate": ([C.c_int, C.POINTER(GenerateParams), _u8, C.POINTER(C.c_int), _dp,
                        C.POINTER(C.c_double)], C.c_int),
    "splbm_generate_device": ([C.c_int, C.POINTER(GenerateParams), C.c_int, _u8, C.POINTER(C.c_int),
                               _dp, C.POINTER(C.c_double)], C.c_int),
    "splbm_geometry_load": ([C.c_char_p, C.POINTER(C.c_int), _i32, C.c_void_p, _dp,
                             C.POINTER(C.c_double)], C.c_int),
    "splbm_geometry_save": ([C.c_char_p, C.c_int, C.c_int, _i32, _u8, _dp, C.c_double], C.c_int),
    "splbm_tile_dims": ([C.c_int, _i32, C.c_int, _i32, _i32], C.c_int),
    "splbm_count_tiles": ([_u8, C.c_int, _i32, C.c_int, C.c_int, C.POINTER(C.c_uint64)], C.c_int),
    "splbm_build_tile_map": ([_u8, C.c_int, _i32, C.c_int, C.c_int, _u32, _i32, _u8, _u32,
                              C.c_void_p], C.c_int),
    "splbm_degenerate_bc_mask": ([_u8, C.c_int, _i32, C.c_int, _u8], C.c_int),
    "splbm_plane_tile_counts": ([_u8, C.c_int, _i32, C.c_int, C.c_int, _u64], C.c_int),
    "splbm_slab_layout": ([_u8, C.c_int, _i32, C.c_int, C.c_int, C.c_int, C.c_int,
                           C.POINTER(SlabLayout), C.c_void_p, C.c_void_p], C.c_int),
    "splbm_dev_create": ([C.POINTER(DevDesc), C.POINTER(_vp)], C.c_int),
    "splbm_dev_destroy": ([_vp], None),
    "splbm_dev_get_info": ([_vp, C.POINTER(DevInfo)], C.c_int),
    "splbm_dev_get_tile_grid": ([_vp, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p], C.c_int),
    "splbm_dev_stored_tiles": ([_vp, _u64], C.c_int),
    "splbm_dev_initialize": ([_vp, _dp, _dp, _dp, _dp], C.c_int),
    "splbm_dev_initialize_uniform": ([_vp, C.c_double, _dp], C.c_int),
    "splbm_dev_step": ([_vp, C.c_long, C.POINTER(C.c_int), C.POINTER(C.c_long)], C.c_int),
    "splbm_dev_step_async": ([_vp, C.c_long], C.c_int),
    "splbm_dev_sync": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_long)], C.c_int),
    "splbm_dev_current_step": ([_vp], C.c_long),
    "splbm_dev_tile_visits": ([_vp], C.c_uint64),
    "splbm_dev_padded_dims": ([_vp, _i32], C.c_int),
    "splbm_dev_fields": ([_vp, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.POINTER(C.c_double)], C.c_int),
    "splbm_dev_reduce": ([_vp, _dp], C.c_int),
    "splbm_dev_get_pdf": ([_vp, C.c_void_p], C.c_int),
    "splbm_dev_set_pdf": ([_vp, C.c_void_p], C.c_int),
    "splbm_dev_stream": ([_vp], C.c_void_p),
    "splbm_dev_last_batch_ms": ([_vp, C.POINTER(C.c_float)], C.c_int),
    "splbm_dev_launch_count": ([_vp], C.c_uint64),
    "splbm_dev_halo_bytes": ([_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], C.c_int),
    "splbm_dev_halo_recv_bytes": ([_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], C.c_int),
    "splbm_dev_halo_pack": ([_vp, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_dev_halo_unpack": ([_vp, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_dev_halo_pack_back": ([_vp, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_dev_halo_unpack_back": ([_vp, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_dev_step_part": ([_vp, C.c_int], C.c_int),
    "splbm_comm_unique_id": ([C.c_void_p], C.c_int),
    "splbm_dev_ipc_blob": ([_vp, C.c_void_p], C.c_int),
    "splbm_dev_p2p_attach": ([_vp, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_dev_comm_attach": ([_vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
    "splbm_dev_halo_pack_next": ([_vp, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_selftest_divide": ([C.c_uint64, _dp, _dp, _dp], C.c_int),
    "splbm_selftest_divide_f32": ([C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "splbm_mrt_kernel": ([C.c_int, C.c_double, C.c_void_p, _dp], C.c_int),
    "splbm_mrt_specialise": ([C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int,
                              C.POINTER(C.c_int)], C.c_int),
}


_fma_lib = None


def lib(arithmetic: str = "exact"):
    """The loaded native library; raises if it was not built (no fallback path exists).
    arithmetic="fma" selects the tolerance-mode build."""
    global _lib, _fma_lib
    if arithmetic == "fma":
        if _fma_lib is None:
            _fma_lib = load(FMA_LIB_PATH)
        return _fma_lib
    if arithmetic != "exact":
        raise errors.ConfigError("arithmetic must be exact or fma")
    if _lib is None:
        _lib = load(LIB_PATH)
    return _lib


def load(path: str):
    """Loads a build of the library at `path` (an experiment build for A/B timing, or the
    in-tree one) with every signature bound."""
    if not os.path.exists(path):
        raise ImportError(
            f"native library {path} is missing; build it with "
            "`python -m paper_1703_08015_b200.build` (the T2C path has no CPU fallback)")
    L = C.CDLL(path)
    missing = []
    for name, (args, res) in SIGNATURES.items():
        if not hasattr(L, name):  # an older experiment build; tests/test_native_abi.py guards
            missing.append(name)
            continue
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    L.missing_symbols = missing
    if hasattr(L, "splbm_dev_info_size") and L.splbm_dev_info_size() != C.sizeof(DevInfo):
        raise ImportError(f"{path} was built from another revision of include/splbm_b200.h "
                          f"(splbm_dev_info is {L.splbm_dev_info_size()} bytes there, "
                          f"{C.sizeof(DevInfo)} here); rebuild it")
    return L


def check(rc: int, step: int | None = None, lib_=None) -> None:
    """Raises the errors.hpp exception for a non-zero status; the message is the thread's last
    error of the library that returned it (`lib_`, default the bit-exact build)."""
    if rc == 0:
        return
    msg = (lib_ or lib()).splbm_last_error().decode(errors="replace")
    raise errors.from_status(rc, msg, step)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
