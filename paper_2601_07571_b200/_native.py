"""ctypes binding of the in-tree CUDA extension `_gazemap_b200.so`.

There is no CPU fallback: if the shared object is missing, or no CUDA device
is visible, every compute call raises `NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConfigError, GazemapError, GazeOutsideFrustumError, InvalidFrustumError

SO_PATH = Path(__file__).resolve().parent / "_gazemap_b200.so"

(GM_OK, GM_ERR_CUDA, GM_ERR_ARG, GM_ERR_INVALID_FRUSTUM, GM_ERR_NO_DEVICE, GM_ERR_OOM, GM_ERR_UNSUPPORTED,
 GM_ERR_GAZE_OUTSIDE) = range(8)

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_U8 = ctypes.POINTER(ctypes.c_uint8)
_VP = ctypes.c_void_p


class NativeUnavailableError(GazemapError, RuntimeError):
    """The CUDA extension could not be loaded or no GPU is visible."""


class GmConfig(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("eps_abs", ctypes.c_double), ("eps_rel", ctypes.c_double),
                ("zbuffer_resolution", ctypes.c_int32), ("filtering", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("flags", ctypes.c_int32)]


class GmTimings(ctypes.Structure):
    _fields_ = [("setup_ms", ctypes.c_double), ("cull_ms", ctypes.c_double), ("rasterize_ms", ctypes.c_double),
                ("accumulate_ms", ctypes.c_double), ("total_ms", ctypes.c_double), ("mark_ms", ctypes.c_double),
                ("texel_ms", ctypes.c_double), ("screen_tris", ctypes.c_int64), ("bin_items", ctypes.c_int64),
                ("batches", ctypes.c_int64), ("retries", ctypes.c_int64)]


# GmFixExact is 26 float64 (gm_types.h); GmFixCull 20 float32
FIX_EXACT_DOUBLES = 26
FIX_CULL_FLOATS = 20

GM_FLAG_STATS = 1
GM_FLAG_ONE_STREAM = 2
GM_FLAG_TWO_STREAMS = 4
STAT_NAMES = ["l1_tests", "l2_tests", "exact_evals", "ndc_candidates", "cone_candidates", "visible",
              "texels", "texel_pairs", "covered_pairs", "tile_occluded", "tx_tiles", "tx_staged", "tx_list", "tx_iter",
              "tx_edge", "tx_crowded",
              "tx_chunked", "tx_chunked_pairs", "tx_chunked_texels", "bbox_px"]

CHECK_NAMES = ["tx_texels", "tx_bound_wrong", "tx_winner_wrong", "cand_pairs", "cand_l1_wrong", "cand_l3_wrong",
               "mask_wrong", "depth_tests", "depth_wrong", "tileocc_wrong", "cull_tris", "cull_texels",
               "cull_wrong"] + [f"reserved{i}" for i in range(3)]

PROGRESS_FN = ctypes.CFUNCTYPE(None, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p)

# every C-ABI entry point (include/gazemap_b200.h) -> (restype, argtypes)
SIGNATURES = {
    "gm_last_error": (ctypes.c_char_p, []),
    "gm_abi_version": (ctypes.c_int, []),
    "gm_device_count": (ctypes.c_int, []),
    "gm_peak_flops": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _D]),
    "gm_layout": (ctypes.c_int, [ctypes.c_int, _D, ctypes.c_int64, ctypes.c_double, _I64, _I64, _I64, _I64]),
    "gm_sample_positions": (ctypes.c_int, [ctypes.c_int, _D, ctypes.c_int64, _I64, _I64, ctypes.c_int64, _D, _D]),
    "gm_normalize": (ctypes.c_int, [ctypes.c_int, _D, ctypes.c_int64, ctypes.c_double, _D]),
    "gm_setup_consts": (None, [ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "gm_fixation_check": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "gm_fixation_setup": (ctypes.c_int, [_D, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D,
                                         ctypes.c_void_p, _I64]),
    "gm_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_VP)]),
    "gm_plan_destroy": (None, [_VP]),
    "gm_plan_set_host_threads": (ctypes.c_int, [_VP, ctypes.c_int]),
    "gm_plan_set_scene": (ctypes.c_int, [_VP, ctypes.c_int, _I64, _D, _D, _I64, _U8]),
    "gm_plan_set_poses": (ctypes.c_int, [_VP, _D]),
    "gm_plan_num_samples": (ctypes.c_int64, [_VP]),
    "gm_plan_num_triangles": (ctypes.c_int64, [_VP]),
    "gm_plan_values_device": (ctypes.c_void_p, [_VP]),
    "gm_plan_accumulate": (ctypes.c_int, [_VP, _D, ctypes.c_int64, ctypes.POINTER(GmConfig), ctypes.c_int,
                                          ctypes.POINTER(GmTimings), PROGRESS_FN, ctypes.c_void_p, _I64]),
    "gm_plan_prepare": (ctypes.c_int, [_VP, _D, ctypes.c_int64, ctypes.POINTER(GmConfig), _I64]),
    "gm_plan_run": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, ctypes.POINTER(GmTimings),
                                   ctypes.POINTER(ctypes.c_float)]),
    "gm_plan_flush_l2": (ctypes.c_int, [_VP, ctypes.c_int64]),
    "gm_plan_stats": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_uint64)]),
    "gm_plan_check": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int)]),
    "gm_plan_set_segment_capacity": (ctypes.c_int, [_VP, ctypes.c_int64]),
    "gm_plan_max": (ctypes.c_int, [_VP, _D]),
    "gm_plan_read": (ctypes.c_int, [_VP, _D, _D, ctypes.c_double]),
    "gm_plan_write": (ctypes.c_int, [_VP, _D]),
    "gm_plan_sync": (ctypes.c_int, [_VP]),
    "gm_plan_ipc_handle": (ctypes.c_int, [_VP, ctypes.c_char_p]),
    "gm_plan_open_peers": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]),
    "gm_plan_reduce_peers": (ctypes.c_int, [_VP, _D, ctypes.POINTER(ctypes.c_float)]),
    "gm_plan_depth_buffer": (ctypes.c_int, [_VP, _D, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            _D]),
    "gm_plan_candidates": (ctypes.c_int, [_VP, _D, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                          _I64, ctypes.c_int64, _I64]),
    "gm_plan_positions": (ctypes.c_int, [_VP, _D]),
    "gm_rasterize": (ctypes.c_int, [ctypes.c_int, _D, ctypes.c_int64, _D, _D, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_double, _D, ctypes.c_void_p, _D]),
    "gm_render_heatmap": (ctypes.c_int, [ctypes.c_int, _D, ctypes.c_int64, _D, _D, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_double, _I64, _I64, _D, ctypes.c_int64, _D, _D, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_void_p]),
    "gm_cull_mask": (ctypes.c_int, [ctypes.c_int, _D, ctypes.c_int64, _D, ctypes.c_int, ctypes.c_void_p]),
    "gm_depth_match": (ctypes.c_int, [_D, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double]),
    "gm_ellipse_intersection": (ctypes.c_int, [_D, ctypes.c_double, ctypes.c_double, _D]),
    "gm_crop_bounds": (ctypes.c_int, [_D, _D]),
    "gm_fixlog_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_VP)]),
    "gm_fixlog_rows": (ctypes.c_int64, [_VP]),
    "gm_fixlog_groups": (ctypes.c_int64, [_VP]),
    "gm_fixlog_copy": (ctypes.c_int, [_VP, _D, _I64, ctypes.c_void_p, _I64, _I64, _D]),
    "gm_fixlog_error": (ctypes.c_int, [_VP, _I64]),
    "gm_fixlog_free": (None, [_VP]),
    "gm_export_format": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, _I64, _I64, ctypes.c_int64, ctypes.c_int64,
                                        _D, _D, _D, ctypes.c_int, ctypes.POINTER(_VP)]),
    "gm_buffer_data": (ctypes.c_void_p, [_VP]),
    "gm_buffer_size": (ctypes.c_int64, [_VP]),
    "gm_buffer_free": (None, [_VP]),
}

_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = True):
    """Load (building first if needed and possible) the CUDA extension."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        so_path = Path(os.environ.get("GAZEMAP_B200_SO", SO_PATH))  # experimental variants (build.py)
        if build_if_missing and so_path == SO_PATH:
            try:
                from . import build as _build

                if _build.needs_build():
                    _build.build()
            except Exception as e:  # no nvcc on this host: only a prebuilt .so can work
                if not SO_PATH.exists():
                    raise NativeUnavailableError(f"CUDA extension missing and build failed: {e}") from e
        if not so_path.exists():
            raise NativeUnavailableError(f"CUDA extension not built: {so_path}")
        try:
            lib = ctypes.CDLL(str(so_path))
        except OSError as e:
            raise NativeUnavailableError(f"cannot load {so_path}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def device_count() -> int:
    return int(load().gm_device_count())


def check(rc: int, what: str = "") -> None:
    if rc == GM_OK:
        return
    msg = load().gm_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == GM_ERR_INVALID_FRUSTUM:
        raise InvalidFrustumError(msg)
    if rc == GM_ERR_GAZE_OUTSIDE:
        raise GazeOutsideFrustumError(msg)
    if rc == GM_ERR_NO_DEVICE:
        raise NativeUnavailableError(msg)
    if rc == GM_ERR_ARG:
        raise ConfigError(msg)
    raise GazemapError(f"CUDA extension error {rc}: {msg}")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_D) if a is not None else None


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_I64) if a is not None else None


def u8ptr(a: np.ndarray):
    return a.ctypes.data_as(_U8) if a is not None else None
