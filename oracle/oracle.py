"""ctypes front end of the CPU oracle (oracle/gm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg as the checker.  The product package
(paper_2601_07571_b200) never imports this module.

Each function restates a reference function (file:line of
/root/reference/pkg/src/gazemap given per function) and works on plain numpy
arrays or on duck-typed scene / fixation / config objects (the reference's own
dataclasses or the product's mirrors both work).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

FS_ROT, FS_TRANS, FS_GAZE, FS_AMP = 0, 9, 12, 15
FS_P00, FS_P11, FS_P02, FS_P12, FS_NEAR, FS_FAR, FS_CROPPED = 16, 17, 18, 19, 20, 21, 22
FS_PROJ, FS_VIEW, FS_LEN = 23, 39, 55

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_U8 = ctypes.POINTER(ctypes.c_uint8)


def build() -> Path:
    """Compile gm_oracle.c (make) if the shared object is missing or stale."""
    src = _HERE / "gm_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.or_layout.argtypes = [_D, ctypes.c_int64, ctypes.c_double, _I64, _I64, _I64, _I64]
        L.or_positions_local.argtypes = [_D, ctypes.c_int64, _I64, _I64, _I64, _D]
        L.or_transform_apply.argtypes = [_D, ctypes.c_int64, _D, _D, _D, _D]
        L.or_fixation_setup.argtypes = [_D, ctypes.c_double, ctypes.c_int, _D]
        L.or_fixation_setup.restype = ctypes.c_int
        L.or_frustum_planes.argtypes = [_D, _D, _D]
        L.or_cull_mask.argtypes = [_D, ctypes.c_int64, _D, _U8]
        L.or_rasterize.argtypes = [_D, ctypes.c_int64, _D, _D] + [ctypes.c_double] * 4 + [
            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, _D]
        L.or_depth_match.argtypes = [_D, ctypes.c_int, ctypes.c_int] + [ctypes.c_double] * 4
        L.or_depth_match.restype = ctypes.c_int
        L.or_accumulate.argtypes = [_D, ctypes.c_int64, _D, _D, _D, ctypes.c_double, ctypes.c_double] + [
            ctypes.c_double] * 4 + [_D, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, _D, _U8, ctypes.c_int]
        L.or_generate.argtypes = [_D, ctypes.c_int64, _D, ctypes.c_int64, _D, ctypes.c_int64,
                                  ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_int, _D, _D, _I64]
        L.or_generate.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, t=_D):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


# ------------------------------------------------------------------ sampling

def layout(tri_local: np.ndarray, k: float):
    """geometry.py:305-320 build_sampled_mesh -> (res, counts, offsets, total)."""
    tri = _f64(tri_local, (-1, 3, 3))
    T = len(tri)
    res = np.zeros(T, np.int64)
    cnt = np.zeros(T, np.int64)
    off = np.zeros(T, np.int64)
    total = np.zeros(1, np.int64)
    lib().or_layout(_p(tri), T, float(k), _p(res, _I64), _p(cnt, _I64), _p(off, _I64), _p(total, _I64))
    return res, cnt, off, int(total[0])


def positions_local(tri_local, res, cnt, off, total):
    """geometry.py:331-346 sample_positions_local."""
    tri = _f64(tri_local, (-1, 3, 3))
    out = np.zeros((total, 3))
    if total:
        lib().or_positions_local(_p(tri), len(tri), _p(np.ascontiguousarray(res, np.int64), _I64),
                                 _p(np.ascontiguousarray(cnt, np.int64), _I64),
                                 _p(np.ascontiguousarray(off, np.int64), _I64), _p(out))
    return out


def transform_apply(pts, translation, rotation, scale):
    """geometry.py:86-89 Transform.apply (dgemm FMA chain + translation)."""
    pts = _f64(pts, (-1, 3))
    out = np.zeros_like(pts)
    if len(pts):
        lib().or_transform_apply(_p(pts), len(pts), _p(_f64(rotation)), _p(_f64(scale)),
                                 _p(_f64(translation)), _p(out))
    return out


# ------------------------------------------------------------ per fixation

def fixation_row(fx) -> np.ndarray:
    """18-float fixation record in the log schema (gaze.py:133-136)."""
    row = np.empty(18)
    row[0] = float(fx.start_time)
    row[1] = float(fx.duration)
    row[2:5] = np.asarray(fx.camera_position, dtype=np.float64)
    row[5:9] = np.asarray(fx.camera_rotation, dtype=np.float64)
    row[9:15] = np.asarray(fx.frustum, dtype=np.float64)
    row[15:18] = np.asarray(fx.gaze_dir, dtype=np.float64)
    return row


def fixation_table(fixations) -> np.ndarray:
    if len(fixations) == 0:
        return np.zeros((0, 18))
    return np.stack([fixation_row(f) for f in fixations])


class OracleFrustumError(Exception):
    pass


def fixation_setup(row, theta: float, filtering: bool) -> np.ndarray:
    """density.py:148-158 + gaze.py:114-127,252-381 -> FS_LEN float64 record."""
    out = np.zeros(FS_LEN)
    rc = lib().or_fixation_setup(_p(_f64(row)), float(theta), int(bool(filtering)), _p(out))
    if rc:
        raise OracleFrustumError(f"invalid frustum (code {rc})")
    return out


def frustum_planes(proj, view):
    out = np.zeros((6, 4))
    lib().or_frustum_planes(_p(_f64(proj)), _p(_f64(view)), _p(out))
    return out


def cull_mask(tris, planes):
    tris = _f64(tris, (-1, 3, 3))
    keep = np.zeros(len(tris), np.uint8)
    if len(tris):
        lib().or_cull_mask(_p(tris), len(tris), _p(_f64(planes)), _p(keep, _U8))
    return keep.astype(bool)


def rasterize(tris, rot, trans, p00, p11, p02, p12, width, height, near, far):
    """kernels.py:140-192 rasterize into a fresh +inf buffer (raster.py:114)."""
    tris = _f64(tris, (-1, 3, 3))
    depth = np.full((height, width), np.inf)
    if len(tris):
        lib().or_rasterize(_p(tris), len(tris), _p(_f64(rot)), _p(_f64(trans)), p00, p11, p02, p12,
                           int(width), int(height), near, far, _p(depth))
    return depth


def depth_match(depth, fx, fy, d, eps) -> bool:
    depth = _f64(depth)
    return bool(lib().or_depth_match(_p(depth), depth.shape[0], depth.shape[1], fx, fy, d, eps))


def accumulate(pos, setup, sigma, depth, eps_abs, eps_rel, values, threads=1):
    """kernels.py:288-340 accumulate (values updated in place)."""
    pos = _f64(pos, (-1, 3))
    depth = _f64(depth)
    s = setup
    lib().or_accumulate(_p(pos), len(pos), _p(_f64(s[FS_ROT:FS_ROT + 9])), _p(_f64(s[FS_TRANS:FS_TRANS + 3])),
                        _p(_f64(s[FS_GAZE:FS_GAZE + 3])), sigma, s[FS_AMP], s[FS_P00], s[FS_P11], s[FS_P02],
                        s[FS_P12], _p(depth), depth.shape[0], depth.shape[1], eps_abs, eps_rel, s[FS_NEAR],
                        s[FS_FAR], _p(values), None, int(threads))
    return values


def candidates(pos, setup) -> np.ndarray:
    """Indices passing the NDC crop filter of kernels.py:302-319 (sorted)."""
    pos = _f64(pos, (-1, 3))
    s = setup
    mask = np.zeros(len(pos), np.uint8)
    if len(pos):
        dummy = np.zeros((1, 1))
        lib().or_accumulate(_p(pos), len(pos), _p(_f64(s[FS_ROT:FS_ROT + 9])), _p(_f64(s[FS_TRANS:FS_TRANS + 3])),
                            _p(_f64(s[FS_GAZE:FS_GAZE + 3])), 1.0, s[FS_AMP], s[FS_P00], s[FS_P11], s[FS_P02],
                            s[FS_P12], _p(dummy), 1, 1, 0.0, 0.0, s[FS_NEAR], s[FS_FAR], None,
                            _p(mask, _U8), 1)
    return np.nonzero(mask)[0].astype(np.int64)


# ------------------------------------------------------------ scene helpers

def _obj_fields(obj):
    tr = obj.transform
    return (np.asarray(obj.mesh.vertices, np.float64).reshape(-1, 3),
            np.asarray(obj.mesh.faces, np.int64).reshape(-1, 3),
            np.asarray(tr.translation, np.float64), np.asarray(tr.rotation, np.float64),
            np.asarray(tr.scale, np.float64))


def scene_world_triangles(scene) -> np.ndarray:
    """raster.py:68-78 scene_world_triangles (no overrides)."""
    parts = []
    for obj in scene.objects:
        v, f, t, q, s = _obj_fields(obj)
        tri = v[f]
        parts.append(transform_apply(tri.reshape(-1, 3), t, q, s).reshape(-1, 3, 3))
    if not parts:
        return np.zeros((0, 3, 3))
    return np.concatenate(parts, axis=0)


def build_layouts(scene, k):
    """geometry.py:323-328 build_sampled_meshes -> {oid: (res, cnt, off, total)}."""
    out = {}
    for obj in scene.objects:
        v, f, *_ = _obj_fields(obj)
        out[obj.object_id] = layout(v[f], k)
    return out


def world_samples(scene, layouts) -> dict:
    """density.py:109-121 _SampleCache.base_world per object."""
    out = {}
    for obj in scene.objects:
        if obj.object_id not in layouts:
            continue
        v, f, t, q, s = _obj_fields(obj)
        res, cnt, off, total = layouts[obj.object_id]
        local = positions_local(v[f], res, cnt, off, total)
        out[obj.object_id] = transform_apply(local, t, q, s)
    return out


def generate(scene, fixations, k=40000.0, theta=math.radians(1.0), zbuffer_resolution=512,
             epsilon_abs=1e-3, epsilon_rel=1e-3, filtering_enabled=True, object_include_list=None,
             threads=1, layouts=None):
    """density.py:203-227 generate -> (values dict, global_max).  No overrides."""
    for fx in fixations:
        if getattr(fx, "overrides", None):
            raise NotImplementedError("oracle: per-fixation overrides not restated")
    layouts = layouts if layouts is not None else build_layouts(scene, k)
    world = world_samples(scene, layouts)
    ids = [o.object_id for o in scene.objects]
    included = ids if object_include_list is None else [o for o in ids if o in object_include_list]
    included = [o for o in included if layouts[o][3] > 0]
    pos = np.concatenate([world[o] for o in included]) if included else np.zeros((0, 3))
    tris = scene_world_triangles(scene)
    fx = fixation_table(fixations)
    vals = np.zeros(len(pos))
    gmax = np.zeros(1)
    bad = np.zeros(1, np.int64)
    rc = lib().or_generate(_p(tris), len(tris), _p(_f64(pos, (-1, 3))), len(pos), _p(_f64(fx, (-1, 18))),
                           len(fx), float(theta), int(zbuffer_resolution), float(epsilon_abs),
                           float(epsilon_rel), int(bool(filtering_enabled)), int(threads), _p(vals),
                           _p(gmax), _p(bad, _I64))
    if rc:
        raise OracleFrustumError(f"fixation {int(bad[0])}: invalid frustum (code {rc})")
    values = {oid: np.zeros(layouts[oid][3]) for oid in layouts}
    o = 0
    for oid in included:
        n = layouts[oid][3]
        values[oid] = vals[o:o + n].copy()
        o += n
    return values, float(gmax[0])


class RowFixation:
    """Duck-typed fixation over one 18-column row (no re-normalisation)."""

    __slots__ = ("start_time", "duration", "camera_position", "camera_rotation", "frustum", "gaze_dir", "overrides")

    def __init__(self, r):
        r = np.asarray(r, dtype=np.float64)
        self.start_time, self.duration = float(r[0]), float(r[1])
        self.camera_position, self.camera_rotation = r[2:5], r[5:9]
        self.frustum, self.gaze_dir, self.overrides = tuple(r[9:15]), r[15:18], {}


def rows_as_fixations(table):
    return [RowFixation(r) for r in np.asarray(table, dtype=np.float64).reshape(-1, 18)]
