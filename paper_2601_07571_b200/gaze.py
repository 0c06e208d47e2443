"""Fixations and the Gaussian gaze cone (drop-in for the reference's gaze.py
data model: GazeCone :52-67, Fixation :70-127).

The per-fixation crop-frustum construction (ref :252-381) runs in the
extension's host setup (csrc/gm_setup.cpp) for the whole fixation table at
once; `fixation_setup()` exposes its output.  Fixations reach the C-ABI as an
(F, 18) float64 table in the fixation-log column order (ref :133-136):
start, duration, position xyz, rotation xyzw, frustum l r t b n f, gaze xyz.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import GazeOutsideFrustumError, InvalidFrustumError

__all__ = ["GazeCone", "Fixation", "world_to_camera", "EllipseParams", "CropFrustum", "DEFAULT_THETA", "SQRT_TWO_PI", "fixation_table",
           "fixation_setup", "perspective_matrix", "frustum_from_matrix", "gaussian_weight", "ellipse_intersection",
           "crop_bounds", "crop_projection_matrix", "build_crop_frustum"]

SQRT_TWO_PI = math.sqrt(2.0 * math.pi)
DEFAULT_THETA = math.radians(1.0)
FIX_COLUMNS = 18


@dataclass(frozen=True)
class GazeCone:
    """theta = one standard deviation; sigma = tan(theta); phi = atan(4 sigma)."""

    theta: float
    sigma: float
    phi: float

    def __post_init__(self):
        if not 0.0 < self.theta < math.pi / 2:
            raise ValueError(f"theta must be in (0, pi/2), got {self.theta}")

    @classmethod
    def from_theta(cls, theta: float) -> "GazeCone":
        s = math.tan(theta)
        return cls(theta=theta, sigma=s, phi=math.atan(4.0 * s))


@dataclass(frozen=True)
class Fixation:
    """One fixation with its camera pose, frustum (l, r, t, b, n, f) and unit
    camera-space gaze direction (normalised here, must point to z < 0)."""

    start_time: float
    duration: float
    camera_position: np.ndarray
    camera_rotation: np.ndarray
    frustum: tuple
    gaze_dir: np.ndarray
    overrides: dict = field(default_factory=dict)

    def __post_init__(self):
        object.__setattr__(self, "camera_position", np.asarray(self.camera_position, dtype=np.float64))
        object.__setattr__(self, "camera_rotation", np.asarray(self.camera_rotation, dtype=np.float64))
        g = np.asarray(self.gaze_dir, dtype=np.float64)
        gn = float(np.linalg.norm(g))
        if gn == 0.0:
            raise ValueError("gaze_dir must be a nonzero vector")
        object.__setattr__(self, "gaze_dir", g / gn)
        left, right, top, bottom, near, far = self.frustum
        if self.duration <= 0:
            raise ValueError("duration must be > 0")
        if not (near > 0 and far > near):
            raise ValueError("frustum needs 0 < near < far")
        if not (left < right and bottom < top):
            raise ValueError("frustum needs left < right and bottom < top")
        if self.gaze_dir[2] >= 0:
            raise ValueError("gaze_dir must point into the viewed half-space (z < 0)")

    @property
    def near(self) -> float:
        return self.frustum[4]

    @property
    def far(self) -> float:
        return self.frustum[5]

    def row(self) -> np.ndarray:
        """This fixation as one 18-column table row."""
        r = np.empty(FIX_COLUMNS)
        r[0] = self.start_time
        r[1] = self.duration
        r[2:5] = self.camera_position
        r[5:9] = self.camera_rotation
        r[9:15] = self.frustum
        r[15:18] = self.gaze_dir
        return r

    def view_matrix(self) -> np.ndarray:
        """World-to-camera 4x4 (host utility, reference gaze.py:114-122)."""
        return world_to_camera(self.camera_position, self.camera_rotation)

    def projection_matrix(self) -> np.ndarray:
        left, right, top, bottom, near, far = self.frustum
        return perspective_matrix(left, right, bottom, top, near, far)


def world_to_camera(position, rotation) -> np.ndarray:
    """4x4 view matrix of a camera at `position` with orientation `rotation`
    (xyzw): rotation block R^T, translation -R^T p (numpy matmul, i.e. the
    BLAS FMA chain the reference's view matrices carry)."""
    from .geometry import quat_to_matrix

    r_inv = quat_to_matrix(rotation).T
    view = np.zeros((4, 4))
    view[3, 3] = 1.0
    view[:3, :3] = r_inv
    view[:3, 3] = -r_inv @ np.asarray(position, dtype=np.float64)
    return view


def fixation_table(fixations) -> np.ndarray:
    """(F, 18) float64 table from Fixation objects (this package's or any
    object with the reference's fields) or pass an (F, 18) array through."""
    table = getattr(fixations, "table", None)  # FixationLog (fixlog.parse_fixation_log)
    if isinstance(table, np.ndarray) and isinstance(fixations, list) and len(table) == len(fixations):
        return table
    if isinstance(fixations, np.ndarray):
        t = np.ascontiguousarray(fixations, dtype=np.float64)
        if t.ndim != 2 or t.shape[1] != FIX_COLUMNS:
            raise ValueError(f"fixation table must be (F, {FIX_COLUMNS}), got {t.shape}")
        return t
    fixations = list(fixations)
    out = np.empty((len(fixations), FIX_COLUMNS))
    for i, f in enumerate(fixations):
        if isinstance(f, Fixation):
            out[i] = f.row()
        else:
            out[i, 0] = f.start_time
            out[i, 1] = f.duration
            out[i, 2:5] = f.camera_position
            out[i, 5:9] = f.camera_rotation
            out[i, 9:15] = f.frustum
            out[i, 15:18] = f.gaze_dir
    return out


def perspective_matrix(l: float, r: float, b: float, t: float, n: float, f: float) -> np.ndarray:
    """Off-centre perspective projection, -z forward (ref gaze.py:323-336)."""
    if not (l < r and b < t):
        raise InvalidFrustumError(f"degenerate bounds l={l} r={r} b={b} t={t}")
    if not 0 < n < f:
        raise InvalidFrustumError(f"invalid near/far n={n} f={f}")
    m = np.zeros((4, 4))
    m[0, 0] = 2.0 * n / (r - l)
    m[0, 2] = (r + l) / (r - l)
    m[1, 1] = 2.0 * n / (t - b)
    m[1, 2] = (t + b) / (t - b)
    m[2, 2] = -(f + n) / (f - n)
    m[2, 3] = -2.0 * f * n / (f - n)
    m[3, 2] = -1.0
    return m


def frustum_from_matrix(m) -> tuple:
    """(l, r, b, t, n, f) of a perspective_matrix (ref gaze.py:345-356)."""
    m = np.asarray(m, dtype=np.float64)
    n = m[2, 3] / (m[2, 2] - 1.0)
    f = m[2, 3] / (m[2, 2] + 1.0)
    width = 2.0 * n / m[0, 0]
    height = 2.0 * n / m[1, 1]
    l = -0.5 * width * (1.0 - m[0, 2])
    b = -0.5 * height * (1.0 - m[1, 2])
    return l, l + width, b, b + height, n, f


def gaussian_weight(p, gaze_dir, duration_t: float, cone: GazeCone) -> float:
    """Scalar duration-weighted Gaussian of a camera-space point (helper; the
    production evaluation is k_accumulate)."""
    p = np.asarray(p, dtype=np.float64)
    g = np.asarray(gaze_dir, dtype=np.float64)
    g = g / np.linalg.norm(g)
    d1 = float(p @ g)
    if d1 <= 0.0:
        return 0.0
    d2 = float(np.linalg.norm(p - d1 * g))
    radius = d1 * cone.sigma
    ratio = 0.0 if radius == 0.0 else d2 / radius
    if ratio > 4.0:
        return 0.0
    return duration_t / (cone.sigma * SQRT_TWO_PI) * math.exp(-0.5 * ratio * ratio)


# ------------------------------------------------ 4-sigma cone crop frustum

@dataclass(frozen=True)
class EllipseParams:
    """The 4-sigma cone's ellipse on the near plane z = -n (ref gaze.py:218-229)."""

    center_E: np.ndarray
    major_a: float
    minor_b: float
    inclination_alpha: float
    A0: np.ndarray
    A1: np.ndarray
    B0: np.ndarray
    B1: np.ndarray

    def packed(self) -> np.ndarray:
        return np.concatenate([self.center_E, [self.major_a, self.minor_b, self.inclination_alpha], self.A0,
                               self.A1, self.B0, self.B1]).astype(np.float64)


_GAZE_OUTSIDE = {1: "gaze cone ray does not reach the near clip plane (z >= 0)",
                 2: "gaze cone does not cut the near plane in an ellipse"}


def ellipse_intersection(gaze_dir, n: float, cone: GazeCone) -> EllipseParams:
    """Near-plane ellipse of the 4-sigma cone (ref gaze.py:252-309), computed
    by the same host code (csrc/gm_setup.cpp) the generation setup uses:
    bit-identical to the reference (glibc trig, OpenBLAS FMA-chain norms).
    Raises GazeOutsideFrustumError like the reference."""
    g = np.ascontiguousarray(np.asarray(gaze_dir, dtype=np.float64).reshape(3))
    out = np.zeros(18)
    rc = _native.load().gm_ellipse_intersection(_native.dptr(g), float(n), float(cone.phi), _native.dptr(out))
    if rc == _native.GM_ERR_GAZE_OUTSIDE:
        raise GazeOutsideFrustumError(_GAZE_OUTSIDE[int(out[0])])
    _native.check(rc, "gm_ellipse_intersection")
    return EllipseParams(out[0:3].copy(), float(out[3]), float(out[4]), float(out[5]), out[6:9].copy(),
                         out[9:12].copy(), out[12:15].copy(), out[15:18].copy())


def crop_bounds(e: EllipseParams) -> tuple:
    """(l', r', b', t') bounding box of the near-plane ellipse (ref gaze.py:312-320)."""
    lrbt = np.zeros(4)
    _native.check(_native.load().gm_crop_bounds(_native.dptr(e.packed()), _native.dptr(lrbt)), "gm_crop_bounds")
    return float(lrbt[0]), float(lrbt[1]), float(lrbt[2]), float(lrbt[3])


def crop_projection_matrix(bounds, n: float, f: float) -> np.ndarray:
    """Perspective matrix of the sub-frustum bounded by the ellipse box (ref gaze.py:339-342)."""
    l, r, b, t = bounds
    return perspective_matrix(l, r, b, t, n, f)


@dataclass(frozen=True)
class CropFrustum:
    """4-sigma-cone-fitted sub-frustum and its projection (ref gaze.py:359-369)."""

    left: float
    right: float
    bottom: float
    top: float
    near: float
    far: float
    projection_matrix: np.ndarray


def build_crop_frustum(fixation, cone: GazeCone) -> CropFrustum:
    """Crop frustum of a fixation's 4-sigma cone (ref gaze.py:372-381); raises
    GazeOutsideFrustumError when the cone does not fully face the near plane."""
    n, f = fixation.frustum[4], fixation.frustum[5]
    e = ellipse_intersection(fixation.gaze_dir, n, cone)
    l, r, b, t = crop_bounds(e)
    return CropFrustum(l, r, b, t, n, f, crop_projection_matrix((l, r, b, t), n, f))


# GmFixExact field offsets (float64 units, 26 per record), csrc/gm_types.h
SETUP_FIELDS = {"rot": slice(0, 9), "trans": slice(9, 12), "gaze": slice(12, 15), "amp": 15, "p00": 16,
                "p11": 17, "p02": 18, "p12": 19, "near": 20, "far": 21, "near_lo": 22, "far_hi": 23,
                "cropped": 24}


def fixation_setup(fixations, theta: float = DEFAULT_THETA, filtering: bool = True,
                   zbuffer_resolution: int = 512) -> np.ndarray:
    """(F, 26) float64 per-fixation setup table exactly as the kernels use it
    (view rotation/translation, crop-or-full projection terms, near'/far',
    amplitude); see SETUP_FIELDS.  Raises InvalidFrustumError like the
    reference's perspective_matrix."""
    table = fixation_table(fixations)
    F = len(table)
    out = np.zeros((max(F, 1), _native.FIX_EXACT_DOUBLES))
    bad = np.zeros(1, np.int64)
    if F:
        lib = _native.load()
        _native.check(lib.gm_fixation_setup(_native.dptr(table), F, float(theta), int(bool(filtering)),
                                            int(zbuffer_resolution), _native.dptr(out), None,
                                            _native.iptr(bad)), f"fixation {int(bad[0])}")
    return out[:F]
