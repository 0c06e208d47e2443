"""Scene data model and area-adaptive surface sampling (drop-in for the
reference's geometry.py).

The data model (Transform, Mesh, SceneObject, Scene, TriangleSampling,
SampledMesh) mirrors /root/reference/pkg/src/gazemap/geometry.py:60-145 and
:261-302 field for field.  The sampling stage itself --
build_sampled_mesh (ref :305-320) and sample_positions_local (ref :331-346) --
runs on the GPU (k_layout + CUB scan, k_positions in csrc/gm_kernels.cu) and
returns bit-identical arrays.  The scalar index helpers below are the
reference's O(1) closed forms, kept for API completeness.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError

__all__ = [
    "Transform", "Mesh", "SceneObject", "Scene", "TriangleSampling", "SampledMesh", "triangle_area",
    "adaptive_resolution", "sample_count", "sample_index_to_rowcol", "rowcol_to_barycentric",
    "build_sampled_mesh", "build_sampled_meshes", "sample_positions_local", "sample_world_position",
    "quat_to_matrix",
]

_QUAT_NORM_TOL = 1e-6


def quat_to_matrix(q) -> np.ndarray:
    """3x3 rotation of a unit quaternion (x, y, z, w) (ref geometry.py:48-57)."""
    x, y, z, w = (float(c) for c in q)
    xx, yy, zz = x * x, y * y, z * z
    return np.array([
        [1 - 2 * (yy + zz), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (xx + zz), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (xx + yy)],
    ])


@dataclass(frozen=True)
class Transform:
    """Object pose: scale, then rotate (unit quaternion xyzw), then translate."""

    translation: np.ndarray
    rotation: np.ndarray
    scale: np.ndarray

    def __post_init__(self):
        for name in ("translation", "rotation", "scale"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        if (self.translation.shape, self.rotation.shape, self.scale.shape) != ((3,), (4,), (3,)):
            raise ValueError("transform components must be xyz / xyzw / xyz")
        qn = float(np.linalg.norm(self.rotation))
        if abs(qn - 1.0) > _QUAT_NORM_TOL:
            raise ValueError(f"rotation quaternion norm {qn} not within {_QUAT_NORM_TOL} of 1")

    @classmethod
    def identity(cls) -> "Transform":
        return cls(np.zeros(3), np.array([0.0, 0.0, 0.0, 1.0]), np.ones(3))

    def matrix(self) -> np.ndarray:
        """Linear part R * diag(scale)."""
        return quat_to_matrix(self.rotation) * self.scale[None, :]

    def packed(self) -> np.ndarray:
        """[t(3), q(4), s(3)]: the layout the C-ABI takes per object."""
        return np.concatenate([self.translation, self.rotation, self.scale])

    def apply(self, points: np.ndarray) -> np.ndarray:
        """Map (N, 3) local points to world space (host-side utility)."""
        return np.asarray(points, dtype=np.float64) @ self.matrix().T + self.translation


@dataclass(frozen=True)
class Mesh:
    """Indexed triangle mesh: (V, 3) float64 vertices, (T, 3) int64 faces."""

    vertices: np.ndarray
    faces: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        f = np.asarray(self.faces, dtype=np.int64).reshape(-1, 3)
        if len(f) and (f.min() < 0 or f.max() >= len(v)):
            raise ValueError("face index out of range")
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "faces", f)

    @property
    def triangle_count(self) -> int:
        return len(self.faces)

    def triangle_vertices(self) -> np.ndarray:
        """(T, 3, 3) corner positions."""
        return self.vertices[self.faces]


@dataclass(frozen=True)
class SceneObject:
    object_id: str
    mesh: Mesh
    transform: Transform = field(default_factory=Transform.identity)

    def world_triangles(self, transform: Transform | None = None) -> np.ndarray:
        t = self.transform if transform is None else transform
        tri = self.mesh.triangle_vertices()
        return t.apply(tri.reshape(-1, 3)).reshape(tri.shape)


@dataclass(frozen=True)
class Scene:
    objects: tuple

    def __post_init__(self):
        objs = tuple(self.objects)
        object.__setattr__(self, "objects", objs)
        ids = [o.object_id for o in objs]
        if len(ids) != len(set(ids)):
            raise ValueError("duplicate object_id in scene")

    def object(self, object_id: str) -> SceneObject:
        for o in self.objects:
            if o.object_id == object_id:
                return o
        raise KeyError(object_id)

    @property
    def object_ids(self) -> list:
        return [o.object_id for o in self.objects]


# ----------------------------------------------------------------- indexing

def sample_count(r: int) -> int:
    """Samples of a triangle at resolution r: (r+1)(r+2)/2 (paper Eq. 1)."""
    return (r + 1) * (r + 2) // 2


def triangle_area(v0, v1, v2) -> float:
    """Heron area of one triangle, radicand clamped at 0 (scalar helper)."""
    p = [np.asarray(v, dtype=np.float64) for v in (v0, v1, v2)]
    a = float(np.linalg.norm(p[1] - p[0]))
    b = float(np.linalg.norm(p[2] - p[1]))
    c = float(np.linalg.norm(p[2] - p[0]))
    s = 0.5 * (a + b + c)
    return math.sqrt(max(s * (s - a) * (s - b) * (s - c), 0.0))


def adaptive_resolution(area: float, k: float) -> int:
    """Smallest r with (r+1)(r+2)/2 >= k * area, at least 1 (paper Eq. 4)."""
    if k <= 0:
        raise ConfigError(f"sampling density k must be > 0, got {k}")
    if area < 0:
        raise ValueError("negative area")
    disc = 1.0 + 8.0 * k * area
    if disc < 25.0:
        return 1
    return max(1, math.ceil((-3.0 + math.sqrt(disc)) / 2.0))


def sample_index_to_rowcol(idx: int) -> tuple:
    """O(1) (row, col) of a within-triangle sample index (paper Eq. 2)."""
    if idx < 0:
        raise IndexError(f"negative sample index {idx}")
    row = math.ceil((-3.0 + math.sqrt(8.0 * idx + 9.0)) / 2.0)
    while idx - row * (row + 1) // 2 < 0:
        row -= 1
    while idx - row * (row + 1) // 2 > row:
        row += 1
    return row, idx - row * (row + 1) // 2


def rowcol_to_barycentric(row: int, col: int, r: int) -> tuple:
    """Weights (col/r, (row-col)/r, 1-row/r) of grid sample (row, col)."""
    if r < 1:
        raise IndexError(f"resolution must be >= 1, got {r}")
    if not 0 <= col <= row <= r:
        raise IndexError(f"sample (row={row}, col={col}) out of range for r={r}")
    return col / r, (row - col) / r, 1.0 - row / r


@dataclass(frozen=True)
class TriangleSampling:
    resolution_r: int
    sample_count: int
    sample_offset: int

    def __post_init__(self):
        if self.resolution_r < 1:
            raise ValueError("resolution must be >= 1")
        if self.sample_count != sample_count(self.resolution_r):
            raise ValueError("sample_count inconsistent with resolution")


@dataclass(frozen=True)
class SampledMesh:
    """Per-triangle sample layout of one object (int64 arrays of length T;
    offsets = exclusive prefix sum of counts)."""

    object_id: str
    resolutions: np.ndarray
    counts: np.ndarray
    offsets: np.ndarray
    total_samples: int
    sampling_density_k: float

    def triangle_sampling(self, triangle_index: int) -> TriangleSampling:
        i = triangle_index
        return TriangleSampling(int(self.resolutions[i]), int(self.counts[i]), int(self.offsets[i]))

    def sample_triangle_arrays(self) -> tuple:
        """(triangle index, index within triangle) of every sample."""
        tri = np.repeat(np.arange(len(self.counts), dtype=np.int64), self.counts)
        return tri, np.arange(self.total_samples, dtype=np.int64) - self.offsets[tri]


def _local_triangles(mesh) -> np.ndarray:
    v = np.asarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(mesh.faces, dtype=np.int64).reshape(-1, 3)
    return np.ascontiguousarray(v[f])


def build_sampled_mesh(mesh, k: float, object_id: str = "", device: int = 0) -> SampledMesh:
    """Adaptive resolution + contiguous sample block per triangle, on the GPU
    (k_layout: Heron area -> r -> count; CUB exclusive scan -> offsets)."""
    if not k > 0:
        raise ConfigError(f"sampling density k must be > 0, got {k}")
    tri = _local_triangles(mesh)
    T = len(tri)
    res = np.zeros(T, np.int64)
    cnt = np.zeros(T, np.int64)
    off = np.zeros(T, np.int64)
    total = np.zeros(1, np.int64)
    if T:
        lib = _native.load()
        _native.check(lib.gm_layout(device, _native.dptr(tri), T, float(k), _native.iptr(res), _native.iptr(cnt),
                                    _native.iptr(off), _native.iptr(total)), "gm_layout")
    return SampledMesh(object_id, res, cnt, off, int(total[0]), float(k))


def build_sampled_meshes(scene, k: float, device: int = 0) -> dict:
    """Layout for every scene object, keyed by object_id in scene order."""
    return {o.object_id: build_sampled_mesh(o.mesh, k, o.object_id, device) for o in scene.objects}


def sample_positions_local(mesh, sampled, transform=None, device: int = 0) -> np.ndarray:
    """(N, 3) sample positions in layout order, on the GPU (k_positions);
    local space, or world space when `transform` is given."""
    n = int(sampled.total_samples)
    out = np.zeros((n, 3))
    if n == 0:
        return out
    tri = _local_triangles(mesh)
    res = np.ascontiguousarray(sampled.resolutions, dtype=np.int64)
    off = np.ascontiguousarray(sampled.offsets, dtype=np.int64)
    xf = None
    if transform is not None:
        xf = np.ascontiguousarray(np.concatenate([transform.translation, transform.rotation, transform.scale]),
                                  dtype=np.float64)
    lib = _native.load()
    _native.check(lib.gm_sample_positions(device, _native.dptr(tri), len(tri), _native.iptr(res),
                                          _native.iptr(off), n, _native.dptr(xf), _native.dptr(out)),
                  "gm_sample_positions")
    return out


def sample_world_position(scene_object, sampled, triangle_index: int, sample_index: int,
                          transform: Transform | None = None) -> np.ndarray:
    """World position of one sample (scalar helper, host side)."""
    if not 0 <= triangle_index < len(sampled.counts):
        raise IndexError(f"triangle index {triangle_index} out of range")
    if not 0 <= sample_index < sampled.counts[triangle_index]:
        raise IndexError(f"sample index {sample_index} out of range")
    r = int(sampled.resolutions[triangle_index])
    w = rowcol_to_barycentric(*sample_index_to_rowcol(sample_index), r)
    v = scene_object.mesh.triangle_vertices()[triangle_index]
    local = w[0] * v[0] + w[1] * v[1] + w[2] * v[2]
    t = scene_object.transform if transform is None else transform
    return t.apply(local[None, :])[0]
