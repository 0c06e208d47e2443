"""Synthetic scenes and fixation streams for tests and bench.py (SURVEY.md
section 8d configs C1-C5).  Geometry is built in world coordinates from
primitive meshes; fixation streams are seeded numpy generators.

Only numpy and the package's data model are used; nothing here computes
densities.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2601_07571_b200 import Mesh, Scene, SceneObject, Transform

FRUSTUM = (-0.1, 0.1, 0.1, -0.1, 0.1, 100.0)  # 90 degree FOV, near 0.1, far 100


# ------------------------------------------------------------- primitives

def quad(half: float = 5.0, z: float = 0.0) -> Mesh:
    v = np.array([[-half, -half, z], [half, -half, z], [half, half, z], [-half, half, z]], dtype=np.float64)
    return Mesh(v, np.array([[0, 1, 2], [0, 2, 3]]))


def grid(nx: int, ny: int, sx: float, sy: float, z: float = 0.0) -> Mesh:
    """nx*ny cells (two triangles each) in the xy plane, centred."""
    xs = np.linspace(-sx / 2, sx / 2, nx + 1)
    ys = np.linspace(-sy / 2, sy / 2, ny + 1)
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    v = np.column_stack([gx.ravel(), gy.ravel(), np.full(gx.size, z)])
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    a = (i * (ny + 1) + j).ravel()
    b = ((i + 1) * (ny + 1) + j).ravel()
    f = np.empty((2 * a.size, 3), np.int64)
    f[0::2] = np.column_stack([a, b, b + 1])
    f[1::2] = np.column_stack([a, b + 1, a + 1])
    return Mesh(v, f)


def box(half: float = 1.0) -> Mesh:
    h = half
    v = np.array([[-h, -h, -h], [h, -h, -h], [h, h, -h], [-h, h, -h],
                  [-h, -h, h], [h, -h, h], [h, h, h], [-h, h, h]], dtype=np.float64)
    f = np.array([[0, 2, 1], [0, 3, 2], [4, 5, 6], [4, 6, 7], [0, 1, 5], [0, 5, 4],
                  [2, 3, 7], [2, 7, 6], [1, 2, 6], [1, 6, 5], [0, 4, 7], [0, 7, 3]])
    return Mesh(v, f)


def icosphere(level: int = 2, radius: float = 1.0) -> Mesh:
    """Subdivided icosahedron projected to the sphere (20 * 4^level faces)."""
    p = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, p, 0), (1, p, 0), (-1, -p, 0), (1, -p, 0), (0, -1, p), (0, 1, p), (0, -1, -p), (0, 1, -p),
             (p, 0, -1), (p, 0, 1), (-p, 0, -1), (-p, 0, 1)]
    verts = [np.array(v, dtype=np.float64) / np.linalg.norm(v) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
             (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        mid = {}

        def m(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in mid:
                c = verts[a] + verts[b]
                verts.append(c / np.linalg.norm(c))
                mid[key] = len(verts) - 1
            return mid[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = m(a, b), m(b, c), m(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return Mesh(np.array(verts) * radius, np.array(faces))


def _moved(mesh: Mesh, offset) -> Mesh:
    return Mesh(mesh.vertices + np.asarray(offset, dtype=np.float64), mesh.faces)


def _rotated(mesh: Mesh, R: np.ndarray, offset=(0.0, 0.0, 0.0)) -> Mesh:
    return Mesh(mesh.vertices @ R.T + np.asarray(offset, dtype=np.float64), mesh.faces)


# ------------------------------------------------------------- cameras

def look_at_quat(position, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """Quaternion (xyzw) of a camera at `position` whose -z looks at target."""
    fwd = np.asarray(target, np.float64) - np.asarray(position, np.float64)
    fwd /= np.linalg.norm(fwd)
    upv = np.asarray(up, np.float64)
    if abs(float(fwd @ upv)) > 0.999:
        upv = np.array([1.0, 0.0, 0.0])
    right = np.cross(fwd, upv)
    right /= np.linalg.norm(right)
    true_up = np.cross(right, fwd)
    m = np.column_stack([right, true_up, -fwd])
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        q = [(m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s, 0.25 * s]
    elif m[0, 0] > m[1, 1] and m[0, 0] > m[2, 2]:
        s = math.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2
        q = [0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s, (m[2, 1] - m[1, 2]) / s]
    elif m[1, 1] > m[2, 2]:
        s = math.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2
        q = [(m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s, (m[0, 2] - m[2, 0]) / s]
    else:
        s = math.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2
        q = [(m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s, (m[1, 0] - m[0, 1]) / s]
    q = np.array(q)
    return q / np.linalg.norm(q)


def tilted_gaze(rng, max_tilt: float) -> np.ndarray:
    """(0,0,-1) rotated by U(0, max_tilt) about a random xy axis (unit)."""
    a = rng.uniform(0.0, 2.0 * math.pi)
    ang = rng.uniform(0.0, max_tilt)
    g = np.array([math.sin(ang) * math.sin(a), -math.sin(ang) * math.cos(a), -math.cos(ang)])
    return g / np.linalg.norm(g)


def fixation_rows(positions, targets, gazes, durations, start_step=0.25) -> np.ndarray:
    """(F, 18) fixation table (log column order) for the given cameras."""
    F = len(positions)
    t = np.empty((F, 18))
    for i in range(F):
        t[i, 0] = start_step * i
        t[i, 1] = durations[i]
        t[i, 2:5] = positions[i]
        t[i, 5:9] = look_at_quat(positions[i], targets[i])
        t[i, 9:15] = FRUSTUM
        t[i, 15:18] = gazes[i]
    return t


def orbit_fixations(n: int, seed: int, r_lo: float, r_hi: float, center=(0.0, 0.0, 0.0), jitter=0.0,
                    max_tilt=0.15) -> np.ndarray:
    """Cameras at radius U(r_lo, r_hi) in uniform directions, looking at the
    centre (+ optional target jitter)."""
    rng = np.random.default_rng(seed)
    c = np.asarray(center, np.float64)
    pos, tgt, gz, dur = [], [], [], []
    for _ in range(n):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        pos.append(c + d * rng.uniform(r_lo, r_hi))
        tgt.append(c + (rng.normal(size=3) * jitter if jitter else 0.0))
        gz.append(tilted_gaze(rng, max_tilt))
        dur.append(rng.uniform(0.1, 0.6))
    return fixation_rows(pos, tgt, gz, dur)


# ------------------------------------------------------------- configs

def c1():
    """C1: icosphere(3) radius 1, k = 1000 (N = 14,400), 200 fixations."""
    scene = Scene((SceneObject("icosphere", icosphere(3, 1.0)),))
    return scene, 1000.0, orbit_fixations(200, 0, 2.5, 4.0)


def room_scene(seed: int = 2) -> Scene:
    """C2 room: 8 x 6 x 3 m, floor/ceiling 120x100 cells, walls 80x30 and
    60x30 cells, 6 icosphere(4) props r=0.4 and 8 icosphere(2) props r=0.25
    (T = 98,080 triangles, 20 objects)."""
    rng = np.random.default_rng(seed)
    Rx = np.array([[1, 0, 0], [0, 0, -1], [0, 1, 0]], dtype=np.float64)    # xy-plane -> xz-plane (normal +y)
    Ry90 = np.array([[0, 0, 1], [0, 1, 0], [-1, 0, 0]], dtype=np.float64)  # xy-plane -> zy-plane (normal +x)
    objs = [SceneObject("floor", _rotated(grid(120, 100, 8.0, 6.0), Rx, (0.0, 0.0, 0.0))),
            SceneObject("ceiling", _rotated(grid(120, 100, 8.0, 6.0), Rx, (0.0, 3.0, 0.0))),
            SceneObject("wall_n", _moved(grid(80, 30, 8.0, 3.0), (0.0, 1.5, -3.0))),
            SceneObject("wall_s", _moved(grid(80, 30, 8.0, 3.0), (0.0, 1.5, 3.0))),
            SceneObject("wall_w", _rotated(grid(60, 30, 6.0, 3.0), Ry90, (-4.0, 1.5, 0.0))),
            SceneObject("wall_e", _rotated(grid(60, 30, 6.0, 3.0), Ry90, (4.0, 1.5, 0.0)))]
    big = icosphere(4, 0.4)
    small = icosphere(2, 0.25)
    for i in range(6):
        objs.append(SceneObject(f"prop{i}", _moved(big, (rng.uniform(-3, 3), 0.8, rng.uniform(-2, 2)))))
    for i in range(8):
        objs.append(SceneObject(f"bowl{i}", _moved(small, (rng.uniform(-3, 3), 1.2, rng.uniform(-2, 2)))))
    return Scene(tuple(objs))


def room_fixations(n: int, seed: int = 1, scene: Scene | None = None) -> np.ndarray:
    """C2 stream: cameras U(-3.5,3.5) x U(1.2,1.9) x U(-2.5,2.5), each looking at
    a random prop centre or wall point, gaze tilted U(0, 0.15) rad."""
    scene = scene or room_scene()
    rng = np.random.default_rng(seed)
    props = [o.mesh.vertices.mean(axis=0) for o in scene.objects if o.object_id.startswith(("prop", "bowl"))]
    pos = np.column_stack([rng.uniform(-3.5, 3.5, n), rng.uniform(1.2, 1.9, n), rng.uniform(-2.5, 2.5, n)])
    tgt, gz, dur = [], [], []
    for i in range(n):
        if rng.uniform() < 0.6:
            t = props[rng.integers(len(props))]
        else:
            t = np.array([rng.uniform(-3.9, 3.9), rng.uniform(0.1, 2.9), rng.choice([-3.0, 3.0])])
        if np.linalg.norm(t - pos[i]) < 0.3:
            t = t + np.array([0.0, 0.0, -1.0])
        tgt.append(t)
        gz.append(tilted_gaze(rng, 0.15))
        dur.append(rng.uniform(0.1, 0.6))
    return fixation_rows(pos, tgt, gz, dur)


def c2(n_fix: int = 100_000):
    scene = room_scene()
    return scene, 10_000.0, room_fixations(n_fix, 1, scene)


def look_at_quats(positions, targets, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """Row-wise look_at_quat for (F, 3) cameras and targets (same formulas,
    vectorised; results can differ from the scalar version in the last bit)."""
    p = np.asarray(positions, np.float64)
    fwd = np.asarray(targets, np.float64) - p
    fwd /= np.sqrt((fwd * fwd).sum(axis=1))[:, None]
    upv = np.broadcast_to(np.asarray(up, np.float64), fwd.shape).copy()
    upv[np.abs(fwd @ np.asarray(up, np.float64)) > 0.999] = (1.0, 0.0, 0.0)
    right = np.cross(fwd, upv)
    right /= np.sqrt((right * right).sum(axis=1))[:, None]
    true_up = np.cross(right, fwd)
    m = np.stack([right, true_up, -fwd], axis=2)  # columns
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    q = np.empty((len(p), 4))
    c0 = tr > 0
    c1 = ~c0 & (m[:, 0, 0] > m[:, 1, 1]) & (m[:, 0, 0] > m[:, 2, 2])
    c2 = ~c0 & ~c1 & (m[:, 1, 1] > m[:, 2, 2])
    c3 = ~(c0 | c1 | c2)
    with np.errstate(invalid="ignore", divide="ignore"):
        s0 = np.sqrt(tr + 1.0) * 2
        s1 = np.sqrt(1.0 + m[:, 0, 0] - m[:, 1, 1] - m[:, 2, 2]) * 2
        s2 = np.sqrt(1.0 + m[:, 1, 1] - m[:, 0, 0] - m[:, 2, 2]) * 2
        s3 = np.sqrt(1.0 + m[:, 2, 2] - m[:, 0, 0] - m[:, 1, 1]) * 2
        cand = [
            (c0, np.stack([(m[:, 2, 1] - m[:, 1, 2]) / s0, (m[:, 0, 2] - m[:, 2, 0]) / s0,
                           (m[:, 1, 0] - m[:, 0, 1]) / s0, 0.25 * s0], axis=1)),
            (c1, np.stack([0.25 * s1, (m[:, 0, 1] + m[:, 1, 0]) / s1, (m[:, 0, 2] + m[:, 2, 0]) / s1,
                           (m[:, 2, 1] - m[:, 1, 2]) / s1], axis=1)),
            (c2, np.stack([(m[:, 0, 1] + m[:, 1, 0]) / s2, 0.25 * s2, (m[:, 1, 2] + m[:, 2, 1]) / s2,
                           (m[:, 0, 2] - m[:, 2, 0]) / s2], axis=1)),
            (c3, np.stack([(m[:, 0, 2] + m[:, 2, 0]) / s3, (m[:, 1, 2] + m[:, 2, 1]) / s3, 0.25 * s3,
                           (m[:, 1, 0] - m[:, 0, 1]) / s3], axis=1)),
        ]
    for mask, val in cand:
        q[mask] = val[mask]
    return q / np.sqrt((q * q).sum(axis=1))[:, None]


def session_fixations(users: int = 50, per_user: int = 20_000, scene: Scene | None = None,
                      first_user: int = 0) -> np.ndarray:
    """C4: users first_user .. first_user + users - 1, concatenated; user u
    (seed 100 + u) walks the room (steps N(0, 0.05) m, eye height 1.6 +- 0.1,
    clamped to the room) and picks a new target every 5 fixations (a prop
    centre with p = 0.6, else a random wall point); gaze tilted U(0, 0.15) rad,
    durations U(0.1, 0.6) s.  Vectorised per user."""
    scene = scene or room_scene()
    props = np.array([o.mesh.vertices.mean(axis=0) for o in scene.objects
                      if o.object_id.startswith(("prop", "bowl"))])
    rows = []
    n = per_user
    for u in range(first_user, first_user + users):
        rng = np.random.default_rng(100 + u)
        p0 = np.array([rng.uniform(-3, 3), 1.6 + rng.uniform(-0.1, 0.1), rng.uniform(-2, 2)])
        steps = rng.normal(0.0, 0.05, (n, 3))
        lo, hi = np.array([-3.7, 1.5, -2.7]), np.array([3.7, 1.7, 2.7])
        pos = np.empty((n, 3))
        p = p0
        for i in range(n):  # clamped random walk (sequential by nature)
            p = np.minimum(np.maximum(p + steps[i], lo), hi)
            pos[i] = p
        n_t = (n + 4) // 5
        pick_prop = rng.uniform(size=n_t) < 0.6
        prop_idx = rng.integers(len(props), size=n_t)
        wall = np.column_stack([rng.uniform(-3.9, 3.9, n_t), rng.uniform(0.1, 2.9, n_t),
                                rng.choice([-3.0, 3.0], n_t)])
        tgt = np.where(pick_prop[:, None], props[prop_idx], wall)[np.arange(n) // 5]
        near = np.sqrt(((tgt - pos) ** 2).sum(axis=1)) <= 0.3
        tgt = tgt + near[:, None] * np.array([0.0, 0.0, -1.0])
        a = rng.uniform(0.0, 2.0 * math.pi, n)
        ang = rng.uniform(0.0, 0.15, n)
        g = np.column_stack([np.sin(ang) * np.sin(a), -np.sin(ang) * np.cos(a), -np.cos(ang)])
        g /= np.sqrt((g * g).sum(axis=1))[:, None]
        dur = rng.uniform(0.1, 0.6, n)
        t = np.empty((n, 18))
        t[:, 0] = 0.25 * np.arange(n)
        t[:, 1] = dur
        t[:, 2:5] = pos
        t[:, 5:9] = look_at_quats(pos, tgt)
        t[:, 9:15] = FRUSTUM
        t[:, 15:18] = g
        rows.append(t)
    return np.concatenate(rows) if rows else np.zeros((0, 18))


def shells_scene() -> Scene:
    """C5: 12 concentric icosphere(6) shells of radius 0.5 + 0.25 i
    (T = 983,040): occlusion-dominated."""
    base = icosphere(6, 1.0)
    return Scene(tuple(SceneObject(f"shell{i}", Mesh(base.vertices * (0.5 + 0.25 * i), base.faces))
                       for i in range(12)))


def c5(n_fix: int = 50_000):
    return shells_scene(), 20_000.0, orbit_fixations(n_fix, 4, 4.5, 6.0, jitter=0.3)


def rotated_object_scene() -> Scene:
    """A small scene whose objects carry non-trivial transforms (exercises
    the FMA-chain world transform)."""
    q = np.array([0.2, 0.3, 0.1, 0.95])
    q /= np.linalg.norm(q)
    q2 = np.array([-0.4, 0.1, 0.3, 0.8])
    q2 /= np.linalg.norm(q2)
    return Scene((SceneObject("statue", icosphere(2, 0.4), Transform([-1.2, 0.1, 0.0], q, [1.0, 1.3, 0.9])),
                  SceneObject("cube", box(0.4), Transform([0.0, 0.0, 0.2], q2, [1.0, 1.0, 1.0])),
                  SceneObject("plane", grid(8, 12, 1.0, 2.0), Transform([1.7, 0.0, -0.5], [0, 0, 0, 1], [2, 1, 1]))))
