"""Golden dynamic-scene case, produced by the REFERENCE's
generate() with per-fixation pose overrides (gazemap/density.py:123-127,
161-165).

    python tests/golden/make_dynamic_golden.py

Scene: workloads.rotated_object_scene (three objects with non-trivial
transforms), k = 3000; 40 orbit fixations.  Overrides: runs that move or
rotate the statue and the cube, one fixation moving both, one naming an
object that is not in the scene (ignored by the reference), and the base
pose in between.  Writes tests/golden/dynamic.npz: scene arrays, the fixation
table, the override specification (fixation, object index or -1, 10 floats)
and the reference's un-normalized values + global max, with filtering on
and off.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GAZEMAP_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import gazemap as R  # noqa: E402

import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "dynamic.npz"


def overrides_spec(n_fix: int):
    """(fixation, object index or -1 for an unknown id, [t q s]) triples."""
    q1 = np.array([0.1, -0.2, 0.05, 0.97])
    q1 /= np.linalg.norm(q1)
    q2 = np.array([0.0, 0.38268343236508984, 0.0, 0.9238795325112867])
    spec = []
    for f in range(n_fix):
        if 8 <= f < 16:  # the statue moves along x, the same pose for the whole run
            spec.append((f, 0, [-0.4, 0.1, 0.3, *q1, 1.0, 1.3, 0.9]))
        if 16 <= f < 22:  # the cube spins a different amount every fixation
            spec.append((f, 1, [0.1 * (f - 16), 0.0, 0.2, *q2, 1.0, 1.0, 1.0]))
        if f == 27:  # both, plus an id the scene does not have
            spec.append((f, 0, [0.8, -0.2, 0.0, 0.0, 0.0, 0.0, 1.0, 0.7, 0.7, 0.7]))
            spec.append((f, 1, [-0.3, 0.0, 0.6, *q1, 1.2, 1.0, 1.0]))
            spec.append((f, -1, [5.0, 5.0, 5.0, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1.0]))
        if f == 33:  # the plane is rescaled
            spec.append((f, 2, [1.7, 0.0, -0.5, 0.0, 0.0, 0.0, 1.0, 1.0, 1.5, 1.0]))
    return spec


def main():
    scene_b = W.rotated_object_scene()
    objs = []
    for o in scene_b.objects:
        t = o.transform
        objs.append(R.SceneObject(o.object_id, R.Mesh(o.mesh.vertices, o.mesh.faces),
                                  R.Transform(t.translation, t.rotation, t.scale)))
    scene = R.Scene(tuple(objs))
    fx_table = W.orbit_fixations(40, 11, 1.2, 4.0, jitter=0.5, max_tilt=0.3)
    spec = overrides_spec(len(fx_table))
    ids = scene.object_ids
    fixations = []
    for f, row in enumerate(fx_table):
        ov = {}
        for ff, oi, v in spec:
            if ff == f:
                oid = ids[oi] if oi >= 0 else "not_in_scene"
                ov[oid] = R.Transform(np.array(v[0:3]), np.array(v[3:7]), np.array(v[7:10]))
        fixations.append(R.Fixation(row[0], row[1], row[2:5], row[5:9], tuple(row[9:15]), row[15:18], overrides=ov))
    d = {"ids": np.array(ids), "fix": fx_table,
         "spec_f": np.array([s[0] for s in spec], np.int64), "spec_o": np.array([s[1] for s in spec], np.int64),
         "spec_v": np.array([s[2] for s in spec], np.float64), "k": np.float64(3000.0)}
    for i, o in enumerate(scene.objects):
        d[f"v{i}"] = o.mesh.vertices
        d[f"f{i}"] = o.mesh.faces
        d[f"t{i}"] = np.concatenate([o.transform.translation, o.transform.rotation, o.transform.scale])
    for filt in (True, False):
        cfg = R.GenerationConfig(k=3000.0, filtering_enabled=filt)
        sm = R.build_sampled_meshes(scene, cfg.k)
        dm = R.generate(scene, sm, fixations, cfg)
        tag = "on" if filt else "off"
        d[f"gmax_{tag}"] = np.float64(dm.global_max)
        for i, oid in enumerate(ids):
            d[f"val_{tag}{i}"] = dm.values[oid]
        static = R.generate(scene, sm, [R.Fixation(f.start_time, f.duration, f.camera_position, f.camera_rotation,
                                                   f.frustum, f.gaze_dir) for f in fixations], cfg)
        diff = sum(int((static.values[o] != dm.values[o]).sum()) for o in ids)
        print(f"filtering {tag}: gmax {dm.global_max:.6g}, {diff} samples differ from the static scene")
    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
