"""Golden export/persistence bytes from the REFERENCE's
write_export (gazemap/io_export.py:63-116) and save_map (:211-229).

    python tests/golden/make_export_golden.py

Scene: workloads.rotated_object_scene (non-trivial transforms: the world
columns exercise the FMA-chain transform), k = 300.  Values are crafted to
hit every '.9g' formatting branch (zeros, -0.0, subnormals, exponent
switch-overs at 1e-5 / 1e9, rounding carries, inf, nan, huge).  Stores the
exact CSV and GAZEMAP1 bytes (zlib-compressed) in tests/golden/export.npz.
"""

from __future__ import annotations

import os
import sys
import tempfile
import zlib
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GAZEMAP_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import gazemap as R  # noqa: E402

import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "export.npz"
SPECIAL = [0.0, -0.0, 5e-324, 2.2250738585072014e-308, 1e-5, 9.9999999995e-06, 0.0001, 123456789.0,
           999999999.5, 1e9, 999999999.4, 0.1, 1.0 / 3.0, 2.0 / 3.0, 12345.6789012345, -1.5, 1e300, -1e-300,
           float("inf"), float("-inf"), float("nan"), 0.99999999995, 9.9999999949e22]


def values_for(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = rng.uniform(0.0, 25.0, n) * 10.0 ** rng.integers(-8, 12, n)
    v[rng.uniform(size=n) < 0.3] = 0.0
    k = min(len(SPECIAL), n)
    v[:k] = SPECIAL[:k]
    return v


def main():
    scene_b = W.rotated_object_scene()
    objs = []
    for o in scene_b.objects:
        t = o.transform
        objs.append(R.SceneObject(o.object_id, R.Mesh(o.mesh.vertices, o.mesh.faces),
                                  R.Transform(t.translation, t.rotation, t.scale)))
    scene = R.Scene(tuple(objs))
    k = 300.0
    sm = R.build_sampled_meshes(scene, k)
    values = {oid: values_for(sm[oid].total_samples, i) for i, oid in enumerate(scene.object_ids)}
    dm = R.DensityMap(values, global_max=12.5, normalized=False)
    d = {"k": np.float64(k), "ids": np.array(scene.object_ids)}
    for i, oid in enumerate(scene.object_ids):
        d[f"val{i}"] = values[oid]
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "export.csv"
        n = R.write_export(dm, scene, sm, p)
        d["csv"] = np.frombuffer(zlib.compress(p.read_bytes(), 9), np.uint8)
        d["count"] = np.int64(n)
        p2 = Path(td) / "sub.csv"
        R.write_export(dm, scene, sm, p2, objects=["plane", "cube"])
        d["csv_sub"] = np.frombuffer(zlib.compress(p2.read_bytes(), 9), np.uint8)
        m = Path(td) / "map.gzm"
        R.save_map(dm, m, "abc123", k)
        d["map"] = np.frombuffer(zlib.compress(m.read_bytes(), 9), np.uint8)
    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}: {n} records")


if __name__ == "__main__":
    main()
