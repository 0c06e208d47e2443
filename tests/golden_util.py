"""Rebuild the golden cases (tests/golden/golden.npz, written by
tests/golden/make_golden.py from the reference) as this package's objects."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2601_07571_b200 import Mesh, Scene, SceneObject, Transform

PATH = Path(__file__).resolve().parent / "golden" / "golden.npz"


class Golden:
    def __init__(self, d):
        self.d = d

    def __getitem__(self, k):
        return self.d[k]

    def scene(self, prefix: str) -> Scene:
        ids = [str(x) for x in self.d[prefix + "ids"]]
        objs = []
        for i, oid in enumerate(ids):
            t = self.d[f"{prefix}t{i}"]
            objs.append(SceneObject(oid, Mesh(self.d[f"{prefix}v{i}"], self.d[f"{prefix}f{i}"]),
                                    Transform(t[0:3], t[3:7], t[7:10])))
        return Scene(tuple(objs))


def load() -> Golden:
    return Golden(dict(np.load(PATH, allow_pickle=False)))
