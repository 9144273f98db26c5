"""Triangle scenes for the tracer that feeds the GBS stage.

Mirror of the generators in the reference ``beamfield.scene``
(/root/reference/pkg/src/beamfield/scene.py:360-413) -- the benchmark scenes
of SURVEY.md 8(d) are built with them.  No BVH is built: the sm_100a tracer
searches all triangles (the same (t, index) lexicographic minimum that
bvh_nearest returns, kernels.py:54-116).  Any object exposing v0/v1/v2/refl/
bounds/diameter (including a reference ``beamfield.scene.Scene``) can be
traced.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

HARD_MATERIAL_ID = 0


@dataclass
class Scene:
    v0: np.ndarray      # (n, 3)
    v1: np.ndarray
    v2: np.ndarray
    refl: np.ndarray    # (n,) reflection coefficient per triangle
    bounds: np.ndarray  # (2, 3) world AABB; zeros for an empty scene
    category: tuple = ()

    @property
    def n_triangles(self) -> int:
        return self.v0.shape[0]

    @property
    def diameter(self) -> float:
        return float(np.linalg.norm(self.bounds[1] - self.bounds[0]))


def _assemble(v0, v1, v2, material_ids=None, categories=()) -> Scene:
    v0 = np.ascontiguousarray(v0, dtype=np.float64).reshape(-1, 3)
    v1 = np.ascontiguousarray(v1, dtype=np.float64).reshape(-1, 3)
    v2 = np.ascontiguousarray(v2, dtype=np.float64).reshape(-1, 3)
    n = v0.shape[0]
    if n:
        allv = np.concatenate([v0, v1, v2])
        bounds = np.stack([allv.min(axis=0), allv.max(axis=0)])
    else:
        bounds = np.zeros((2, 3))
    # Only the rigid material exists in the reference (scene.py:29-30): coefficient +1.
    return Scene(v0=v0, v1=v1, v2=v2, refl=np.ones(n), bounds=bounds,
                 category=tuple(categories))


def empty_scene() -> Scene:
    return _assemble(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)))


def make_ground_plane(half_extent: float = 1000.0, z: float = 0.0) -> Scene:
    """Two-triangle rigid square at height z (scene.py:360-367)."""
    h = half_extent
    a, b, c, d = (np.array(p, dtype=np.float64)
                  for p in ([-h, -h, z], [h, -h, z], [h, h, z], [-h, h, z]))
    return _assemble(np.stack([a, a]), np.stack([b, c]), np.stack([c, d]),
                     categories=("terrain", "terrain"))


def _box(cx, cy, sx, sy, h):
    """Five faces (no bottom) of an axis-aligned box on z=0, two triangles each."""
    x0, x1, y0, y1 = cx - sx / 2, cx + sx / 2, cy - sy / 2, cy + sy / 2
    lo = [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]
    bot = [np.array([x, y, 0.0]) for x, y in lo]
    top = [np.array([x, y, h]) for x, y in lo]
    quads = [(bot[i], bot[(i + 1) % 4], top[(i + 1) % 4], top[i]) for i in range(4)]
    quads.append((top[0], top[1], top[2], top[3]))
    for q in quads:
        yield q[0], q[1], q[2]
        yield q[0], q[2], q[3]


def make_city(nx: int = 6, ny: int = 6, spacing: float = 40.0, footprint: float = 20.0,
              ground_half: float = 250.0) -> Scene:
    """Block-grid city on a rigid ground plane (scene.py:388-413).

    Triangle order, vertex order and building heights h = 10 + 5*((3i + 5j) % 6)
    follow the reference generator, so traced paths carry the same bits.
    """
    g = make_ground_plane(ground_half)
    v0, v1, v2 = list(g.v0), list(g.v1), list(g.v2)
    cats = ["terrain"] * 2
    x_off = -(nx - 1) * spacing / 2
    y_off = -(ny - 1) * spacing / 2
    for i in range(nx):
        for j in range(ny):
            h = 10.0 + 5.0 * ((i * 3 + j * 5) % 6)
            for a, b, c in _box(x_off + i * spacing, y_off + j * spacing, footprint, footprint, h):
                v0.append(a)
                v1.append(b)
                v2.append(c)
                cats.append("building")
    return _assemble(np.array(v0), np.array(v1), np.array(v2), categories=cats)
