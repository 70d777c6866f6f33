"""Seeded synthetic wall meshes (input generation only — no method arithmetic).

The paper's benchmark geometry is an ideal cylinder, D = 4 cm, L = 30 cm, with both
ends fully fixed (§3.1).  Its meshes are unstructured (5,074 /
15,136 / 32,994 / 131,552 triangles) and not published,
so this module builds a structured "offset-ring" triangulation with the same
topology (an open tube, Euler characteristic 0) — recipe in SURVEY.md §8(d), c1-c3:

    node = r * n_circ + i,  theta = 2*pi*(i + 0.5*[r odd]) / n_circ,  z = L*r/(n_axial-1)

Triangles are oriented counter-clockwise about the outward normal (the ABI contract,
include/ens.h), so (X2-X1)x(X3-X1) points out of the lumen.

"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FIX_ALL = 7  # bit c set => displacement component c fixed (include/ens.h)


@dataclass
class Mesh:
    xyz: np.ndarray           # [V][3] float64, cm
    tris: np.ndarray          # [F][3] int32, 0-based, CCW about the outward normal
    fixed: np.ndarray         # [V] uint8 bitmask
    name: str = "mesh"
    meta: dict = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_tris(self) -> int:
        return int(self.tris.shape[0])


def _orient_outward(xyz: np.ndarray, tris: np.ndarray, inside_point_fn) -> np.ndarray:
    """Swap nodes 2/3 of every triangle whose normal points towards inside_point_fn(centroid)."""
    X = xyz[tris]
    n = np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0])
    c = X.mean(axis=1)
    out = c - inside_point_fn(c)
    flip = np.einsum("ij,ij->i", n, out) < 0
    tris = tris.copy()
    tris[flip, 1], tris[flip, 2] = tris[flip, 2].copy(), tris[flip, 1].copy()
    return tris


def cylinder(n_circ: int, n_axial: int, D: float = 4.0, L: float = 30.0,
             fix_ends: bool = True) -> Mesh:
    """Structured offset-ring cylinder: V = n_circ*n_axial, F = 2*n_circ*(n_axial-1).

    c1: cylinder(12, 23)  -> V = 276,    F = 528
    c2: cylinder(96, 262) -> V = 25,152, F = 50,112
    """
    if n_circ < 3 or n_axial < 2:
        raise ValueError("cylinder needs n_circ >= 3 and n_axial >= 2")
    R = 0.5 * D
    r = np.arange(n_axial)
    i = np.arange(n_circ)
    rr, ii = np.meshgrid(r, i, indexing="ij")
    theta = 2.0 * np.pi * (ii + 0.5 * (rr % 2)) / n_circ
    z = L * rr / (n_axial - 1)
    xyz = np.stack([R * np.cos(theta), R * np.sin(theta), z], axis=-1).reshape(-1, 3)

    tris = []
    for ring in range(n_axial - 1):
        a = ring * n_circ + i
        b = (ring + 1) * n_circ + i
        a1 = ring * n_circ + (i + 1) % n_circ
        b1 = (ring + 1) * n_circ + (i + 1) % n_circ
        if ring % 2 == 0:   # upper ring offset by +half a cell
            tris.append(np.stack([a, a1, b], 1))
            tris.append(np.stack([b, a1, b1], 1))
        else:               # lower ring offset by +half a cell
            tris.append(np.stack([a, a1, b1], 1))
            tris.append(np.stack([a, b1, b], 1))
    tris = np.concatenate(tris).astype(np.int32)
    tris = _orient_outward(xyz, tris, lambda c: np.stack([0 * c[:, 0], 0 * c[:, 1], c[:, 2]], 1))

    fixed = np.zeros(xyz.shape[0], np.uint8)
    if fix_ends:
        fixed[:n_circ] = FIX_ALL
        fixed[-n_circ:] = FIX_ALL
    return Mesh(np.ascontiguousarray(xyz), np.ascontiguousarray(tris), fixed,
                name=f"cylinder_{n_circ}x{n_axial}",
                meta=dict(kind="cylinder", R=R, L=L, n_circ=n_circ, n_axial=n_axial))


def perturb(mesh: Mesh, amplitude: float, seed: int) -> Mesh:
    """Jitter every node by a seeded uniform offset (for tests on irregular elements)."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    xyz = mesh.xyz + amplitude * rng.uniform(-1.0, 1.0, mesh.xyz.shape)
    return Mesh(xyz, mesh.tris.copy(), mesh.fixed.copy(), name=mesh.name + "_jit", meta=dict(mesh.meta))


def shuffle_nodes(mesh: Mesh, seed: int) -> Mesh:
    """Randomly renumber nodes (and triangles) — exercises the RCM reordering."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    V = mesh.n_nodes
    p = rng.permutation(V)           # new id of old node k is inv[k]
    inv = np.empty(V, np.int64)
    inv[p] = np.arange(V)
    xyz = mesh.xyz[p]
    tris = inv[mesh.tris].astype(np.int32)
    tris = tris[rng.permutation(tris.shape[0])]
    fixed = mesh.fixed[p]
    return Mesh(np.ascontiguousarray(xyz), np.ascontiguousarray(tris), fixed,
                name=mesh.name + "_shuf", meta=dict(mesh.meta))
