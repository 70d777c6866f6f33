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


# --------------------------------------------------------------------------------------
# Synthetic branched aorta (configs c4 / c5).
# Main vessel: offset-ring tube swept along a centreline (ascending 5 cm, arch of bend
# radius 3 cm, descending 30 cm; radius 1.5 -> 1.2 -> 1.0 cm).  Each side branch replaces
# a patch of the main tube's triangles: the patch's boundary loop (a closed chain of
# existing nodes) becomes the branch's first ring, and further rings are extruded along
# the outward normal, blending from the loop's shape to a circle of radius R_b.  All open
# ends (aortic inlet/outlet and every branch end) are fully fixed.
# --------------------------------------------------------------------------------------

def _rmf(P):
    """Tangents and a rotation-minimising normal/binormal along polyline P[n][3]."""
    T = np.gradient(P, axis=0)
    T /= np.linalg.norm(T, axis=1, keepdims=True)
    a = np.array([1.0, 0.0, 0.0]) if abs(T[0, 0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    N = [np.cross(T[0], a) / np.linalg.norm(np.cross(T[0], a))]
    for k in range(1, len(P)):
        n = N[-1] - np.dot(N[-1], T[k]) * T[k]
        N.append(n / np.linalg.norm(n))
    N = np.array(N)
    return T, N, np.cross(T, N)


def _ring_tube_tris(n_rings, n_circ, base=0):
    """Offset-ring triangulation of rings 0..n_rings-1 (n_circ nodes each), CCW about
    the outward normal when ring nodes advance counter-clockwise about the tangent."""
    i = np.arange(n_circ)
    out = []
    for r in range(n_rings - 1):
        a = base + r * n_circ + i
        b = base + (r + 1) * n_circ + i
        a1 = base + r * n_circ + (i + 1) % n_circ
        b1 = base + (r + 1) * n_circ + (i + 1) % n_circ
        if r % 2 == 0:
            out += [np.stack([a, a1, b], 1), np.stack([b, a1, b1], 1)]
        else:
            out += [np.stack([a, a1, b1], 1), np.stack([a, b1, b], 1)]
    return np.concatenate(out) if out else np.zeros((0, 3), np.int64)


def _aorta_centreline(ds):
    pts = []
    n = max(2, int(round(5.0 / ds)))
    pts += [[0.0, 0.0, 5.0 * k / n] for k in range(n)]
    n = max(4, int(round(np.pi * 3.0 / ds)))
    pts += [[3.0 - 3.0 * np.cos(np.pi * k / n), 0.0, 5.0 + 3.0 * np.sin(np.pi * k / n)] for k in range(n)]
    n = max(2, int(round(30.0 / ds)))
    pts += [[6.0, 0.0, 5.0 - 30.0 * k / n] for k in range(n + 1)]
    P = np.array(pts)
    s = np.concatenate([[0.0], np.cumsum(np.linalg.norm(np.diff(P, axis=0), axis=1))])
    return P, s


def _boundary_loop(tris_removed, tris_kept_edges):
    """Ordered closed loop of nodes bounding a removed triangle patch (edges of exactly
    one removed triangle), walked in the removed triangles' winding direction."""
    from collections import Counter
    cnt = Counter()
    directed = {}
    for t in tris_removed:
        for k in range(3):
            a, b = int(t[k]), int(t[(k + 1) % 3])
            cnt[(min(a, b), max(a, b))] += 1
            directed[(a, b)] = True
    nxt = {}
    for (a, b) in directed:
        if cnt[(min(a, b), max(a, b))] == 1:
            nxt[a] = b
    start = min(nxt)
    loop = [start]
    while len(loop) <= len(nxt):
        v = nxt[loop[-1]]
        if v == start:
            break
        loop.append(v)
    if len(loop) != len(nxt):
        raise ValueError("patch boundary is not a single loop")
    return loop


def aorta(target_tris: int = 500_000, with_branches: bool = True) -> Mesh:
    """Synthetic patient-like aorta (~target_tris triangles), see the section comment."""
    L_main = 5.0 + 3.0 * np.pi + 30.0
    ds = float(np.sqrt(2.0 * L_main * 2 * np.pi * 1.25 / target_tris))
    m = _aorta(ds, with_branches)
    ds *= float(np.sqrt(m.n_tris / target_tris))        # one size correction
    return _aorta(ds, with_branches)


def _aorta(ds: float, with_branches: bool) -> Mesh:
    L_main = 5.0 + 3.0 * np.pi + 30.0
    P, s = _aorta_centreline(ds)
    n_circ = max(16, 2 * int(round(np.pi * 1.25 / ds)))
    R = np.interp(s, [0.0, 5.0, 5.0 + 3 * np.pi, L_main], [1.5, 1.5, 1.2, 1.0])
    T, N, B = _rmf(P)
    n_rings = len(P)
    ring = np.arange(n_rings)[:, None]
    th = 2 * np.pi * (np.arange(n_circ)[None, :] + 0.5 * (ring % 2)) / n_circ
    xyz = (P[:, None, :] + R[:, None, None] * (np.cos(th)[..., None] * N[:, None, :]
                                               + np.sin(th)[..., None] * B[:, None, :])).reshape(-1, 3)
    tris = _ring_tube_tris(n_rings, n_circ)
    # orient the main tube outward
    X = xyz[tris]
    nrm = np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0])
    cen = X.mean(1)
    rr = np.repeat(np.arange(n_rings - 1), 2 * n_circ)
    flip = np.einsum("ij,ij->i", nrm, cen - P[rr]) < 0
    tris[flip, 1], tris[flip, 2] = tris[flip, 2].copy(), tris[flip, 1].copy()
    fixed = np.zeros(len(xyz), np.uint8)
    fixed[:n_circ] = FIX_ALL
    fixed[(n_rings - 1) * n_circ:] = FIX_ALL
    keep = np.ones(len(tris), bool)
    new_xyz, new_tris, new_fixed = [xyz], [], [fixed]
    n_nodes = len(xyz)
    if with_branches:
        s_arch = 5.0 + 1.5 * np.pi                  # arch apex
        s_desc = 5.0 + 3.0 * np.pi
        # (arc position, angle about the tangent, radius, length)
        branches = [(s_arch - 2.2, 0.25, 0.60, 8.0), (s_arch, 0.25, 0.35, 8.0), (s_arch + 2.2, 0.25, 0.45, 8.0),
                    (s_desc + 12.0, 0.75, 0.35, 5.0), (s_desc + 16.0, 0.75, 0.35, 5.0),
                    (s_desc + 20.0, 0.0, 0.30, 5.0), (s_desc + 20.6, 0.5, 0.30, 5.0)]
        tri_ring = rr
        tri_cell = np.tile(np.repeat(np.arange(n_circ), 2), n_rings - 1)
        for (s_b, ang, Rb, Lb) in branches:
            r_c = int(np.searchsorted(s, s_b))
            th_c = 2 * np.pi * ang
            centre = P[r_c] + R[r_c] * (np.cos(th_c) * N[r_c] + np.sin(th_c) * B[r_c])
            loop = None
            for fac in (1.0, 1.08, 0.93, 1.17, 0.86):
                inner = np.linalg.norm(xyz - centre, axis=1) < fac * Rb
                sel = inner[tris].any(axis=1) & keep
                try:
                    loop = _boundary_loop(tris[sel], None)
                    break
                except ValueError:
                    continue
            if loop is None or not sel.any():
                continue
            keep &= ~sel
            loop = np.array(loop)
            Lxyz = xyz[loop]
            c = Lxyz.mean(0)
            axis = c - P[r_c]
            axis -= np.dot(axis, T[r_c]) * T[r_c]
            axis /= np.linalg.norm(axis)
            m = len(loop)
            nb = max(3, int(round(Lb / ds)))
            # loop direction: removed triangles' winding == outward CCW -> loop is CW seen
            # from outside along +axis; branch rings follow the loop order
            rel = Lxyz - c
            rel -= np.outer(rel @ axis, axis)
            dirs = rel / np.linalg.norm(rel, axis=1, keepdims=True)
            rings = [loop]
            bxyz = []
            for k in range(1, nb + 1):
                w = min(1.0, k / 3.0)                 # blend loop shape -> circle in 3 rings
                pos = (c + axis * (k * ds) + (1 - w) * (rel + 0.0) + w * Rb * dirs)
                ids = n_nodes + np.arange(m)
                n_nodes += m
                bxyz.append(pos)
                rings.append(ids)
            new_xyz.append(np.concatenate(bxyz))
            bf = np.zeros(m * nb, np.uint8)
            bf[-m:] = FIX_ALL
            new_fixed.append(bf)
            for k in range(nb):
                a, b = np.asarray(rings[k]), np.asarray(rings[k + 1])
                a1, b1 = np.roll(a, -1), np.roll(b, -1)
                new_tris += [np.stack([a, a1, b1], 1), np.stack([a, b1, b], 1)]
    all_xyz = np.concatenate(new_xyz)
    all_fixed = np.concatenate(new_fixed)
    parts = [tris[keep]] + new_tris
    all_tris = np.concatenate(parts).astype(np.int64)
    used = np.zeros(len(all_xyz), bool)
    used[all_tris.ravel()] = True
    newid = -np.ones(len(all_xyz), np.int64)
    newid[used] = np.arange(int(used.sum()))
    all_tris = newid[all_tris]
    all_xyz, all_fixed = all_xyz[used], all_fixed[used]
    all_tris = _orient_consistently(all_tris)
    return Mesh(np.ascontiguousarray(all_xyz), np.ascontiguousarray(all_tris.astype(np.int32)), all_fixed,
                name=f"aorta_{len(all_tris)}", meta=dict(kind="aorta", n_circ=n_circ, ds=ds))


def _orient_consistently(tris):
    """Flip triangles so every interior edge is traversed once in each direction, by BFS
    over the triangle adjacency from triangle 0 (outward by construction)."""
    from collections import deque
    F = len(tris)
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
    key = np.minimum(e[:, 0], e[:, 1]) * (int(tris.max()) + 1) + np.maximum(e[:, 0], e[:, 1])
    order = np.argsort(key, kind="stable")
    ks = key[order]
    tri_of = order % F
    pairs = {}
    same = np.nonzero(ks[1:] == ks[:-1])[0]
    nbr = [[] for _ in range(F)]
    for k in same:
        t1, t2 = int(tri_of[k]), int(tri_of[k + 1])
        nbr[t1].append(t2)
        nbr[t2].append(t1)
    tris = tris.copy()
    seen = np.zeros(F, bool)
    for root in range(F):
        if seen[root]:
            continue
        seen[root] = True
        q = deque([root])
        while q:
            f = q.popleft()
            tf = tris[f]
            dir_f = {(int(tf[k]), int(tf[(k + 1) % 3])) for k in range(3)}
            for g in nbr[f]:
                if seen[g]:
                    continue
                tg = tris[g]
                if any((int(tg[k]), int(tg[(k + 1) % 3])) in dir_f for k in range(3)):
                    tris[g, 1], tris[g, 2] = tg[2], tg[1]
                seen[g] = True
                q.append(g)
    return tris
