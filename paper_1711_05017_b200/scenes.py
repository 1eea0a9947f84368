"""Built-in geometry: primitives, extrusion, pair grids, demo scenes.

API-compatible with the reference's `geofield.scenes`
(/root/reference/pkg/src/geofield/scenes.py): the same primitives with the
same vertex/face order (so fields agree with the reference on identical
inputs), the same random polygon draw order, the same pair-grid sizing.
Added for the BASELINE.json configurations, which the reference does not
ship: a cylinder peg and a bored block
(peg-in-hole), an extruded gear pair, and a threaded bolt and nut -- all
closed, consistently oriented meshes that pass TriangleMesh validation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .descriptor import IntegrationPolicy, KernelSpec, SampleGrid, affinity_field
from .energy import PartAsset
from .solids import Polygon2, Solid, TriangleMesh

__all__ = [
    "box_mesh",
    "icosphere",
    "lbracket",
    "extrude_polygon",
    "random_polygon",
    "grid_for_pair",
    "build_pair_assets",
    "Scene",
    "SCENES",
    "get_scene",
    "regular_polygon",
    "cylinder_peg",
    "bored_block",
    "gear_profile",
    "gear",
    "threaded_bolt",
    "threaded_nut",
]


# ---------------------------------------------------------------------------
# primitives (scenes.py:31-94)

_BOX_FACES = np.array([
    [4, 6, 7], [4, 7, 5],   # +x
    [0, 1, 3], [0, 3, 2],   # -x
    [2, 3, 7], [2, 7, 6],   # +y
    [0, 4, 5], [0, 5, 1],   # -y
    [1, 5, 7], [1, 7, 3],   # +z
    [0, 2, 6], [0, 6, 4],   # -z
], dtype=np.int64)


def box_mesh(extents=(1.0, 1.0, 1.0), center=(0.0, 0.0, 0.0)):
    """Axis-aligned box; vertex i has the coordinate signs of bits (x, y, z) of i."""
    half = 0.5 * np.asarray(extents, dtype=np.float64)
    signs = np.array([[sx, sy, sz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)], dtype=np.float64)
    return Solid(TriangleMesh(signs * half + np.asarray(center, dtype=np.float64), _BOX_FACES.copy()))


_ICO_FACES = [
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
]


def icosphere(radius=1.0, subdivisions=3, center=(0.0, 0.0, 0.0)):
    """Geodesic sphere with 20 * 4^subdivisions faces."""
    t = (1.0 + np.sqrt(5.0)) / 2.0
    base = [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
            [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]]
    verts = [np.asarray(v, dtype=np.float64) / np.linalg.norm(v) for v in base]
    faces = list(_ICO_FACES)
    for _ in range(subdivisions):
        midpoint_of = {}

        def mid(i, j):
            key = (i, j) if i < j else (j, i)
            if key not in midpoint_of:
                m = verts[i] + verts[j]
                verts.append(m / np.linalg.norm(m))
                midpoint_of[key] = len(verts) - 1
            return midpoint_of[key]

        refined = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            refined += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = refined
    V = np.asarray(verts) * radius + np.asarray(center, dtype=np.float64)
    return Solid(TriangleMesh(V, np.asarray(faces, dtype=np.int64)))


_LBRACKET_LOOP = [(-0.5, -0.5), (0.5, -0.5), (0.5, -0.2), (-0.2, -0.2), (-0.2, 0.5), (-0.5, 0.5)]


def lbracket(height=0.4, scale=1.0):
    return extrude_polygon([np.asarray(_LBRACKET_LOOP, dtype=np.float64) * scale], height)


# ---------------------------------------------------------------------------
# extrusion (scenes.py:101-164)


def _point_in_tri(p, a, b, c):
    def side(u, v):
        return (v[0] - u[0]) * (p[1] - u[1]) - (v[1] - u[1]) * (p[0] - u[0])

    s = (side(a, b), side(b, c), side(c, a))
    return not (min(s) < 0 and max(s) > 0)


def _ear_clip(loop):
    """Triangulate one simple CCW loop (index triples)."""
    n = len(loop)
    idx = list(range(n))
    scale = float(np.max(np.abs(loop))) or 1.0
    tris = []
    guard = 0
    while len(idx) > 3:
        guard += 1
        if guard > n * n + 16:
            raise ValueError("ear clipping stalled; loop may be non-simple")
        m = len(idx)
        for k in range(m):
            i0, i1, i2 = idx[k - 1], idx[k], idx[(k + 1) % m]
            a, b, c = loop[i0], loop[i1], loop[i2]
            if (b[0] - a[0]) * (c[1] - b[1]) - (b[1] - a[1]) * (c[0] - b[0]) <= 1e-12 * scale * scale:
                continue  # reflex or degenerate corner
            if any(_point_in_tri(loop[j], a, b, c) for j in idx if j not in (i0, i1, i2)):
                continue
            tris.append((i0, i1, i2))
            del idx[k]
            break
        else:
            raise ValueError("no ear found; loop may be non-simple")
    tris.append(tuple(idx))
    return tris


def extrude_polygon(loops, height):
    """Prism over a single-loop polygon, centred on z = 0, outward normals."""
    poly = Polygon2(loops)
    if len(poly.loops) != 1:
        raise ValueError("extrusion supports a single loop")
    loop = poly.loops[0]
    n = len(loop)
    h = 0.5 * float(height)
    verts = np.vstack([np.column_stack([loop, np.full(n, -h)]), np.column_stack([loop, np.full(n, h)])])
    faces = []
    for i0, i1, i2 in _ear_clip(loop):
        faces.append((i2, i1, i0))
        faces.append((n + i0, n + i1, n + i2))
    for i in range(n):
        j = (i + 1) % n
        faces.append((i, j, n + j))
        faces.append((i, n + j, n + i))
    return Solid(TriangleMesh(verts, np.asarray(faces, dtype=np.int64)))


def random_polygon(rng, n_vertices=9, r_min=0.4, r_max=1.0):
    """Star-shaped polygon about the origin; draw order jitter then radii."""
    jitter = rng.uniform(0.15, 0.85, n_vertices)
    theta = (np.arange(n_vertices) + jitter) * (2.0 * np.pi / n_vertices)
    r = rng.uniform(r_min, r_max, n_vertices)
    return Solid(Polygon2([np.column_stack([r * np.cos(theta), r * np.sin(theta)])]))


# ---------------------------------------------------------------------------
# BASELINE.json geometry (new): peg-in-hole, gear pair, bolt and nut


def regular_polygon(n, radius, phase=0.0):
    th = phase + 2.0 * np.pi * np.arange(n) / n
    return np.column_stack([radius * np.cos(th), radius * np.sin(th)])


def cylinder_peg(radius=0.15, length=0.6, segments=64, center=(0.0, 0.0, 0.0)):
    """Cylinder along z: an extruded regular n-gon."""
    s = extrude_polygon([regular_polygon(segments, radius)], length)
    if np.any(np.asarray(center) != 0.0):
        m = s.mesh
        s = Solid(TriangleMesh(m.vertices + np.asarray(center, dtype=np.float64), m.faces))
    return s


def _annulus_prism(outer, inner, z0, z1):
    """Closed genus-1 prism between an outer loop and an inner loop (both CCW,
    equal vertex counts, radially matched), from z0 to z1."""
    n = len(outer)
    assert len(inner) == n
    V = np.vstack([np.column_stack([outer, np.full(n, z0)]), np.column_stack([outer, np.full(n, z1)]),
                   np.column_stack([inner, np.full(n, z0)]), np.column_stack([inner, np.full(n, z1)])])
    ob, ot, ib, it = 0, n, 2 * n, 3 * n
    F = []
    for i in range(n):
        j = (i + 1) % n
        F += [(ob + i, ob + j, ot + j), (ob + i, ot + j, ot + i)]      # outer wall, facing out
        F += [(ib + i, it + j, ib + j), (ib + i, it + i, it + j)]      # bore wall, facing the axis
        F += [(ot + i, ot + j, it + j), (ot + i, it + j, it + i)]      # top annulus (+z)
        F += [(ob + i, ib + j, ob + j), (ob + i, ib + i, ib + j)]      # bottom annulus (-z)
    return V, np.asarray(F, dtype=np.int64)


def bored_block(extents=(0.8, 0.8, 0.5), bore_radius=0.15, segments=64):
    """Box (x, y, z extents) with a cylindrical through-bore along z (genus 1).

    The square outline is sampled at the bore's angles (segments divisible by
    4, starting at 45 degrees, so the corners are vertices)."""
    if segments % 4:
        raise ValueError("segments must be a multiple of 4")
    th = np.pi / 4 + 2.0 * np.pi * np.arange(segments) / segments
    c, s = np.cos(th), np.sin(th)
    ax, ay = 0.5 * extents[0], 0.5 * extents[1]
    r_out = 1.0 / np.maximum(np.abs(c) / ax, np.abs(s) / ay)
    outer = np.column_stack([r_out * c, r_out * s])
    inner = np.column_stack([bore_radius * c, bore_radius * s])
    V, F = _annulus_prism(outer, inner, -0.5 * extents[2], 0.5 * extents[2])
    return Solid(TriangleMesh(V, F))


def gear_profile(teeth=24, r_root=0.42, r_tip=0.5, points_per_tooth=8, phase=0.0):
    """Single-loop gear outline: trapezoidal teeth with smoothed flanks."""
    n = teeth * points_per_tooth
    t = np.arange(n) / points_per_tooth  # tooth coordinate
    frac = t - np.floor(t)
    # radius profile over one tooth period: root, rising flank, tip, falling flank
    rise = np.clip((frac - 0.15) / 0.2, 0.0, 1.0)
    fall = np.clip((0.85 - frac) / 0.2, 0.0, 1.0)
    prof = np.minimum(rise, fall)
    prof = prof * prof * (3.0 - 2.0 * prof)  # smoothstep flanks (involute-like)
    r = r_root + (r_tip - r_root) * prof
    th = phase + 2.0 * np.pi * np.arange(n) / n
    return np.column_stack([r * np.cos(th), r * np.sin(th)])


def gear(teeth=24, r_root=0.42, r_tip=0.5, thickness=0.3, points_per_tooth=8, phase=0.0, center=(0.0, 0.0)):
    loop = gear_profile(teeth, r_root, r_tip, points_per_tooth, phase) + np.asarray(center, dtype=np.float64)
    return extrude_polygon([loop], thickness)


def _thread_radius(theta, z, r_minor, r_major, pitch):
    """Radius of a single-start triangular thread at (theta, z)."""
    u = (z - pitch * theta / (2.0 * np.pi)) / pitch
    frac = u - np.floor(u)
    tri = 1.0 - np.abs(2.0 * frac - 1.0)  # 0 at roots, 1 at crests
    return r_minor + (r_major - r_minor) * tri


def threaded_bolt(r_minor=0.17, r_major=0.2, pitch=0.1, turns=4, n_theta=256, n_z=None, cap_center=True):
    """Threaded rod along z (length turns * pitch), closed by flat end caps."""
    length = turns * pitch
    n_z = n_z or max(8, int(round(turns * 48)))
    th = 2.0 * np.pi * np.arange(n_theta) / n_theta
    zs = np.linspace(-0.5 * length, 0.5 * length, n_z + 1)
    T, Z = np.meshgrid(th, zs, indexing="ij")  # (n_theta, n_z+1)
    Rr = _thread_radius(T, Z, r_minor, r_major, pitch)
    side = np.stack([Rr * np.cos(T), Rr * np.sin(T), Z], axis=-1).reshape(-1, 3)
    idx = lambda i, k: (i % n_theta) * (n_z + 1) + k  # noqa: E731
    F = []
    for i in range(n_theta):
        for k in range(n_z):
            a, b, c, d = idx(i, k), idx(i + 1, k), idx(i + 1, k + 1), idx(i, k + 1)
            F += [(a, b, c), (a, c, d)]
    V = [side]
    nb = len(side)
    bot_c, top_c = nb, nb + 1
    V.append(np.array([[0.0, 0.0, -0.5 * length], [0.0, 0.0, 0.5 * length]]))
    for i in range(n_theta):
        F.append((bot_c, idx(i + 1, 0), idx(i, 0)))          # bottom cap (-z)
        F.append((top_c, idx(i, n_z), idx(i + 1, n_z)))      # top cap (+z)
    return Solid(TriangleMesh(np.vstack(V), np.asarray(F, dtype=np.int64)))


def threaded_nut(r_minor=0.17, r_major=0.2, pitch=0.1, turns=3, outer=0.4, n_theta=256, n_z=None, clearance=0.0):
    """Hexagonal nut (circumradius `outer`) with a matched internal thread
    (the bolt's thread surface offset outward by `clearance`); genus 1."""
    length = turns * pitch
    n_z = n_z or max(8, int(round(turns * 48)))
    if n_theta % 6:
        raise ValueError("n_theta must be a multiple of 6")
    th = 2.0 * np.pi * np.arange(n_theta) / n_theta
    zs = np.linspace(-0.5 * length, 0.5 * length, n_z + 1)
    # hexagon sampled at the thread angles (corners at multiples of 60 degrees)
    sector = np.mod(th, np.pi / 3) - np.pi / 6
    r_hex = outer * np.cos(np.pi / 6) / np.cos(sector)
    hx, hy = r_hex * np.cos(th), r_hex * np.sin(th)
    T, Z = np.meshgrid(th, zs, indexing="ij")
    Rt = _thread_radius(T, Z, r_minor + clearance, r_major + clearance, pitch)
    inner = np.stack([Rt * np.cos(T), Rt * np.sin(T), Z], axis=-1).reshape(-1, 3)
    outer_b = np.column_stack([hx, hy, np.full(n_theta, zs[0])])
    outer_t = np.column_stack([hx, hy, np.full(n_theta, zs[-1])])
    V = np.vstack([inner, outer_b, outer_t])
    ii = lambda i, k: (i % n_theta) * (n_z + 1) + k  # noqa: E731
    ob = lambda i: len(inner) + (i % n_theta)  # noqa: E731
    ot = lambda i: len(inner) + n_theta + (i % n_theta)  # noqa: E731
    F = []
    for i in range(n_theta):
        for k in range(n_z):  # thread wall, facing the axis
            a, b, c, d = ii(i, k), ii(i + 1, k), ii(i + 1, k + 1), ii(i, k + 1)
            F += [(a, c, b), (a, d, c)]
        F += [(ob(i), ob(i + 1), ot(i + 1)), (ob(i), ot(i + 1), ot(i))]                  # hex wall
        F += [(ot(i), ot(i + 1), ii(i + 1, n_z)), (ot(i), ii(i + 1, n_z), ii(i, n_z))]   # top annulus
        F += [(ob(i), ii(i + 1, 0), ob(i + 1)), (ob(i), ii(i, 0), ii(i + 1, 0))]         # bottom annulus
    return Solid(TriangleMesh(V, np.asarray(F, dtype=np.int64)))


# ---------------------------------------------------------------------------
# pair grids and assets (scenes.py:185-221)


def grid_for_pair(fixed, moving, n, domain=None, center="cell"):
    """Shared grid sized for clean translations at any rotation."""
    d = fixed.dimension
    if moving.dimension != d:
        raise ValueError("mixed dimensions")
    if domain is None:
        lo1, hi1 = fixed.bbox
        lo2, hi2 = moving.bbox
        rho1 = float(np.max(np.abs(np.stack([lo1, hi1]))))
        rho2 = float(np.linalg.norm(np.maximum(np.abs(lo2), np.abs(hi2))))
        r1 = 0.5 * float(np.linalg.norm(hi1 - lo1))
        domain = 2.0 * 1.25 * (max(rho1, rho2) + rho2 + r1)
    h = float(domain) / n
    if center not in ("cell", "node"):
        raise ValueError("center must be 'cell' or 'node'")
    shift = 0.5 * h if center == "cell" else 0.0
    return SampleGrid(dimension=d, dims=(n,) * d, origin=(-0.5 * float(domain) + shift,) * d, spacing=h)


def build_pair_assets(fixed, moving, grid, kernel=KernelSpec(), policy=IntegrationPolicy(), m_prime=None,
                      threads=None):
    f1 = affinity_field(fixed, grid, kernel, policy, threads=threads)
    f2 = affinity_field(moving, grid, kernel, policy, threads=threads)
    a1 = PartAsset.from_field("fixed", f1, movable=False, m_prime=m_prime, solid_box=fixed.bbox)
    a2 = PartAsset.from_field("moving", f2, movable=True, m_prime=m_prime, solid_box=moving.bbox)
    return a1, a2


# ---------------------------------------------------------------------------
# scenes (scenes.py:227-302) plus the BASELINE.json pairs

_SOCKET_LOOP = [(-0.55, -0.35), (0.55, -0.35), (0.55, 0.25), (0.15, 0.25),
                (0.15, -0.15), (-0.15, -0.15), (-0.15, 0.25), (-0.55, 0.25)]
_PEG_LOOP = [(-0.15, -0.15), (0.15, -0.15), (0.15, 0.25), (0.3, 0.25),
             (0.3, 0.35), (-0.3, 0.35), (-0.3, 0.25), (-0.15, 0.25)]


@dataclass
class Scene:
    name: str
    fixed: Solid
    moving: Solid
    kernel: KernelSpec
    domain: float
    default_n: int
    snap_translation: np.ndarray
    grid_center: str = "cell"

    @property
    def dimension(self):
        return self.fixed.dimension

    def grid(self, n=None):
        return grid_for_pair(self.fixed, self.moving, n or self.default_n, domain=self.domain,
                             center=self.grid_center)

    def build_assets(self, n=None, m_prime=None, threads=None, policy=IntegrationPolicy()):
        return build_pair_assets(self.fixed, self.moving, self.grid(n), self.kernel, policy, m_prime, threads)


def _peg2d():
    return Scene("peg2d", Solid(Polygon2([np.asarray(_SOCKET_LOOP, dtype=np.float64)])),
                 Solid(Polygon2([np.asarray(_PEG_LOOP, dtype=np.float64)])),
                 KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0), 6.0, 256, np.array([0.0, 0.0]), "node")


def _peg3d():
    return Scene("peg3d", extrude_polygon([np.asarray(_SOCKET_LOOP, dtype=np.float64)], 0.5),
                 extrude_polygon([np.asarray(_PEG_LOOP, dtype=np.float64)], 0.5),
                 KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0), 6.0, 32, np.array([0.0, 0.0, 0.0]), "node")


def _peg_in_hole(clearance=0.0, default_n=64):
    """C1/C2: 64-gon cylinder peg (r 0.15, length 0.6) in a bored block
    (0.8 x 0.8 x 0.5, bore r 0.15 (+ clearance)); seated at t = 0."""
    bore = 0.15
    fixed = bored_block((0.8, 0.8, 0.5), bore + clearance, 64)
    moving = cylinder_peg(bore, 0.6, 64)
    return Scene("peg_in_hole" if clearance == 0 else "peg_in_hole_lowclear", fixed, moving,
                 KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0), 3.46, default_n,
                 np.array([0.0, 0.0, 0.0]), "node")


def _gear_pair():
    """C3: 24-tooth gear and a meshing 24-tooth partner (half-tooth phase)."""
    fixed = gear(24, 0.42, 0.5, 0.3, 8, 0.0)
    moving = gear(24, 0.42, 0.5, 0.3, 8, np.pi / 24)
    return Scene("gear_pair", fixed, moving, KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0), 5.42, 256,
                 np.array([0.92, 0.0, 0.0]), "node")


def _bolt_nut():
    """C5: threaded bolt (pitch 0.1, 4 turns) and matched nut."""
    fixed = threaded_nut(0.17, 0.2, 0.1, 3, 0.4, 258 - 258 % 6)
    moving = threaded_bolt(0.17, 0.2, 0.1, 4, 256)
    return Scene("bolt_nut", fixed, moving, KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0), 4.37, 256,
                 np.array([0.0, 0.0, 0.0]), "node")


SCENES = {
    "peg2d": _peg2d,
    "peg3d": _peg3d,
    "peg_in_hole": _peg_in_hole,
    "peg_in_hole_lowclear": lambda: _peg_in_hole(clearance=0.01 * 0.15, default_n=128),
    "gear_pair": _gear_pair,
    "bolt_nut": _bolt_nut,
}


def get_scene(name):
    try:
        return SCENES[name]()
    except KeyError:
        raise ValueError(f"unknown scene {name!r}; have {sorted(SCENES)}") from None
