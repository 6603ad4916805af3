"""Seeded synthetic scene generators.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2407_00046_b200/``).  It holds none of the method's
arithmetic: it only lays out tetrahedral meshes, fixed-node flags, materials,
initial positions/velocities and scene parameters, drawing every random number
from ``numpy.random.default_rng(seed)`` in a fixed order.  Surface extraction,
masses, Lamé parameters, energies etc. are computed independently by each side.

Scene defaults follow Table 1 of the paper: nu = 0.4,
rho = 1e3 kg/m^3, dhat = eps_v = 1e-3, h = 1/30 s; gravity (0, -9.81, 0)
(SURVEY Q4 reading).
"""
from __future__ import annotations

import numpy as np

DEFAULT_PARAMS = dict(
    h=1.0 / 30.0,
    gravity=(0.0, -9.81, 0.0),
    dhat=1e-3,
    eps_v=1e-3,
    chi=0.0,
    newton_rel_tol=1e-4,   # Alg. 1 line 9
    pcg_rel_tol=1e-4,      # App. B
    pcg_stall_window=100,  # App. B
    pcg_resume_iters=100,  # App. B
    alpha_min=1e-9,        # App. B
    ws_rel_tol=1e-2,
    ws_max_iters=100,
    max_newton=1000,
    max_pcg=20000,
    max_constraints=1 << 26,
)


# --------------------------------------------------------------------------
# primitive builders
# --------------------------------------------------------------------------
def _kuhn_tets(v):
    """6-tet Kuhn split of a hex whose 8 corner ids are v[(i,j,k)] (bits x,y,z)."""
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    out = []
    for a, b, _c in perms:
        p0 = (0, 0, 0)
        p1 = [0, 0, 0]
        p1[a] = 1
        p2 = list(p1)
        p2[b] = 1
        out.append([v[p0], v[tuple(p1)], v[tuple(p2)], v[(1, 1, 1)]])
    return out


def _orient(x, tets):
    """Swap two vertices of every tet with negative signed volume."""
    a, b, c, d = (x[tets[:, i]] for i in range(4))
    vol = np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a)
    neg = vol < 0
    t = tets.copy()
    t[neg, 2], t[neg, 3] = tets[neg, 3], tets[neg, 2]
    return t


def hex_block(nx, ny, nz, size):
    """Structured hex grid of nx*ny*nz cells over [0,size]^3 (anisotropic if size is a 3-tuple),
    each cell split into 6 Kuhn tets.  Returns (x (N,3), tets (T,4))."""
    size = np.broadcast_to(np.asarray(size, dtype=np.float64), (3,))
    gx = np.linspace(0.0, size[0], nx + 1)
    gy = np.linspace(0.0, size[1], ny + 1)
    gz = np.linspace(0.0, size[2], nz + 1)
    X, Y, Z = np.meshgrid(gx, gy, gz, indexing="ij")
    x = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)

    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    tets = []
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                v = {}
                for di in (0, 1):
                    for dj in (0, 1):
                        for dk in (0, 1):
                            v[(di, dj, dk)] = nid(i + di, j + dj, k + dk)
                tets.extend(_kuhn_tets(v))
    tets = np.asarray(tets, dtype=np.int64)
    return x, _orient(x, tets)


def voxel_mesh(occ, voxel):
    """Tet mesh of the occupied voxels of a boolean grid occ[nx,ny,nz] (6 Kuhn tets per voxel),
    with shared corner nodes deduplicated.  Returns (x (N,3), tets (T,4))."""
    occ = np.asarray(occ, dtype=bool)
    nx, ny, nz = occ.shape
    idx = np.argwhere(occ)
    if len(idx) == 0:
        return np.zeros((0, 3)), np.zeros((0, 4), dtype=np.int64)
    corner_offsets = np.array([(di, dj, dk) for di in (0, 1) for dj in (0, 1) for dk in (0, 1)])
    corners = (idx[:, None, :] + corner_offsets[None, :, :]).reshape(-1, 3)
    lin = (corners[:, 0] * (ny + 1) + corners[:, 1]) * (nz + 1) + corners[:, 2]
    uniq, inv = np.unique(lin, return_inverse=True)
    inv = inv.reshape(-1, 8)
    ci = uniq // ((ny + 1) * (nz + 1))
    cj = (uniq // (nz + 1)) % (ny + 1)
    ck = uniq % (nz + 1)
    x = np.stack([ci, cj, ck], axis=1).astype(np.float64) * voxel
    # Kuhn split with vectorised corner lookup
    code = {tuple(o): n for n, o in enumerate(corner_offsets)}
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    tl = []
    for a, b, _c in perms:
        p1 = [0, 0, 0]
        p1[a] = 1
        p2 = list(p1)
        p2[b] = 1
        tl.append(np.stack([inv[:, code[(0, 0, 0)]], inv[:, code[tuple(p1)]],
                            inv[:, code[tuple(p2)]], inv[:, code[(1, 1, 1)]]], axis=1))
    tets = np.stack(tl, axis=1).reshape(-1, 4).astype(np.int64)
    return x, _orient(x, tets)


def rot_y(theta):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def rot_axis(axis, theta):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(theta) * K + (1 - np.cos(theta)) * (K @ K)


def random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


class SceneBuilder:
    """Accumulates bodies (tet meshes), fixed obstacle triangles and per-node velocities."""

    def __init__(self):
        self.x = []
        self.tets = []
        self.mat = []
        self.fixed = []
        self.v = []
        self.obst_tris = []
        self.n = 0

    def add_body(self, x, tets, material, v0=(0.0, 0.0, 0.0), fixed=None):
        x = np.asarray(x, dtype=np.float64)
        self.x.append(x)
        self.tets.append(np.asarray(tets, dtype=np.int64) + self.n)
        self.mat.append(np.full(len(tets), material, dtype=np.int32))
        f = np.zeros(len(x), dtype=np.uint8) if fixed is None else np.asarray(fixed, dtype=np.uint8)
        self.fixed.append(f)
        self.v.append(np.broadcast_to(np.asarray(v0, dtype=np.float64), x.shape).copy())
        self.n += len(x)

    def add_obstacle(self, x, tris):
        """Surface-only static obstacle: nodes are fixed, triangles are listed explicitly."""
        x = np.asarray(x, dtype=np.float64)
        self.x.append(x)
        self.fixed.append(np.ones(len(x), dtype=np.uint8))
        self.v.append(np.zeros_like(x))
        self.obst_tris.append(np.asarray(tris, dtype=np.int64) + self.n)
        self.n += len(x)

    def build(self, materials, name, **params):
        p = dict(DEFAULT_PARAMS)
        p.update(params)
        x = np.concatenate(self.x, axis=0)
        tets = np.concatenate(self.tets, axis=0) if self.tets else np.zeros((0, 4), np.int64)
        return dict(
            name=name,
            rest_x=x.copy(),
            x0=x.copy(),
            v0=np.concatenate(self.v, axis=0),
            tets=tets.astype(np.int32),
            tet_material=(np.concatenate(self.mat) if self.mat else np.zeros(0, np.int32)).astype(np.int32),
            node_fixed=np.concatenate(self.fixed).astype(np.uint8),
            obstacle_tris=(np.concatenate(self.obst_tris, axis=0) if self.obst_tris
                           else np.zeros((0, 3), np.int64)).astype(np.int32),
            materials=np.asarray(materials, dtype=np.float64).reshape(-1, 3),  # (E, nu, rho)
            params=p,
        )


def _plane(half, y=0.0, cx=0.0, cz=0.0):
    """Two triangles at height y, normal +y (counter-clockwise seen from above)."""
    x = np.array([[cx - half, y, cz - half], [cx + half, y, cz - half],
                  [cx + half, y, cz + half], [cx - half, y, cz + half]])
    tris = np.array([[0, 2, 1], [0, 3, 2]])
    return x, tris


# --------------------------------------------------------------------------
# C1: two stacked soft cubes dropped on a plane (BASELINE.json configs[0])
# --------------------------------------------------------------------------
def make_cubes(seed=1, cells=5, edge=1.0, E=1e5, nu=0.4, rho=1e3, gap=0.01, speed=1.0):
    """C1 recipe: 2 cubes of 5x5x5 hex cells (Kuhn split, T=1500),
    yaws ~U(10,35) deg, top tilt ~U(0.5,2) deg about a random horizontal axis; bottom base at
    y = gap, top cube `gap` above; v0 = (0,-speed,0); static 10x10 m plane (2 tris) at y = 0."""
    rng = np.random.default_rng(seed)
    yaw0 = np.deg2rad(rng.uniform(10.0, 35.0))
    yaw1 = np.deg2rad(rng.uniform(10.0, 35.0))
    tilt = np.deg2rad(rng.uniform(0.5, 2.0))
    phi = rng.uniform(0.0, 2 * np.pi)
    axis = np.array([np.cos(phi), 0.0, np.sin(phi)])

    xb, tb = hex_block(cells, cells, cells, edge)
    c = np.array([edge / 2, edge / 2, edge / 2])
    sb = SceneBuilder()
    # bottom cube
    x0 = (xb - c) @ rot_y(yaw0).T
    x0[:, 1] += -x0[:, 1].min() + gap
    # top cube
    R1 = rot_axis(axis, tilt) @ rot_y(yaw1)
    x1 = (xb - c) @ R1.T
    x1[:, 1] += -x1[:, 1].min() + x0[:, 1].max() + gap
    sb.add_body(x0, tb, 0, v0=(0.0, -speed, 0.0))
    sb.add_body(x1, tb, 0, v0=(0.0, -speed, 0.0))
    px, pt = _plane(5.0)
    sb.add_obstacle(px, pt)
    return sb.build([(E, nu, rho)], "C1-cubes", chi=0.0)


def make_single_tet(seed=0, height=0.05, E=1e5, nu=0.4, rho=1e3, speed=0.0, vt=0.0, chi=0.0):
    """Tiny fixture: one generically rotated tet above a plane.  The gap is made generic
    (height * (1 + U(0.05, 0.15))): with an exact decimal gap and a vertical approach the CCD
    backtracking (x0.9 of the time of coplanarity, i.e. x0.1 of the gap) produces distances of
    exactly 1e-3, 1e-4, 1e-5 = 1e-2 dhat, a tie on Alg. 1's strict 'min d < 1e-2 dhat' test."""
    rng = np.random.default_rng(seed)
    x = np.array([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0], [0, 0, 0.1]], dtype=np.float64)
    x = (x - x.mean(0)) @ random_rotation(rng).T
    x[:, 1] += -x[:, 1].min() + height * (1.0 + rng.uniform(0.05, 0.15))
    tets = _orient(x, np.array([[0, 1, 2, 3]]))
    sb = SceneBuilder()
    sb.add_body(x, tets, 0, v0=(vt, -speed, 0.0))
    px, pt = _plane(1.0)
    sb.add_obstacle(px, pt)
    return sb.build([(E, nu, rho)], "tet", chi=chi)


def make_incline(seed=0, ratio=0.8, chi=0.3, E=1e5, nu=0.4, rho=1e3, gap=5e-4, size=0.1):
    """Friction fixture (acceptance 9): one tet resting on a fixed plane inclined at
    tan(theta) = ratio * chi about the z axis.  The tet's base face is parallel to the incline, `gap`
    above it, at rest; a small generic yaw about the incline normal and an offset from the plane's
    diagonal keep the base vertices inside the plane triangles (no type-resolution ties, Q27).
    Returns the scene; scene["incline_normal"] / ["incline_down"] are the unit normal and the unit
    downhill direction (geometry only, no method arithmetic)."""
    rng = np.random.default_rng(seed)
    theta = np.arctan(ratio * chi)
    c, s = np.cos(theta), np.sin(theta)
    down = np.array([c, -s, 0.0])     # downhill along the slope (x decreasing height)
    nrm = np.array([s, c, 0.0])       # upward unit normal of the incline
    side = np.array([0.0, 0.0, 1.0])
    yaw = rng.uniform(0.2, 0.6)
    cy, sy = np.cos(yaw), np.sin(yaw)
    base = size * np.array([[-0.5, -0.4], [0.5, -0.3], [0.05, 0.6]])  # (downhill, side) coordinates
    base = base @ np.array([[cy, sy], [-sy, cy]]).T + np.array([0.31, 0.13])
    pts = [gap * nrm + b[0] * down + b[1] * side for b in base]
    apex = gap * nrm + 0.8 * size * nrm + (base.mean(0)[0] * down + base.mean(0)[1] * side)
    x = np.array(pts + [apex])
    tets = _orient(x, np.array([[0, 1, 2, 3]]))
    sb = SceneBuilder()
    sb.add_body(x, tets, 0)
    half = 2.0
    px = np.array([-half * down - half * side, half * down - half * side, half * down + half * side,
                   -half * down + half * side])
    sb.add_obstacle(px, np.array([[0, 2, 1], [0, 3, 2]]) if np.dot(np.cross(px[2] - px[0], px[1] - px[0]), nrm) > 0
                    else np.array([[0, 1, 2], [0, 2, 3]]))
    sc = sb.build([(E, nu, rho)], f"incline-{ratio:g}chi", chi=chi)
    sc["incline_normal"] = nrm
    sc["incline_down"] = down
    return sc


def perturbed(scene, seed, scale):
    """Copy of `scene` with x0 randomly perturbed (free nodes only) by N(0, scale^2)."""
    rng = np.random.default_rng(seed)
    s = dict(scene)
    x = scene["x0"].copy()
    free = scene["node_fixed"] == 0
    x[free] += rng.normal(scale=scale, size=(free.sum(), 3))
    s["x0"] = x
    return s


def make_two_tets(seed=0, gap=0.004, speed=0.3, E=1e5, nu=0.4, rho=1e3):
    """Gravity-free, frictionless, obstacle-free two-tet collision (momentum test, SURVEY c.3)."""
    rng = np.random.default_rng(seed)
    base = np.array([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0], [0, 0, 0.1]], dtype=np.float64)
    xa = (base - base.mean(0)) @ random_rotation(rng).T
    xb = (base - base.mean(0)) @ random_rotation(rng).T
    xb[:, 0] += xa[:, 0].max() - xb[:, 0].min() + gap
    sb = SceneBuilder()
    sb.add_body(xa, _orient(xa, np.array([[0, 1, 2, 3]])), 0, v0=(speed, 0.0, 0.0))
    sb.add_body(xb, _orient(xb, np.array([[0, 1, 2, 3]])), 0, v0=(-speed, 0.0, 0.0))
    return sb.build([(E, nu, rho)], "two-tets", gravity=(0.0, 0.0, 0.0))


def make_free_cube(seed=0, cells=3, E=1e5, nu=0.4, rho=1e3):
    """One rest-shape cube in free fall, no obstacles (free-fall test, SURVEY c.3)."""
    rng = np.random.default_rng(seed)
    xb, tb = hex_block(cells, cells, cells, 0.5)
    xb = (xb - 0.25) @ random_rotation(rng).T
    sb = SceneBuilder()
    sb.add_body(xb, tb, 0, v0=tuple(rng.normal(size=3)))
    return sb.build([(E, nu, rho)], "free-cube")


# --------------------------------------------------------------------------
# C4: puffer balls on a chain-net (BASELINE.json configs[3])
# --------------------------------------------------------------------------
def _ring_xz(L):
    """1-voxel-thick square ring of outer size L in the xz plane (height 1 voxel)."""
    occ = np.zeros((L, 1, L), bool)
    occ[:, 0, :] = True
    occ[1:L - 1, 0, 1:L - 1] = False
    return occ


def _ring_xy(Lx, Ly):
    occ = np.zeros((Lx, Ly, 1), bool)
    occ[:, :, 0] = True
    occ[1:Lx - 1, 1:Ly - 1, 0] = False
    return occ


def _ring_zy(Lz, Ly):
    occ = np.zeros((1, Ly, Lz), bool)
    occ[0, :, :] = True
    occ[0, 1:Ly - 1, 1:Lz - 1] = False
    return occ


def _fib_dirs(n):
    k = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * k / n)
    th = np.pi * (1 + 5 ** 0.5) * k
    return np.stack([np.cos(th) * np.sin(phi), np.cos(phi), np.sin(th) * np.sin(phi)], axis=1)


def spiky_ball_occ(R, n_spikes, spike_len, spike_r=0.75):
    """Voxel occupancy of a solid sphere of radius R (voxels) with radial cylindrical spikes."""
    ext = int(np.ceil(R + spike_len + 2))
    g = np.arange(-ext, ext) + 0.5
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    r2 = X * X + Y * Y + Z * Z
    occ = r2 <= R * R
    P = np.stack([X, Y, Z], axis=-1)
    for d in _fib_dirs(n_spikes):
        t = P @ d
        perp2 = r2 - t * t
        occ |= (t >= R - 1) & (t <= R + spike_len) & (perp2 <= spike_r * spike_r)
    return occ, ext


def make_puffer_net(seed=4, nx=40, nz=40, L=8, spacing=10, voxel=0.01, ball_R=20.4, n_spikes=110,
                    spike_len=15.0, n_balls=4, E_ball=5e5, E_net=1e9, nu=0.4, rho=1e3, chi=0.3, drop_gap=0.002,
                    jitter_deg=(0.2, 0.8), settled=False, rest_gap=(0.4e-3, 0.7e-3)):
    """C4 recipe (Table 1 row 1 P:664 for the statistics): a chain-net of
    interlocked 1-voxel-thick square rings (horizontal rings on an nx x nz lattice plus vertical
    connector rings threading neighbours through their holes; outermost horizontal rings fixed)
    and n_balls spiky balls (voxel core + radial spikes on a Fibonacci direction set) dropped onto
    it.  Every ring gets a small generic rotation so no cross-body edges are exactly parallel.
    Defaults target T ~ 1.76M tets, N ~ 0.8M nodes.
    settled=True: the contact-rich start the paper's statistics describe (228K avg constraints,
    P:664): every connector ring hangs on the two rings it threads (its top beam rests on their
    beams with a clearance drawn from rest_gap, below d_hat) and the balls start rest_gap above the
    net; rotations are reduced to 0.05-0.1 deg so the clearances stay positive."""
    rng = np.random.default_rng(seed)
    sb = SceneBuilder()
    assert L == 8 and spacing == 10, "connector layout below is laid out for L=8, spacing=10"
    xr, tr = voxel_mesh(_ring_xz(L), voxel)
    # Hole of every horizontal ring: [1,7)^2 (voxels, ring-local).  Vertical beams threading it:
    #   x-connector (xy plane, z in [4.5,5.5)): own near beam x in [4.5,5.5), incoming far beam [1.5,2.5)
    #   z-connector (zy plane, x in [3,4)):     own near beam z in [4.5,5.5), incoming far beam [1.5,2.5)
    # -> every pair of distinct rings is >= 0.5 voxel apart before the jitter rotations.
    conn_len = 8
    xcx, tcx = voxel_mesh(_ring_xy(conn_len, 9), voxel)
    xcz, tcz = voxel_mesh(_ring_zy(conn_len, 9), voxel)

    if settled:
        jitter_deg = (0.05, 0.1)

    def jitter(x):
        c = x.mean(0)
        ax = rng.normal(size=3)
        R = rot_axis(ax, np.deg2rad(rng.uniform(*jitter_deg)))
        return (x - c) @ R.T + c

    def hang(xc, host_top):
        """settled: lower a connector so its top beam rests rest_gap above the host beams' top."""
        if not settled:
            return xc
        top_beam = xc[:, 1] > xc[:, 1].max() - 1.5 * voxel
        return xc - np.array([0.0, xc[top_beam, 1].min() - host_top - rng.uniform(*rest_gap), 0.0])

    # bodies in the original interleaved order (ring, x-connector, z-connector per lattice site; the
    # node numbering and the rotation draws of the default scene are unchanged by `settled`)
    bodies, tops = [], {}
    for i in range(nx):
        for k in range(nz):
            o = np.array([i * spacing, 0.0, k * spacing]) * voxel
            border = i == 0 or k == 0 or i == nx - 1 or k == nz - 1
            x = xr + o
            if not border:
                x = jitter(x)
            tops[i, k] = float(x[:, 1].max())
            bodies.append(("ring", x, tr, np.full(len(xr), 1 if border else 0, np.uint8), None))
            if i + 1 < nx:
                # vertical ring in the xy plane through the holes of rings (i,k) and (i+1,k)
                oc = o + np.array([4.5, -4.0, 4.5]) * voxel
                bodies.append(("conn", jitter(xcx + oc), tcx, None, ((i, k), (i + 1, k))))
            if k + 1 < nz:
                oc = o + np.array([3.0, -4.0, 4.5]) * voxel
                bodies.append(("conn", jitter(xcz + oc), tcz, None, ((i, k), (i, k + 1))))
    for kind, x, t, fx, hosts in bodies:
        if kind == "conn":
            x = hang(x, max(tops[hosts[0]], tops[hosts[1]]))
        sb.add_body(x, t, 1, fixed=fx)
    occ, ext = spiky_ball_occ(ball_R, n_spikes, spike_len)
    xb, tb = voxel_mesh(occ, voxel)
    xb = xb - ext * voxel
    span = np.array([(nx - 1) * spacing + L, (nz - 1) * spacing + L]) * voxel
    top = 6 * voxel  # above the connector rings
    if settled:  # balls rest_gap above the highest point of the net (the hanging connectors' tops)
        top = max(float(b_x[:, 1].max()) for b_x in sb.x)
        drop_gap = rest_gap[0]
    for b in range(n_balls):
        fx = (0.3 + 0.4 * (b % 2)) * span[0]
        fz = (0.3 + 0.4 * (b // 2 % 2)) * span[1]
        xbb = xb @ random_rotation(rng).T
        xbb = xbb + np.array([fx, top - xbb[:, 1].min() + drop_gap, fz])
        sb.add_body(xbb, tb, 0, v0=(0.0, -1.0, 0.0))
    return sb.build([(E_ball, nu, rho), (E_net, nu, rho)], "C4-puffer-net", chi=chi)


# --------------------------------------------------------------------------
# C2 / C3
# --------------------------------------------------------------------------
def _ellipsoid_occ(shape, voxel, shapes):
    """Union of ellipsoids / capsules on a voxel grid: each entry (kind, a, b, r) with centres in
    metres; kind 'e' = ellipsoid centre a, semi-axes b; kind 'c' = capsule a->b radius r."""
    nx, ny, nz = shape
    g = (np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1) + 0.5) * voxel
    occ = np.zeros(shape, bool)
    for kind, a, b, r in shapes:
        a = np.asarray(a, float)
        b = np.asarray(b, float)
        if kind == "e":
            occ |= (((g - a) / b) ** 2).sum(-1) <= 1.0
        else:
            ab = b - a
            t = np.clip(((g - a) @ ab) / (ab @ ab), 0.0, 1.0)
            occ |= np.linalg.norm(g - (a + t[..., None] * ab), axis=-1) <= r
    return occ


def make_armadillo_like(seed=2, voxel=0.0095, E=1e6, nu=0.4, rho=1e3, chi=0.9, gap=0.01):
    """C2 recipe: an 'armadillo-like' creature (no paper mesh available: P:672 roller row, 100K tets)
    = union of 9 ellipsoids / capsules (torso, head, 2 ears, 4 limbs, tail) voxelised, 6 Kuhn tets
    per voxel, generically rotated, `gap` above a static plane, v0 = (0.5, -1, 0), chi = 0.9."""
    rng = np.random.default_rng(seed)
    shapes = [("e", (0.30, 0.28, 0.20), (0.17, 0.11, 0.10), 0),      # torso
              ("e", (0.50, 0.36, 0.20), (0.07, 0.07, 0.065), 0),     # head
              ("c", (0.50, 0.41, 0.16), (0.53, 0.50, 0.13), 0.022),  # ears
              ("c", (0.50, 0.41, 0.24), (0.53, 0.50, 0.27), 0.022),
              ("c", (0.20, 0.22, 0.12), (0.17, 0.03, 0.09), 0.035),  # legs
              ("c", (0.20, 0.22, 0.28), (0.17, 0.03, 0.31), 0.035),
              ("c", (0.40, 0.22, 0.12), (0.44, 0.03, 0.09), 0.035),
              ("c", (0.40, 0.22, 0.28), (0.44, 0.03, 0.31), 0.035),
              ("c", (0.14, 0.28, 0.20), (0.02, 0.20, 0.20), 0.03)]   # tail
    n = (int(0.62 / voxel), int(0.56 / voxel), int(0.42 / voxel))
    occ = _ellipsoid_occ(n, voxel, shapes)
    x, t = voxel_mesh(occ, voxel)
    x = (x - x.mean(0)) @ rot_axis(rng.normal(size=3), np.deg2rad(rng.uniform(2, 5))).T
    x[:, 1] += -x[:, 1].min() + gap * (1.0 + rng.uniform(0.05, 0.15))
    sb = SceneBuilder()
    sb.add_body(x, _orient(x, t), 0, v0=(0.5, -1.0, 0.0))
    px, pt = _plane(2.0)
    sb.add_obstacle(px, pt)
    return sb.build([(E, nu, rho)], "C2-armadillo-like", chi=chi)


def make_impact(seed=3, nx=78, ny=8, nz=78, slab_voxel=0.02, R=0.1, sphere_voxel=0.01, E_slab=1e9, E_sphere=1e7,
                nu=0.4, rho=1e3, gap=0.05, speed=10.0):
    """C3 recipe: stiff slab nx x ny x nz voxels of slab_voxel (side faces fixed, E = 1 GPa) and a
    voxelised sphere of radius R (sphere_voxel, E = 1e7) `gap` above it moving at v0 = (0, -speed, 0)
    (0.33 m/step, so CCD bounds the first steps); both generically rotated by a small angle."""
    rng = np.random.default_rng(seed)
    xs, ts = voxel_mesh(np.ones((nx, ny, nz), bool), slab_voxel)
    c = xs.mean(0)
    ext = xs.max(0) - xs.min(0)
    side = (np.abs(xs[:, 0] - c[0]) > 0.5 * ext[0] - 1e-9) | (np.abs(xs[:, 2] - c[2]) > 0.5 * ext[2] - 1e-9)
    xs = (xs - c) @ rot_axis(rng.normal(size=3), np.deg2rad(rng.uniform(0.2, 0.6))).T
    m = int(np.ceil(2 * R / sphere_voxel))
    g = (np.stack(np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij"), -1) + 0.5) * sphere_voxel
    occ = np.linalg.norm(g - R, axis=-1) <= R
    xb, tb = voxel_mesh(occ, sphere_voxel)
    xb = (xb - xb.mean(0)) @ random_rotation(rng).T
    xb[:, 1] += xs[:, 1].max() - xb[:, 1].min() + gap * (1.0 + rng.uniform(0.05, 0.15))
    xb[:, [0, 2]] += rng.uniform(-0.05, 0.05, 2)
    sb = SceneBuilder()
    sb.add_body(xs, _orient(xs, ts), 1, fixed=side.astype(np.uint8))
    sb.add_body(xb, _orient(xb, tb), 0, v0=(0.0, -speed, 0.0))
    return sb.build([(E_sphere, nu, rho), (E_slab, nu, rho)], "C3-impact", chi=0.0)


def make_puffer_tiles(seed=5, tiles=(3, 2), gap=0.1, **kw):
    """C5 recipe (configs[4]): the C4 tile replicated tiles[0] x tiles[1] in the x-z plane with `gap`
    metres between tiles, tile i generated with seed 500 + i (its own fixed border frame, balls,
    jitter); ~10.5M tets for 3 x 2."""
    del seed  # the per-tile seeds are 500 + i (SURVEY d.2)
    parts = []
    off = np.zeros(3)
    k = 0
    for i in range(tiles[0]):
        for j in range(tiles[1]):
            sc = make_puffer_net(seed=500 + k, **kw)
            parts.append((sc, np.array([i, 0.0, j])))
            k += 1
    span = parts[0][0]["rest_x"].max(0) - parts[0][0]["rest_x"].min(0) + gap
    sb = SceneBuilder()
    for sc, ij in parts:
        off = ij * span
        x = sc["rest_x"] + off
        sb.x.append(x)
        sb.tets.append(sc["tets"].astype(np.int64) + sb.n)
        sb.mat.append(sc["tet_material"])
        sb.fixed.append(sc["node_fixed"])
        sb.v.append(sc["v0"])
        sb.n += len(x)
    first = parts[0][0]
    return sb.build(first["materials"], "C5-puffer-tiles", chi=first["params"]["chi"])


# --------------------------------------------------------------------------
# NEXT-2: twisting rods (PAPER.md:299-304 fig:rods, Table 1 row P:679)
# --------------------------------------------------------------------------
TWIST_OMEGA = 2.0 * np.pi * 5.0 / 12.0  # 5/12 revolutions per second


def make_twisting_rods(seed=6, n=12, length=103, voxel=0.0025, gap=0.01, E=1e7, nu=0.4, rho=1e3,
                       omega=TWIST_OMEGA):
    """NEXT-2 recipe: four stiff rods (E = 10 MPa; Table 1: 355K tets / 70.4K nodes)
    along z in a 2 x 2 bundle, each n x n x length voxels of `voxel` (6 Kuhn tets per voxel: 12 x 12 x
    103 gives T = 355,968, N = 70,304), `gap` between neighbouring rods, a generic 0.05-0.15 degree
    rotation per rod.  The first and last node layers of every rod are Dirichlet nodes (node_fixed)
    scripted by twist_targets(): the z = 0 ends rotate about the bundle axis at +omega, the far ends
    at -omega (torsion from both ends).  chi = 0 (Table 1)."""
    rng = np.random.default_rng(seed)
    x0, t0 = voxel_mesh(np.ones((n, n, length), bool), voxel)
    zl = x0[:, 2]
    ends = np.where(np.abs(zl - zl.min()) < 1e-12, 1, np.where(np.abs(zl - zl.max()) < 1e-12, 2, 0))
    half = 0.5 * n * voxel
    sb = SceneBuilder()
    end_side = []
    for cx, cy in ((-1, -1), (1, -1), (-1, 1), (1, 1)):
        x = x0 - np.array([half, half, 0.5 * length * voxel])
        x = x @ rot_axis(rng.normal(size=3), np.deg2rad(rng.uniform(0.05, 0.15))).T
        x[:, 0] += cx * (half + 0.5 * gap)
        x[:, 1] += cy * (half + 0.5 * gap)
        sb.add_body(x, _orient(x, t0), 0, fixed=(ends > 0).astype(np.uint8))
        end_side.append(ends)
    sc = sb.build([(E, nu, rho)], "twisting-rods", chi=0.0)
    sc["twist_end"] = np.concatenate(end_side).astype(np.int8)  # 1 = near end (+omega), 2 = far end (-omega)
    sc["twist_omega"] = float(omega)
    return sc


def twist_targets(scene, t):
    """Scripted Dirichlet positions of the rod ends at time t (scene boundary condition, no method
    arithmetic): rest positions rotated about the z axis by +omega t (near ends) / -omega t (far ends).
    Returns the (N, 3) array of target positions of all nodes (non-end rows = rest positions)."""
    x = scene["rest_x"].copy()
    for side, sign in ((1, 1.0), (2, -1.0)):
        m = scene["twist_end"] == side
        x[m] = x[m] @ rot_axis((0.0, 0.0, 1.0), sign * scene["twist_omega"] * t).T
    return x


# --------------------------------------------------------------------------
# NEXT-4: Neo-Hookean / ARAP coupling (fig:bunny-balls)
# --------------------------------------------------------------------------
def make_nh_arap_cubes(seed=1, E_arap=1e6, E_nh=1e4, **kw):
    """The C1 layout with the bottom cube ARAP (stiff, E = 1 MPa) and the top cube Neo-Hookean (soft,
    E = 10 kPa) -- the contrast of the paper's NH bunnies in ARAP balls on a scene the
    oracle steps in seconds.  material_model: 0 = Neo-Hookean, 1 = ARAP (per material)."""
    sc = make_cubes(seed, **kw)
    nt = len(sc["tets"]) // 2  # two equal cubes, bottom first
    nu, rho = sc["materials"][0][1], sc["materials"][0][2]
    sc["materials"] = np.array([[E_arap, nu, rho], [E_nh, nu, rho]])
    sc["material_model"] = np.array([1, 0])
    tm = np.zeros(len(sc["tets"]), np.int32)
    tm[nt:] = 1
    sc["tet_material"] = tm
    sc["name"] = "NH-ARAP-cubes"
    return sc
