"""2D isotropic elastic-wave DG (velocity-stress) as a loop chain.

The paper's application (Seigen elastic-wave timestep, ``PAPER.md:762``) is not
in the reference (SPEC.md:14 excludes it), so this is the project's own
discretisation, declared on the loop-chain API and run by
the native kernels ``dg_{vol,iflux,eflux,minv,axpy}_p{1..4}``:

    rho dv/dt = div(sigma)
    dsigma/dt = lambda tr(eps(v)) I + 2 mu eps(v)

* Orthonormal modal basis of degree P on the reference triangle
  (-1,-1),(1,-1),(-1,1) (Gram-Schmidt of monomials, so M_ref = I and the
  inverse-mass loop is a per-cell scaling by 1/(rho |J|) resp. 1/|J|).
* Strong form: volume term |J| (r_x S_r + s_x S_s) Q per field; facet term
  = lift of the flux correction at P+1 Gauss-Legendre points per facet.
* Upwind (exact Riemann) flux with P/S impedances of both sides; free
  surface on exterior facets by a mirror state (traction-free).
* Forward Euler ("axpy update").

Chain per timestep (5 loops, seed = cells):
  L0 cells    dg_vol    [cgeo R, mat R, u R, s R, ru W, rs W]
  L1 ifacets  dg_iflux  [fgeo R, mat R@if2c, u R@if2c, s R@if2c, ru I@if2c, rs I@if2c]
  L2 efacets  dg_eflux  [fgeo R, mat R@ef2c, u R@ef2c, s R@ef2c, ru I@ef2c, rs I@ef2c]
  L3 cells    dg_minv   [cgeo R, mat R, ru RW, rs RW]
  L4 cells    dg_axpy   [u RW, s RW, ru R, rs R]                      (param: dt)
``c2v`` is declared (unused by the loops) so the seed loop has a tile
adjacency map (SURVEY section 7 "Seed adjacency for DG").

Data layout (element-major, like the reference Dataset): u = [vx(nd), vy(nd)],
s = [sxx(nd), syy(nd), sxy(nd)], cgeo = [rx, ry, sx, sy, detJ],
mat = [rho, lambda, mu, Zp, Zs] (impedances rho*c_p, rho*c_s precomputed), fgeo = [nx, ny, |f|/2, face_a, face_b] (face_b = -1 on
exterior facets).  The operator tables (``dg_tables``) are generated once in
float64 and are the same arrays the CUDA kernels and the CPU oracle use.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .chain import AccessMode, Descriptor, IterationSpace, Loop, MeshMap, build_chain
from .mesh import (CELLS, EDGES, EFACETS, IFACETS, VERTS, Mesh, cell_edge_map, facet_topology,
                   generate_rect_mesh, renumber)

R, W, I, RW = AccessMode.READ, AccessMode.WRITE, AccessMode.INC, AccessMode.RW
REF_VERTS = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0]])


def n_dofs(p: int) -> int:
    return (p + 1) * (p + 2) // 2


def _monomial_exponents(p):
    return [(i, d - i) for d in range(p + 1) for i in range(d, -1, -1)]


def _monomials(p, r, s):
    ex = _monomial_exponents(p)
    v = np.stack([r ** i * s ** j for i, j in ex], axis=-1)
    dr = np.stack([i * r ** max(i - 1, 0) * s ** j if i else 0 * r for i, j in ex], axis=-1)
    ds = np.stack([j * r ** i * s ** max(j - 1, 0) if j else 0 * r for i, j in ex], axis=-1)
    return v, dr, ds


def triangle_quadrature(n: int):
    """Collapsed Gauss-Legendre rule on the reference triangle (n x n points)."""
    x, w = np.polynomial.legendre.leggauss(n)
    a, b = np.meshgrid(x, x, indexing="ij")
    wa, wb = np.meshgrid(w, w, indexing="ij")
    r = (1 + a) * (1 - b) / 2 - 1
    s = b
    wt = wa * wb * (1 - b) / 2
    return r.ravel(), s.ravel(), wt.ravel()


@dataclass(frozen=True)
class DGTables:
    p: int
    nd: int
    nq: int
    coef: np.ndarray      # psi = monomials @ coef  (nd x nd)
    Sr: np.ndarray        # int psi_i d_r psi_j   (nd x nd)
    Ss: np.ndarray
    E: np.ndarray         # face traces  (3, nq, nd)
    LIFT: np.ndarray      # w_q psi_i(face pt) (3, nd, nq)

    def basis(self, r, s):
        v, dr, ds = _monomials(self.p, np.asarray(r, float), np.asarray(s, float))
        return v @ self.coef, dr @ self.coef, ds @ self.coef

    def vol_params(self) -> np.ndarray:
        return np.concatenate([self.Sr.ravel(), self.Ss.ravel()])

    def flux_params(self) -> np.ndarray:
        return np.concatenate([self.E.ravel(), self.LIFT.ravel()])


@lru_cache(maxsize=None)
def dg_tables(p: int) -> DGTables:
    if not 1 <= p <= 4:
        raise ValueError("DG degree must be 1..4")
    nd = n_dofs(p)
    r, s, w = triangle_quadrature(p + 3)
    V, Vr, Vs = _monomials(p, r, s)
    coef = np.eye(nd)
    for _ in range(2):  # Gram-Schmidt by Cholesky, repeated once for full accuracy
        P = V @ coef
        G = P.T @ (w[:, None] * P)
        coef = coef @ np.linalg.inv(np.linalg.cholesky(G)).T  # psi = V @ coef orthonormal
    P, Pr, Ps = V @ coef, Vr @ coef, Vs @ coef
    Sr = P.T @ (w[:, None] * Pr)
    Ss = P.T @ (w[:, None] * Ps)
    nq = p + 1
    t, wq = np.polynomial.legendre.leggauss(nq)
    E = np.empty((3, nq, nd))
    LIFT = np.empty((3, nd, nq))
    for f in range(3):
        a, b = REF_VERTS[f], REF_VERTS[(f + 1) % 3]
        pts = ((1 - t)[:, None] * a + (1 + t)[:, None] * b) / 2
        Vf, _, _ = _monomials(p, pts[:, 0], pts[:, 1])
        E[f] = Vf @ coef
        LIFT[f] = (E[f] * wq[:, None]).T
    return DGTables(p, nd, nq, coef, Sr, Ss, E, LIFT)


# ---- geometry ------------------------------------------------------------------------

def cell_geometry(mesh: Mesh) -> np.ndarray:
    """Per-cell [rx, ry, sx, sy, detJ] of the affine map from the reference triangle."""
    X = mesh.vertex_coords[mesh.cells_to_vertices.reshape(-1, 3)]
    xr = (X[:, 1] - X[:, 0]) / 2
    xs = (X[:, 2] - X[:, 0]) / 2
    det = xr[:, 0] * xs[:, 1] - xs[:, 0] * xr[:, 1]
    if np.any(det <= 0):
        raise ValueError("cells must be counter-clockwise")
    return np.stack([xs[:, 1] / det, -xs[:, 0] / det, -xr[:, 1] / det, xr[:, 0] / det, det],
                    axis=1)


def facet_geometry(mesh: Mesh, cells: np.ndarray, faces: np.ndarray,
                   faces_b: np.ndarray | None = None) -> np.ndarray:
    """[nx, ny, |f|/2, face_a, face_b] with n outward from the first flank."""
    tri = mesh.cells_to_vertices.reshape(-1, 3)
    P0 = mesh.vertex_coords[tri[cells, faces]]
    P1 = mesh.vertex_coords[tri[cells, (faces + 1) % 3]]
    d = P1 - P0
    length = np.hypot(d[:, 0], d[:, 1])
    out = np.stack([d[:, 1] / length, -d[:, 0] / length, length / 2, faces.astype(float),
                    -np.ones(len(cells)) if faces_b is None else faces_b.astype(float)], axis=1)
    return out


# ---- problem ---------------------------------------------------------------------------

@dataclass
class ElasticSetup:
    """Host-side description of one elastic DG instance (no device state)."""

    p: int
    mesh: Mesh
    steps_per_chain: int
    dt: float
    spaces: dict
    maps: dict
    loops: list
    bindings: tuple
    data: dict          # name -> numpy values
    vpe: dict           # name -> values per element
    space_of: dict      # dataset -> space name
    tables: DGTables
    chain: object = None
    facets: object = None       # global FacetTopology (for rank-local restriction)
    local_mesh: object = None   # set on rank-local setups
    global_ids: dict | None = None

    num_cells: int | None = None  # device-generated setups carry no host Mesh

    @property
    def n_cells(self) -> int:
        return self.mesh.num_cells if self.mesh is not None else self.num_cells

    @property
    def dofs(self) -> int:
        return self.n_cells * 5 * n_dofs(self.p)


def _gaussian_projection(mesh: Mesh, tab: DGTables, centre, sigma: float) -> np.ndarray:
    """L2 projection of exp(-|x-c|^2 / (2 sigma^2)) on each cell (modal coefficients)."""
    r, s, w = triangle_quadrature(tab.p + 3)
    psi, _, _ = tab.basis(r, s)                           # (nqv, nd)
    X = mesh.vertex_coords[mesh.cells_to_vertices.reshape(-1, 3)]
    out = np.empty((mesh.num_cells, tab.nd))
    chunk = 1 << 20
    lam0, lam1, lam2 = -(r + s) / 2, (1 + r) / 2, (1 + s) / 2
    for c0 in range(0, mesh.num_cells, chunk):
        Xc = X[c0:c0 + chunk]
        x = lam0 * Xc[:, 0, 0:1] + lam1 * Xc[:, 1, 0:1] + lam2 * Xc[:, 2, 0:1]
        y = lam0 * Xc[:, 0, 1:2] + lam1 * Xc[:, 1, 1:2] + lam2 * Xc[:, 2, 1:2]
        g = np.exp(-((x - centre[0]) ** 2 + (y - centre[1]) ** 2) / (2 * sigma ** 2))
        out[c0:c0 + chunk] = (g * w) @ psi
    return out


def elastic_setup(nx: int, ny: int, p: int, steps_per_chain: int = 1,
                  material="homogeneous", noise_seed: int | None = 1, sigma: float = 8.0,
                  dt: float | None = None, renumbering: str | None = None,
                  mesh: Mesh | None = None, centre=None,
                  cell_offset: int = 0) -> ElasticSetup:
    """Build the BASELINE elastic DG instance on an nx x ny right-diagonal mesh (h = 1).

    ``material``: "homogeneous" (rho=1, lambda=2, mu=1) or ("uniform", seed) for
    per-cell rho, lambda, mu ~ U[1, 2] drawn as rng.uniform(1, 2, (cells, 3)).

    ``mesh``/``centre``/``cell_offset`` build a window of a larger mesh (the
    strips of ``strips.py``): the pulse centre is the global one and the random
    streams are advanced past the ``cell_offset`` cells before the window, so
    the window's draws are the global draws of its cells.
    """
    tab = dg_tables(p)
    nd = tab.nd
    if mesh is None:
        mesh = renumber(generate_rect_mesh(nx, ny), renumbering)
    c2e = cell_edge_map(mesh)
    ft = facet_topology(mesh, c2e)
    C, Fi, Fe = mesh.num_cells, ft.n_interior, ft.n_exterior
    spaces = {CELLS: IterationSpace(CELLS, C), IFACETS: IterationSpace(IFACETS, Fi),
              EFACETS: IterationSpace(EFACETS, Fe), VERTS: IterationSpace(VERTS, mesh.num_vertices)}
    maps = {
        "c2v": MeshMap("c2v", spaces[CELLS], spaces[VERTS], 3, mesh.cells_to_vertices),
        "if2c": MeshMap("if2c", spaces[IFACETS], spaces[CELLS], 2, ft.if2c),
        "ef2c": MeshMap("ef2c", spaces[EFACETS], spaces[CELLS], 1, ft.ef2c),
    }
    # geometry
    cgeo = cell_geometry(mesh)
    rows = ft.if2c.reshape(-1, 2)
    faces = ft.iface.reshape(-1, 2)
    fig = facet_geometry(mesh, rows[:, 0], faces[:, 0], faces[:, 1])
    tri = mesh.cells_to_vertices.reshape(-1, 3)
    # the second flank must traverse the facet in the opposite direction
    assert np.array_equal(tri[rows[:, 1], faces[:, 1]], tri[rows[:, 0], (faces[:, 0] + 1) % 3])
    feg = facet_geometry(mesh, ft.ef2c, ft.eface)
    # material
    if material == "homogeneous":
        mat = np.tile([1.0, 2.0, 1.0], (C, 1))
    else:
        kind, seed = material
        assert kind == "uniform"
        rng = np.random.default_rng(seed)
        rng.bit_generator.advance(3 * cell_offset)  # one 64-bit draw per double
        mat = rng.uniform(1.0, 2.0, size=(C, 3))
    if dt is None:
        cp = np.sqrt((mat[:, 1] + 2 * mat[:, 2]) / mat[:, 0]).max()
        dt = 0.1 * 1.0 / (cp * (2 * p + 1))
    zp = np.sqrt(mat[:, 0] * (mat[:, 1] + 2 * mat[:, 2]))
    zs = np.sqrt(mat[:, 0] * mat[:, 2])
    mat = np.column_stack([mat, zp, zs])
    # initial condition: Gaussian pulse at the domain centre on all components
    X = mesh.vertex_coords
    if centre is None:
        centre = ((X[:, 0].min() + X[:, 0].max()) / 2, (X[:, 1].min() + X[:, 1].max()) / 2)
    g = _gaussian_projection(mesh, tab, centre, sigma)
    q = np.repeat(g[:, None, :], 5, axis=1)                # (C, 5, nd)
    if noise_seed is not None:
        rng = np.random.default_rng(noise_seed)
        rng.bit_generator.advance(5 * nd * cell_offset)
        q = q + rng.uniform(-1e-3, 1e-3, size=q.shape)
    data = {
        "cgeo": cgeo.ravel(), "mat": mat.ravel(),
        "u": q[:, 0:2, :].reshape(-1).copy(), "s": q[:, 2:5, :].reshape(-1).copy(),
        "ru": np.zeros(C * 2 * nd), "rs": np.zeros(C * 3 * nd),
        "figeo": fig.ravel(), "fegeo": feg.ravel(),
    }
    vpe = {"cgeo": 5, "mat": 5, "u": 2 * nd, "s": 3 * nd, "ru": 2 * nd, "rs": 3 * nd,
           "figeo": 5, "fegeo": 5}
    space_of = {"cgeo": CELLS, "mat": CELLS, "u": CELLS, "s": CELLS, "ru": CELLS, "rs": CELLS,
                "figeo": IFACETS, "fegeo": EFACETS}
    loops, bindings = chain_loops(p, steps_per_chain, spaces, maps)
    return ElasticSetup(p, mesh, steps_per_chain, float(dt), spaces, maps, loops, bindings,
                        data, vpe, space_of, tab, facets=ft)


# ---- device-side generation (configs 3-4: 8.4M-67M cells) ---------------------------

def rect_mesh_device(nx: int, ny: int, device) -> dict:
    """The right-diagonal nx x ny mesh generated on ``device`` (torch), in the
    numbering of ``mesh.generate_rect_mesh`` + ``facet_topology``.

    Vertex (i, j) = j*(nx+1)+i; quad (i, j) gives lower (v00, v10, v11) = cell
    2q and upper (v00, v11, v01) = cell 2q+1, q = j*nx+i.  Edges are the sorted
    unique sides: per vertex, right (v, v+1), up (v, v+nx+1), diagonal
    (v, v+nx+2) where they exist -- the order ``generate_rect_mesh`` emits.
    Flanks of each edge in closed form (ascending cell ids, local face
    0: v0v1, 1: v1v2, 2: v2v0):
      right of (i, j): upper cell of quad (i, j-1), face 1 | lower of (i, j), face 0
      up of (i, j):    lower cell of quad (i-1, j), face 1 | upper of (i, j), face 2
      diagonal:        lower of quad (i, j), face 2        | upper of (i, j), face 0
    Interior facets are the two-flank edges in edge order, exterior the rest.
    Returns int64 tensors c2v (C*3), if2c/iface (Fi*2), ef2c/eface (Fe).
    ``tests/test_dg_device_setup.py`` checks equality with the host generator.
    """
    import torch
    L = dict(dtype=torch.int64, device=device)
    nvx = nx + 1
    q = torch.arange(nx * ny, **L)
    qi, qj = q % nx, q // nx
    v00 = qj * nvx + qi
    v10, v01 = v00 + 1, v00 + nvx
    v11 = v01 + 1
    c2v = torch.stack([v00, v10, v11, v00, v11, v01], dim=1).reshape(-1)
    del q, qi, qj, v00, v10, v01, v11
    nv = nvx * (ny + 1)
    v = torch.arange(nv, **L)
    vi, vj = v % nvx, v // nvx
    del v
    lower = lambda i, j: 2 * (j * nx + i)
    neg = torch.full_like(vi, -1)
    # per vertex, slots (right, up, diagonal): flank a/b (cell or -1) and faces
    fa = torch.stack([torch.where(vj > 0, lower(vi, vj - 1) + 1, neg),
                      torch.where(vi > 0, lower(vi - 1, vj), neg),
                      lower(vi, vj)], dim=1)
    fb = torch.stack([torch.where(vj < ny, lower(vi, vj), neg),
                      torch.where(vi < nx, lower(vi, vj) + 1, neg),
                      lower(vi, vj) + 1], dim=1)
    has = torch.stack([vi < nx, vj < ny, (vi < nx) & (vj < ny)], dim=1)
    del vi, vj, neg
    face_a = torch.tensor([1, 1, 2], **L).expand(nv, 3)
    face_b = torch.tensor([0, 2, 0], **L).expand(nv, 3)
    fa, fb = fa[has], fb[has]
    face_a, face_b = face_a[has], face_b[has]
    del has
    inter = (fa >= 0) & (fb >= 0)
    if2c = torch.stack([fa[inter], fb[inter]], dim=1).reshape(-1)
    iface = torch.stack([face_a[inter], face_b[inter]], dim=1).reshape(-1)
    ext = ~inter
    one = torch.where(fa[ext] >= 0, fa[ext], fb[ext])
    oneface = torch.where(fa[ext] >= 0, face_a[ext], face_b[ext])
    return {"nv": nv, "c2v": c2v, "if2c": if2c, "iface": iface, "ef2c": one, "eface": oneface}


def morton_renumber_device(m: dict, nx: int, ny: int, block=None) -> dict:
    """Locality renumbering of a device mesh (north star item 3, the layout
    pass): quads in Morton (Z-curve) order of (i, j), the two cells of a quad
    kept adjacent, so ``ts`` consecutive cells form a compact block of quads
    instead of a one-quad-high strip of the row-major numbering (smaller tile
    footprints after projection across the chain).  Facet flanks are re-sorted
    to ascending cell ids (the convention of ``facet_topology``) and facets
    ordered by their first cell.  Returns the renumbered mesh plus
    ``old_of_new`` (cells) for permuting per-cell inputs drawn in the
    generator's order."""
    import torch
    dev = m["c2v"].device
    q = torch.arange(nx * ny, dtype=torch.int64, device=dev)

    def spread(v):  # bit k of v -> bit 2k
        out = torch.zeros_like(v)
        for k in range(max(nx, ny).bit_length()):
            out |= ((v >> k) & 1) << (2 * k)
        return out

    if block is None:
        code = spread(q % nx) | (spread(q // nx) << 1)
    else:
        # bx x by blocks of quads, blocks and the quads inside them row-major:
        # 2*bx*by consecutive cells are one block (seed tiles of any such size)
        bx, by = block
        qi, qj = q % nx, q // nx
        nbx = (nx + bx - 1) // bx
        code = ((qj // by) * nbx + qi // bx) * (bx * by) + (qj % by) * bx + qi % bx
        del qi, qj
    qs = torch.argsort(code)
    del code, q
    old_of_new = torch.stack([2 * qs, 2 * qs + 1], dim=1).reshape(-1)
    del qs
    new_of_old = torch.empty_like(old_of_new)
    new_of_old[old_of_new] = torch.arange(old_of_new.numel(), dtype=torch.int64, device=dev)
    out = {"nv": m["nv"], "old_of_new": old_of_new}
    out["c2v"] = m["c2v"].reshape(-1, 3)[old_of_new].reshape(-1)
    f = new_of_old[m["if2c"]].reshape(-1, 2)
    fc = m["iface"].reshape(-1, 2)
    swap = f[:, 0] > f[:, 1]
    f = torch.where(swap[:, None], f.flip(1), f)
    fc = torch.where(swap[:, None], fc.flip(1), fc)
    order = torch.argsort(f[:, 0] * 4 + fc[:, 0])      # first cell, then its face: unique
    out["if2c"], out["iface"] = f[order].reshape(-1), fc[order].reshape(-1)
    e = new_of_old[m["ef2c"]]
    order = torch.argsort(e * 4 + m["eface"])
    out["ef2c"], out["eface"] = e[order], m["eface"][order]
    return out


def _coords_of(v, nx):
    import torch
    return torch.stack([(v % (nx + 1)).to(torch.float64), (v // (nx + 1)).to(torch.float64)], -1)


def _cell_geometry_device(c2v, nx):
    import torch
    X = _coords_of(c2v.reshape(-1, 3), nx)              # (C, 3, 2)
    xr = (X[:, 1] - X[:, 0]) / 2
    xs = (X[:, 2] - X[:, 0]) / 2
    det = xr[:, 0] * xs[:, 1] - xs[:, 0] * xr[:, 1]
    return torch.stack([xs[:, 1] / det, -xs[:, 0] / det, -xr[:, 1] / det, xr[:, 0] / det, det],
                       dim=1)


def _facet_geometry_device(c2v, cells, faces, faces_b, nx):
    import torch
    tri = c2v.reshape(-1, 3)
    P0 = _coords_of(tri[cells, faces], nx)
    P1 = _coords_of(tri[cells, (faces + 1) % 3], nx)
    d = P1 - P0
    length = torch.hypot(d[:, 0], d[:, 1])
    fb = torch.full_like(length, -1.0) if faces_b is None else faces_b.to(torch.float64)
    return torch.stack([d[:, 1] / length, -d[:, 0] / length, length / 2,
                        faces.to(torch.float64), fb], dim=1)


def _gaussian_projection_device(c2v, nx, tab: DGTables, centre, sigma, device):
    import torch
    r, s, w = triangle_quadrature(tab.p + 3)
    psi, _, _ = tab.basis(r, s)
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=device)
    psi, w = T(psi), T(w)
    lam = [T(-(r + s) / 2), T((1 + r) / 2), T((1 + s) / 2)]
    tri = c2v.reshape(-1, 3)
    C = tri.shape[0]
    out = torch.empty((C, tab.nd), dtype=torch.float64, device=device)
    chunk = 1 << 21
    for c0 in range(0, C, chunk):
        X = _coords_of(tri[c0:c0 + chunk], nx)
        x = lam[0] * X[:, 0, 0:1] + lam[1] * X[:, 1, 0:1] + lam[2] * X[:, 2, 0:1]
        y = lam[0] * X[:, 0, 1:2] + lam[1] * X[:, 1, 1:2] + lam[2] * X[:, 2, 1:2]
        g = torch.exp(-((x - centre[0]) ** 2 + (y - centre[1]) ** 2) / (2 * sigma ** 2))
        out[c0:c0 + chunk] = (g * w) @ psi
    return out


def elastic_setup_device(nx: int, ny: int, p: int, steps_per_chain: int = 1,
                         material="homogeneous", noise_seed: int | None = 1,
                         sigma: float = 8.0, dt: float | None = None,
                         device=None, renumber: str | None = None) -> ElasticSetup:
    """:func:`elastic_setup` with the mesh, geometry, material and initial state
    generated on the GPU (no host mesh: the 67M-cell configuration needs no
    host pass over its cells).  Same numbering, datasets and chain; maps are
    device tensors (``MeshMap`` validates and fingerprints them on the device).
    Random draws (per-cell material, initial noise) use the host generator of
    :func:`elastic_setup` so both setups draw identical values."""
    import torch
    device = torch.device(device if device is not None else "cuda")
    tab = dg_tables(p)
    nd = tab.nd
    m = rect_mesh_device(nx, ny, device)
    C = 2 * nx * ny
    old_of_new = None
    if renumber == "morton":
        m = morton_renumber_device(m, nx, ny)
        old_of_new = m.pop("old_of_new")
    elif isinstance(renumber, str) and renumber.startswith("block:"):   # "block:3x2"
        bx, by = (int(v) for v in renumber[6:].split("x"))
        m = morton_renumber_device(m, nx, ny, block=(bx, by))
        old_of_new = m.pop("old_of_new")
    elif renumber not in (None, "none"):
        raise ValueError(f"unknown device renumbering {renumber!r}")
    Fi, Fe = m["if2c"].numel() // 2, m["ef2c"].numel()
    spaces = {CELLS: IterationSpace(CELLS, C), IFACETS: IterationSpace(IFACETS, Fi),
              EFACETS: IterationSpace(EFACETS, Fe), VERTS: IterationSpace(VERTS, m["nv"])}
    maps = {
        "c2v": MeshMap("c2v", spaces[CELLS], spaces[VERTS], 3, m["c2v"]),
        "if2c": MeshMap("if2c", spaces[IFACETS], spaces[CELLS], 2, m["if2c"]),
        "ef2c": MeshMap("ef2c", spaces[EFACETS], spaces[CELLS], 1, m["ef2c"]),
    }
    cgeo = _cell_geometry_device(m["c2v"], nx)
    rows, faces = m["if2c"].reshape(-1, 2), m["iface"].reshape(-1, 2)
    fig = _facet_geometry_device(m["c2v"], rows[:, 0], faces[:, 0], faces[:, 1], nx)
    feg = _facet_geometry_device(m["c2v"], m["ef2c"], m["eface"], None, nx)
    del rows, faces
    # impedances on the host (numpy's correctly rounded sqrt, as elastic_setup)
    if material == "homogeneous":
        row = np.array([1.0, 2.0, 1.0])
        cp_max = float(np.sqrt((row[1] + 2 * row[2]) / row[0]))
        row = np.concatenate([row, [np.sqrt(row[0] * (row[1] + 2 * row[2])),
                                    np.sqrt(row[0] * row[2])]])
        mat = torch.from_numpy(row).to(device).repeat(C, 1)
    else:
        kind, seed = material
        assert kind == "uniform"
        host = np.random.default_rng(seed).uniform(1.0, 2.0, size=(C, 3))
        cp_max = float(np.sqrt((host[:, 1] + 2 * host[:, 2]) / host[:, 0]).max())
        host = np.column_stack([host, np.sqrt(host[:, 0] * (host[:, 1] + 2 * host[:, 2])),
                                np.sqrt(host[:, 0] * host[:, 2])])
        mat = torch.from_numpy(host).to(device)
        if old_of_new is not None:          # drawn per cell of the generator's numbering
            mat = mat[old_of_new]
        del host
    if dt is None:
        dt = 0.1 * 1.0 / (cp_max * (2 * p + 1))
    centre = (nx / 2.0, ny / 2.0)
    g = _gaussian_projection_device(m["c2v"], nx, tab, centre, sigma, device)
    u = g.repeat(1, 2)                                   # (C, 2*nd): [vx(nd) vy(nd)]
    s_ = g.repeat(1, 3)
    del g
    if noise_seed is not None:
        # the host draw of elastic_setup, (C, 5, nd) row-major, in cell chunks
        rng = np.random.default_rng(noise_seed)
        chunk = 1 << 20
        new_of_old = None
        if old_of_new is not None:
            new_of_old = torch.empty_like(old_of_new)
            new_of_old[old_of_new] = torch.arange(C, dtype=torch.int64, device=device)
        for c0 in range(0, C, chunk):
            n = min(chunk, C - c0)
            z = torch.from_numpy(rng.uniform(-1e-3, 1e-3, size=(n, 5, nd))).to(device)
            if new_of_old is None:
                u[c0:c0 + n] += z[:, 0:2].reshape(n, -1)
                s_[c0:c0 + n] += z[:, 2:5].reshape(n, -1)
            else:                           # rows of the generator's cells c0..c0+n
                rows = new_of_old[c0:c0 + n]
                u[rows] += z[:, 0:2].reshape(n, -1)
                s_[rows] += z[:, 2:5].reshape(n, -1)
        del new_of_old
    data = {
        "cgeo": cgeo.reshape(-1), "mat": mat.reshape(-1), "u": u.reshape(-1),
        "s": s_.reshape(-1), "ru": torch.zeros(C * 2 * nd, dtype=torch.float64, device=device),
        "rs": torch.zeros(C * 3 * nd, dtype=torch.float64, device=device),
        "figeo": fig.reshape(-1), "fegeo": feg.reshape(-1),
    }
    vpe = {"cgeo": 5, "mat": 5, "u": 2 * nd, "s": 3 * nd, "ru": 2 * nd, "rs": 3 * nd,
           "figeo": 5, "fegeo": 5}
    space_of = {"cgeo": CELLS, "mat": CELLS, "u": CELLS, "s": CELLS, "ru": CELLS, "rs": CELLS,
                "figeo": IFACETS, "fegeo": EFACETS}
    loops, bindings = chain_loops(p, steps_per_chain, spaces, maps)
    del m
    # the generator's temporaries go back to the driver: the library allocates
    # its plan from its own stream-ordered pool, not from torch's cache
    torch.cuda.empty_cache()
    return ElasticSetup(p, None, steps_per_chain, float(dt), spaces, maps, loops, bindings,
                        data, vpe, space_of, tab, num_cells=C)


def local_elastic_setup(setup: ElasticSetup, lm) -> ElasticSetup:
    """Restrict a global elastic instance to one rank's extended-halo mesh.

    Cells keep the partition's region order (core | owned+exec | non-exec);
    local edges split into interior/exterior facets by their *global* flank
    count, flank maps through local ids, a missing flank pointing at the
    present cell (only possible in the non-exec strip).
    Dataset rows are the global rows of the local elements, so halo rows of
    constant data (geometry, material) are exact without any exchange.
    """
    ft = setup.facets
    iid, if2c, eid, ef2c, isz, esz = lm.facets()
    egid = lm.global_ids[EDGES]
    # global facet index of every global edge
    inv_i = np.full(setup.mesh.num_edges, -1, dtype=np.int64)
    inv_i[ft.iedge] = np.arange(ft.n_interior)
    inv_e = np.full(setup.mesh.num_edges, -1, dtype=np.int64)
    inv_e[ft.eedge] = np.arange(ft.n_exterior)
    gi, ge = inv_i[egid[iid]], inv_e[egid[eid]]
    assert np.all(gi >= 0) and np.all(ge >= 0)
    cs, vs = lm.sizes[CELLS], lm.sizes[VERTS]
    spaces = {CELLS: IterationSpace(CELLS, cs.core, cs.owned + cs.exec, cs.nonexec),
              IFACETS: IterationSpace(IFACETS, *isz),
              EFACETS: IterationSpace(EFACETS, *esz),
              VERTS: IterationSpace(VERTS, vs.core, vs.owned + vs.exec, vs.nonexec)}
    maps = {
        "c2v": MeshMap("c2v", spaces[CELLS], spaces[VERTS], 3, lm.cells_to_vertices),
        "if2c": MeshMap("if2c", spaces[IFACETS], spaces[CELLS], 2, if2c),
        "ef2c": MeshMap("ef2c", spaces[EFACETS], spaces[CELLS], 1, ef2c),
    }
    cg = lm.global_ids[CELLS]
    rows = {CELLS: cg, IFACETS: gi, EFACETS: ge}
    data = {n: v.reshape(-1, setup.vpe[n])[rows[setup.space_of[n]]].ravel().copy()
            for n, v in setup.data.items()}
    loops, bindings = chain_loops(setup.p, setup.steps_per_chain, spaces, maps)
    local = ElasticSetup(setup.p, setup.mesh, setup.steps_per_chain, setup.dt, spaces, maps,
                         loops, bindings, data, dict(setup.vpe), dict(setup.space_of),
                         setup.tables, facets=None, local_mesh=lm,
                         global_ids={CELLS: cg, IFACETS: gi, EFACETS: ge})
    return local


def chain_loops(p, steps, spaces, maps, loop_cls=Loop, desc_cls=Descriptor, binding_cls=None,
                modes=None):
    """Loops + bindings of ``steps`` timesteps (5 loops each)."""
    if binding_cls is None:
        from .executor import KernelBinding as binding_cls
    m = modes or {"R": R, "W": W, "I": I, "RW": RW}
    C, FI, FE = spaces[CELLS], spaces[IFACETS], spaces[EFACETS]
    if2c, ef2c = maps["if2c"], maps["ef2c"]
    step = [
        (C, f"dg_vol_p{p}", [(None, "R", "cgeo"), (None, "R", "mat"), (None, "R", "u"),
                             (None, "R", "s"), (None, "W", "ru"), (None, "W", "rs")]),
        (FI, f"dg_iflux_p{p}", [(None, "R", "figeo"), (if2c, "R", "mat"), (if2c, "R", "u"),
                                (if2c, "R", "s"), (if2c, "I", "ru"), (if2c, "I", "rs")]),
        (FE, f"dg_eflux_p{p}", [(None, "R", "fegeo"), (ef2c, "R", "mat"), (ef2c, "R", "u"),
                                (ef2c, "R", "s"), (ef2c, "I", "ru"), (ef2c, "I", "rs")]),
        (C, f"dg_minv_p{p}", [(None, "R", "cgeo"), (None, "R", "mat"), (None, "RW", "ru"),
                              (None, "RW", "rs")]),
        (C, f"dg_axpy_p{p}", [(None, "RW", "u"), (None, "RW", "s"), (None, "R", "ru"),
                              (None, "R", "rs")]),
    ]
    loops, bindings = [], []
    for _ in range(steps):
        for space, kern, acc in step:
            loops.append(loop_cls(len(loops), space,
                                  tuple(desc_cls(mp, m[md]) for mp, md, _ in acc), kern))
            bindings.append(binding_cls(kern, tuple(n for _, _, n in acc)))
    return loops, tuple(bindings)


def kernel_params(setup: ElasticSetup) -> dict[str, np.ndarray]:
    """Per-kernel parameter blocks: operator tables and dt."""
    p, tab = setup.p, setup.tables
    return {f"dg_vol_p{p}": tab.vol_params(), f"dg_iflux_p{p}": tab.flux_params(),
            f"dg_eflux_p{p}": tab.flux_params(), f"dg_minv_p{p}": np.zeros(1),
            f"dg_axpy_p{p}": np.array([setup.dt])}


@dataclass
class ElasticProblem:
    """Device instance: chain + HBM datasets + registry with installed parameters."""

    setup: ElasticSetup
    chain: object
    datasets: dict
    bindings: tuple
    registry: object
    schedules: dict = field(default_factory=dict)

    def install_params(self):
        from . import _lib
        for name, prm in kernel_params(self.setup).items():
            kid, _ = _lib.kernel_lookup(name)
            _lib.set_kernel_params(kid, prm)

    def inspect(self, ts: int, mode=None):
        from .inspector import ExecMode, inspect_chain
        mode = mode or ExecMode.SHARED
        key = (ts, mode)
        if key not in self.schedules:
            self.schedules[key] = inspect_chain(self.chain, ts, mode)
        return self.schedules[key]

    def run_tiled(self, schedule, n_chains: int = 1, use_local_maps: bool = True):
        from .executor import execute_schedule
        self.install_params()
        for _ in range(n_chains):
            execute_schedule(schedule, self.chain, self.bindings, self.datasets, self.registry,
                             use_local_maps=use_local_maps)

    def run_untiled(self, n_chains: int = 1):
        from .executor import execute_untiled
        self.install_params()
        for _ in range(n_chains):
            execute_untiled(self.chain, self.bindings, self.datasets, self.registry)


def elastic_problem(setup: ElasticSetup, depth: int | None = None) -> ElasticProblem:
    from .executor import Dataset
    from .problems import default_registry
    chain = build_chain(tuple(setup.spaces.values()), tuple(setup.maps.values()),
                        setup.loops, depth or len(setup.loops))
    setup.chain = chain
    ds = {n: Dataset(n, setup.spaces[setup.space_of[n]], setup.vpe[n], v)
          for n, v in setup.data.items()}
    return ElasticProblem(setup, chain, ds, setup.bindings, default_registry())


def compulsory_bytes(chain, bindings, vpe: dict, space_total: dict) -> int:
    """Algorithmic HBM bytes of one chain execution.

    Every dataset the chain reads before writing is read once, every dataset
    it writes is written once (float64), and every map a loop uses is read
    once (int32).  This is the B_chain of DESIGN.md (section "Roofline").
    """
    first = {}
    written = set()
    maps = {}
    for loop, b in zip(chain.loops, bindings):
        for d, name in zip(loop.descriptors, b.args):
            if name not in first:
                first[name] = d.mode
            if d.mode is not AccessMode.READ:
                written.add(name)
            if d.map is not None:
                maps[d.map.name] = d.map.source.total * d.map.arity * 4
    total = 0
    for name, mode in first.items():
        size = space_total[name] * vpe[name] * 8
        if mode in (AccessMode.READ, AccessMode.RW, AccessMode.INC):
            total += size
        if name in written:
            total += size
    return total + sum(maps.values())


def constant_datasets(chain, bindings) -> set[str]:
    """Datasets no loop of the chain writes (their halo rows never go stale)."""
    written = {n for lp, b in zip(chain.loops, bindings)
               for d, n in zip(lp.descriptors, b.args) if d.mode is not AccessMode.READ}
    return {n for b in bindings for n in b.args} - written


def run_elastic_distributed(setup: ElasticSetup, nranks: int, depth: int, ts: int,
                            n_chains: int = 1, mode=None, poison_halo: bool = False,
                            use_local_maps: bool = True):
    """The elastic chain on ``nranks`` virtual ranks sharing one GPU.

    Partition (strips + ``depth`` halo strips), rank-local problems, mixed-mode
    (SHARED) inspection per rank, one halo exchange per chain execution
    (reference ``distsim.run_distributed`` semantics; constant datasets are not
    exchanged).  Returns the gathered owned rows of ``u`` and ``s``.
    """
    from .distributed import (HaloEndpoint, _PreStaged, check_exchange_symmetry,
                              exchanged_from_chain)
    from .executor import execute_schedule
    from .inspector import ExecMode
    from .partition import partition_for_ranks
    mode = mode or ExecMode.SHARED
    ranks = []
    for lm in partition_for_ranks(setup.mesh, nranks, depth):
        loc = local_elastic_setup(setup, lm)
        pb = elastic_problem(loc, depth=len(loc.loops))
        owned = lm.sizes[CELLS].owned_total
        if poison_halo:
            for n in ("u", "s", "ru", "rs"):
                pb.datasets[n].values[owned * loc.vpe[n]:] = 1e30
        sched = pb.inspect(ts, mode)
        const = constant_datasets(pb.chain, pb.bindings)
        exchanged = tuple(n for n in exchanged_from_chain(pb.chain, pb.bindings) if n not in const)
        ranks.append((lm, pb, sched, HaloEndpoint(lm, pb.datasets, exchanged)))
    eps = [r[3] for r in ranks]
    for e in eps:
        e.link(eps)
    check_exchange_symmetry(eps)
    ranks[0][1].install_params()
    for _ in range(n_chains):
        for e in eps:
            e.begin()
        for lm, pb, sched, ep in ranks:
            execute_schedule(sched, pb.chain, pb.bindings, pb.datasets, pb.registry,
                             exchange=_PreStaged(ep), use_local_maps=use_local_maps)
    out = {}
    for n in ("u", "s"):
        k = setup.vpe[n]
        vals = np.full(setup.mesh.num_cells * k, np.nan)
        for lm, pb, _, _ in ranks:
            owned = lm.sizes[CELLS].owned_total
            vals.reshape(-1, k)[lm.global_ids[CELLS][:owned]] = \
                pb.datasets[n].numpy().reshape(-1, k)[:owned]
        out[n] = vals
    return out, ranks
