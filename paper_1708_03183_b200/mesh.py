"""Synthetic triangle meshes, facet derivation and locality renumbering.

Host-side fixtures and the data-layout pass.  Entity numbering matches the
reference generator exactly (``pkg/src/looptile/mesh.py:65-101``): vertex
(i, j) is ``j*(nx+1)+i``, quad (i, j) yields the lower triangle
``(v00, v10, v11)`` then the upper ``(v00, v11, v01)``, row-major, and edges
are the sorted unique cell sides.  The generator here is vectorised (the
reference builds Python sets), so it reaches the 67M-cell configurations:
for this diagonal every sorted side ``(a, b)`` has ``a`` = its lower-left
vertex, so the sorted edge list is emitted directly in order without a sort.

Renumbering: ``rcm_renumber`` reproduces the reference Reverse Cuthill-McKee
(``mesh.py:104-206``: lowest-id minimum-degree start, neighbours by
(degree, id), cells/edges ordered by sorted new-vertex tuples) through the
native BFS in ``libltcuda`` (``lt_rcm_order``).  ``morton_renumber`` is the
locality alternative the paper names as future work (``PAPER.md:967``).

Builder helpers the BASELINE workloads need and the reference lacks
(SURVEY Appendix C): ``cell_edge_map`` (c2e, side order (v0,v1),(v1,v2),(v0,v2))
and ``facet_topology`` (interior/exterior facets, if2c/ef2c, local face ids).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .chain import IterationSpace, MeshMap


@dataclass(frozen=True, eq=False)
class Mesh:
    """A 2D triangulation: flat connectivity arrays plus coordinates (``mesh.py:17-53``)."""

    num_vertices: int
    num_cells: int
    num_edges: int
    cells_to_vertices: np.ndarray  # flat, arity 3
    edges_to_vertices: np.ndarray  # flat, arity 2
    vertex_coords: np.ndarray      # shape (num_vertices, 2)

    def cell_vertices(self, c: int) -> np.ndarray:
        return self.cells_to_vertices[3 * c: 3 * c + 3]

    def edge_vertices(self, e: int) -> np.ndarray:
        return self.edges_to_vertices[2 * e: 2 * e + 2]

    def validate(self) -> None:
        c2v = self.cells_to_vertices
        e2v = self.edges_to_vertices
        assert len(c2v) == 3 * self.num_cells
        assert len(e2v) == 2 * self.num_edges
        if self.num_cells:
            assert 0 <= c2v.min() and c2v.max() < self.num_vertices
        assert 0 <= e2v.min() and e2v.max() < self.num_vertices
        tri = c2v.reshape(-1, 3)
        assert np.all(tri[:, 0] != tri[:, 1])
        assert np.all(tri[:, 1] != tri[:, 2])
        assert np.all(tri[:, 0] != tri[:, 2])
        pairs = e2v.reshape(-1, 2)
        assert np.all(pairs[:, 0] != pairs[:, 1])
        sides = np.unique(_side_keys(tri, self.num_vertices))
        stored = np.sort(np.minimum(pairs[:, 0], pairs[:, 1]) * self.num_vertices
                         + np.maximum(pairs[:, 0], pairs[:, 1]))
        assert len(stored) == self.num_edges
        assert np.array_equal(sides, stored), "edge set does not match cell sides"


def _side_keys(tri: np.ndarray, nv: int) -> np.ndarray:
    """Undirected side keys min*nv+max of every cell side, in (cell, side) order."""
    a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
    sides = np.stack([np.stack([a, b], 1), np.stack([b, c], 1),
                      np.stack([a, c], 1)], 1)  # (C, 3, 2), side order of mesh.py:58-61
    lo = sides.min(axis=2)
    hi = sides.max(axis=2)
    return (lo * nv + hi).ravel()


def generate_rect_mesh(nx: int, ny: int) -> Mesh:
    """Triangulate an nx-by-ny quad grid into 2*nx*ny triangles (``mesh.py:65-101``)."""
    if nx < 1 or ny < 1:
        raise ValueError(f"mesh dimensions must be positive, got {nx}x{ny}")
    nvx, nvy = nx + 1, ny + 1
    nv = nvx * nvy
    ii, jj = np.meshgrid(np.arange(nvx), np.arange(nvy))
    coords = np.column_stack([ii.ravel().astype(float), jj.ravel().astype(float)])

    j, i = np.meshgrid(np.arange(ny, dtype=np.int64), np.arange(nx, dtype=np.int64),
                       indexing="ij")
    v00 = (j * nvx + i).ravel()
    v10 = v00 + 1
    v01 = v00 + nvx
    v11 = v01 + 1
    tri = np.empty((nx * ny, 2, 3), dtype=np.int64)
    tri[:, 0, 0], tri[:, 0, 1], tri[:, 0, 2] = v00, v10, v11   # lower triangle
    tri[:, 1, 0], tri[:, 1, 1], tri[:, 1, 2] = v00, v11, v01   # upper triangle

    # sorted unique sides: per vertex v (ascending) its partners v+1 (right),
    # v+nvx (up), v+nvx+1 (diagonal), which are already in ascending order
    vi = np.arange(nv, dtype=np.int64) % nvx
    vj = np.arange(nv, dtype=np.int64) // nvx
    has = np.stack([vi < nx, vj < ny, (vi < nx) & (vj < ny)], axis=1)
    partner = np.arange(nv, dtype=np.int64)[:, None] + np.array([1, nvx, nvx + 1])
    src = np.broadcast_to(np.arange(nv, dtype=np.int64)[:, None], (nv, 3))
    e2v = np.stack([src[has], partner[has]], axis=1).ravel()

    return Mesh(num_vertices=nv, num_cells=2 * nx * ny, num_edges=len(e2v) // 2,
                cells_to_vertices=tri.reshape(-1), edges_to_vertices=e2v,
                vertex_coords=coords)


def vertex_adjacency_csr(mesh: Mesh) -> tuple[np.ndarray, np.ndarray]:
    """Vertex graph over the edge set as CSR (offsets, sorted neighbour ids)."""
    pairs = mesh.edges_to_vertices.reshape(-1, 2)
    a = np.concatenate([pairs[:, 0], pairs[:, 1]])
    b = np.concatenate([pairs[:, 1], pairs[:, 0]])
    order = np.lexsort((b, a))
    counts = np.bincount(a, minlength=mesh.num_vertices)
    offsets = np.zeros(mesh.num_vertices + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, b[order]


def adjacency_bandwidth(mesh: Mesh) -> int:
    """max |i - j| over connected vertex pairs."""
    pairs = mesh.edges_to_vertices.reshape(-1, 2)
    return int(np.abs(pairs[:, 0] - pairs[:, 1]).max()) if len(pairs) else 0


@dataclass(frozen=True)
class MeshRenumbering:
    """Old-to-new index maps for each entity space; all bijections (``mesh.py:148-154``)."""

    vertex_perm: np.ndarray
    cell_perm: np.ndarray
    edge_perm: np.ndarray


def _induced_perms(mesh: Mesh, vertex_perm: np.ndarray) -> MeshRenumbering:
    """Cells/edges relabelled by the sorted tuple of their new vertex ids (``mesh.py:167-179``)."""
    tri = np.sort(vertex_perm[mesh.cells_to_vertices.reshape(-1, 3)], axis=1)
    cell_order = np.lexsort((tri[:, 2], tri[:, 1], tri[:, 0]))
    cell_perm = np.empty(mesh.num_cells, dtype=np.int64)
    cell_perm[cell_order] = np.arange(mesh.num_cells)
    pairs = np.sort(vertex_perm[mesh.edges_to_vertices.reshape(-1, 2)], axis=1)
    edge_order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    edge_perm = np.empty(mesh.num_edges, dtype=np.int64)
    edge_perm[edge_order] = np.arange(mesh.num_edges)
    return MeshRenumbering(vertex_perm=vertex_perm, cell_perm=cell_perm,
                           edge_perm=edge_perm)


def rcm_ordering(mesh: Mesh) -> np.ndarray:
    """Reverse Cuthill-McKee order: position k holds the old id placed k-th.

    Native BFS (``lt_rcm_order``) with the reference tie-breaks
    (``mesh.py:123-145``); raises ValueError on a disconnected graph.
    """
    from . import _lib
    offsets, nbrs = vertex_adjacency_csr(mesh)
    return _lib.rcm_order(offsets, nbrs)


def rcm_permutations(mesh: Mesh) -> MeshRenumbering:
    order = rcm_ordering(mesh)
    vertex_perm = np.empty(mesh.num_vertices, dtype=np.int64)
    vertex_perm[order] = np.arange(mesh.num_vertices)
    return _induced_perms(mesh, vertex_perm)


def morton_permutations(mesh: Mesh) -> MeshRenumbering:
    """Z-order (Morton) vertex relabelling by coordinates; cells/edges induced.

    Compact 2D tiles from contiguous seed chunks, at the price of more colours
    than RCM's bands (SURVEY §7 "Colours = launch phases").
    """
    xy = mesh.vertex_coords
    lo = xy.min(axis=0)
    span = np.maximum(xy.max(axis=0) - lo, 1e-300)
    q = np.minimum(((xy - lo) / span * 65535.0).astype(np.uint64), 65535)

    def spread(v):
        v = v & np.uint64(0xFFFF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v

    key = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))
    order = np.lexsort((np.arange(mesh.num_vertices), key))
    vertex_perm = np.empty(mesh.num_vertices, dtype=np.int64)
    vertex_perm[order] = np.arange(mesh.num_vertices)
    return _induced_perms(mesh, vertex_perm)


def apply_renumbering(mesh: Mesh, renum: MeshRenumbering) -> Mesh:
    """Relabel every entity (``mesh.py:184-201``)."""
    vperm, cperm, eperm = renum.vertex_perm, renum.cell_perm, renum.edge_perm
    tri = vperm[mesh.cells_to_vertices.reshape(-1, 3)]
    new_tri = np.empty_like(tri)
    new_tri[cperm] = tri
    pairs = np.sort(vperm[mesh.edges_to_vertices.reshape(-1, 2)], axis=1)
    new_pairs = np.empty_like(pairs)
    new_pairs[eperm] = pairs
    coords = np.empty_like(mesh.vertex_coords)
    coords[vperm] = mesh.vertex_coords
    return Mesh(num_vertices=mesh.num_vertices, num_cells=mesh.num_cells,
                num_edges=mesh.num_edges, cells_to_vertices=new_tri.ravel(),
                edges_to_vertices=new_pairs.ravel(), vertex_coords=coords)


def rcm_renumber(mesh: Mesh) -> Mesh:
    """Relabel all entity spaces by reverse Cuthill-McKee over the edge graph."""
    return apply_renumbering(mesh, rcm_permutations(mesh))


def morton_renumber(mesh: Mesh) -> Mesh:
    return apply_renumbering(mesh, morton_permutations(mesh))


def renumber(mesh: Mesh, scheme: str | None) -> Mesh:
    if scheme in (None, "", "none"):
        return mesh
    if scheme == "rcm":
        return rcm_renumber(mesh)
    if scheme == "morton":
        return morton_renumber(mesh)
    raise ValueError(f"unknown renumbering {scheme!r}")


# -- chain-building helpers (mesh.py:209-227) ---------------------------------

CELLS, EDGES, VERTS = "cells", "edges", "verts"
IFACETS, EFACETS = "ifacets", "efacets"


def mesh_spaces(mesh: Mesh) -> dict[str, IterationSpace]:
    """Single-rank iteration spaces: everything core, no halo regions."""
    return {
        CELLS: IterationSpace(CELLS, mesh.num_cells),
        EDGES: IterationSpace(EDGES, mesh.num_edges),
        VERTS: IterationSpace(VERTS, mesh.num_vertices),
    }


def mesh_maps(mesh: Mesh, spaces: dict[str, IterationSpace]) -> dict[str, MeshMap]:
    return {
        "c2v": MeshMap("c2v", spaces[CELLS], spaces[VERTS], 3, mesh.cells_to_vertices),
        "e2v": MeshMap("e2v", spaces[EDGES], spaces[VERTS], 2, mesh.edges_to_vertices),
    }


def cell_edge_map(mesh: Mesh) -> np.ndarray:
    """c2e rows: edge ids of sides (v0,v1), (v1,v2), (v0,v2) per cell (flat, arity 3)."""
    nv = mesh.num_vertices
    pairs = mesh.edges_to_vertices.reshape(-1, 2)
    ekeys = np.minimum(pairs[:, 0], pairs[:, 1]) * nv + np.maximum(pairs[:, 0], pairs[:, 1])
    order = np.argsort(ekeys, kind="stable")
    skeys = _side_keys(mesh.cells_to_vertices.reshape(-1, 3), nv)
    pos = np.searchsorted(ekeys[order], skeys)
    return order[pos].astype(np.int64)


@dataclass(frozen=True, eq=False)
class FacetTopology:
    """Interior/exterior facets in edge order with their flanking cells.

    ``if2c`` rows are (lower cell id, higher cell id); ``iface`` the local face
    index (0: v0v1, 1: v1v2, 2: v2v0) of the facet in each flank; ``ef2c`` /
    ``eface`` likewise for the single flank of an exterior facet.
    ``iedge``/``eedge`` give the originating edge ids.
    """

    if2c: np.ndarray
    iface: np.ndarray
    iedge: np.ndarray
    ef2c: np.ndarray
    eface: np.ndarray
    eedge: np.ndarray

    @property
    def n_interior(self) -> int:
        return len(self.iedge)

    @property
    def n_exterior(self) -> int:
        return len(self.eedge)


def facet_topology(mesh: Mesh, c2e: np.ndarray | None = None) -> FacetTopology:
    c2e = cell_edge_map(mesh) if c2e is None else c2e
    flat_cell = np.repeat(np.arange(mesh.num_cells, dtype=np.int64), 3)
    flat_face = np.tile(np.array([0, 1, 2], dtype=np.int64), mesh.num_cells)
    order = np.lexsort((flat_cell, c2e))  # by edge, then ascending cell id
    edges_sorted = c2e[order]
    counts = np.bincount(c2e, minlength=mesh.num_edges)
    first = np.zeros(mesh.num_edges + 1, dtype=np.int64)
    np.cumsum(counts, out=first[1:])
    interior = np.flatnonzero(counts == 2)
    exterior = np.flatnonzero(counts == 1)
    assert np.all((counts == 1) | (counts == 2)), "non-manifold mesh"
    del edges_sorted
    fi = first[interior]
    if2c = np.stack([flat_cell[order[fi]], flat_cell[order[fi + 1]]], 1).ravel()
    iface = np.stack([flat_face[order[fi]], flat_face[order[fi + 1]]], 1).ravel()
    fe = first[exterior]
    return FacetTopology(if2c=if2c, iface=iface, iedge=interior,
                         ef2c=flat_cell[order[fe]], eface=flat_face[order[fe]],
                         eedge=exterior)
