"""Partitioner parity with the reference (CPU only)."""

import numpy as np
import pytest

from conftest import golden_npz

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.partition import partition_for_ranks


CASES = [("fig2_8x4_rcm", 2), ("fig2_8x4_rcm", 4), ("p_16x8_none", 3), ("p_12x10_rcm", 4),
         ("p_16x8_rcm", 8), ("p_9x7_none", 5)]


@pytest.mark.parametrize("tag,nranks", CASES)
def test_partition_matches_reference_fixtures(tag, nranks):
    ref = golden_npz("distributed.npz")
    _, d, ren = tag.split("_")
    mesh = lt.generate_rect_mesh(*(int(v) for v in d.split("x")))
    if ren == "rcm":
        mesh = lt.rcm_renumber(mesh)
    pre = f"{tag}/n{nranks}"
    lms = partition_for_ranks(mesh, nranks, int(ref[f"{pre}/depth"][0]))
    for lm in lms:
        r = lm.rank
        for space, sz in lm.sizes.items():
            np.testing.assert_array_equal([sz.core, sz.owned, sz.exec, sz.nonexec],
                                          ref[f"{pre}/r{r}/{space}/sizes"], err_msg=(r, space))
            np.testing.assert_array_equal(lm.global_ids[space], ref[f"{pre}/r{r}/{space}/gids"])
        np.testing.assert_array_equal(lm.cells_to_vertices, ref[f"{pre}/r{r}/c2v"])
        np.testing.assert_array_equal(lm.edges_to_vertices, ref[f"{pre}/r{r}/e2v"])
        keys = {k for k in ref if k.startswith(f"{pre}/r{r}/x/")}
        assert len(keys) == len(lm.exchange_table)
        for (space, nbr), table in lm.exchange_table.items():
            np.testing.assert_array_equal(table, ref[f"{pre}/r{r}/x/{space}/{nbr}"])


@pytest.mark.parametrize("dims,nranks,depth", [((8, 4), 2, 1), ((12, 6), 3, 2), ((10, 10), 4, 4)])
def test_partition_invariants(dims, nranks, depth):
    mesh = lt.generate_rect_mesh(*dims)
    lms = partition_for_ranks(mesh, nranks, depth)
    for space, total in (("cells", mesh.num_cells), ("edges", mesh.num_edges),
                         ("verts", mesh.num_vertices)):
        owned = np.concatenate([lm.global_ids[space][:lm.sizes[space].owned_total] for lm in lms])
        assert sorted(owned.tolist()) == list(range(total)), space  # owners partition the space
    for lm in lms:
        for (space, nbr), table in lm.exchange_table.items():
            mirror = lms[nbr].exchange_table[(space, lm.rank)]
            np.testing.assert_array_equal(lm.global_ids[space][table[:, 0]],
                                          lms[nbr].global_ids[space][mirror[:, 0]])
        # local connectivity resolves locally
        assert lm.cells_to_vertices.max() < lm.sizes["verts"].total
        c2e = lm.cell_edges()
        assert c2e.max() < lm.sizes["edges"].total


def test_partition_rejects_bad_arguments():
    mesh = lt.generate_rect_mesh(2, 1)
    with pytest.raises(ValueError):
        partition_for_ranks(mesh, 0, 1)
    with pytest.raises(ValueError):
        partition_for_ranks(mesh, 2, 0)
    with pytest.raises(ValueError):
        partition_for_ranks(mesh, 5, 1)
