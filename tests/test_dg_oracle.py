"""Elastic-wave DG: tables, oracle vs reference-executor goldens (CPU only)."""

import numpy as np
import pytest

from conftest import golden_npz, golden_schedule_text, golden_schedules, parse_case
from cases import build_case, dg_setup

from paper_1708_03183_b200.dg import dg_tables, n_dofs, triangle_quadrature
from oracle import looptile_oracle as O

DG_CASES = sorted(c for c in golden_schedules()["schedules"] if c.startswith("dg"))


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_tables_orthonormal_and_exact(p):
    t = dg_tables(p)
    r, s, w = triangle_quadrature(p + 4)
    psi, dr, ds = t.basis(r, s)
    np.testing.assert_allclose(psi.T @ (w[:, None] * psi), np.eye(n_dofs(p)), atol=1e-12)
    # integration by parts on the reference triangle: S_r + S_r^T = boundary term
    assert t.Sr.shape == (n_dofs(p), n_dofs(p))
    # constants are annihilated by the derivative matrices
    const = np.linalg.lstsq(psi, np.ones_like(r), rcond=None)[0]
    np.testing.assert_allclose(t.Sr @ const, 0, atol=1e-12)
    np.testing.assert_allclose(t.Ss @ const, 0, atol=1e-12)
    # face traces of the constant are the constant
    for f in range(3):
        np.testing.assert_allclose(t.E[f] @ const, 1.0, atol=1e-12)


@pytest.mark.parametrize("case", DG_CASES)
def test_oracle_dg_schedule_matches_reference(case):
    prob, dims, ren, ts, mode = parse_case(case)
    _, (chain, _, _, _) = build_case(prob, dims, ren)
    assert O.inspect(chain, ts, mode).serialize() == golden_schedule_text(case)


@pytest.mark.parametrize("tag", sorted({c.rsplit("_", 2)[0] for c in DG_CASES}))
def test_oracle_dg_untiled_matches_reference_executor(tag):
    st, chain = dg_setup(tag)
    data = {n: v.copy() for n, v in st.data.items()}
    O.execute_untiled(chain, st.bindings, data, st.vpe, O.kernel_table(dg=(st.p, st.dt)))
    ref = golden_npz("values.npz")
    for n in ("u", "s", "ru", "rs"):
        np.testing.assert_array_equal(data[n], ref[f"{tag}/untiled/{n}"], err_msg=n)


@pytest.mark.parametrize("case", DG_CASES)
def test_oracle_dg_tiled_matches_reference_executor(case):
    tag = case.rsplit("_", 2)[0]
    st, chain = dg_setup(tag)
    _, _, _, ts, mode = parse_case(case)
    data = {n: v.copy() for n, v in st.data.items()}
    s = O.inspect(chain, ts, mode)
    O.execute_tiled(s, chain, st.bindings, data, st.vpe, O.kernel_table(dg=(st.p, st.dt)))
    ref = golden_npz("values.npz")
    for n in ("u", "s", "ru", "rs"):
        np.testing.assert_array_equal(data[n], ref[f"{case}/tiled/{n}"], err_msg=n)


def test_dg_pulse_propagates_and_stays_bounded():
    st, chain = dg_setup("dg1s1_8x6_none")
    data = {n: v.copy() for n, v in st.data.items()}
    k = O.kernel_table(dg=(st.p, st.dt))
    e0 = np.sum(data["u"] ** 2) + np.sum(data["s"] ** 2)
    for _ in range(3):
        O.execute_untiled(chain, st.bindings, data, st.vpe, k)
    e1 = np.sum(data["u"] ** 2) + np.sum(data["s"] ** 2)
    assert np.isfinite(e1) and 0.5 * e0 < e1 < 1.5 * e0
