"""CEM-GMsFEM basis build on the GPU (msbasis.py:296-394) against the
reference's offline build.

A CEM basis is defined up to the choices its auxiliary eigenproblems leave open: the sign
of an eigenvector whose largest entries tie in magnitude (mirror-symmetric blocks), and the
basis of an eigenspace of a repeated eigenvalue (homogeneous blocks: the cos(pi x) /
cos(pi y) pair).  The reference resolves both by rounding (LAPACK's), any other
implementation by its own; the basis functions of a block then differ by an orthogonal
n_eig x n_eig transform, which parareal is equivariant to.  So the bar is:

* the auxiliary eigenvalues of every block against the reference's (1e-9);
* config 0: every block's n_eig columns against the reference's Psi (fine_cfg0.npz, from
  the unmodified reference) up to one orthogonal transform per block (1e-9), and the
  dominant / complementary split itself wherever the reference's eigenvalues n_dom - 1 and
  n_dom differ (config 0 has two blocks where they coincide exactly, 12 and 15);
* config 2 (no such block: smallest relative gap 0.039): the projected CoarseSystem's
  invariants under those transforms -- the generalized eigenvalues of (A11, M11) and
  (A22, M22), the mass and energy principal-angle cosines between the two subspaces, and
  the load norms f^T M^-1 f -- against the reference-built sys_cfg2.npz (5e-8: contrast
  1e6 makes both builds conditioning-limited; config 3 agrees to 1e-11,
  tools/cem_build_bench.py).
The fine operators come from the harness's Q1 assembly (oracle/configs.py), pinned to the
reference's in tests/test_oracle_pins.py.
"""

import json

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle.configs import CONFIGS, assemble_fine, corner_load, kappa_field
from tests.conftest import golden

pytestmark = pytest.mark.gpu


def _csr(z, prefix):
    return sp.csr_matrix((z[prefix + "_val"], z[prefix + "_idx"], z[prefix + "_ptr"]),
                         shape=tuple(z[prefix + "_shape"]))


def _space(name):
    import paper_2411_09244_b200 as P

    c = CONFIGS[name]
    return P.build_cem_space(c["nx"], c["nb"], c["layers"], kappa_field(name), c["n_dom"],
                             c["n_comp"])


def _procrustes_residual(ref, mine):
    """min over orthogonal Q of ||mine - ref Q|| / ||ref||, and Q."""
    u, _, vt = np.linalg.svd(ref.T @ mine)
    q = u @ vt
    return np.linalg.norm(mine - ref @ q) / np.linalg.norm(ref), q


def _invariants(s, f1, f2):
    """Quantities unchanged by orthogonal transforms within Psi1 and within Psi2."""
    out = {}
    out["eig11"] = np.sort(sla.eigh(s["A11"], s["M11"], eigvals_only=True))
    out["eig22"] = np.sort(sla.eigh(s["A22"], s["M22"], eigvals_only=True))
    for key, X11, X12, X22 in (("mass", s["M11"], s["M12"], s["M22"]),
                               ("energy", s["A11"], s["A12"], s["A22"])):
        l1 = np.linalg.cholesky(X11)
        l2 = np.linalg.cholesky(X22)
        c = sla.solve_triangular(l1, sla.solve_triangular(l2, X12.T, lower=True).T, lower=True)
        out[key] = np.linalg.svd(c, compute_uv=False)
    out["f1"] = np.array([f1 @ np.linalg.solve(s["M11"], f1)])
    out["f2"] = np.array([f2 @ np.linalg.solve(s["M22"], f2)])
    return out


def test_cem_aux_eigenvalues_match_reference():
    g = golden("cem_aux.npz")
    for name in ("cfg0", "cfg2"):
        sp_ = _space(name)
        ref = g[f"{name}_eig"]
        assert sp_.eigenvalues.shape == ref.shape
        assert np.abs(sp_.eigenvalues - ref).max() <= 1e-9 * np.abs(ref).max(), name
        assert sp_.constraint_residual <= 1e-8


def test_cem_basis_config0_matches_reference_columns():
    z = golden("fine_cfg0.npz")
    eig = golden("cem_aux.npz")["cfg0_eig"]
    c = CONFIGS["cfg0"]
    nd, nc = c["n_dom"], c["n_comp"]
    sp_ = _space("cfg0")
    r1, r2 = _csr(z, "P1").toarray(), _csr(z, "P2").toarray()
    m1, m2 = sp_.Psi1.toarray(), sp_.Psi2.toarray()
    assert m1.shape == r1.shape and m2.shape == r2.shape
    straddle = 0
    for b in range(c["nb"] ** 2):
        ref = np.hstack([r1[:, nd * b: nd * (b + 1)], r2[:, nc * b: nc * (b + 1)]])
        mine = np.hstack([m1[:, nd * b: nd * (b + 1)], m2[:, nc * b: nc * (b + 1)]])
        res, q = _procrustes_residual(ref, mine)
        assert res <= 1e-9, (b, res)
        if abs(eig[b, nd] - eig[b, nd - 1]) > 1e-6 * abs(eig[b, nd]):
            # a unique split: the transform does not mix dominant and complementary columns
            assert np.abs(q[:nd, nd:]).max() <= 1e-8 and np.abs(q[nd:, :nd]).max() <= 1e-8, b
        else:
            straddle += 1
    assert straddle == 2  # blocks 12 and 15 (repeated eigenvalue across the split)


def test_cem_basis_config2_projected_invariants_match_reference():
    import paper_2411_09244_b200 as P

    c = CONFIGS["cfg2"]
    sysz = golden("sys_cfg2.npz")
    scale = json.loads(str(sysz["meta"]))["kappa_scale"]
    sp_ = _space("cfg2")
    assert sp_.Psi1.shape == (99 * 99, 300) and sp_.Psi2.shape == (99 * 99, 300)
    kap = kappa_field("cfg2")
    M, A = assemble_fine(c["nx"], kap)
    ops = type("Ops", (), {})()
    ops.M, ops.A = M, A * scale
    cs = P.project_coarse(sp_.Psi1, sp_.Psi2, ops)
    f1, f2 = P.project_load(sp_, corner_load(c["nx"], np.ones(c["nx"] ** 2)))
    mine = _invariants({k: getattr(cs, k) for k in ("M11", "A11", "M12", "A12", "M22", "A22")},
                       f1, f2)
    ref = _invariants(sysz, sysz["f1"], sysz["f2"])
    # contrast 1e6: both builds are conditioning-limited at ~1e-9 (the reference's sparse LU
    # of the KKT system, libpe's refined Schur complement); measured 6e-9 on the pencil
    # eigenvalues, 1.1e-8 on the angles, 7e-11 on the loads (config 3, contrast 1e4: 1e-11)
    for k in ref:
        assert np.abs(mine[k] - ref[k]).max() <= 5e-8 * np.abs(ref[k]).max(), k


def test_cem_basis_rejects_bad_geometry():
    import paper_2411_09244_b200 as P

    with pytest.raises(ValueError):
        P.build_cem_space(40, 3, 2, np.ones(1600), 2, 2)
    with pytest.raises(ValueError):
        P.build_cem_space(40, 4, 2, np.ones(10), 2, 2)
    with pytest.raises(P.PeError):
        P.build_cem_space(40, 4, 2, -np.ones(1600), 2, 2)
