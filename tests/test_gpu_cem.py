"""CEM-GMsFEM basis build on the GPU (msbasis.py:296-394) against the
reference's offline build.

* config 0: the basis columns themselves against the reference's Psi1 / Psi2
  (tests/golden/fine_cfg0.npz, written by oracle/make_fine_golden.py with the unmodified
  reference), and the projected CoarseSystem against sys_cfg0.npz;
* config 2: the projected CoarseSystem (GPU basis -> GPU projection) against the
  reference-built sys_cfg2.npz.
The fine operators come from the harness's Q1 assembly (oracle/configs.py), pinned to the
reference's in tests/test_oracle_pins.py.
"""

import json

import numpy as np
import pytest
import scipy.sparse as sp

from oracle.configs import CONFIGS, assemble_fine, kappa_field
from tests.conftest import golden

pytestmark = pytest.mark.gpu

BLOCKS = ("M11", "A11", "M12", "A12", "M22", "A22")


def _csr(z, prefix):
    return sp.csr_matrix((z[prefix + "_val"], z[prefix + "_idx"], z[prefix + "_ptr"]),
                         shape=tuple(z[prefix + "_shape"]))


def _space(name):
    import paper_2411_09244_b200 as P

    c = CONFIGS[name]
    return P.build_cem_space(c["nx"], c["nb"], c["layers"], kappa_field(name), c["n_dom"],
                             c["n_comp"])


def _compare_system(P, name, space, sysz, tol):
    c = CONFIGS[name]
    M, A = assemble_fine(c["nx"], kappa_field(name))
    scale = json.loads(str(sysz["meta"]))["kappa_scale"]
    ops = type("Ops", (), {})()
    ops.M, ops.A = M, A * scale
    cs = P.project_coarse(space.Psi1, space.Psi2, ops)
    for k in BLOCKS:
        g, r = getattr(cs, k), sysz[k]
        assert g.shape == r.shape, k
        assert np.abs(g - r).max() <= tol * np.abs(r).max(), (k, np.abs(g - r).max() / np.abs(r).max())


def test_cem_basis_config0_matches_reference_columns():
    import paper_2411_09244_b200 as P

    z = golden("fine_cfg0.npz")
    sp_ = _space("cfg0")
    assert sp_.constraint_residual <= 1e-8
    for mine, ref in ((sp_.Psi1, _csr(z, "P1")), (sp_.Psi2, _csr(z, "P2"))):
        assert mine.shape == ref.shape
        d = abs(mine - ref).max()
        assert d <= 1e-9 * abs(ref).max(), d
    _compare_system(P, "cfg0", sp_, golden("sys_cfg0.npz"), 1e-10)


def test_cem_basis_config2_projected_system_matches_reference():
    import paper_2411_09244_b200 as P

    sp_ = _space("cfg2")
    assert sp_.constraint_residual <= 1e-8
    assert sp_.Psi1.shape == (99 * 99, 300) and sp_.Psi2.shape == (99 * 99, 300)
    _compare_system(P, "cfg2", sp_, golden("sys_cfg2.npz"), 1e-9)


def test_cem_basis_rejects_bad_geometry():
    import paper_2411_09244_b200 as P

    with pytest.raises(ValueError):
        P.build_cem_space(40, 3, 2, np.ones(1600), 2, 2)
    with pytest.raises(ValueError):
        P.build_cem_space(40, 4, 2, np.ones(10), 2, 2)
    with pytest.raises(P.PeError):
        P.build_cem_space(40, 4, 2, -np.ones(1600), 2, 2)
