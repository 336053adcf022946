"""Auxiliary-eigenvalue golden vectors for the GPU CEM build (TEST INFRASTRUCTURE).

Runs the UNMODIFIED reference's `aux_eigen_cem` (msbasis.py:296-328) on every block of
configs 0 and 2 (the kappa fields of oracle/configs.py) and records the n_dom + n_comp
smallest eigenvalues per block.  Output: tests/golden/cem_aux.npz.
"""

import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from paradiff.fem import Channel, assemble_fine, build_fine_grid, generate_field  # noqa: E402
from paradiff.msbasis import aux_eigen_cem, build_coarse_partition  # noqa: E402

from oracle.configs import CONFIGS, rectangles  # noqa: E402


def main():
    out = {}
    for name in ("cfg0", "cfg2"):
        c = CONFIGS[name]
        rects, contrast, _ = rectangles(name)
        grid = build_fine_grid(c["nx"])
        fld = generate_field(grid, 1.0, contrast, [Channel(*r) for r in rects])
        ops = assemble_fine(grid, fld)
        part = build_coarse_partition(grid, c["nb"], c["layers"])
        ne = c["n_dom"] + c["n_comp"]
        out[f"{name}_eig"] = np.array([aux_eigen_cem(part, ops, fld, b, ne).eigenvalues
                                       for b in range(part.n_blocks)])
        print(name, out[f"{name}_eig"].shape)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cem_aux.npz"), **out)


if __name__ == "__main__":
    main()
