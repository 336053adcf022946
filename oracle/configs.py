"""Seeded coefficient-field / load generators for the BASELINE.json configs.

TEST / BENCH INFRASTRUCTURE.  The reference only accepts explicit
channel rectangles (`fem.py:106-120`, `generate_field` `fem.py:150-162`) and
constant/box/point sources (`fem.py:165-193`); these helpers turn the configs'
seeded descriptions into those rectangles and into per-cell source values that are
assembled with the reference's own corner rule (`assemble_load`, `fem.py:237-250`).

Pure NumPy; no reference import, so the descriptions are reproducible anywhere.
"""

from __future__ import annotations

import numpy as np

# name -> geometry / basis / time parameters (SURVEY §8 "Config sizes")
CONFIGS = {
    "cfg0": dict(nx=40, nb=4, layers=2, n_dom=2, n_comp=2, T=1.0, N=10, J=10,
                 kind="sequential", alpha=0.1),
    "cfg1": dict(nx=40, nb=4, layers=2, n_dom=2, n_comp=2, T=1.0, N=10, J=10,
                 kind="all-at-once", alpha=0.1),
    "cfg2": dict(nx=100, nb=10, layers=3, n_dom=3, n_comp=3, T=1.0, N=64, J=64,
                 kind="all-at-once", alpha=0.1),
    "cfg3": dict(nx=256, nb=32, layers=3, n_dom=4, n_comp=4, T=2.0, N=128, J=100,
                 kind="all-at-once", alpha=0.1),
    "cfg4": dict(nx=100, nb=10, layers=3, n_dom=3, n_comp=3, T=1.0, N=32, J=32,
                 kind="sequential", alpha=0.1, E=64),
}

R_STABILITY = 0.4      # coarse step Dt = 0.4 * explicit bound after kappa rescaling (F2)
STOP_REL_EPS = 1e-8    # relative-increment stop (F5)
FINE_TOL = 1e-12       # WR tolerance passed explicitly (F5)


def channel_rows(rng, nx, count):
    """Distinct horizontal channel rows in [1, nx-1), sorted (cfg0/cfg3/cfg4)."""
    return sorted(int(r) for r in rng.choice(np.arange(1, nx - 1), count, replace=False))


def place_inclusions(rng, nx, count, high):
    """`count` non-overlapping 2x2 cell squares, lower-left corner in [1, nx-2).

    `high` is an (nx, nx) bool cell mask (row = y) of cells already at high
    contrast; candidates touching any high cell are rejected.  Returns the
    list of (x0, y0) corners and updates `high` in place.
    """
    out = []
    tries = 0
    while len(out) < count:
        tries += 1
        if tries > 200 * count + 10000:
            raise RuntimeError("could not place inclusions")
        x0, y0 = (int(v) for v in rng.integers(1, nx - 2, 2))
        if high[y0:y0 + 2, x0:x0 + 2].any():
            continue
        high[y0:y0 + 2, x0:x0 + 2] = True
        out.append((x0, y0))
    return out


def rectangles(name, member=0):
    """Channel rectangles (x0, x1, y0, y1) in cell indices plus contrast.

    Returns (rects, contrast, source) where source is "constant" or
    ("gaussian", x, y, sigma).
    """
    c = CONFIGS[name]
    nx = c["nx"]
    high = np.zeros((nx, nx), dtype=bool)
    rects = []
    if name in ("cfg0", "cfg1"):
        rng = np.random.default_rng(0)
        for r in channel_rows(rng, nx, 8):
            rects.append((1, nx - 1, r, r + 1))
        return rects, 1e4, "constant"
    if name == "cfg2":
        rng = np.random.default_rng(0)
        n_inc = int(round(0.20 * nx * nx / 4))
        for x0, y0 in place_inclusions(rng, nx, n_inc, high):
            rects.append((x0, x0 + 2, y0, y0 + 2))
        return rects, 1e6, "constant"
    if name == "cfg3":
        rng = np.random.default_rng(0)
        for r in channel_rows(rng, nx, 32):
            rects.append((1, nx - 1, r, r + 1))
            high[r, 1:nx - 1] = True
        n_inc = int(round(0.15 * nx * nx / 4))
        for x0, y0 in place_inclusions(rng, nx, n_inc, high):
            rects.append((x0, x0 + 2, y0, y0 + 2))
        return rects, 1e4, ("gaussian", 0.3, 0.7, 0.05)
    if name == "cfg4":
        rng = np.random.default_rng(member)
        contrast = float(10.0 ** rng.uniform(2.0, 8.0))
        for r in channel_rows(rng, nx, 8):
            rects.append((1, nx - 1, r, r + 1))
            high[r, 1:nx - 1] = True
        n_inc = int(round(0.10 * nx * nx / 4))
        for x0, y0 in place_inclusions(rng, nx, n_inc, high):
            rects.append((x0, x0 + 2, y0, y0 + 2))
        return rects, contrast, "constant"
    raise KeyError(name)


def gaussian_cell_values(nx, x, y, sigma):
    """exp(-((cx-x)^2 + (cy-y)^2) / (2 sigma^2)) at cell centres, row-major cells."""
    h = 1.0 / nx
    cx = (np.arange(nx) + 0.5) * h
    xx, yy = np.meshgrid(cx, cx)
    return np.exp(-((xx - x) ** 2 + (yy - y) ** 2) / (2 * sigma ** 2)).ravel()


def corner_load(nx, f_cells):
    """Interior-node load by the assemble_load corner rule (fem.py:237-250)."""
    h = 1.0 / nx
    n1 = nx + 1
    b = np.zeros(n1 * n1)
    cells = np.arange(nx * nx)
    cx, cy = cells % nx, cells // nx
    n00 = cy * n1 + cx
    contrib = f_cells * h * h / 4.0
    for off in (0, 1, n1 + 1, n1):
        np.add.at(b, n00 + off, contrib)
    ix = np.arange(1, nx)
    interior = (ix[:, None] * n1 + ix[None, :]).ravel()
    return b[interior]


def kappa_field(name, member=0, background=1.0):
    """Cell-wise coefficient of a config (generate_field, fem.py:150-162): background
    everywhere, background * contrast on every channel / inclusion rectangle (half-open cell
    ranges, row-major cells)."""
    nx = CONFIGS[name]["nx"]
    rects, contrast, _ = rectangles(name, member)
    k = np.full((nx, nx), background)
    for x0, x1, y0, y1 in rects:
        k[y0:y1, x0:x1] = background * contrast
    return k.ravel()


Q1_STIFF = np.array([[4.0, -1.0, -2.0, -1.0], [-1.0, 4.0, -1.0, -2.0],
                     [-2.0, -1.0, 4.0, -1.0], [-1.0, -2.0, -1.0, 4.0]]) / 6.0
Q1_MASS = np.array([[4.0, 2.0, 1.0, 2.0], [2.0, 4.0, 2.0, 1.0],
                    [1.0, 2.0, 4.0, 2.0], [2.0, 1.0, 2.0, 4.0]]) / 36.0


def assemble_fine(nx, kappa):
    """Interior-node Q1 mass and stiffness (fem.py:196-206, 277-289): element matrices
    summed over cells (nodes SW, SE, NE, NW), symmetrised as (X + X^T) / 2, boundary rows
    and columns removed.  Returns scipy CSR (M, A)."""
    import scipy.sparse as sp

    n1 = nx + 1
    cells = np.arange(nx * nx)
    cx, cy = cells % nx, cells // nx
    n00 = cy * n1 + cx
    conn = np.stack([n00, n00 + 1, n00 + n1 + 1, n00 + n1], axis=1)
    rows = np.broadcast_to(conn[:, :, None], (nx * nx, 4, 4)).ravel()
    cols = np.broadcast_to(conn[:, None, :], (nx * nx, 4, 4)).ravel()

    def asm(data_cells, ref):
        data = (data_cells[:, None, None] * ref[None]).ravel()
        m = sp.coo_matrix((data, (rows, cols)), shape=(n1 * n1, n1 * n1)).tocsr()
        return (m + m.T) * 0.5

    h = 1.0 / nx
    full_m = asm(np.full(nx * nx, h * h), Q1_MASS)
    full_a = asm(np.asarray(kappa, dtype=float), Q1_STIFF)
    ix = np.arange(1, nx)
    idx = (ix[:, None] * n1 + ix[None, :]).ravel()
    return full_m[idx][:, idx].tocsr(), full_a[idx][:, idx].tocsr()
