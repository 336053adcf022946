"""Compact on-disk form of a `CoarseSystem` (+ loads): what the offline build hands over.

The reduced operators of the larger configs are mostly structural zeros (a CEM basis
function lives on its oversampled patch, so two columns couple only when their patches
overlap: 13 % of the entries at config 3) and the diagonal blocks are symmetric (the
reference symmetrises them, msbasis.py:560-566).  A block is stored as

* a bit mask of its nonzero entries (the upper triangle only for an exactly symmetric
  block), and
* the nonzero values in row-major order, byte-shuffled (the eight bytes of every double
  grouped by significance, so exponents and leading mantissa bytes sit together) and
  zlib-compressed.

Decoding is exact (bitwise), so a packed system reproduces the reference's operators
bit for bit.  Pure NumPy/zlib host code, no GPU; used to ship the reference-built
operators of configs 3 and 4 with the repository (`data/`).
"""

from __future__ import annotations

import json
import os
import zlib

import numpy as np

BLOCKS = ("M11", "A11", "M12", "A12", "M22", "A22")
FORMAT = "pesys-1"


def _shuffle(v: np.ndarray) -> bytes:
    b = np.ascontiguousarray(v, dtype="<f8").view(np.uint8).reshape(-1, 8)
    return zlib.compress(np.ascontiguousarray(b.T).tobytes(), 9)


def _unshuffle(blob: bytes, count: int) -> np.ndarray:
    raw = np.frombuffer(zlib.decompress(blob), dtype=np.uint8)
    if raw.size != 8 * count:
        raise ValueError("packed block is corrupt (value count mismatch)")
    return np.ascontiguousarray(raw.reshape(8, count).T).view("<f8").reshape(count)


def pack_block(X: np.ndarray) -> dict:
    """Arrays describing one dense block (see the module docstring)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    r, c = X.shape
    sym = r == c and r > 0 and np.array_equal(X, X.T)
    mask = X != 0.0
    if sym:
        mask &= np.triu(np.ones((r, c), dtype=bool))
    vals = X[mask]
    return {"shape": np.array([r, c], dtype=np.int64), "sym": np.array(int(sym)),
            "mask": np.frombuffer(zlib.compress(np.packbits(mask.ravel()).tobytes(), 9),
                                  dtype=np.uint8),
            "vals": np.frombuffer(_shuffle(vals), dtype=np.uint8),
            "nnz": np.array(vals.size, dtype=np.int64)}


def unpack_block(z, prefix: str = "") -> np.ndarray:
    r, c = (int(v) for v in z[prefix + "shape"])
    nnz = int(z[prefix + "nnz"])
    bits = np.frombuffer(zlib.decompress(z[prefix + "mask"].tobytes()), dtype=np.uint8)
    mask = np.unpackbits(bits, count=r * c).astype(bool).reshape(r, c)
    X = np.zeros((r, c))
    X[mask] = _unshuffle(z[prefix + "vals"].tobytes(), nnz)
    if int(z[prefix + "sym"]):
        iu = np.triu_indices(r, 1)
        X[iu[1], iu[0]] = X[iu]
    return X


def save_system(path: str, blocks: dict, f1, f2, meta: dict | None = None,
                split: bool = False) -> list:
    """Write a packed system.  `split=False`: one file `path` (.npz).  `split=True`: a
    directory `path` holding one file per block plus `loads.npz` (keeps every file small
    enough for any repository host).  Returns the written paths."""
    out = []
    loads = {"f1": np.asarray(f1, dtype=np.float64), "f2": np.asarray(f2, dtype=np.float64),
             "meta": np.array(json.dumps(meta or {})), "format": np.array(FORMAT)}
    if split:
        os.makedirs(path, exist_ok=True)
        for k in BLOCKS:
            p = os.path.join(path, f"{k}.npz")
            np.savez(p, **pack_block(blocks[k]))
            out.append(p)
        p = os.path.join(path, "loads.npz")
        np.savez(p, **loads)
        out.append(p)
        return out
    arrs = dict(loads)
    for k in BLOCKS:
        for n, a in pack_block(blocks[k]).items():
            arrs[f"{k}.{n}"] = a
    np.savez(path, **arrs)
    return [path]


def load_system(path: str):
    """(blocks dict, f1, f2, meta) from `save_system` output (file or directory)."""
    if os.path.isdir(path):
        blocks = {}
        for k in BLOCKS:
            with np.load(os.path.join(path, f"{k}.npz")) as z:
                blocks[k] = unpack_block(z)
        with np.load(os.path.join(path, "loads.npz")) as z:
            return blocks, z["f1"].copy(), z["f2"].copy(), json.loads(str(z["meta"]))
    with np.load(path) as z:
        if str(z["format"]) != FORMAT:
            raise ValueError(f"{path}: unknown format {z['format']!r}")
        blocks = {k: unpack_block(z, k + ".") for k in BLOCKS}
        return blocks, z["f1"].copy(), z["f2"].copy(), json.loads(str(z["meta"]))
