"""Deterministic Matrix Market inputs for the ingest golden fixtures (test
infrastructure).  ``make_golden.py mm`` reads every case with the
UNMODIFIED reference (io.py:96-206 read_matrix_market, 209-230
write_matrix_market, 278-299 permutation files) and stores digests in
``mm.json``; tests/test_io_cli.py reads the same texts with this repo's
ingest (native body parser, host or device canonicalisation) and compares.

Sizes: the small cases stay below the native-parser threshold (16 K
entries), the large ones pass it and, after symmetric expansion, the
device COO -> CSR threshold (64 K triplets)."""

from __future__ import annotations

import numpy as np

CASES = {
    # name: (field, symmetry, n, entries, seed)
    "real_general_small": ("real", "general", 300, 2000, 1),
    "integer_symmetric_small": ("integer", "symmetric", 200, 1500, 2),
    "pattern_general_small": ("pattern", "general", 250, 1800, 3),
    "real_skew_small": ("real", "skew-symmetric", 220, 1600, 4),
    "real_general_large": ("real", "general", 20000, 90000, 5),
    "real_symmetric_large": ("real", "symmetric", 30000, 70000, 6),
    "pattern_symmetric_large": ("pattern", "symmetric", 25000, 60000, 7),
    "integer_general_dups_large": ("integer", "general", 5000, 80000, 8),
}


def mm_text(name: str) -> str:
    """The Matrix Market text of a case: random coordinates (duplicates
    included, summed by the reader), values spanning 60 decades, comments,
    blank lines and irregular spacing."""
    field, symmetry, n, m, seed = CASES[name]
    rng = np.random.default_rng(seed)
    r = rng.integers(1, n + 1, m)
    c = rng.integers(1, n + 1, m)
    if symmetry != "general":  # lower triangle only, no diagonal for skew
        lo, hi = np.minimum(r, c), np.maximum(r, c)
        r, c = hi, lo
        if symmetry == "skew-symmetric":
            keep = r != c
            r, c = r[keep], c[keep]
    m = len(r)
    if field == "integer":
        v = rng.integers(-9, 10, m)
    else:
        v = rng.standard_normal(m) * 10.0 ** rng.uniform(-30, 30, m)
    lines = [f"%%MatrixMarket matrix coordinate {field} {symmetry}", "% generated",
             f"{n} {n} {m}"]
    for k in range(m):
        if field == "pattern":
            e = f"{r[k]} {c[k]}"
        elif field == "integer":
            e = f"{r[k]} {c[k]} {int(v[k])}"
        else:
            e = f"{r[k]} {c[k]} {float(v[k])!r}"
        if k % 11 == 0:
            e = "  " + e.replace(" ", "\t", 1) + "  "
        lines.append(e)
        if k == 17:
            lines.append("% a comment inside the body")
        if k == 40:
            lines.append("")
    return "\n".join(lines) + "\n"


def perm_of(n: int, seed: int = 0) -> np.ndarray:
    """A fixed permutation (forward map) for the permutation-file check."""
    return np.random.default_rng(seed).permutation(n).astype(np.int64)
