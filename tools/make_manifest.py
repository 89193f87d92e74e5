"""Write paper_2203_05096_b200/data/manifest.csv -- the paper's benchmark
suite (PAPER.md Table "Benchmark suite", tab:testsuite: 35 regular and 29
irregular SuiteSparse matrices) in the loader's CSV schema
``id,name,n,nnz,max,class`` (reference io.py:237-275).

Run in the build container (PAPER.md is read from /root/reference):
    python tools/make_manifest.py
The table truncates five SuiteSparse names; they are completed from the
SuiteSparse collection's own names below.  MAX values written as 1.2K /
2.3M in the table become integers."""

from __future__ import annotations

import os
import re
import sys

PAPER = "/root/reference/PAPER.md"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2203_05096_b200", "data", "manifest.csv")
FULL_NAMES = {  # table truncations -> SuiteSparse names
    "packing...": "packing-500x100x100-b050",
    "wikipedia-2005110": "wikipedia-20051105",
    "wikipedia-2006092": "wikipedia-20060925",
    "wikipedia-2006110": "wikipedia-20061104",
    "wikipedia-2007020": "wikipedia-20070206",
}


def count(text: str) -> int:
    m = re.fullmatch(r"([0-9.]+)([kKM]?)", text.strip())
    if not m:
        raise ValueError(f"bad MAX entry {text!r}")
    scale = {"": 1, "k": 1000, "K": 1000, "M": 1000000}[m.group(2)]
    return int(round(float(m.group(1)) * scale))


def main() -> None:
    rows = []
    for line in open(PAPER, encoding="utf-8"):
        m = re.match(r"^([ri]\d+)\s*&", line)
        if not m or line.count("&") != 6:
            continue
        cells = [c.strip() for c in line.split("\\\\")[0].split("&")]
        mid, _sy, name, n, nnz, mx, _r = cells
        name = name.replace("\\_", "_")
        name = FULL_NAMES.get(name, name)
        cls = "regular" if mid.startswith("r") else "irregular"
        rows.append(f"{mid},{name},{n},{nnz},{count(mx)},{cls}")
    if len(rows) != 64:
        raise SystemExit(f"expected 64 table rows, parsed {len(rows)}")
    with open(OUT, "w", encoding="ascii") as fh:
        fh.write("id,name,n,nnz,max,class\n")
        fh.write("\n".join(rows) + "\n")
    print(f"wrote {OUT} ({len(rows)} matrices)")


if __name__ == "__main__":
    sys.exit(main())
