"""Tables from tools/mapping_ab.py output (JSON lines): the held-out model
table (B200 model pick vs Volta / Ampere picks vs the per-matrix grid
optimum) and the mapping A/B (row cuts vs SSR-aligned cuts vs the paper's
literal Listing 3 / 4 launch).

    python tools/ab_table.py profiles/r02_mapping_ab_*.jsonl
"""

from __future__ import annotations

import json
import sys


def load(paths):
    rows = []
    for p in paths:
        for line in open(p):
            if line.startswith("{"):
                rows.append(json.loads(line))
    return rows


def main(paths):
    rows = load(paths)
    seen = {}
    for r in rows:  # later files win (re-runs)
        seen[(r["config"], r["ssrs"], r["srs"], r["order"], r["nx"])] = r
    rows = list(seen.values())
    configs = sorted({r["config"] for r in rows})
    print("| Config | order | grid optimum (SSRS, SRS) ms | B200 model pick ms (x opt) |"
          " Volta pick ms (x opt) | Ampere pick ms (x opt) | points within 2 % of optimum |")
    print("|---|---|---|---|---|---|---|")
    for c in configs:
        rs = [r for r in rows if r["config"] == c and r["order_of"] == "b200"]
        if not rs:
            continue
        best = min(rs, key=lambda r: r["auto_ms"])
        t0 = best["auto_ms"]
        near = sum(1 for r in rs if r["auto_ms"] <= 1.02 * t0)

        def pick(name):
            p = [r for r in rs if name in r["picked_by"]]
            if not p:
                return "-"
            r = p[0]
            return f"({r['ssrs']}, {r['srs']}) {r['auto_ms']:.4f} ({r['auto_ms'] / t0:.3f})"
        order = best["order"] + (f" nx={best['nx']}" if best["order"] == "strided" else "")
        print(f"| {c} | {order} | ({best['ssrs']}, {best['srs']}) {t0:.4f} | {pick('b200')} |"
              f" {pick('volta')} | {pick('ampere')} | {near} / {len(rs)} |")
    print()
    print("| Config | pair (picked by) | row cuts ms | SSR-aligned cuts ms (tile) |"
          " paper Listing 3/4 ms (dims) | streaming / listing |")
    print("|---|---|---|---|---|---|")
    for c in configs:
        for r in sorted((r for r in rows if r["config"] == c and r["picked_by"]
                         and r["order_of"] == "b200"), key=lambda r: (r["ssrs"], r["srs"])):
            for name in r["picked_by"]:
                lm = r.get(f"listing_{name}_ms")
                ld = r.get(f"listing_{name}_dims")
                lo = r.get(f"listing_{name}_order")
                g = (f"{r['groups_ms']:.4f} ({r['groups_tile']})" if "groups_ms" in r
                     else "stage overflow")
                ratio = f"{lm / r['auto_ms']:.2f}x slower" if lm else "-"
                print(f"| {c} | ({r['ssrs']}, {r['srs']}) {name} | {r['rows_ms']:.4f} | {g} |"
                      f" {lm if lm else '-'} ({lo} {ld}) | {ratio} |")
    print()
    # SSR-aligned vs row cuts over every grid point where groups fit a stage
    print("| Config | grid points with SSR-aligned tiles fitting | aligned faster | "
          "median aligned / rows |")
    print("|---|---|---|---|")
    for c in configs:
        rs = [r for r in rows if r["config"] == c and r["order_of"] == "b200" and "groups_ms" in r
              and r["groups_ms"] < 3 * r["rows_ms"]]
        if not rs:
            continue
        ratios = sorted(r["groups_ms"] / r["rows_ms"] for r in rs)
        faster = sum(1 for x in ratios if x < 0.99)
        print(f"| {c} | {len(rs)} | {faster} | {ratios[len(ratios) // 2]:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
