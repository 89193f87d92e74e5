"""Tabulate plan_sweep JSON lines: python tools/sweep_table.py FILE"""
import collections
import json
import sys

t = collections.defaultdict(dict)
text = open(sys.argv[1]).read()
recs = json.loads(text) if text.lstrip().startswith("[") else \
    [json.loads(line) for line in text.splitlines() if line.startswith("{")]
for r in recs:
    key = (r["config"], r["dtype"], r["variant"] + ("%d" % r["nx"] if r.get("nx") else ""),
           "G%d" % r["gather"], "C%d" % r.get("ctas", 0), "L%d" % r.get("layout", 2))
    t[key]["T%dS%d" % (r["tile_cost"], r["stages"])] = (r["gbs"], r["bitwise_equal"])
for k, v in t.items():
    print(" ".join(k), " ".join("%s:%.0f%s" % (a, b[0], "" if b[1] else "!") for a, b in v.items()))
