"""profiles/ncu_traffic.json[key] = dram__bytes_read.sum + dram__bytes_write.sum of
the (first) kernel in an ncu report:  python tools/ncu_traffic_update.py KEY REPORT [SOURCE]"""
import csv
import io
import json
import subprocess
import sys

key, rep = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
tot = 0
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    tot += float(vals[hdr.index(name)].replace(",", ""))
path = "profiles/ncu_traffic.json"
d = json.load(open(path))
d[key] = int(tot)
d.setdefault("_sources", {})[key] = src
json.dump(d, open(path, "w"), indent=1)
print(key, int(tot))
