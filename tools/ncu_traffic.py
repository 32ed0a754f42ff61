"""Sum an ncu launch list (--csv, metrics gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum)
over one bench step and record the DRAM traffic per step in profiles/r02/traffic.json under `key`
(bench.py's roofline.traffic reads it).

    python tools/ncu_traffic.py <ncu.csv> <key> <launches_per_step>

The ncu per-launch times are serialised and cold-cache; only the DRAM bytes and the kernels' share of the
step are used."""
import csv
import collections
import io
import json
import os
import sys

path, key, per_step = sys.argv[1], sys.argv[2], int(sys.argv[3])
txt = open(path).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
iid, ik, im, iv = (hdr.index(h) for h in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
d = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    d[int(r[iid])][r[im]] = v * scale
    names[int(r[iid])] = r[ik]
ids = sorted(d)[:per_step]
traffic = sum(d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0) for i in ids)
ns = sum(d[i].get("gpu__time_duration.sum", 0) for i in ids)
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02", "traffic.json")
t = json.load(open(out)) if os.path.exists(out) else {}
t[key] = round(traffic)
json.dump(t, open(out, "w"), indent=1, sort_keys=True)
kinds = collections.Counter(names[i].split("(")[0] for i in ids)
print(json.dumps({"key": key, "launches": len(ids), "traffic_bytes": round(traffic), "serialised_ms": round(ns / 1e6, 4),
                  "kernels": dict(kinds)}))
