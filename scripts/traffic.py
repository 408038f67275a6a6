"""Per-launch DRAM traffic of the step's kernels from an ncu CSV (NVTX-renamed launches):
    python scripts/traffic.py gpurun_out/X_traffic.csv CONFIG_NAME CAPTURE_LABEL
updates profiles/roofline_traffic.json: "<config>:<kernel>" -> {"bytes": median per launch of
dram__bytes_read.sum + dram__bytes_write.sum, "us": median gpu__time_duration, "capture": label}."""
import collections
import csv
import json
import os
import statistics
import sys

path, cfg, label = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.defaultdict(dict)
for r in rows[1:]:
    try:
        per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
agg = collections.defaultdict(lambda: {"bytes": [], "us": []})
for (_, name), m in per.items():
    name = name.split("/")[0].strip() if "/" in name.split("(")[0] else name.strip()
    if "dram__bytes_read.sum" not in m:
        continue
    agg[name]["bytes"].append(m["dram__bytes_read.sum"] + m.get("dram__bytes_write.sum", 0.0))
    agg[name]["us"].append(m.get("gpu__time_duration.sum", 0.0) / 1e3)
out_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "roofline_traffic.json")
tj = json.load(open(out_p)) if os.path.exists(out_p) else {}
for name, v in sorted(agg.items()):
    tj[f"{cfg}:{name}"] = {"bytes": statistics.median(v["bytes"]), "us": statistics.median(v["us"]),
                           "launches": len(v["bytes"]), "capture": label}
    print(f"{name:28s} {statistics.median(v['bytes']) / 1e6:9.2f} MB  {statistics.median(v['us']):8.2f} us  n={len(v['bytes'])}")
json.dump(tj, open(out_p, "w"), indent=1, sort_keys=True)
