"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
bench's roofline kernels from an ncu launch list of one config-2 step:

  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py
  python tools/traffic_json.py gpurun_out/launches.csv > profiles/traffic_<config>.json
"""
import collections
import csv
import json
import sys

GROUPS = {"gemm": ("gemm_tc_kernel", "gemm_pair_kernel"), "attention": ("attn_tc_kernel", "attn_pp_kernel"),
          "gather_rope": ("gather_rope_kernel", "gather_rope_bulk_kernel")}

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[i], rows[i + 1:]
ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.defaultdict(dict)
for r in data:
    per[r[idi]]["name"] = r[ki]
    v = float(r[vi].replace(",", ""))
    if r[mi].startswith("dram__bytes"):
        v *= scale.get(r[ui], 1)
    per[r[idi]][r[mi]] = v
out = {"source": sys.argv[1].split("/")[-1], "how": __doc__.strip().splitlines()[0], "kernels": {}}
for g, pat in GROUPS.items():
    ls = [p for p in per.values() if any(x in p["name"] for x in pat)]
    if not ls:
        continue
    tot = sum(p.get("dram__bytes_read.sum", 0) + p.get("dram__bytes_write.sum", 0) for p in ls)
    out["kernels"][g] = {"launches": len(ls), "dram_bytes_per_launch": int(tot / len(ls)),
                         "us_per_launch": round(sum(p["gpu__time_duration.sum"] for p in ls) / len(ls) / 1e3, 2)}
print(json.dumps(out, indent=1))
