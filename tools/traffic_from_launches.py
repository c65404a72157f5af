"""profiles/ncu_traffic.json from an ncu launch list of one bench step (gpu__time_duration,
dram__bytes_read, dram__bytes_write per launch): per kernel family (conv_fwd / conv_dgrad /
conv_wgrad = the tensor-core kernel in mode 0 / 1 / 2), the DRAM bytes per launch -- the
`traffic` field of bench.py's roofline (bench.py uses an entry only for the workload it names).
Usage: python tools/traffic_from_launches.py list.csv out.json [workload, default cfg3]"""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
iK, iM, iV, iU, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) > iV:
        per[r[iID]][r[iM]] = float(r[iV].replace(",", "")) * B.get(r[iU], 1)
        names[r[iID]] = r[iK]
fam = collections.defaultdict(list)
for i, m in per.items():
    mm = re.search(r"igemm_kernel<(?:\(int\))?(\d)", names[i])
    if not mm:
        continue
    f = {"0": "conv_fwd", "1": "conv_dgrad", "2": "conv_wgrad"}.get(mm.group(1))
    if f:
        fam[f].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
wl = sys.argv[3] if len(sys.argv) > 3 else "cfg3"
out = {f: {"launches": len(v), "dram_bytes_per_launch": sum(v) / len(v),
           "source": "ncu launch list of one %s step (%s)" % (wl, sys.argv[1]), "workload": wl} for f, v in fam.items()}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
