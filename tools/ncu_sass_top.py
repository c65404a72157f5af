"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv --print-source sass`
export (gzip ok), with the dominant stall reasons of each. Usage: python tools/ncu_sass_top.py f.csv.gz [N]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
lines = raw.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
agg = {}
for c in stall_cols:
    agg[c] = sum(float(r[c] or 0) for r in rows)
print("total samples %d; by reason: %s" % (tot, ", ".join("%s %.1f%%" % (k[6:], 100 * v / tot)
                                                          for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8])))
rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
for r in rows[:n]:
    s = float(r["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((float(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print("%5.1f%%  %-6s %-60s %s" % (100 * s / tot, r["Address"], r["Source"][:60], " ".join("%s:%.0f" % (b, a) for a, b in top)))
