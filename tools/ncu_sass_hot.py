"""Hottest SASS instructions of an `ncu --page source --csv --print-source sass` export (by warp
stall samples and by executed count), with the code around them. Usage: ncu_sass_hot.py file.csv.gz [n]"""
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
H = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[H[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0


S, NI, EX = "Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed"
tot = sum(f(r, S) for r in data) or 1.0
print("total stall samples %.0f, instructions executed %.0f" % (tot, sum(f(r, EX) for r in data)))
idx = sorted(range(len(data)), key=lambda i: -f(data[i], S))[:n]
for i in idx:
    r = data[i]
    print("%6.0f %5.1f%% %10.0f  [%5d] %s" % (f(r, S), 100 * f(r, S) / tot, f(r, EX), i, r[H["Source"]].strip()[:100]))
