"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes) by kernel."""
import collections, csv, re, sys

src, dst, title = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]
iK, iM, iV, iU, iID = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= iV:
        continue
    per[r[iID]][r[iM]] = (float(r[iV].replace(',', '')), r[iU])
    names[r[iID]] = r[iK]
T = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
B = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}


def key(k):
    m = re.search(r'igemm_kernel<\(int\)(\d), \(int\)(\d+), \(int\)(\d), \(bool\)(\d)(?:, \(bool\)(\d))?>', k)
    if m:
        return 'igemm<%s,BN=%s,stages=%s,x3=%s,tma=%s>' % (
            {'0': 'FWD', '1': 'DGRAD', '2': 'WGRAD', '3': 'TEST'}[m.group(1)],
            m.group(2), m.group(3), m.group(4), m.group(5) or '0')
    k = re.sub(r'\(.*', '', k)
    return k.replace('void ', '').replace('pooch::', '').replace('(anonymous namespace)::', '').replace('<unnamed>::', '')


agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for i, m in per.items():
    t, u = m['gpu__time_duration.sum']
    ms = t * T.get(u, 1e-6)
    b = sum(m[q][0] * B.get(m[q][1], 1) for q in ('dram__bytes_read.sum', 'dram__bytes_write.sum') if q in m)
    a = agg[key(names[i])]
    a[0] += 1
    a[1] += ms
    a[2] += b
    tot += ms
out = [title, "%-44s %6s %10s %7s %9s %8s" % ("kernel", "count", "ms", "share", "DRAM GB", "GB/s")]
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append("%-44s %6d %10.3f %6.1f%% %9.2f %8.0f" % (k, c, t, 100 * t / tot, b / 1e9, b / 1e9 / (t / 1e3) if t else 0))
out.append("total: %d launches, %.3f ms (serialised, cold cache)" % (sum(a[0] for a in agg.values()), tot))
open(dst, 'w').write("\n".join(out) + "\n")
print("\n".join(out))
