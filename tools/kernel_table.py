"""Per-kernel totals (time, DRAM bytes, GB/s) of an ncu --csv launch list
taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # e.g. repetitions in the run
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
seen = set()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r'(k_\w+)', r[ki])
    name = m.group(1) if m else r[ki][:40]
    agg[name][r[mi]] += float(r[vi].replace(',', ''))
    if r[idi] not in seen:
        seen.add(r[idi])
        cnt[name] += 1
print(f"{'kernel':24s} {'n':>5s} {'ms':>9s} {'GB rd':>8s} {'GB wr':>8s} {'GB/s':>8s}")
for k, d in sorted(agg.items(), key=lambda x: -x[1]['gpu__time_duration.sum']):
    t = d['gpu__time_duration.sum'] / 1e6 / div
    rd, wr = d['dram__bytes_read.sum'] / 1e9 / div, d['dram__bytes_write.sum'] / 1e9 / div
    print(f"{k:24s} {cnt[k] / div:5.0f} {t:9.3f} {rd:8.3f} {wr:8.3f} {(rd + wr) / t * 1e3 if t else 0:8.1f}")
