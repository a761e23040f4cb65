"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel."""
import csv, collections, json, sys
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]
ki, mi, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
SC = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1, 'msecond': 1, 's': 1e3, 'second': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].split('(')[0].replace('void ', '').split('<')[0][:60]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', '')) * SC[r[ui]]
tot = sum(v[1] for v in agg.values())
out = [{"kernel": k, "launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
       for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
for o in out[:16]:
    print(o)
if len(sys.argv) > 2:
    json.dump({"source": path, "total_ms": tot, "kernels": out}, open(sys.argv[2], "w"), indent=1)
