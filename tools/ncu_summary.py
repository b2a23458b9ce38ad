"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv, collections, io, sys
lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r['Kernel Name'].split('(')[0]
    v = float(r['Metric Value'].replace(',', ''))
    u = r['Metric Unit']
    v = v / 1000 if u in ('nsecond', 'ns') else v * 1000 if u in ('msecond', 'ms') else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':58s} {'count':>6s} {'total':>10s} {'share':>6s} {'avg':>10s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:58]:58s} {c:6d} {t/1e3:8.2f}ms {100*t/tot:5.1f}% {t/c:8.1f}us")
print(f"total {tot/1e3:.2f} ms over {len(rows)} launches")
