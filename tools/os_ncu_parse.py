"""Print the mean gpu__time_duration (us) per kernel name of an ncu --csv log."""
import csv, sys, collections
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith('=='))]
h = rows[0]; ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] == 'gpu__time_duration.sum':
        d[r[ki].split('(')[0]].append(float(r[vi].replace(',', '')) / 1e3)
for k, v in d.items():
    print(f"{k:45s} n={len(v)} mean={sum(v)/len(v):.2f} us")
