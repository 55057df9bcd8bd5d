"""From an ncu launch-list csv, the ordinal (among launches whose name matches
`pattern`) of the longest launch whose name also contains `sub`: the -s value
for a follow-up `ncu -k regex:<pattern> -s <n> -c 1` capture."""
import csv, sys
path, pattern, sub = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
K, V = h.index("Kernel Name"), h.index("Metric Value")
U = h.index("Metric Unit") if "Metric Unit" in h else None
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
M = h.index("Metric Name") if "Metric Name" in h else None
best, best_v, k = 0, -1.0, 0
for r in rows[hi + 1:]:
    if len(r) <= V or pattern not in r[K] or (M is not None and r[M] != "gpu__time_duration.sum"):
        continue
    v = float(r[V].replace(",", "")) * (SCALE.get(r[U], 1.0) if U is not None else 1.0)
    if sub in r[K] and v > best_v:
        best, best_v = k, v
    k += 1
print(best)
