"""From an ncu launch-list csv, the ordinal (among launches whose name matches
`pattern`) of the longest launch whose name also contains `sub`: the -s value
for a follow-up `ncu -k regex:<pattern> -s <n> -c 1` capture."""
import csv, sys
path, pattern, sub = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
K, V = h.index("Kernel Name"), h.index("Metric Value")
M = h.index("Metric Name") if "Metric Name" in h else None
best, best_v, k = 0, -1.0, 0
for r in rows[hi + 1:]:
    if len(r) <= V or pattern not in r[K] or (M is not None and r[M] != "gpu__time_duration.sum"):
        continue
    v = float(r[V].replace(",", ""))
    if sub in r[K] and v > best_v:
        best, best_v = k, v
    k += 1
print(best)
