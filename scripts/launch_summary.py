"""Summarises an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, re, sys
def summarize(path, top=16):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", "")) * scale[r[ui]]
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = re.sub(r"<.*", "", name.split("(")[0]).replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"{path}: {sum(cnt.values())} launches, {T:.2f} ms total device time"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"  {k:52s} {v:10.3f} ms {100 * v / T:5.1f}%  n={cnt[k]}")
    return "\n".join(out)
if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))
