"""Per-launch DRAM traffic of the rotation write pass from an ncu csv
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
over one factorization): writes profiles/merge_traffic_r01.json."""
import collections, csv, json, sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def is_write(name):
    if "k_merge2" in name:
        return any(t in name for t in ("k_merge2<1", "k_merge2<(bool)1", "k_merge2<true"))
    return "k_merge_p" in name and any(t in name for t in ("(bool)1", ", 1>", ", true>"))


def main(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ID, K, M, U, V = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= V:
            continue
        per[r[ID]][r[M]] = float(r[V].replace(",", "")) * UNITS.get(r[U], 1.0)
        names[r[ID]] = r[K]
    w = [per[i] for i in per if is_write(names[i])]
    tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in w)
    ms = sum(d.get("gpu__time_duration.sum", 0) for d in w)
    res = {"kernel": "k_merge2<true> (k = 2 rotation stream, write pass)", "launches": len(w),
           "dram_bytes_total": tot, "dram_bytes_per_launch": tot / max(len(w), 1), "kernel_ms_total_ncu": ms,
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     f"--clock-control none over every write-pass launch of one config-4 factorization ({path})"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/merge_traffic_r01.json")
