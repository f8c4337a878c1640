"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel and grid."""
import collections
import csv
import sys


def summarise(path, top=30):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]
        key = (name, r["Grid Size"], r["Block Size"])
        v = float(r["Metric Value"]) / 1e3
        agg[key][0] += 1
        agg[key][1] += v
        tot += v
    out = [f"# {path}: {sum(a[0] for a in agg.values())} launches, {tot:.1f} us total (cold-cache, serialised)",
           "# share    total_us   launches  avg_us   kernel grid block"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{t / tot * 100:6.2f}% {t:11.1f} {n:9d} {t / n:8.2f}   {k[0]} {k[1]} {k[2]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
