"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total time, share and launch count."""
import collections
import csv
import io
import sys


def summarise(path, top=25):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    t = collections.defaultdict(float)
    n = collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        t[k] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
        n[k] += 1
    tot = sum(t.values())
    out = [f"launches {sum(n.values())}  total kernel time {tot:.1f} us (serialised, cold-cache ncu replay)",
           f"{'us':>10} {'share':>6} {'count':>6}  kernel"]
    for k, v in sorted(t.items(), key=lambda x: -x[1])[:top]:
        out.append(f"{v:10.1f} {100 * v / tot:5.1f}% {n[k]:6d}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
