"""Turn the ncu outputs of tools/gpu_profile.sh (gpurun_out/) into the
committed summaries under profiles/:
  profiles/<tag>_solve_launches.txt   per-kernel share of one solve step
  profiles/<tag>_spmv_ncu.txt         --set full key metrics, level-0 SpMV
  profiles/<tag>_fres1_ncu.txt        --set full key metrics, level-4 F residual
  profiles/dram_bytes.json            DRAM bytes per step / per SpMV (bench traffic)
"""
import collections
import csv
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from ncu_summary import summary  # noqa: E402

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    by = collections.OrderedDict()
    for r in rows:
        d = by.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", ""),
                                    "grid": r["Grid Size"]})
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v * SCALE[u]
        elif r["Metric Name"].startswith("dram__bytes"):
            d["dram"] = d.get("dram", 0.0) + v * BYTES.get(u, 1)
    return list(by.values())


def main(tag="r1"):
    out = os.path.join(REPO, "gpurun_out")
    prof = os.path.join(REPO, "profiles")
    L = launches(os.path.join(out, f"{tag}_solve_launches.csv"))
    t = collections.defaultdict(float)
    b = collections.defaultdict(float)
    n = collections.Counter()
    for d in L:
        t[d["name"]] += d.get("us", 0.0)
        b[d["name"]] += d.get("dram", 0.0)
        n[d["name"]] += 1
    tot = sum(t.values())
    totb = sum(b.values())
    lines = [f"ncu launch list of one C2 solve (tools/profile_solve.py --what solve): {len(L)} launches,",
             f"serialised cold-cache kernel time {tot:.1f} us, DRAM bytes {totb / 1e6:.1f} MB",
             "(ncu flushes caches before every kernel: bytes are an upper bound of the warm step)",
             f"{'us':>10} {'share':>6} {'count':>6} {'DRAM MB':>9}  kernel"]
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        lines.append(f"{v:10.1f} {100 * v / tot:5.1f}% {n[k]:6d} {b[k] / 1e6:9.1f}  {k}")
    open(os.path.join(prof, f"{tag}_solve_launches.txt"), "w").write("\n".join(lines) + "\n")
    res = {"solve_dram_bytes_per_step": totb, "solve_kernel_us_serialised": tot, "launches": len(L)}
    for what in ("spmv", "fres1"):
        rep = os.path.join(out, f"{tag}_{what}_full.ncu-rep")
        if os.path.exists(rep):
            s = summary(rep)
            open(os.path.join(prof, f"{tag}_{what}_ncu.txt"), "w").write(s + "\n")
            if what == "spmv":
                rd = wr = 0.0
                for line in s.splitlines():
                    f = line.split()
                    if f and f[0] in ("dram_rd", "dram_wr"):
                        val = float(f[1]) * BYTES.get(f[2], 1)
                        rd, wr = (val, wr) if f[0] == "dram_rd" else (rd, val)
                res["spmv_dram_bytes_per_launch"] = rd + wr
    # CF split of all C2 levels (tools/ncu_cf.py): launch list + level-3 captures
    cfl = os.path.join(out, f"{tag}_cf_launches.csv")
    if os.path.exists(cfl):
        L = launches(cfl)
        t = collections.defaultdict(float)
        b = collections.defaultdict(float)
        n = collections.Counter()
        for d in L:
            t[d["name"]] += d.get("us", 0.0)
            b[d["name"]] += d.get("dram", 0.0)
            n[d["name"]] += 1
        tot, totb = sum(t.values()), sum(b.values())
        lines = [f"ncu launch list of one batched CF split of all C2 levels (tools/ncu_cf.py): {len(L)} launches,",
                 f"serialised cold-cache kernel time {tot:.1f} us, DRAM bytes {totb / 1e6:.1f} MB",
                 f"{'us':>10} {'share':>6} {'count':>6} {'DRAM MB':>9}  kernel"]
        for k, v in sorted(t.items(), key=lambda x: -x[1]):
            lines.append(f"{v:10.1f} {100 * v / tot:5.1f}% {n[k]:6d} {b[k] / 1e6:9.1f}  {k}")
        rep = os.path.join(out, f"{tag}_cf_l3.ncu-rep")
        if os.path.exists(rep):
            lines += ["", "--set full of the three row passes at level 3 (n = 947,182, nnz = 16,719,437):",
                      summary(rep)]
        open(os.path.join(prof, f"{tag}_cf_ncu.txt"), "w").write("\n".join(lines) + "\n")
        res["cf_split_dram_bytes_all_levels"] = totb
    json.dump(res, open(os.path.join(prof, "dram_bytes.json"), "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:])
