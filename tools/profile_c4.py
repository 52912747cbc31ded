"""Summaries of tools/gpu_profile_r2.sh (gpurun_out/) into profiles/:
r2_c4_solve_launches.txt (per-kernel share + DRAM bytes of one C4 solve),
r2_c4_cf_launches.txt (all-level CF split), r2_<name>_ncu.txt (--set full
key metrics) and the C4 entry of profiles/dram_bytes.json (bench traffic)."""
import collections
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from make_profiles import launches  # noqa: E402
from ncu_summary import summary  # noqa: E402

OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")


def table(L, head):
    t, b, n = collections.defaultdict(float), collections.defaultdict(float), collections.Counter()
    for d in L:
        t[d["name"]] += d.get("us", 0.0)
        b[d["name"]] += d.get("dram", 0.0)
        n[d["name"]] += 1
    tot, totb = sum(t.values()), sum(b.values())
    lines = head + [f"launches {len(L)}  serialised cold-cache kernel time {tot:.1f} us  DRAM bytes {totb:.4e}",
                    f"{'us':>10} {'share':>6} {'count':>6} {'DRAM MB':>10}  kernel"]
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        lines.append(f"{v:10.1f} {100 * v / tot:5.1f}% {n[k]:6d} {b[k] / 1e6:10.1f}  {k}")
    return lines, tot, totb


def main():
    res = json.load(open(os.path.join(PROF, "dram_bytes.json")))
    c4 = {}
    L = launches(os.path.join(OUT, "r2_c4_solve_launches.csv"))
    lines, tot, totb = table(L, [
        "ncu launch list of ONE C4 solve in the bench's configuration (fast mode: one-pass ascent on the",
        "levels fused.cu picks, composed coarse solve, device GMRES(30) with the Gram-corrected CGS2 over the",
        "unnormalised basis; kernels launched one by one: AIRG_GM_FLAT=1 -- the timed bench runs the same",
        "kernels inside one nested conditional graph). tools/gpu_profile_r2.sh: ncu --metrics",
        "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none.",
        "Times are cold-cache and serialised: compare SHARES with the bench step."])
    open(os.path.join(PROF, "r2_c4_solve_launches.txt"), "w").write("\n".join(lines) + "\n")
    c4.update(solve_dram_bytes_per_step=totb, solve_kernel_us_serialised=tot, launches=len(L))
    sp = os.path.join(OUT, "r2_c4_spmv.csv")
    if os.path.exists(sp):
        S = launches(sp)
        if S:
            c4["spmv_dram_bytes_per_launch"] = sum(d.get("dram", 0.0) for d in S) / len(S)
    cf = os.path.join(OUT, "r2_c4_cf.csv")
    if os.path.exists(cf):
        C = launches(cf)
        lines, _, cb = table(C, ["ncu launch list of one batched CF split of all C4 levels (tools/ncu_cf.py,",
                                 "CF_CONFIG=4), cold-cache serialised"])
        open(os.path.join(PROF, "r2_c4_cf_launches.txt"), "w").write("\n".join(lines) + "\n")
        c4["cf_split_dram_bytes_all_levels"] = cb
    for name in ("desc0", "fusedx0", "fusedx4", "sweep"):
        rep = os.path.join(OUT, f"r2_{name}_full.ncu-rep")
        if os.path.exists(rep):
            open(os.path.join(PROF, f"r2_{name}_ncu.txt"), "w").write(
                f"ncu --set full --clock-control none --import-source on (tools/gpu_profile_r2.sh): {name}\n"
                + summary(rep) + "\n")
    c4["note"] = "round 2 (final): fast mode, one-pass ascent, composed coarse solve, lazy GMRES basis"
    res["C4"] = c4
    json.dump(res, open(os.path.join(PROF, "dram_bytes.json"), "w"), indent=1)
    print(json.dumps(c4))


if __name__ == "__main__":
    main()
