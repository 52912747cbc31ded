"""Render profiles/results_{gpu,cpu}.json (tools/results_table.py) as the
BASELINE.md §4 table (markdown on stdout)."""
import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    g = json.load(open(os.path.join(REPO, "profiles", "results_gpu.json")))
    c = json.load(open(os.path.join(REPO, "profiles", "results_cpu.json")))
    rows = ["| Config | GPUs | CF split (ms) GPU / CPU | Setup (ms) GPU / CPU | Solve DOFs/s GPU fast (exact) / CPU | "
            "Its GPU / CPU | SpMV % HBM | Weak-scaling eff. |",
            "|---|---|---|---|---|---|---|---|"]
    for k in sorted(g):
        a, b = g[k], c.get(k, {})
        note = "" if b.get("scale", 1.0) == 1.0 else f" (CPU at {b['n']:,} unknowns)"
        rows.append(f"| {k} ({a['n']:,}; {a['outer']}){note} | 1 | {a['cf_split_ms']:.2f} / {b.get('cf_split_ms', 0):.0f} "
                    f"| {a['setup_ms']:.0f} / {b.get('setup_ms', 0):.0f} | {a['dofs'] / 1e6:.1f} M "
                    f"({a.get('exact_dofs', 0) / 1e6:.1f} M) / "
                    f"{b.get('dofs', 0) / 1e6:.2f} M | {a['iterations']} / {b.get('iterations', '—')} "
                    f"| {100 * a['spmv_hbm_frac']:.0f} % | not measured (1 GPU) |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
