"""Run reports in the reference's schema (reports.cpp:18-133):
the GPU hierarchy's hierarchy_report, csv_header and csv_row equal the
reference's own (oracle/_ref, same hierarchy through coefficient injection)."""
import glob
import json
import os

import numpy as np
import pytest

import refpy
from paper_2408_08262_b200 import airg, reports

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.fixture(scope="module")
def ref():
    r = refpy.ref()
    if r is None:
        pytest.skip("reference build (oracle/_ref) not available")
    return r


def _injection(oh, prm):
    info = oh.info()
    return {"levels": [(list(oh.level(l).coefficients[: prm["poly_order"] + 1]), oh.level(l).effective_order)
                       for l in range(info.n_levels)],
            "coarse": (list(info.coarse_coefficients[: prm["coarse_poly_order"] + 1]),
                       info.coarse_effective_order)}


@pytest.mark.parametrize("path", GOLDEN[:4], ids=lambda p: os.path.basename(p)[:-4])
def test_reports_match_reference(ref, path, tmp_path):
    g = np.load(path)
    prm = dict(eval(str(g["params"][0])))
    prm.setdefault("poly_order", 6)
    prm.setdefault("coarse_poly_order", 12)
    n = len(g["rp"]) - 1
    oh = refpy.setup(ref, ref.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    a = airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])
    h = airg.setup(a, injection=_injection(oh, prm), **prm)
    theirs = json.loads(oh.report())
    ours = json.loads(json.dumps(reports.hierarchy_report(h)))
    # injection skips the growth guard, whose results are compared in native mode below
    native_only = ("smoother_growth", "poly_attempts", "solver_growth")

    def strip(rep):
        rep = json.loads(json.dumps(rep))
        for lv in rep["levels"]:
            for k in native_only:
                lv.pop(k, None)
        rep["coarse"].pop("solver_growth", None)
        return rep
    assert strip(ours) == strip(theirs)
    hn = airg.setup(a, **prm)  # native: the guard's numbers agree to rounding
    nat = reports.hierarchy_report(hn)
    assert hn.n_levels == oh.info().n_levels
    for lo, lt in zip(nat["levels"], theirs["levels"]):
        assert lo["poly_attempts"] == lt["poly_attempts"]
        # native coefficients differ from the long-double fit in the last
        # digits: the same accept / reject side of 0.5, values close
        assert (lo["smoother_growth"] <= 0.5) == (lt["smoother_growth"] <= 0.5)
        assert abs(lo["smoother_growth"] - lt["smoother_growth"]) <= 1e-3 * max(1.0, lt["smoother_growth"])
    res = airg.richardson_solve(h, g["b"], coarse_iterations=prm.get("coarse_iterations", 3))
    assert reports.csv_row(h, res.stats, prm["strength_alpha"], "pmisr-ddc", 7) == \
        oh.csv_row(res.stats, prm["strength_alpha"], "pmisr-ddc", 7)
    sr = reports.solve_report(res)
    assert sr["iterations"] == res.stats.iterations and len(sr["residual_history"]) == len(res.residual_history)
    f = tmp_path / "runs.csv"
    reports.append_csv(f, reports.csv_row(h, res.stats, 0.5, "pmisr-ddc", 0))
    reports.append_csv(f, reports.csv_row(h, res.stats, 0.5, "pmisr-ddc", 1))
    lines = f.read_text().splitlines()
    assert lines[0] == reports.csv_header() and len(lines) == 3


@pytest.mark.parametrize("P,threshold", [(2, 2.0), (4, 50.0), (8, 1e9), (3, 500.0)])
@pytest.mark.parametrize("path", GOLDEN[:4], ids=lambda p: os.path.basename(p)[:-4])
def test_rank_halving_matches_reference_replay(ref, path, P, threshold):
    """The GPU distribution's active-rank decisions (dist.cu dist_create) are
    the reference's replay rule (partition_model.cpp:77-112): on the same
    hierarchy (coefficient injection), every level's active ranks, trigger,
    locality ratios and local share equal partition_report(replay_triggers)
    bit for bit; the coarsest grid is gathered on one GPU (the reference's
    model applies the rule once more there)."""
    g = np.load(path)
    prm = dict(eval(str(g["params"][0])))
    n = len(g["rp"]) - 1
    oh = refpy.setup(ref, ref.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    h = airg.setup(airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"]), injection=_injection(oh, prm),
                   **prm)
    theirs = json.loads(oh.partition_report(P, threshold))
    d = airg.Dist(h, P, threshold=threshold)
    ours = reports.partition_report(d, P, threshold)
    assert len(ours["levels"]) == len(theirs["levels"]) == h.n_levels + 1
    for lo, lt in zip(ours["levels"][:-1], theirs["levels"][:-1]):
        for k in ("level", "n", "nnz", "active_ranks", "triggered", "ratio", "ratio_before_trigger", "local_share"):
            assert lo[k] == lt[k], (lo["level"], k, lo[k], lt[k])
    assert ours["trigger_levels"] == [l for l in theirs["trigger_levels"] if l < h.n_levels]
    assert ours["levels"][-1]["active_ranks"] == 1 and ours["levels"][-1]["n"] == theirs["levels"][-1]["n"]
