"""One C4 setup (fast-mode fused operators included) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r2_setup_launches.csv python tools/ncu_setup.py
  python tools/launch_summary.py gpurun_out/r2_setup_launches.csv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

CFG = int(os.environ.get("SETUP_CONFIG", "4"))
p = problems.make(CFG)
prm = dict(problems.setup_params(CFG), fused_smooths=2)
h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
print("levels", h.n_levels)
