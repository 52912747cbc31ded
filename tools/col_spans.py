import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2408_08262_b200 import airg, problems
p = problems.make(2); prm = problems.setup_params(2)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
h = airg.setup(a, **prm)
for l in range(0, h.n_levels, 2):
    out = []
    for w in ("a", "r", "ff_inv", "a_ff"):
        m = h.matrix(l, w)
        rows = np.repeat(np.arange(m.nrows), np.diff(m.row_offsets))
        if w == "r":  # R rows are coarse; compare against the row's first column
            first = np.repeat(m.col_indices[m.row_offsets[:-1][np.diff(m.row_offsets) > 0]], np.diff(m.row_offsets)[np.diff(m.row_offsets) > 0])
            d = m.col_indices - first
        else:
            d = m.col_indices - rows
        out.append(f"{w}: max|d|={int(np.abs(d).max()) if d.size else 0}")
    print(l, h.level(l).n, ' '.join(out))
