"""Nested condition estimates of stored Gram matrices (tools/_*.npy) on the
GPU (k_small's eigensolver, sscg_nested_conds) next to numpy's eigvalsh."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1908_04081_b200.kernels import nested_basis_conds
path = sys.argv[1] if len(sys.argv) > 1 else "tools/_c4j_grams.npy"
s_bar = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for k, g in enumerate(np.load(path)):
    gpu = nested_basis_conds(g, s_bar)
    cols = lambda i: list(range(i + 1)) + list(range(s_bar + 1, s_bar + 1 + i))
    ref = [np.nan] + [np.sqrt(np.max(np.linalg.eigvalsh(g[np.ix_(cols(i), cols(i))])) /
                              np.min(np.abs(np.linalg.eigvalsh(g[np.ix_(cols(i), cols(i))]))))
                      for i in range(1, s_bar + 1)]
    print(k, "gpu  ", np.array2string(gpu, precision=3))
    print(k, "numpy", np.array2string(np.array(ref), precision=3))
