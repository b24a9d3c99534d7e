"""Compare saved (dq, dp) RHS outputs of two A/B variants: python tools/ab_compare.py a.npz b.npz"""

import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in ("dq", "dp"):
    d = np.abs(a[k] - b[k]).max() / max(np.abs(b[k]).max(), 1e-300)
    print(f"{sys.argv[1]} vs {sys.argv[2]} {k}: rel {d:.3e} bitwise {np.array_equal(a[k], b[k])}")
