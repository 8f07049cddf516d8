"""Which constraint gates look-back resolution?  R_i (prefix known) vs
R_{i-W} (the window chain) and the latest aggregate in the window."""
import sys
import numpy as np

for f in sys.argv[1:]:
    W = int(f.split("=")[1]) if "=" in f else 32
    f = f.split("=")[0]
    t = np.load(f).astype(np.float64)
    n = len(t)
    A, R, S = t[:, 1], t[:, 2], t[:, 0]
    mid = slice(n // 4, 3 * n // 4)
    runmax = np.maximum.accumulate(A)
    chain = np.r_[np.zeros(W), R[:-W]]
    print(f, "W", W)
    print("  R_i - R_{i-W} median/mean", np.median((R - chain)[mid]), np.mean((R - chain)[mid]))
    print("  R_i - runmaxA_i p10/50/90", np.percentile((R - runmax)[mid], [10, 50, 90]))
    bind_chain = (chain >= runmax)[mid].mean()
    print("  fraction where chain binds (R_{i-W} >= runmaxA)", bind_chain)
    print("  claim->load-done p50", np.median((A - S)[mid]))
    span = R[mid].max() - R[mid].min()
    print("  resolved tiles/us (mid)", (n // 2) / span)
