"""Debug helper: first mismatches of K3/K4 vs numpy at a few sizes, with the
tile-level aggregates/prefixes the sweeper published (dense layout)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import numpy_oracle as no, synthetic  # noqa: E402
from paper_2112_10034_b200 import _lib, ops  # noqa: E402

T = 8192
for n in [int(v) for v in sys.argv[1:]] or [8193, 16384 + 5, 3 * 8192, 1048579]:
    a = synthetic.generate("i32_full", n, seed=n + 1)
    got = ops.scan_inclusive_i32(torch.from_numpy(a).cuda()).cpu().numpy()
    want = no.scan_inclusive_i32(a)
    bad = np.nonzero(got != want)[0]
    nt = (n + T - 1) // T
    ws = ops.workspace(_lib.OP_SCAN_INCLUSIVE_I32, n, torch.device("cuda", 0))
    d = ws[8192:8192 + 8 * 2 * ((nt + 15) // 16 * 16)].view(torch.int64).cpu().numpy().view(np.uint64)
    agg = (d[:nt] & 0xFFFFFFFF).astype(np.uint32)
    pref = (d[(nt + 15) // 16 * 16:][:nt] & 0xFFFFFFFF).astype(np.uint32)
    true_agg = np.array([np.uint32(a[i * T:(i + 1) * T].astype(np.int64).sum() & 0xFFFFFFFF)
                         for i in range(nt)], dtype=np.uint32)
    true_pref = (np.concatenate([[0], np.cumsum(true_agg.astype(np.int64))[:-1]]) & 0xFFFFFFFF).astype(np.uint32)
    print(f"n={n} tiles={nt} bad={len(bad)} first={bad[:5].tolist()} tiles_bad={sorted(set((bad // T).tolist()))[:10]}")
    print("  agg ok:", np.array_equal(agg, true_agg), " pref ok:", np.array_equal(pref, true_pref),
          " epochs:", sorted(set((d[:nt] >> np.uint64(34)).tolist()))[:4])
    if len(bad):
        t = int(bad[0] // T)
        print("  tile", t, "agg", agg[t], true_agg[t], "pref", pref[t], true_pref[t])
    r, c = ops.compact_gt0_i32(torch.from_numpy(a).cuda())
    m = int(c.cpu()[0])
    w = no.compact_gt0_i32(a)
    print("  compact ok:", m == len(w) and np.array_equal(r[:m].cpu().numpy(), w))
