"""Parity of the round-1 scan/compaction kernels kept as variant builds
(tools/variants/*.cu, not in the product library).  Run on a GPU box:

    python tools/build_variants.py smem="-DWF_SCAN_IMPL=1" tile="-DWF_SCAN_IMPL=2" \\
        twopass="-DWF_SCAN_IMPL=3 -DWF_2P_MIN_N=1"
    python tools/variants/check_variants.py

Each variant is checked in its own process (WF_LIB selects the library)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import numpy_oracle as no, synthetic
from paper_2112_10034_b200 import ops
for n in [1, 4097, 8192 * 5 + 3, (1 << 20) + 3, (1 << 22) + 13]:
    a = synthetic.generate("i32_full", n, seed=n + 9)
    for view in (0, 1):
        d = torch.from_numpy(np.concatenate([[5] * view, a]).astype(np.int32)).cuda()[view:]
        assert np.array_equal(ops.scan_inclusive_i32(d).cpu().numpy(), no.scan_inclusive_i32(a)), n
        out, cnt = ops.compact_gt0_i32(d)
        want = no.compact_gt0_i32(a)
        m = int(cnt.cpu()[0])
        assert m == len(want) and np.array_equal(out[:m].cpu().numpy(), want), n
print("ok")
'''

rc = 0
for lib in sorted((ROOT / "build" / "variants").glob("*.so")):
    env = dict(os.environ, WF_LIB=str(lib))
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=600)
    print(lib.name, r.stdout.strip() or r.stderr.strip()[-400:])
    rc |= r.returncode
sys.exit(rc)
