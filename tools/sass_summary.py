"""Per-kernel SASS instruction-class counts of the product library (proof of
what the kernels execute: tcgen05 TMEM traffic STTM/LDTM, TMA bulk copies
UBLKCP, mbarrier SYNCS, REDUX/VOTE/SHFL warp collectives, 128-bit global
loads/stores).  usage: python tools/sass_summary.py [lib.so] > profiles/r02_sass_ops.md"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2112_10034_b200" / "libwarpfold_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
CLASSES = ["STTM", "LDTM", "UTCMMA", "UBLKCP", "UTMALDG", "SYNCS", "REDUX", "VOTE", "SHFL",
           "LDG.128", "LDG", "STG.128", "STG", "LDS", "STS", "ATOMS", "ATOMG", "RED", "BAR", "NANOSLEEP"]
per = defaultdict(Counter)
fn = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if not m or fn is None:
        continue
    op = m.group(2)
    base = op.split(".")[0]
    if base in ("LDG", "STG"):
        per[fn][base + (".128" if ".128" in op or "E.128" in op else "")] += 1
    elif base in CLASSES:
        per[fn][base] += 1


def short(name: str) -> str:
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"wf::\(anonymous namespace\)::", "", d)
    return d.split("(")[0][:60]


rows = sorted(per.items(), key=lambda kv: short(kv[0]))
print("# SASS instruction classes per kernel (`cuobjdump -sass` of the product library)\n")
print(f"Library: `{Path(lib).name}` built for sm_100a.  Counts are static instructions in each kernel's SASS.\n")
print("| kernel | " + " | ".join(CLASSES) + " |")
print("|---|" + "---|" * len(CLASSES))
for fname, c in rows:
    print(f"| `{short(fname)}` | " + " | ".join(str(c.get(k, 0)) for k in CLASSES) + " |")
tot = Counter()
for _, c in per.items():
    tot.update(c)
print("| **total** | " + " | ".join(str(tot.get(k, 0)) for k in CLASSES) + " |")
