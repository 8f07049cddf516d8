"""Build experimental variants of the library into build/variants/ (travels to
the GPU box; gitignored).  Usage: python tools/build_variants.py name="-DA=1 -DB=2" ...

Variant builds also compile tools/variants/*.cu (the round-1 scan/compaction
kernels that are not in the product library); select them with
-DWF_SCAN_IMPL=1 (smem-stage persistent), 2 (register tile) or 3 (two-pass)."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2112_10034_b200 import build  # noqa: E402

out_dir = ROOT / "build" / "variants"
out_dir.mkdir(parents=True, exist_ok=True)
for old in out_dir.glob("*.so"):
    old.unlink()


def one(spec):
    name, flags = spec.split("=", 1)
    cmd = [build.nvcc_path(), *build.NVCC_FLAGS, f"-I{build.INCLUDE}", f"-I{build.CSRC}",
           *flags.split(), "-o", str(out_dir / f"lib_{name}.so"), *map(str, build.sources()),
           *map(str, sorted((ROOT / "tools" / "variants").glob("*.cu"))), *build.LINK_FLAGS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-500:]


with ThreadPoolExecutor(8) as ex:
    for name, rc, err in ex.map(one, sys.argv[1:]):
        print(name, "OK" if rc == 0 else f"FAILED\n{err}")
