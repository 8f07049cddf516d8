"""INTEGRATION.md §2 executed: the ctypes stub a warpfold maintainer would add
(`warpfold/runtime/b200.py`), run verbatim against the reference's own
`DeviceMemory` from the `baseline/_ref` install, and checked against the
reference's `run_oracle` on the same buffer.  Skips when the reference is not
installed (it is git-ignored; bench.py's reference arm uses the same copy)."""

import ctypes
import re
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2. The ctypes stub"):text.index("### 2b.")]
    code = re.findall(r"```python\n(.*?)```", sec, re.S)[0]
    lib = ROOT / "paper_2112_10034_b200" / "libwarpfold_b200.so"
    return code.replace('C.CDLL("libwarpfold_b200.so")', f'C.CDLL("{lib}")')


@pytest.fixture(scope="module")
def warpfold():
    if not (REF / "warpfold").is_dir():
        pytest.skip("reference not installed in baseline/_ref")
    from paper_2112_10034_b200 import build
    build.build_library()
    torch.zeros(1, device="cuda")  # libcudart loaded by torch: the stub's CDLL finds it
    sys.path.insert(0, str(REF))
    import warpfold
    return warpfold


def test_integration_stub_runs_on_reference_memory(warpfold):
    from oracle import synthetic
    ns = {"__name__": "warpfold.runtime.b200"}
    exec(compile(_stub_source(), "INTEGRATION.md#2", "exec"), ns)
    n = (1 << 20) + 37
    mem = warpfold.DeviceMemory()
    buf = mem.alloc(4 * n)
    data = synthetic.generate("i32_full", n, seed=11)
    mem.view(buf, "i32")[:] = data
    got = ns["reduce_sum_i32"](mem, buf, n)
    want = int(np.int64(data.astype(np.int64).sum()) & 0xFFFFFFFF)
    assert got & 0xFFFFFFFF == want


def test_integration_stub_matches_reference_oracle(warpfold):
    """Same buffer through the reference's own oracle (the C1 kernel text,
    run_oracle, host wrap-fold) and through the stub."""
    from warpfold import LaunchConfig, parse_module, run_oracle
    from warpfold.runtime.launch import bind_args
    ns = {"__name__": "warpfold.runtime.b200"}
    exec(compile(_stub_source(), "INTEGRATION.md#2", "exec"), ns)
    n, grid, block = 4096 + 7, 4, 64
    mem = warpfold.DeviceMemory()
    a, out = mem.alloc(4 * n), mem.alloc(4 * grid * block // 32)
    mem.view(a, "i32")[:] = np.arange(n, dtype=np.int32) * 7919 - 123456
    kernel = parse_module((ROOT / "tests" / "golden" / "C1_I32.spk").read_text()).kernel()
    cfg = LaunchConfig(grid_size=grid, block_size=block, warp_size=32, workers=1)
    run_oracle(kernel, cfg, bind_args(kernel.params, mem, [a, out, n]))
    ref = int(mem.view(out, "i32").astype(np.int64).sum()) & 0xFFFFFFFF
    assert ns["reduce_sum_i32"](mem, a, n) & 0xFFFFFFFF == ref


def test_c_consumer_host_paths_end_to_end(tmp_path):
    """A plain C program (tests/c_consumer/abi_consumer.c) drives the
    host-buffer entry points of C2-C5 through the header and the .so alone —
    no Python or torch in that process — and checks every result against
    serial C loops (fp32 sum exact by construction, wrapping int32 sum,
    carried scan, ordered compaction, 256 bins)."""
    import subprocess
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_host import build_c_consumer
    r = subprocess.run([str(build_c_consumer(tmp_path)), "gpu"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "OK gpu", r.stdout + r.stderr
