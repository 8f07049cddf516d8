"""Randomised stress of the product ops against torch references, for a time
budget: K1 / K3 / K4 / K5 (and K2's reproducibility) at random sizes
(log-uniform up to 2^27), random 4-byte misalignments, random data
(full-range, selectivity permille, constant / geometric / uniform bytes),
random K5 grids, and runs of dependent launches (WF_FLAG_INPUT_STABLE) on
one input behind unrelated kernels.  Every result is checked exactly (K2:
bitwise equal to a plain launch and within the fp64 bound).
usage: python tools/fuzz_ops.py [seconds] [seed]"""
import json
import math
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = random.Random(seed)
torch.cuda.set_device(0)
CAP = (1 << 27) + 64
xi = torch.empty(CAP, dtype=torch.int32, device="cuda")
xf = torch.empty(CAP, dtype=torch.float32, device="cuda")
xu = torch.empty(4 * CAP, dtype=torch.uint8, device="cuda")
yi = torch.empty(CAP, dtype=torch.int32, device="cuda")
noise = torch.empty(1 << 22, dtype=torch.float32, device="cuda")


def size():
    return max(0, int(2 ** rng.uniform(0, 27)) + rng.choice([0, 0, 1, -1, 3, 8191, 8193]))


stats = {"iterations": 0, "checks": 0, "failures": []}
t_end = time.time() + budget
while time.time() < t_end:
    op = rng.choice(["scan", "compact", "hist", "reduce_i32", "reduce_f32"])
    n, off = size(), rng.randrange(4)
    n = min(n, CAP - 4)
    stable = rng.random() < 0.5
    reps = rng.randrange(1, 4)
    case = {"op": op, "n": n, "off": off, "stable": stable, "reps": reps}
    try:
        if op in ("scan", "compact", "reduce_i32"):
            gen = rng.choice(["i32_full", "i32_select"])
            param = rng.choice([0, 1, 10, 500, 999, 1000]) if gen == "i32_select" else 0
            case.update(gen=gen, param=param)
            x = xi[off:off + n]
            if n:
                ops.fill_synthetic(gen, n, seed=rng.randrange(1 << 30), param=param, out=x)
            torch.cuda.synchronize()
            x64 = x.to(torch.int64)
            for r in range(reps):
                noise.mul_(0.5)  # an unrelated kernel right before (the dependent launch's predecessor)
                if op == "scan":
                    yo = yi[rng.randrange(4):][:n]
                    ops.scan_inclusive_i32(x, yo, input_stable=stable)
                    want = torch.cumsum(x64, 0).to(torch.int32) if n else x
                    ok = torch.equal(yo, want)
                elif op == "compact":
                    yo = yi[:n]
                    _, cnt = ops.compact_gt0_i32(x, yo, input_stable=stable)
                    want = x[x > 0]
                    c = int(cnt.item())
                    ok = c == want.numel() and torch.equal(yo[:c], want)
                else:
                    got = ops.reduce_sum_i32(x, grid=rng.choice([0, 0, 1, 5, 300]))
                    ok = int(got.reshape(-1)[0].item()) == (
                        (int(x64.sum().item()) + (1 << 31)) % (1 << 32)) - (1 << 31)
                stats["checks"] += 1
                if not ok:
                    stats["failures"].append(dict(case, rep=r))
        elif op == "hist":
            gen = rng.choice(["u8_uniform", "u8_const", "u8_geom"])
            nb = min(size() * 4, 4 * CAP - off)
            grid = rng.choice([0, 0, 1, 7, 148, 296, 1000])
            case.update(gen=gen, n=nb, grid=grid)
            u = xu[off:off + nb]
            if nb:
                ops.fill_synthetic(gen, nb, seed=rng.randrange(1 << 30), out=u)
            torch.cuda.synchronize()
            want = torch.bincount(u.to(torch.int64), minlength=256) if nb else torch.zeros(
                256, dtype=torch.int64, device="cuda")
            for r in range(reps):
                noise.mul_(0.5)
                got = ops.histogram256_u8(u, grid=grid, input_stable=stable)
                stats["checks"] += 1
                if not torch.equal(got, want):
                    stats["failures"].append(dict(case, rep=r))
        else:
            x = xf[off:off + n]
            if n:
                ops.fill_synthetic("f32_unit", n, seed=rng.randrange(1 << 30), out=x)
            torch.cuda.synchronize()
            base = ops.reduce_sum_f32(x).clone()
            exact = float(x.to(torch.float64).sum().item()) if n else 0.0
            bound = 2 * max(1, math.ceil(math.log2(max(n, 2)))) * 2 ** -24 * (
                float(x.abs().to(torch.float64).sum().item()) if n else 0.0)
            for r in range(reps):
                noise.mul_(0.5)
                got = ops.reduce_sum_f32(x, input_stable=stable)
                stats["checks"] += 1
                if not (torch.equal(got, base) and abs(float(got.item()) - exact) <= bound + 1e-30):
                    stats["failures"].append(dict(case, rep=r))
    except Exception as e:  # noqa: BLE001
        stats["failures"].append(dict(case, error=f"{type(e).__name__}: {e}"))
    stats["iterations"] += 1
stats["seconds"] = budget
stats["seed"] = seed
print(json.dumps(stats), flush=True)
sys.exit(1 if stats["failures"] else 0)
