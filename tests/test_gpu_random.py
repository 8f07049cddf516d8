"""Seeded randomized parity sweep of K1-K5 against the oracle: random sizes
(one element to several waves of tiles), random 4-byte view offsets, random
selectivities / byte distributions / block sizes, and random interleavings
of plain and WF_FLAG_INPUT_STABLE (programmatic dependent) launches on one
stream, every result checked bit for bit (fp32 within the a-priori bound and
bitwise against the plain launch).  The case list is a pure function of the
seed, so a failure names a reproducible case."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import numpy_oracle as no, synthetic  # noqa: E402

N_CASES = 60


@pytest.fixture(scope="module")
def ops():
    from paper_2112_10034_b200 import build
    build.build_library()
    from paper_2112_10034_b200 import ops as _ops
    torch.cuda.init()
    return _ops


def _cases(seed: int):
    rng = np.random.default_rng(seed)
    for i in range(N_CASES):
        op = ["reduce_i32", "reduce_f32", "scan", "compact", "hist"][i % 5]
        scale = int(rng.integers(0, 5))  # size regime
        n = int([rng.integers(1, 40), rng.integers(40, 9000), rng.integers(9000, 300_000),
                 rng.integers(300_000, 5_000_000), rng.integers(5_000_000, 12_000_000)][scale])
        off = int(rng.integers(0, 4))
        block = int(rng.choice([128, 256, 512, 1024]))
        permille = int(rng.choice([0, 1, 10, 300, 500, 999, 1000]))
        hgen = str(rng.choice(["u8_uniform", "u8_const", "u8_geom"]))
        flagged = bool(rng.integers(0, 2))
        yield i, op, n, off, block, permille, hgen, flagged


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_kernel_parity(ops, seed):
    for i, op, n, off, block, permille, hgen, flagged in _cases(seed):
        case = dict(seed=seed, i=i, op=op, n=n, off=off, block=block, permille=permille,
                    hgen=hgen, flagged=flagged)
        if op in ("reduce_i32", "scan", "compact"):
            gen, param = ("i32_select", permille) if op == "compact" else ("i32_full", 0)
            full = synthetic.generate(gen, n + off, seed=seed * 1000 + i, param=param)
            a = full[off:]
            xd = torch.from_numpy(full).cuda()[off:]
            torch.cuda.synchronize()
            if op == "reduce_i32":
                got = int(ops.reduce_sum_i32(xd, block=block).cpu()[0])
                assert got == no.reduce_sum_i32(a), case
            elif op == "scan":
                y = ops.scan_inclusive_i32(xd, input_stable=flagged)
                y2 = ops.scan_inclusive_i32(xd, input_stable=flagged)  # back to back
                want = no.scan_inclusive_i32(a)
                assert np.array_equal(y.cpu().numpy(), want), case
                assert torch.equal(y, y2), case
            else:
                out, cnt = ops.compact_gt0_i32(xd, input_stable=flagged)
                out2, cnt2 = ops.compact_gt0_i32(xd, input_stable=flagged)
                want = no.compact_gt0_i32(a)
                m = int(cnt.cpu()[0])
                assert m == len(want) and int(cnt2.cpu()[0]) == m, case
                assert np.array_equal(out[:m].cpu().numpy(), want), case
                assert torch.equal(out[:m], out2[:m]), case
        elif op == "reduce_f32":
            full = synthetic.generate("f32_unit", n + off, seed=seed * 1000 + i)
            a = full[off:]
            xd = torch.from_numpy(full).cuda()[off:]
            torch.cuda.synchronize()
            r1 = ops.reduce_sum_f32(xd, block=block)
            r2 = ops.reduce_sum_f32(xd, block=block, input_stable=flagged)
            got = float(r1.cpu()[0])
            tol = no.f32_tolerance(n, no.abs_sum(a), chain=max(1, n // 1000))
            assert abs(got - no.reduce_sum_f32_exact(a)) <= tol + 1e-30, case
            assert torch.equal(r1.view(torch.int32), r2.view(torch.int32)), case
        else:
            full = synthetic.generate(hgen, 4 * n + off, seed=seed * 1000 + i, param=i)
            a = full[off:]
            xd = torch.from_numpy(full).cuda()[off:]
            torch.cuda.synchronize()
            b1 = ops.histogram256_u8(xd, input_stable=flagged)
            b2 = ops.histogram256_u8(xd, input_stable=flagged)
            want = no.histogram256_u8(a)
            assert np.array_equal(b1.cpu().numpy().view(np.uint64), want), case
            assert torch.equal(b1, b2), case
