"""Single-process multi-GPU C ABI (``wf_mg_*``) through
``paper_2112_10034_b200.multidevice``: one host thread, one rank per listed
device, each rank's kernel with its exchange fused in over peer memory.  On a
one-GPU box the ranks share cuda:0 (their kernels run concurrently from
different streams); the distinct-device case runs where >= 2 GPUs exist.
Every result is checked against the single-GPU ops on the whole input."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import numpy_oracle as no, synthetic  # noqa: E402


@pytest.fixture(scope="module")
def md():
    from paper_2112_10034_b200 import build
    build.build_library()
    from paper_2112_10034_b200 import multidevice, ops
    return multidevice, ops


def _devices(world):
    n = torch.cuda.device_count()
    return [r % n for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("n", [1, 4096 * 3 + 5, (1 << 20) + 7])
def test_multidevice_ops_equal_single_gpu(md, world, n):
    multidevice, ops = md
    with multidevice.MultiDevice(_devices(world)) as mg:
        # fp32 sum: the rank-order fold of the per-rank K2 partials, on every rank
        f = ops.fill_synthetic("f32_unit", n, seed=n)
        fs = mg.split(f)
        got = mg.reduce_sum_f32(fs)
        parts = torch.stack([ops.reduce_sum_f32(s.to("cuda:0"), block=512)[0] for s in fs])
        want = ops.fold(parts)
        for g in got:
            assert torch.equal(g.cpu().view(torch.int32), want.cpu().view(torch.int32))
        fh = f.cpu().numpy()
        assert abs(float(want.item()) - no.reduce_sum_f32_exact(fh)) <= no.f32_tolerance(
            n, no.abs_sum(fh))
        # scan: the global scan, shard by shard
        x = ops.fill_synthetic("i32_full", n, seed=n + 1)
        xs = mg.split(x)
        ys = mg.scan_inclusive_i32(xs)
        assert torch.equal(torch.cat([y.cpu() for y in ys]), ops.scan_inclusive_i32(x).cpu())
        # compaction: concatenation == x[x > 0], counts / offsets / total
        outs, c3 = mg.compact_gt0_i32(xs)
        want_c = torch.masked_select(x, x > 0).cpu()
        off = 0
        pieces = []
        for o, c in zip(outs, c3):
            cnt, goff, tot = (int(v) for v in c.cpu())
            assert goff == off and tot == want_c.numel()
            pieces.append(o[:cnt].cpu())
            off += cnt
        assert torch.equal(torch.cat(pieces), want_c)
        # histogram: global bins on every rank
        u = ops.fill_synthetic("u8_uniform", 4 * n + 3, seed=n + 2)
        bins = mg.histogram256_u8(mg.split(u))
        want_b = ops.histogram256_u8(u).cpu()
        for b in bins:
            assert torch.equal(b.cpu(), want_b)


def test_multidevice_repeated_calls_and_reuse(md):
    """Epoch sequences across many calls of mixed ops on one context."""
    multidevice, ops = md
    with multidevice.MultiDevice(_devices(2)) as mg:
        for i in range(6):
            n = 50000 + 977 * i
            x = ops.fill_synthetic("i32_small", n, seed=i)
            xs = mg.split(x)
            ys = mg.scan_inclusive_i32(xs)
            assert torch.equal(torch.cat([y.cpu() for y in ys]), ops.scan_inclusive_i32(x).cpu())
            u = ops.fill_synthetic("u8_geom", n, seed=i)
            bins = mg.histogram256_u8(mg.split(u))
            assert np.array_equal(bins[1].cpu().numpy().view(np.uint64),
                                  no.histogram256_u8(synthetic.generate("u8_geom", n, seed=i)))


def test_multidevice_rejects_bad_shards(md):
    multidevice, ops = md
    from paper_2112_10034_b200.errors import LaunchError
    with multidevice.MultiDevice(_devices(2)) as mg:
        x = ops.fill_synthetic("i32_full", 100, seed=0)
        with pytest.raises(LaunchError):
            mg.scan_inclusive_i32([x])  # one shard for two ranks
        with pytest.raises(LaunchError):
            mg.reduce_sum_f32([x, x])   # wrong dtype


def test_multidevice_distinct_devices(md):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    multidevice, ops = md
    with multidevice.MultiDevice([0, 1]) as mg:
        x = ops.fill_synthetic("i32_full", (1 << 22) + 11, seed=5)
        ys = mg.scan_inclusive_i32(mg.split(x))
        assert torch.equal(torch.cat([y.cpu() for y in ys]), ops.scan_inclusive_i32(x).cpu())


def test_launch_config_device_must_match_memory(md):
    import paper_2112_10034_b200 as wf
    from paper_2112_10034_b200.errors import ConfigError
    mem = wf.DeviceMemory(0)
    a, out = mem.alloc(4 * 64), mem.alloc(4)
    cfg = wf.LaunchConfig(grid_size=1, block_size=64, device=1)
    with pytest.raises(ConfigError, match="device"):
        wf.launch(wf.PROGRAMS["reduce_sum_i32"], cfg, mem, [a, out, 64])
    cfg.device = 0
    wf.launch(wf.PROGRAMS["reduce_sum_i32"], cfg, mem, [a, out, 64])
