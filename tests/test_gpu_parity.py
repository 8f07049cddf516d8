"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the reference's golden vectors.  Bit-exact for integer work; fp32 within the
a-priori bound stated in oracle/numpy_oracle.f32_tolerance."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import numpy_oracle as no, semantics, synthetic  # noqa: E402


@pytest.fixture(scope="module")
def ops():
    from paper_2112_10034_b200 import build
    build.build_library()
    from paper_2112_10034_b200 import ops as _ops
    torch.cuda.init()
    return _ops


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


SIZES = [0, 1, 3, 4, 5, 31, 1000, 4095, 4096, 4097, 65536 + 7, (1 << 20) + 3]


# ---- synthetic generator -----------------------------------------------------

@pytest.mark.parametrize("gen", synthetic.GENS)
def test_generator_bit_exact(ops, gen):
    for n, base in ((1, 0), (1027, 0), (100003, 12345678901)):
        g = host(ops.fill_synthetic(gen, n, seed=0xABCDEF, base=base, param=437))
        want = synthetic.generate(gen, n, seed=0xABCDEF, base=base, param=437)
        assert np.array_equal(g.view(np.uint8), want.view(np.uint8)), (gen, n)


# ---- K1 ----------------------------------------------------------------------

@pytest.mark.parametrize("n", SIZES)
def test_reduce_i32_sizes(ops, n):
    a = synthetic.generate("i32_full", n, seed=n)
    got = host(ops.reduce_sum_i32(dev(a)))[0]
    assert got == no.reduce_sum_i32(a)


@pytest.mark.parametrize("block", [128, 256, 512, 1024])
@pytest.mark.parametrize("grid", [0, 1, 7, 148])
def test_reduce_i32_blocks_grids(ops, block, grid):
    a = synthetic.generate("i32_small", 300001, seed=block + grid)
    assert host(ops.reduce_sum_i32(dev(a), block=block, grid=grid))[0] == no.reduce_sum_i32(a)


def test_reduce_i32_misaligned_views(ops):
    a = synthetic.generate("i32_full", 100000, seed=9)
    d = dev(a)
    for off in (1, 2, 3, 5):
        assert host(ops.reduce_sum_i32(d[off:]))[0] == no.reduce_sum_i32(a[off:])


def test_reduce_i32_matches_reference_c1_pin(ops, golden):
    g = np.load(golden / "c1c2_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    for gen in ("i32_full", "i32_small"):
        a = ops.fill_synthetic(gen, n, seed=seed)
        want = no.reduce_sum_i32(g[f"{gen}_partials"])  # reference partials, wrap-folded
        assert host(ops.reduce_sum_i32(a, block=256))[0] == want


def test_reduce_i32_c1_config(ops):
    """BASELINE config 1: 2^20 int32, block 256."""
    n = 1 << 20
    a = ops.fill_synthetic("i32_full", n, seed=0)
    want = no.reduce_sum_i32(synthetic.generate("i32_full", n, seed=0))
    for _ in range(3):  # workspace reuse across launches
        assert host(ops.reduce_sum_i32(a, block=256))[0] == want


# ---- K2 ----------------------------------------------------------------------

@pytest.mark.parametrize("n", SIZES)
def test_reduce_f32_within_bound(ops, n):
    a = synthetic.generate("f32_unit", n, seed=n)
    got = float(host(ops.reduce_sum_f32(dev(a)))[0])
    tol = no.f32_tolerance(max(n, 1), no.abs_sum(a), chain=max(1, n // 1000))
    assert abs(got - no.reduce_sum_f32_exact(a)) <= tol + 1e-30


def test_reduce_f32_reproducible_and_pinned(ops, golden):
    g = np.load(golden / "c1c2_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    x = ops.fill_synthetic("f32_unit", n, seed=seed)
    r1 = host(ops.reduce_sum_f32(x)).view(np.int32)[0]
    r2 = host(ops.reduce_sum_f32(x)).view(np.int32)[0]
    assert r1 == r2  # bitwise reproducible
    ref_total = np.float32(0)
    for p in g["f32_unit_partials"]:  # the reference's own result
        ref_total = np.float32(ref_total + p)
    a = synthetic.generate("f32_unit", n, seed=seed)
    tol = no.f32_tolerance(n, no.abs_sum(a), chain=n // (grid * block))
    assert abs(float(np.int32(r1).view(np.float32)) - float(ref_total)) <= 2 * tol


@pytest.mark.slow
@pytest.mark.parametrize("block", [256, 512, 1024])  # 256: bench.py C2 block
def test_reduce_f32_full_config(ops, block):
    """BASELINE config 2 on one GPU: 2^30 fp32."""
    n = 1 << 30
    x = ops.fill_synthetic("f32_unit", n, seed=1)
    got = float(host(ops.reduce_sum_f32(x, block=block))[0])
    exact = float(torch.sum(x, dtype=torch.float64))
    absx = float(torch.sum(x.abs(), dtype=torch.float64))
    # per-thread chains: n / (148 SMs * resident threads * 16 chains) elements
    chain = n // (148 * 1024 * 16) + 16
    assert abs(got - exact) <= no.f32_tolerance(n, absx, chain=chain)
    assert abs(got - exact) <= no.f32_tolerance(n, absx)  # SURVEY §8c contract
    assert float(host(ops.reduce_sum_f32(x, block=block))[0]) == got
    del x


@pytest.mark.parametrize("block", [256, 512, 1024])
def test_reduce_f32_input_stable_launches(ops, block):
    """WF_FLAG_INPUT_STABLE (programmatic dependent launch): a chain of
    back-to-back launches, each streaming while the previous one drains, over
    several inputs, each result into its own output — every one bit-identical
    to the plain launch.  The workspace is shared by the whole chain, so a
    dependent launch that touched it before its predecessor finished would
    corrupt the folds."""
    n = (1 << 24) + 5
    xs = [ops.fill_synthetic("f32_unit", n, seed=s) for s in range(3)]
    want = [host(ops.reduce_sum_f32(x, block=block)).view(np.int32)[0] for x in xs]
    outs = torch.empty(30, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for k in range(30):
        ops.reduce_sum_f32(xs[k % 3], outs[k:k + 1], block=block, input_stable=True)
    got = host(outs).view(np.int32)
    assert [int(v) for v in got] == [int(want[k % 3]) for k in range(30)]


def test_reduce_f32_input_stable_after_a_writer_and_sync(ops):
    """The promise covers the kernel issued just before: after a synchronise,
    a writer of the input followed by a plain launch then flagged launches,
    the flagged results follow the new data."""
    n = 1 << 22
    x = ops.fill_synthetic("f32_unit", n, seed=1)
    torch.cuda.synchronize()
    a = host(ops.reduce_sum_f32(x, input_stable=True)).view(np.int32)[0]
    ops.fill_synthetic("f32_unit", n, seed=2, out=x)  # writes x
    ops.reduce_sum_f32(x)  # plain launch after the writer
    b = host(ops.reduce_sum_f32(x, input_stable=True)).view(np.int32)[0]
    want_a = host(ops.reduce_sum_f32(ops.fill_synthetic("f32_unit", n, seed=1))).view(np.int32)[0]
    want_b = host(ops.reduce_sum_f32(ops.fill_synthetic("f32_unit", n, seed=2))).view(np.int32)[0]
    assert (a, b) == (want_a, want_b)


def test_reduce_f32_ex_rejects_unknown_flags(ops):
    from paper_2112_10034_b200 import _lib
    x = torch.zeros(16, dtype=torch.float32, device="cuda")
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    rc = _lib.load().wf_reduce_sum_f32_ex(x.data_ptr(), 16, out.data_ptr(), 256, 0, None, 0, 6,
                                          None)
    assert rc == _lib.WF_ERR_ARG and b"flags" in _lib.load().wf_last_error()


# ---- K3 ----------------------------------------------------------------------

@pytest.mark.parametrize("n", SIZES)
def test_scan_sizes(ops, n):
    a = synthetic.generate("i32_full", n, seed=n + 1)
    assert np.array_equal(host(ops.scan_inclusive_i32(dev(a))), no.scan_inclusive_i32(a))


def test_scan_carry_inplace_misaligned(ops):
    a = synthetic.generate("i32_full", 50000, seed=4)
    carry = torch.tensor([123456789], dtype=torch.int32, device="cuda")
    got = host(ops.scan_inclusive_i32(dev(a), carry=carry))
    assert np.array_equal(got, no.scan_inclusive_i32(a, carry=123456789))
    d = dev(a)
    ops.scan_inclusive_i32(d, out=d)
    assert np.array_equal(host(d), no.scan_inclusive_i32(a))
    d = dev(a)
    out = torch.empty(50001, dtype=torch.int32, device="cuda")
    got = host(ops.scan_inclusive_i32(d[1:], out=out[2:50001]))  # both misaligned
    assert np.array_equal(got, no.scan_inclusive_i32(a[1:]))


def test_scan_repeated_launches(ops):
    # epoch/ticket reuse: many launches on one workspace, varying sizes
    for i, n in enumerate([4096 * 3, 10, 4096 * 17 + 5, 1 << 16, 7]):
        a = synthetic.generate("i32_small", n, seed=i)
        assert np.array_equal(host(ops.scan_inclusive_i32(dev(a))), no.scan_inclusive_i32(a))


def test_scan_matches_reference_warp_prefix(ops, golden):
    g = np.load(golden / "c3_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    a = synthetic.generate("i32_full", n, seed=seed)
    got = host(ops.scan_inclusive_i32(dev(a)))
    # global scan minus the carry of each 32-element warp segment == the
    # reference's warp prefix
    seg_start = np.concatenate([[0], got[31::32][:-1]]).astype(np.int64)
    local = (got.reshape(-1, 32).astype(np.int64) - seg_start[:, None]) & 0xFFFFFFFF
    assert np.array_equal(local.astype(np.uint32).view(np.int32).reshape(-1), g["warp_prefix_out"])


@pytest.mark.slow
def test_scan_full_config_properties(ops):
    """BASELINE config 3 on one GPU: 2^28 int32."""
    n = 1 << 28
    x = ops.fill_synthetic("i32_full", n, seed=2)
    y = ops.scan_inclusive_i32(x)
    torch.cuda.synchronize()
    # checksum: last element == wrapping total (K1), first == x[0]
    total = host(ops.reduce_sum_i32(x))[0]
    assert host(y[-1:])[0] == total and host(y[:1])[0] == host(x[:1])[0]
    # linearity: y[i] - y[i-1] == x[i] (mod 2^32) everywhere
    d = (y[1:].to(torch.int64) - y[:-1].to(torch.int64) - x[1:].to(torch.int64)) % (1 << 32)
    assert int(d.count_nonzero()) == 0
    # sampled slices vs numpy with the right carry
    xs = synthetic.generate("i32_full", 1 << 20, seed=2, base=(1 << 27))
    carry = int(host(y[(1 << 27) - 1:(1 << 27)])[0])
    want = no.scan_inclusive_i32(xs, carry=carry)
    assert np.array_equal(host(y[1 << 27:(1 << 27) + (1 << 20)]), want)


# ---- K4 ----------------------------------------------------------------------

@pytest.mark.parametrize("n", SIZES)
def test_compact_sizes(ops, n):
    a = synthetic.generate("i32_full", n, seed=n + 2)
    out, cnt = ops.compact_gt0_i32(dev(a))
    m = int(host(cnt)[0])
    want = no.compact_gt0_i32(a)
    assert m == len(want)
    assert np.array_equal(host(out)[:m], want)


@pytest.mark.parametrize("permille", [0, 10, 500, 1000])
def test_compact_selectivity(ops, permille):
    n = 300007
    x = ops.fill_synthetic("i32_select", n, seed=11, param=permille)
    out, cnt = ops.compact_gt0_i32(x)
    a = synthetic.generate("i32_select", n, seed=11, param=permille)
    want = no.compact_gt0_i32(a)
    assert int(host(cnt)[0]) == len(want)
    assert np.array_equal(host(out)[:len(want)], want)


@pytest.mark.slow
def test_compact_full_config(ops):
    """BASELINE config 4: 2^28 int32, ordered output."""
    n = 1 << 28
    x = ops.fill_synthetic("i32_full", n, seed=3)
    out, cnt = ops.compact_gt0_i32(x)
    want = torch.masked_select(x, x > 0)
    m = int(host(cnt)[0])
    assert m == want.numel()
    assert torch.equal(out[:m], want)


# ---- K3/K4 many launches on one workspace ----------------------------------

def test_tmem_kernel_many_launches(ops):
    """TMEM-parked kernel: epochs/tickets survive back-to-back launches on one
    workspace, sizes from one ragged tile to many tiles.  (The round-1
    smem-stage / register-tile / two-pass kernels are variant builds now:
    tools/variants/check_variants.py.)"""
    for i, n in enumerate([8192 * 148 * 3 + 17, 5, 8192, 8193, 1 << 21, 77777]):
        a = synthetic.generate("i32_select", n, seed=i, param=700)
        assert np.array_equal(host(ops.scan_inclusive_i32(dev(a))), no.scan_inclusive_i32(a))
        out, cnt = ops.compact_gt0_i32(dev(a))
        want = no.compact_gt0_i32(a)
        assert int(host(cnt)[0]) == len(want) and np.array_equal(host(out)[:len(want)], want)


# tile counts around the early L2 prefetch of the first claims (4 stages x 148
# CTAs = 592 tiles of 8192): fewer tiles than CTAs, exactly / one past, many
TILE_EDGE_SIZES = [1, 8192 * 3 + 5, 8192 * 148, 8192 * 592, 8192 * 592 + 1, 8192 * 600 - 3,
                   (1 << 23) + 77]


def test_tmem_kernels_input_stable_chain(ops):
    """K3/K4 with WF_FLAG_INPUT_STABLE: a back-to-back chain of dependent
    launches over inputs of every tile-count regime, alternating scan and
    compaction on one stream, every output in its own buffer; equal to the
    oracle.  Only the L2 prefetch of the first tiles precedes
    griddepcontrol.wait; the tickets, epochs, descriptors and outputs are
    touched after it, so a launch that raced its predecessor would corrupt the
    shared workspace."""
    xs = [ops.fill_synthetic("i32_select", n, seed=i, param=600)
          for i, n in enumerate(TILE_EDGE_SIZES)]
    ys = [torch.empty_like(x) for x in xs]
    outs = [torch.empty_like(x) for x in xs]
    cnts = [torch.empty(1, dtype=torch.int64, device="cuda") for _ in xs]
    torch.cuda.synchronize()
    for _ in range(2):
        for x, y, o, c in zip(xs, ys, outs, cnts):
            ops.scan_inclusive_i32(x, y, input_stable=True)
            ops.compact_gt0_i32(x, o, c, input_stable=True)
    torch.cuda.synchronize()
    for i, n in enumerate(TILE_EDGE_SIZES):
        a = synthetic.generate("i32_select", n, seed=i, param=600)
        assert np.array_equal(host(ys[i]), no.scan_inclusive_i32(a)), n
        want = no.compact_gt0_i32(a)
        assert int(host(cnts[i])[0]) == len(want), n
        assert np.array_equal(host(outs[i])[:len(want)], want), n


def test_scan_input_stable_carry_from_predecessor(ops):
    """The flagged scan reads its device carry only after the previous kernel
    (which wrote it) has completed: the sharded scan's pass 1 -> scan pair."""
    n = (1 << 22) + 9
    x = ops.fill_synthetic("i32_full", n, seed=4)
    a = synthetic.generate("i32_full", n, seed=4)
    torch.cuda.synchronize()
    y = torch.empty_like(x)
    for c in (0, 12345, -7, 2 ** 31 - 1):
        carry = torch.full((1,), 0, dtype=torch.int32, device="cuda")
        carry.fill_(c)  # a kernel that writes the carry right before the scan
        ops.scan_inclusive_i32(x, y, carry=carry, input_stable=True)
        want = (no.scan_inclusive_i32(a).astype(np.int64) + c).astype(np.int32)
        assert np.array_equal(host(y), want), c


# ---- K5 ----------------------------------------------------------------------

@pytest.mark.parametrize("n", SIZES + [(1 << 22) + 13])
def test_hist_sizes(ops, n):
    a = synthetic.generate("u8_uniform", n, seed=n)
    got = host(ops.histogram256_u8(dev(a))).view(np.uint64)
    assert np.array_equal(got, no.histogram256_u8(a))


@pytest.mark.parametrize("gen,param", [("u8_const", 0), ("u8_const", 255), ("u8_geom", 0)])
def test_hist_skewed(ops, gen, param):
    n = 5_000_011
    x = ops.fill_synthetic(gen, n, seed=5, param=param)
    want = no.histogram256_u8(synthetic.generate(gen, n, seed=5, param=param))
    assert np.array_equal(host(ops.histogram256_u8(x)).view(np.uint64), want)


def test_hist_input_stable_launches(ops):
    """K5 with WF_FLAG_INPUT_STABLE: a back-to-back chain of dependent
    launches over three inputs (uniform, constant, skewed), each into its own
    bins, all equal to the oracle; the shared workspace accumulators would be
    corrupted by a launch that touched them before its predecessor ended."""
    n = (1 << 24) + 13
    gens = [("u8_uniform", 0), ("u8_const", 7), ("u8_geom", 0)]
    xs = [ops.fill_synthetic(g, n, seed=5, param=p) for g, p in gens]
    want = [no.histogram256_u8(synthetic.generate(g, n, seed=5, param=p)) for g, p in gens]
    bins = torch.empty(12, 256, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    for k in range(12):
        ops.histogram256_u8(xs[k % 3], bins[k], input_stable=True)
    got = host(bins).view(np.uint64)
    for k in range(12):
        assert np.array_equal(got[k], want[k % 3]), k


def test_hist_misaligned_and_grids(ops):
    a = synthetic.generate("u8_uniform", 1 << 20, seed=6)
    d = dev(a)
    for off in (1, 7, 15):
        got = host(ops.histogram256_u8(d[off:])).view(np.uint64)
        assert np.array_equal(got, no.histogram256_u8(a[off:]))
    for grid in (1, 3, 296):
        got = host(ops.histogram256_u8(d, grid=grid)).view(np.uint64)
        assert np.array_equal(got, no.histogram256_u8(a))


def _bincount_slices(x, parts=16):
    """Independent check: sum of torch.bincount over ``parts`` slices."""
    total = torch.zeros(256, dtype=torch.int64, device=x.device)
    step = (x.numel() + parts - 1) // parts
    for lo in range(0, x.numel(), step):
        total += torch.bincount(x[lo:lo + step].to(torch.int32), minlength=256)
    return total.cpu().numpy().astype(np.uint64)


@pytest.mark.slow
def test_hist_full_config(ops):
    """BASELINE config 5 on one GPU: 2^32 uint8 (4 GiB), the whole histogram
    against 16 independent torch.bincount slices, plus linearity."""
    n = 1 << 32
    x = ops.fill_synthetic("u8_uniform", n, seed=4)
    bins = host(ops.histogram256_u8(x)).view(np.uint64)
    assert int(bins.sum()) == n
    assert np.array_equal(bins, _bincount_slices(x))
    parts = np.zeros(256, dtype=np.uint64)
    step = n // 8
    for k in range(8):
        parts += host(ops.histogram256_u8(x[k * step:(k + 1) * step])).view(np.uint64)
    assert np.array_equal(parts, bins)
    del x


@pytest.mark.slow
def test_hist_full_config_single_value(ops):
    """All-same-value bytes at 2^32: one bin reaches 2^32 (overflows any u32
    count) — exact on the auto grid."""
    n = 1 << 32
    x = ops.fill_synthetic("u8_const", n, seed=4)
    v = int(host(x[:1])[0])
    bins = host(ops.histogram256_u8(x)).view(np.uint64)
    want = np.zeros(256, dtype=np.uint64)
    want[v] = n
    assert np.array_equal(bins, want)
    del x


@pytest.mark.slow
def test_hist_one_block_counts_2p32_of_one_byte(ops):
    """grid=1 over 2^32 equal bytes: the single block's per-bin fold is
    64-bit (a u32 fold wraps to 0 here), and the per-(bin, lane) u32
    counters stay below 2^32 (2^27 each)."""
    n = 1 << 32
    x = torch.full((n,), 0xA5, dtype=torch.uint8, device="cuda")
    bins = host(ops.histogram256_u8(x, grid=1)).view(np.uint64)
    assert int(bins[0xA5]) == n and int(bins.sum()) == n
    del x


def test_hist_grid_floor_keeps_counters_exact(ops):
    """A caller grid below the counter-overflow floor is raised to it
    (grid >= n / 2^36); below 2^36 bytes the floor is one block, so any
    grid >= 1 is exact."""
    a = synthetic.generate("u8_const", (1 << 20) + 5, seed=2)
    for g in (1, 2, 3, 7, 1000):
        got = host(ops.histogram256_u8(dev(a), grid=g)).view(np.uint64)
        assert np.array_equal(got, no.histogram256_u8(a)), g


# ---- P: warp collectives -----------------------------------------------------

def test_shfl_down_golden_table(ops, golden):
    t = json.loads((golden / "warp_semantics.json").read_text())["shfl_down"]
    buf = np.array(t["buffer"], dtype=np.int32)
    for j, off in enumerate(t["offsets"]):
        got = host(ops.warp_collective("shfl_down", dev(buf), operand=off, block=32))
        assert got.tolist() == [t["table"][lane][j] for lane in range(32)], off


def test_oracle_kats_on_gpu(ops, golden):
    kat = np.load(golden / "oracle_kat.npz")
    got = host(ops.warp_collective("shfl_down", dev(np.arange(32, dtype=np.int32)), operand=1))
    assert np.array_equal(got, kat["kat_shfl_out"])
    pred = (kat["kat_vote_any_in"] == 9).astype(np.int32)
    got = host(ops.warp_collective("vote_any", dev(pred), block=64))
    assert np.array_equal(got, kat["kat_vote_any_out"])
    got = host(ops.warp_collective("vote_all", dev(np.ones(32, dtype=np.int32))))
    assert np.array_equal(got, kat["kat_vote_all_out"])


KINDS = ["shfl_down", "shfl_up", "shfl_xor", "shfl_idx", "vote_all", "vote_any", "ballot",
         "reduce_add"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("block,width,mask", [
    (32, 32, 0xFFFFFFFF), (64, 32, 0xFFFFFFFF), (256, 32, 0xFFFFFFFF),
    (48, 32, 0xFFFFFFFF), (100, 32, 0xFFFFFFFF),          # partial warps
    (64, 32, 0x0F0F00FF), (96, 32, 0xAAAAAAAA),            # non-full masks
    (64, 4, 0xFFFFFFFF), (64, 8, 0x00FFFF00), (40, 16, 0xFFFFFFFF), (32, 1, 0xFFFFFFFF),
])
def test_collectives_vs_semantics(ops, kind, block, width, mask):
    rng = np.random.default_rng(block * 131 + width)
    n = block * 3
    a = rng.integers(-3, 4, n).astype(np.int32)
    a[rng.random(n) < 0.3] = 0
    b = rng.integers(-40, 40, n).astype(np.int32)
    init = np.full(n, -777, dtype=np.int32)
    got = host(ops.warp_collective(kind, dev(a), dev(b), block=block, width=width, mask=mask,
                                   out=dev(init)))
    want = semantics.collective(kind, a, b, 0, block, width, mask, out_init=init)
    assert np.array_equal(got, want)


# ---- launch() drop-in API ----------------------------------------------------

def test_launch_named_programs(ops):
    from paper_2112_10034_b200 import DeviceMemory, LaunchConfig, launch, PROGRAMS
    mem = DeviceMemory()
    n = 10007
    a = synthetic.generate("i32_full", n, seed=1)
    ab = mem.alloc(4 * n)
    mem.write(ab, a, "i32")
    ob = mem.alloc(4)
    launch(PROGRAMS["reduce_sum_i32"], LaunchConfig(grid_size=1, block_size=256), mem, [ab, ob, n])
    assert mem.host_view(ob, "i32")[0] == no.reduce_sum_i32(a)
    sb = mem.alloc(4 * n)
    launch(PROGRAMS["scan_inclusive_i32"], LaunchConfig(block_size=256), mem, [ab, sb, n])
    assert np.array_equal(mem.host_view(sb, "i32"), no.scan_inclusive_i32(a))
    cb, kb = mem.alloc(4 * n), mem.alloc(8)
    launch(PROGRAMS["compact_gt0_i32"], LaunchConfig(), mem, [ab, cb, kb, n])
    m = int(mem.host_view(kb, "u64")[0])
    assert np.array_equal(mem.host_view(cb, "i32")[:m], no.compact_gt0_i32(a))
    u = synthetic.generate("u8_uniform", n, seed=2)
    ub, hb = mem.alloc(n), mem.alloc(256 * 8)
    mem.copy_in(ub, u.tobytes())
    launch(PROGRAMS["histogram256_u8"], LaunchConfig(), mem, [ub, hb, n])
    assert np.array_equal(mem.host_view(hb, "u64"), no.histogram256_u8(u))


def test_launch_errors_follow_reference(ops):
    from paper_2112_10034_b200 import (DeviceMemory, ExecutionError, LaunchConfig, LaunchError,
                                       launch, PROGRAMS)
    mem = DeviceMemory()
    ab, ob = mem.alloc(40), mem.alloc(4)
    with pytest.raises(LaunchError, match="kernel takes 3 arguments, got 2"):
        launch(PROGRAMS["reduce_sum_i32"], LaunchConfig(), mem, [ab, ob])
    with pytest.raises(ExecutionError, match=r"out-of-bounds read a\[10\], length 10"):
        launch(PROGRAMS["reduce_sum_i32"], LaunchConfig(), mem, [ab, ob, 11])
    launch(PROGRAMS["reduce_sum_i32"], LaunchConfig(grid_size=0), mem, [ab, ob, 11])  # no-op


def test_launch_warp_program_partial_warps(ops):
    from paper_2112_10034_b200 import DeviceMemory, LaunchConfig, launch, warp_program
    mem = DeviceMemory()
    grid, block = 3, 48
    n = grid * block
    a = np.arange(n, dtype=np.int32)
    off = np.full(n, 2, dtype=np.int32)
    ab, bb, ob = mem.alloc(4 * n), mem.alloc(4 * n), mem.alloc(4 * n)
    mem.write(ab, a, "i32")
    mem.write(bb, off, "i32")
    launch(warp_program("shfl_down"), LaunchConfig(grid_size=grid, block_size=block), mem,
           [ab, bb, ob])
    want = semantics.collective("shfl_down", a, off, 0, block, 32, 0xFFFFFFFF)
    assert np.array_equal(mem.host_view(ob, "i32"), want)


def test_device_memory_numpy_view_contract(ops):
    """`view` is the reference's writable numpy view (runtime/memory.py:83-85):
    writes through it reach the next launch, a view held across a launch
    shows the kernel's output, and copy_in / copy_out / copy stay coherent
    with it — the reference test idiom `mem.view(b, kind)[:] = init`."""
    from paper_2112_10034_b200 import DeviceMemory, LaunchConfig, launch, PROGRAMS
    mem = DeviceMemory()
    n = 5000
    a = synthetic.generate("i32_full", n, seed=4)
    ab, sb = mem.alloc(4 * n), mem.alloc(4 * n)
    va = mem.view(ab, "i32")
    assert isinstance(va, np.ndarray) and va.flags.writeable and not va.any()
    va[:] = a                                # host write through the view
    vs = mem.view(sb, "i32")                 # held across the launch
    launch(PROGRAMS["scan_inclusive_i32"], LaunchConfig(), mem, [ab, sb, n])
    assert np.array_equal(vs, no.scan_inclusive_i32(a))
    va[0] += 1                               # write again, after the launch
    launch(PROGRAMS["scan_inclusive_i32"], LaunchConfig(), mem, [ab, sb, n])
    b = a.copy()
    b[0] += 1
    assert np.array_equal(vs, no.scan_inclusive_i32(b))
    mem.copy_in(ab, np.zeros(2, dtype=np.int32), offset=8)   # copy_in shows in the view
    assert va[2] == 0 and va[3] == 0 and va[4] == b[4]
    assert mem.copy_out(ab, 4, offset=0) == np.int32(b[0]).tobytes()
    mem.copy(sb, ab, 16)
    assert np.array_equal(vs[:4], va[:4])
    assert np.array_equal(mem.host_view(sb, "i32")[:4], va[:4])
    # large copies stream through the pinned chunks, both directions
    big = synthetic.generate("u8_uniform", (70 << 20) + 3, seed=5)
    bb = mem.alloc(big.size)
    mem.copy_in(bb, big)
    assert mem.copy_out(bb) == big.tobytes()


def test_device_memory_roundtrip(ops):
    from paper_2112_10034_b200 import DeviceMemory, LaunchError
    mem = DeviceMemory()
    b = mem.alloc(16)
    mem.copy_in(b, bytes(range(16)))
    assert mem.copy_out(b, 4, offset=2) == bytes([2, 3, 4, 5])
    c = mem.clone()
    assert c.equal_bytes(mem)
    with pytest.raises(LaunchError, match="exceeds buffer"):
        mem.copy_in(b, bytes(17))
    mem.free(b)
    with pytest.raises(LaunchError, match="unknown buffer"):
        mem.raw(b)


# ---- host-buffer (end-to-end) entry points -----------------------------------

def test_host_entry_points(ops):
    n = (64 << 20) + 5  # several staging chunks
    f = synthetic.generate("f32_unit", n, seed=8)
    got = ops.reduce_sum_f32_host(torch.from_numpy(f).pin_memory())
    assert abs(got - no.reduce_sum_f32_exact(f)) <= no.f32_tolerance(n, no.abs_sum(f))
    a = synthetic.generate("i32_full", n, seed=8)
    assert ops.reduce_sum_i32_host(a) == no.reduce_sum_i32(a)
    u = synthetic.generate("u8_uniform", 3 * (128 << 20) + 11, seed=8)
    assert np.array_equal(ops.histogram256_u8_host(u), no.histogram256_u8(u))


@pytest.mark.parametrize("n", [0, 1, 5, 8191, (1 << 20) + 3, 3 * 22369536 + 7])
def test_host_scan_and_compaction(ops, n):
    """wf_scan_inclusive_i32_host / wf_compact_gt0_i32_host: host buffer in,
    host buffer out, through the 8-slot H2D / kernel / D2H ring; the
    largest size spans several chunks (carry chain, output offsets)."""
    a = synthetic.generate("i32_full", n, seed=n + 21)
    pinned = torch.from_numpy(a).pin_memory()
    out = torch.empty(n, dtype=torch.int32).pin_memory()
    got = ops.scan_inclusive_i32_host(pinned, out)
    assert np.array_equal(got.numpy(), no.scan_inclusive_i32(a))
    assert np.array_equal(ops.scan_inclusive_i32_host(a, carry=-5), no.scan_inclusive_i32(a, carry=-5))
    want = no.compact_gt0_i32(a)
    res, m = ops.compact_gt0_i32_host(pinned, out)
    assert m == len(want) and np.array_equal(res.numpy()[:m], want)
    res, m = ops.compact_gt0_i32_host(a)  # pageable in / out
    assert m == len(want) and np.array_equal(res[:m], want)


@pytest.mark.parametrize("permille", [0, 10, 1000])
def test_host_compaction_selectivity(ops, permille):
    n = 2 * 11184768 + 333  # several 16 MiB chunks of the compaction ring
    a = synthetic.generate("i32_select", n, seed=3, param=permille)
    res, m = ops.compact_gt0_i32_host(a)
    want = no.compact_gt0_i32(a)
    assert m == len(want) and np.array_equal(res[:m], want)


def test_host_entry_points_from_concurrent_threads(ops):
    """Host-buffer calls from several threads on one device share the copy
    streams (and, through ops, the staging buffer); the library serialises
    them, so every thread gets its own exact result."""
    from concurrent.futures import ThreadPoolExecutor
    n = (40 << 20) + 3
    arrays = [synthetic.generate("i32_full", n, seed=100 + t) for t in range(4)]
    bytes_ = [synthetic.generate("u8_uniform", n, seed=200 + t) for t in range(4)]
    want = [no.reduce_sum_i32(a) for a in arrays]
    want_h = [no.histogram256_u8(u) for u in bytes_]

    def work(t):
        torch.cuda.set_device(0)
        for _ in range(3):
            assert ops.reduce_sum_i32_host(arrays[t]) == want[t]
            assert np.array_equal(ops.histogram256_u8_host(bytes_[t]), want_h[t])
        return True

    with ThreadPoolExecutor(4) as ex:
        assert all(ex.map(work, range(4)))


@pytest.mark.slow
def test_scan_beyond_2p32_elements(ops):
    """Maximum-size check: > 2^32 elements (16 GiB in + 16 GiB out), so tile
    offsets, descriptors and stores need 64-bit addressing.  Verified in
    2^28-element slices: first differences == input and the carry across
    slice boundaries is continuous (wrapping)."""
    n = (1 << 32) + 4097
    free, _ = torch.cuda.mem_get_info()
    if free < 40 << 30:
        pytest.skip("needs ~40 GiB of free HBM")
    x = ops.fill_synthetic("i32_small", n, seed=21)
    y = ops.scan_inclusive_i32(x)
    torch.cuda.synchronize()
    step = 1 << 28
    prev = 0
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        xs = x[lo:hi].to(torch.int64)
        ys = y[lo:hi].to(torch.int64)
        want_first = (prev + int(xs[0].item())) & 0xFFFFFFFF
        assert int(ys[0].item()) & 0xFFFFFFFF == want_first, lo
        d = (ys[1:] - ys[:-1] - xs[1:]) % (1 << 32)
        assert int(d.count_nonzero().item()) == 0, lo
        prev = int(ys[-1].item())
        del xs, ys, d
    total = int(ops.reduce_sum_i32(x).item()) & 0xFFFFFFFF
    assert prev & 0xFFFFFFFF == total


@pytest.mark.slow
def test_compact_max_size(ops):
    """Largest compaction one call takes (n < 2^32): count and ordered
    output checked slice by slice against masked_select."""
    n = (1 << 32) - 5
    free, _ = torch.cuda.mem_get_info()
    if free < 40 << 30:
        pytest.skip("needs ~40 GiB of free HBM")
    x = ops.fill_synthetic("i32_full", n, seed=22)
    out, cnt = ops.compact_gt0_i32(x)
    m = int(cnt.item())
    step = 1 << 28
    pos = 0
    for lo in range(0, n, step):
        want = torch.masked_select(x[lo:lo + step], x[lo:lo + step] > 0)
        assert torch.equal(out[pos:pos + want.numel()], want), lo
        pos += want.numel()
        del want
    assert pos == m


def test_c4_c5_reference_pins_on_gpu(ops, golden):
    """K4 / K5 reproduce the reference-produced vectors of
    tests/golden/c4c5_pin.npz (the reference's expressible serial compaction
    and per-bin counting kernels)."""
    g = np.load(golden / "c4c5_pin.npz")
    for tag in [k[:-3] for k in g.files if k.endswith("_in")]:
        a = g[f"{tag}_in"]
        if tag.startswith("c4_"):
            out, cnt = ops.compact_gt0_i32(dev(a))
            m = int(host(cnt)[0])
            assert m == int(g[f"{tag}_count"][0]) and np.array_equal(host(out)[:m], g[f"{tag}_out"]), tag
        else:
            bins = host(ops.histogram256_u8(dev(a))).view(np.uint64)
            assert np.array_equal(bins.astype(np.int64), g[f"{tag}_bins"].astype(np.int64)), tag


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("n", [1, 3, 5, 8189, 8192, 8195, 3 * 8192 + 1, (1 << 20) + 3])
def test_tmem_kernel_misaligned_views(ops, k, n):
    """4-byte-aligned views (x[k:]) take the TMEM kernel with the first 0-3
    virtual elements masked: nothing before the view is stored, results equal
    the oracle; the scan also in place and with a carry."""
    a = synthetic.generate("i32_full", n + 8, seed=n + k)
    x = dev(a)
    y = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
    got = ops.scan_inclusive_i32(x[k:k + n], out=y[k:k + n])
    assert np.array_equal(host(got), no.scan_inclusive_i32(a[k:k + n]))
    assert not host(y[:k]).any() and not host(y[k + n:]).any()  # no stray stores
    carry = torch.tensor([99], dtype=torch.int32, device="cuda")
    z = dev(a)
    ops.scan_inclusive_i32(z[k:k + n], out=z[k:k + n], carry=carry)
    zz = host(z)
    assert np.array_equal(zz[k:k + n], no.scan_inclusive_i32(a[k:k + n], carry=99))
    assert np.array_equal(zz[:k], a[:k]) and np.array_equal(zz[k + n:], a[k + n:])
    for ko in (0, 1, 3):  # compaction: any output offset
        buf = torch.full((n + 8,), -7, dtype=torch.int32, device="cuda")
        out, cnt = ops.compact_gt0_i32(x[k:k + n], out=buf[ko:ko + n])
        want = no.compact_gt0_i32(a[k:k + n])
        m = int(host(cnt)[0])
        assert m == len(want) and np.array_equal(host(out)[:m], want)
        assert (host(buf[:ko]) == -7).all()


@pytest.mark.gpu
def test_ops_follow_the_current_torch_stream(ops):
    """ops.* enqueue on the current stream (fast raw-handle lookup), including
    inside a `torch.cuda.stream` context."""
    side = torch.cuda.Stream()
    assert ops._stream_handle() == torch.cuda.current_stream().cuda_stream
    with torch.cuda.stream(side):
        assert ops._stream_handle() == side.cuda_stream
        x = torch.arange(1 << 20, dtype=torch.int32, device="cuda") % 7 - 3
        out = ops.reduce_sum_i32(x)
    side.synchronize()
    assert int(out.item()) == int(x.long().sum())


@pytest.mark.gpu
def test_two_devices_in_one_process(ops):
    """Every op on a tensor of a non-current GPU: the op switches to the
    tensor's device, and each kernel's dynamic-smem opt-in is set per device
    (scan / compaction use 192 KiB), so a second GPU in the same process
    gives the same results as the first."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs in one process")
    torch.cuda.set_device(0)
    n = (1 << 22) + 5
    a = synthetic.generate("i32_full", n, seed=11)
    u = synthetic.generate("u8_geom", n, seed=11, param=0)
    for d in (1, 0, 1):
        x = torch.from_numpy(a).to(f"cuda:{d}")
        assert torch.cuda.current_device() == 0
        assert np.array_equal(host(ops.scan_inclusive_i32(x)), no.scan_inclusive_i32(a))
        out, cnt = ops.compact_gt0_i32(x)
        want = no.compact_gt0_i32(a)
        assert int(host(cnt)[0]) == len(want) and np.array_equal(host(out)[:len(want)], want)
        assert host(ops.reduce_sum_i32(x))[0] == no.reduce_sum_i32(a)
        bins = host(ops.histogram256_u8(torch.from_numpy(u).to(f"cuda:{d}"))).view(np.uint64)
        assert np.array_equal(bins, no.histogram256_u8(u))
        assert out.device.index == d and cnt.device.index == d
