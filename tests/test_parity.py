"""GPU parity: every path of libconv.so against the CPU oracle (Eq. 1,
PAPER.md:54), through the C ABI.  Tolerances are north_star's (BASELINE.json):
relative L2 <= 1e-5 (FP32 SIMT), <= 5e-3 (TF32, BF16); bit-exact on the
integer twin.  Tensor paths are additionally checked against the oracle run on
the path's rounded inputs (reading R5), which isolates the
accumulation error (fp32, <= 1e-5 relative) from the input rounding.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, Shape, make_inputs

pytestmark = pytest.mark.gpu

TOL = {"fp32_simt": 1e-5, "fp32_tc": 1e-5, "tf32": 5e-3, "bf16": 5e-3}
ROUND = {"fp32_simt": lambda x: x, "fp32_tc": lambda x: x, "tf32": oracle.round_tf32_rna,
         "bf16": oracle.round_bf16_rne}
PATHS = ["fp32_simt", "fp32_tc", "tf32", "bf16"]


def rel_l2(got, ref):
    d = np.linalg.norm((got.astype(np.float64) - ref).ravel())
    n = np.linalg.norm(ref.ravel())
    return d / n if n else d


def coop_ok(sh):
    """The fused (cooperative) In transform TMA-loads NCHW planes: their byte
    size must be a multiple of 16."""
    return ((sh.H + sh.R - 1) * (sh.W + sh.S - 1)) % 4 == 0


def run(shape, inp, ker, path, tile=None):
    plan = conv.ConvPlan(*shape.as_tuple(), path=path, tile=tile, **shape.plan_kwargs())
    out = plan.run(inp.cuda(), ker.cuda())
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


ODD = [
    Shape(N=1, K=5, C=3, H=7, W=9, R=3, S=3),
    Shape(N=2, K=7, C=5, H=6, W=5, R=2, S=3),
    Shape(N=3, K=33, C=17, H=11, W=13, R=3, S=1),
    Shape(N=1, K=1, C=1, H=1, W=1, R=1, S=1),
    Shape(N=2, K=40, C=70, H=9, W=10, R=1, S=1),
    Shape(N=1, K=130, C=36, H=5, W=37, R=5, S=4),
    Shape(N=5, K=64, C=40, H=3, W=3, R=3, S=3),
    Shape(N=1, K=300, C=8, H=20, W=3, R=1, S=3),
]
SMALL = [CONFIGS["tiny"], CONFIGS["r2"], CONFIGS["pw"], CONFIGS["det"]]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", SMALL + ODD, ids=lambda s: "x".join(map(str, s.as_tuple())))
def test_real_inputs(path, shape):
    inp, ker = make_inputs(shape, seed=0)
    got, _ = run(shape, inp, ker, path)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert rel_l2(got, ref) <= TOL[path]
    # Against the oracle on the path's rounded inputs: only fp32 accumulation
    # differs, whatever the precision of the products.
    ref_r = oracle.conv_eq1(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()))
    assert rel_l2(got, ref_r) <= 1e-5


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", SMALL + ODD, ids=lambda s: "x".join(map(str, s.as_tuple())))
def test_integer_twin_bit_exact(path, shape):
    inp, ker = make_inputs(shape, seed=1, kind="int")
    got, _ = run(shape, inp, ker, path)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert np.array_equal(got.astype(np.float64), ref)


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("fuse", [0, 1])
@pytest.mark.parametrize("shape", SMALL + ODD, ids=lambda s: "x".join(map(str, s.as_tuple())))
def test_tensor_cta_group_variants(path, cg, fuse, shape):
    """Both the 1-CTA (M=128) and the CTA-pair (M=256) kernels, with the In
    transform as a separate launch (fuse=0) or inside the kernel (fuse=1,
    cooperative chunk transform; needs a TMA-legal NCHW plane)."""
    spec = f"cg={cg},fuse={fuse}"
    inp, ker = make_inputs(shape, seed=1, kind="int")
    if fuse and not coop_ok(shape):
        with pytest.raises(conv.ConvError) as e:
            run(shape, inp, ker, path, tile=spec)
        assert e.value.status == conv.CONV_ERR_INFEASIBLE
        return
    got, plan = run(shape, inp, ker, path, tile=spec)
    assert plan.describe()["tile"]["cg"] == cg and plan.describe()["tile"]["fuse"] == fuse
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert np.array_equal(got.astype(np.float64), ref)
    inp, ker = make_inputs(shape, seed=0)
    got, _ = run(shape, inp, ker, path, tile=spec)
    ref = oracle.conv_eq1(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()))
    assert rel_l2(got, ref) <= 1e-5


@pytest.mark.parametrize("path", PATHS)
def test_p1_identity(path):
    """P1: 1x1 identity kernel reproduces round_path(In) exactly."""
    sh = Shape(N=2, K=48, C=48, H=9, W=13, R=1, S=1)
    inp, _ = make_inputs(sh, seed=5)
    ker = torch.eye(48).reshape(48, 48, 1, 1).contiguous()
    got, _ = run(sh, inp, ker, path)
    assert np.array_equal(got, ROUND[path](inp.numpy()))


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("r0,s0", [(0, 0), (1, 2), (2, 1), (2, 2)])
def test_p2_shifted_delta(path, r0, s0):
    """P2: Ker = delta_kc delta_{r r0} delta_{s s0} => Out = shifted In (no
    kernel flip, correct h+r / w+s indexing incl. the last row/column)."""
    sh = Shape(N=2, K=16, C=16, H=10, W=12, R=3, S=3)
    inp, _ = make_inputs(sh, seed=6)
    ker = torch.zeros(sh.ker_shape)
    for k in range(16):
        ker[k, k, r0, s0] = 1.0
    got, _ = run(sh, inp, ker, path)
    exp = ROUND[path](inp.numpy())[:, :, r0:r0 + sh.H, s0:s0 + sh.W]
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_p10_tile_invariance_tensor(path):
    """P10: the k-loop order does not depend on BN, so every BN gives
    bit-identical results."""
    sh = Shape(N=2, K=256, C=256, H=12, W=12, R=3, S=3)
    inp, ker = make_inputs(sh, seed=7)
    outs = []
    for cg in (1, 2):
        for bn, kbs, fuse in ((32, 1, 0), (64, 2, 1), (128, 4, 0), (192, 1, 1), (256, 2, 1), (64, 3, 0), (128, 6, 1)):
            try:
                got, plan = run(sh, inp, ker, path, tile=f"bn={bn},cg={cg},kbs={kbs},fuse={fuse},splits=1")
            except conv.ConvError as e:           # e.g. kbs=4 stages do not fit smem
                assert e.status == conv.CONV_ERR_INFEASIBLE
                continue
            d = plan.describe()["tile"]
            assert (d["bn"], d["cg"], d["kbs"]) == (bn, cg, kbs)
            outs.append(got)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


# ---- split-K (small-M layers: the k loop of a few tiles over idle SMs) ------
SPLITK = [
    # (shape, splits): long k loops with few tiles, ragged K / M, uneven split ranges
    (Shape(N=1, K=512, C=512, H=7, W=7, R=3, S=3), 8),        # Table-1 R12-like
    (Shape(N=1, K=100, C=300, H=9, W=11, R=3, S=3), 5),       # ragged K and C; 45 stages over 5
    (Shape(N=2, K=64, C=448, H=10, W=10, R=1, S=1), 3),       # 1x1; 7 (bf16) / 14 (tf32) stages over 3
    (Shape(N=1, K=256, C=1024, H=5, W=5, R=3, S=3), 16),      # M9-like, 16 splits
]


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("case", range(len(SPLITK)))
def test_splitk_parity(path, case):
    """Split-K against the oracle (1e-5 on the path's rounded inputs, TOL on
    real ones), bit-exact on the integer twin, deterministic run to run."""
    sh, sp = SPLITK[case]
    inp, ker = make_inputs(sh, seed=101 + case)
    got, plan = run(sh, inp, ker, path, tile=f"splits={sp}")
    assert plan.describe()["tile"]["splits"] == sp
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert rel_l2(got, ref) <= TOL[path]
    assert rel_l2(got, oracle.conv_eq1(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()))) <= 1e-5
    again, _ = run(sh, inp, ker, path, tile=f"splits={sp}")
    assert np.array_equal(got, again)
    xi, wi = make_inputs(sh, seed=111 + case, kind="int")
    goti, _ = run(sh, xi, wi, path, tile=f"splits={sp}")
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_splitk_fixed_split_tile_invariance_and_graph_replay(path):
    """P10 for a fixed split count: BN and kbs do not change the bits
    (each split's k range and the split-order sum are tiling-independent
    when the stage-aligned ranges coincide: kbs = 1 vs 3 with 72 = 8 x 9
    k-blocks); and a captured graph replays correctly (the arrival counters
    are re-zeroed by every launch)."""
    sh = Shape(N=1, K=256, C=512, H=7, W=7, R=3, S=3)   # 9 taps x 8 c-blocks (bf16) = 72 k-iterations
    inp, ker = make_inputs(sh, seed=121)
    ref, _ = run(sh, inp, ker, path, tile="splits=8,bn=32,cg=1,kbs=1")
    for spec in ("splits=8,bn=64,cg=1,kbs=3", "splits=8,bn=128,cg=1,kbs=1", "splits=8,bn=128,cg=1,kbs=3"):
        got, _ = run(sh, inp, ker, path, tile=spec)
        assert np.array_equal(got, ref), spec
    plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile="splits=8")
    i, k = inp.cuda(), ker.cuda()
    out, ws = plan.new_output(), plan.new_workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.run(i, k, out, ws)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(i, k, out, ws, stream=s)
    for seed in (122, 123, 124):
        inp2, ker2 = make_inputs(sh, seed=seed)
        i.copy_(inp2)
        k.copy_(ker2)
        g.replay()
        torch.cuda.synchronize()
        r2 = oracle.conv_eq1(ROUND[path](inp2.numpy()), ROUND[path](ker2.numpy()))
        assert rel_l2(out.cpu().numpy(), r2) <= 1e-5


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_p10_whole_row_stages(path):
    """kbs = 7 / 9 (one stage = a 7-tap kernel row / the whole 3x3 window of
    a tiny-C layer) gives the same bits as one k-block per stage (P10), and
    matches the oracle: a 7x7 stride-2 stem (R1-like) and a 3-channel 3x3."""
    for sh, kbs in ((Shape.strided(2, 64, 3, 40, 38, 7, 7, 2), 7), (Shape(N=2, K=32, C=3, H=30, W=27, R=3, S=3), 9)):
        inp, ker = make_inputs(sh, seed=141)
        ref, _ = run(sh, inp, ker, path, tile="kbs=1,splits=1,expand=0")
        got, plan = run(sh, inp, ker, path, tile=f"kbs={kbs},splits=1,expand=0")
        assert plan.describe()["tile"]["kbs"] == kbs
        assert np.array_equal(got, ref)
        r64 = oracle.conv_eq1_strided(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), sh.U)
        assert rel_l2(got, r64) <= 1e-5


@pytest.mark.parametrize("splits", [2, 3, 8])
def test_simt_split_c(splits):
    """FP32 SIMT split-C (a deep-C, small-output layer; v2 and v1 kernels):
    relL2 <= 1e-5 against the oracle, bit-exact on the integer twin,
    deterministic run to run, one extra (reduce) kernel."""
    for sh, ver in ((Shape(N=1, K=64, C=256, H=7, W=7, R=3, S=3), 2), (Shape.strided(1, 40, 96, 15, 13, 3, 3, 2), 1)):
        inp, ker = make_inputs(sh, seed=171)
        got, plan = run(sh, inp, ker, "fp32_simt", tile=f"splits={splits}")
        d = plan.describe()
        assert d["tile"]["splits"] == splits and d["tile"]["ver"] == ver and plan.num_kernels == 3
        ref = oracle.conv_eq1_strided(inp.numpy(), ker.numpy(), sh.U)
        assert rel_l2(got, ref) <= 1e-5
        again, _ = run(sh, inp, ker, "fp32_simt", tile=f"splits={splits}")
        assert np.array_equal(got, again)
        xi, wi = make_inputs(sh, seed=172, kind="int")
        goti, _ = run(sh, xi, wi, "fp32_simt", tile=f"splits={splits}")
        assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1_strided(xi.numpy(), wi.numpy(), sh.U))
        # conv_run_events brackets all three kernels
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(plan.num_kernels + 1)]
        out = plan.new_output()
        plan.run_events(inp.cuda(), ker.cuda(), out, plan.new_workspace(), ev)
        torch.cuda.synchronize()
        assert all(ev[j].elapsed_time(ev[j + 1]) >= 0 for j in range(plan.num_kernels))
        assert np.array_equal(out.cpu().numpy(), got)
        # conv_run_host (pinned host buffers, the plan's workspace layout)
        dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
        out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
        plan.run_host(inp.pin_memory(), ker.pin_memory(), out_h, dbuf)
        torch.cuda.synchronize()
        assert np.array_equal(out_h.numpy(), got)


def test_p10_tile_invariance_simt():
    sh = Shape(N=2, K=32, C=24, H=12, W=12, R=3, S=3)
    inp, ker = make_inputs(sh, seed=8)
    outs = []
    for spec in ("tk=4,tw=4,kg=2,pw=2", "tk=8,tw=8,kg=4,pw=1,bc=4", "tk=8,tw=2,kg=1,pw=4,bc=16"):
        got, _ = run(sh, inp, ker, "fp32_simt", tile=spec)
        outs.append(got)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("W", [62, 61], ids=["vec4", "scalar"])
def test_simt_v2_row_loop_copy(W):
    """v2 tiles whose In tile has more copy units than 4 per thread take the
    per-row copy loop (16-B copies when Win % 4 == 0, else 4-B).  Against the
    oracle, and bit-identical to a tile whose copies fit the slotted plan (the
    per-output accumulation order does not depend on the tile)."""
    sh = Shape(N=2, K=8, C=20, H=30, W=W, R=3, S=3)
    inp, ker = make_inputs(sh, seed=12)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    row = "ver=2,tk=4,tw=4,kg=1,pw=2,tn=1,th=4,bc=16"        # 64 threads, 16*6*(Win/4 or Win) units
    slot = "ver=2,tk=4,tw=4,kg=2,pw=1,tn=1,th=2,bc=4"        # 64 threads, 4*4*16 = 256 units (vec4)
    win = W + 2
    units = lambda bc, rows: bc * rows * (win // 4 if win % 4 == 0 else win)
    assert units(16, 6) > 4 * 64
    got, _ = run(sh, inp, ker, "fp32_simt", tile=row)
    assert rel_l2(got, ref) <= TOL["fp32_simt"]
    if win % 4 == 0:
        assert units(4, 4) <= 4 * 64
        got_s, _ = run(sh, inp, ker, "fp32_simt", tile=slot)
        assert np.array_equal(got, got_s)
    xi, wi = make_inputs(sh, seed=12, kind="int")
    goti, _ = run(sh, xi, wi, "fp32_simt", tile=row)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


@pytest.mark.parametrize("path", PATHS)
def test_p10_batch_shards_bit_identical(path):
    """Shards over n equal the slices of the full result
    (plans without split-K: P10 holds for a fixed split count)."""
    sh = Shape(N=8, K=64, C=32, H=14, W=14, R=3, S=3)
    inp, ker = make_inputs(sh, seed=9)
    full, _ = run(sh, inp, ker, path, tile="splits=1")
    for p in (2, 4):
        step = sh.N // p
        for r in range(p):
            sub = Shape(N=step, K=sh.K, C=sh.C, H=sh.H, W=sh.W, R=sh.R, S=sh.S)
            got, _ = run(sub, inp[r * step:(r + 1) * step].contiguous(), ker, path, tile="splits=1")
            assert np.array_equal(got, full[r * step:(r + 1) * step])


@pytest.mark.parametrize("path", PATHS)
def test_batched_full_size_sampled(path):
    """BASELINE configs[4] at full size, in the bench's launch configuration:
    two whole images against the oracle, 256 sampled points against the
    correctly rounded brute-force sum, and the integer twin exact everywhere
    the oracle is cheap (first image) plus all-integer everywhere."""
    sh = CONFIGS["batched"]
    inp, ker = make_inputs(sh, seed=0)
    got, plan = run(sh, inp, ker, path)
    x, w = inp.numpy(), ker.numpy()
    ref2 = oracle.conv_eq1(x[:2], w)
    assert rel_l2(got[:2], ref2) <= TOL[path]
    rng = np.random.default_rng(0)
    pts = [(rng.integers(sh.N), rng.integers(sh.K), rng.integers(sh.H), rng.integers(sh.W)) for _ in range(256)]
    ref_pts = np.array([oracle.conv_eq1_point(x, w, *p) for p in pts])
    got_pts = np.array([got[p] for p in pts], dtype=np.float64)
    assert np.linalg.norm(got_pts - ref_pts) / np.linalg.norm(ref_pts) <= TOL[path]
    # integer twin
    xi, wi = make_inputs(sh, seed=1, kind="int")
    goti, _ = run(sh, xi, wi, path)
    assert np.all(goti == np.round(goti))
    refi = oracle.conv_eq1(xi.numpy()[:1], wi.numpy())
    assert np.array_equal(goti[:1].astype(np.float64), refi)
    for p in pts[:64]:
        assert goti[p] == oracle.conv_eq1_point(xi.numpy(), wi.numpy(), *p)


def test_auto_path_and_describe():
    for name, sh in CONFIGS.items():
        plan = conv.ConvPlan(*sh.as_tuple())
        d = plan.describe()
        assert d["path"] in ("fp32_simt", "fp32_tc")      # AUTO: fp32 precision only
        assert d["problem"]["N"] == sh.N and d["problem"]["W"] == sh.W
        assert d["model"]["model_us"] > 0
        assert d["kernels"] == plan.num_kernels


def test_argument_errors():
    sh = CONFIGS["tiny"]
    plan = conv.ConvPlan(*sh.as_tuple(), path="tf32", tile="halo=0")
    inp, ker = make_inputs(sh, seed=0)
    i, k = inp.cuda(), ker.cuda()
    out = plan.new_output()
    ws = plan.new_workspace()
    lib = conv.load_library()
    st = torch.cuda.current_stream().cuda_stream
    # misaligned input pointer
    assert lib.conv_run(plan._h, i.data_ptr() + 4, k.data_ptr(), out.data_ptr(), ws.data_ptr(), st) == 1
    # NULL output
    assert lib.conv_run(plan._h, i.data_ptr(), k.data_ptr(), None, ws.data_ptr(), st) == 1
    # out aliases in
    assert lib.conv_run(plan._h, i.data_ptr(), k.data_ptr(), i.data_ptr(), ws.data_ptr(), st) == 1
    # missing workspace on a tensor path
    assert lib.conv_run(plan._h, i.data_ptr(), k.data_ptr(), out.data_ptr(), None, st) == 1
    assert "NULL" in conv.last_error()
    with pytest.raises(conv.ConvError):
        conv.ConvPlan(1, 1, 1, 0, 1, 1, 1)
    with pytest.raises(conv.ConvError) as e:
        conv.ConvPlan(1, 4, 64, 4, 4, 130, 1, path="tf32")   # R > 128: past the TMA im2col box
    assert e.value.status == conv.CONV_ERR_INFEASIBLE


def test_run_host_end_to_end():
    sh = CONFIGS["r2"]
    inp, ker = make_inputs(sh, seed=0)
    plan = conv.ConvPlan(*sh.as_tuple(), path="tf32")
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    plan.run_host(inp.pin_memory(), ker.pin_memory(), out_h, dbuf)
    torch.cuda.synchronize()
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert rel_l2(out_h.numpy(), ref) <= TOL["tf32"]


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_run_host_split_k_plans(path):
    """conv_run_host with split-K plans: a batch-1 deep-C layer (the AUTO plan
    splits it) and a forced split count over a batch that the host pipeline
    cuts into image chunks (each chunk a smaller sub-problem of the plan):
    bit-identical to conv_run on device pointers, and within tolerance of
    the oracle."""
    from paper_2101_09808_b200.inputs import TABLE1
    cases = ((TABLE1["M9"], None), (Shape(N=3, K=256, C=512, H=7, W=7, R=3, S=3), "splits=4"))
    for sh, tile in cases:
        inp, ker = make_inputs(sh, seed=151)
        plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile, **sh.plan_kwargs())
        assert plan.describe()["tile"]["splits"] > 1
        dev_out = plan.run(inp.cuda(), ker.cuda())
        dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
        out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
        plan.run_host(inp.pin_memory(), ker.pin_memory(), out_h, dbuf)
        torch.cuda.synchronize()
        assert torch.equal(out_h, dev_out.cpu())
        ref = oracle.conv_eq1_strided(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), sh.U)
        assert rel_l2(out_h.numpy(), ref) <= 1e-5


def test_run_events_records_each_kernel():
    sh = CONFIGS["det"]
    inp, ker = make_inputs(sh, seed=0)
    for path in PATHS:
        plan = conv.ConvPlan(*sh.as_tuple(), path=path)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(plan.num_kernels + 1)]
        out = plan.new_output()
        plan.run_events(inp.cuda(), ker.cuda(), out, plan.new_workspace(), ev)
        torch.cuda.synchronize()
        ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(plan.num_kernels)]
        assert all(t >= 0 for t in ts)


@pytest.mark.parametrize("path", PATHS)
def test_run_host_pipelined_chunks_bit_identical(path):
    """conv_run_host splits a large batch into image chunks pipelined over
    three streams; every chunk runs the same k-order, so the result is
    bit-identical to the device-pointer conv_run."""
    sh = Shape(N=16, K=64, C=128, H=32, W=32, R=3, S=3)      # In = 9.5 MB -> 8 chunks
    inp, ker = make_inputs(sh, seed=13)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path)
    dev_out = plan.run(inp.cuda(), ker.cuda())
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(2):                                         # reuse the plan's pipeline
        out_h.zero_()
        plan.run_host(inp.pin_memory(), ker.pin_memory(), out_h, dbuf)
        torch.cuda.synchronize()
        assert np.array_equal(out_h.numpy(), dev_out.cpu().numpy())
    ref = oracle.conv_eq1(inp.numpy()[:2], ker.numpy())
    assert rel_l2(out_h.numpy()[:2], ref) <= TOL[path]


# FP32 SIMT v2 TMA staging (Win % 4 == 0): ragged image, row, channel-chunk
# and k tiles, row mode and pixel-group mode, 3x3 and 1x1, split-C
SIMT_TMA_CASES = [
    (Shape(N=5, K=44, C=13, H=9, W=14, R=3, S=3), "ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=9,bc=8"),
    (Shape(N=3, K=20, C=9, H=10, W=30, R=3, S=3), "ver=2,tk=4,tw=8,kg=2,pw=2,tn=1,th=10,bc=4"),
    (Shape(N=2, K=36, C=21, H=13, W=22, R=3, S=3), "ver=2,tk=8,tw=4,kg=2,pw=2,tn=1,th=7,bc=8"),
    (Shape(N=3, K=24, C=10, H=7, W=12, R=1, S=1), "ver=2,tk=4,tw=4,kg=2,pw=2,tn=2,th=7,bc=4"),
    (Shape(N=1, K=32, C=40, H=14, W=14, R=3, S=3), "ver=2,tk=4,tw=14,kg=4,pw=1,tn=1,th=14,bc=4,splits=4"),
]


@pytest.mark.parametrize("shape,tile", SIMT_TMA_CASES, ids=lambda x: x if isinstance(x, str) else "x".join(map(str, x.as_tuple())))
def test_simt_tma_staging_ragged(shape, tile):
    """The v2 TMA staging (one 4-D box of In per chunk, OOB zero-fill for
    columns >= Win, rows >= Hin, channels >= C, images >= N, plus one bulk
    copy of the packed Ker slab) on tiles that are ragged in every dimension:
    1e-5 against the double oracle and bit-exact on the integer twin."""
    inp, ker = make_inputs(shape, seed=31)
    got, plan = run(shape, inp, ker, "fp32_simt", tile=tile)
    assert plan.describe()["tile"]["staging"] == "tma"
    assert rel_l2(got, oracle.conv_eq1(inp.numpy(), ker.numpy())) <= TOL["fp32_simt"]
    xi, wi = make_inputs(shape, seed=32, kind="int")
    goti, _ = run(shape, xi, wi, "fp32_simt", tile=tile)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


# FP32 SIMT flat row mode (tile key flat=1): a CTA's 32*pw lanes take
# consecutive (image, row) slots across image boundaries; ragged batches
# (slot tiles past N), ragged k and channel chunks, H not a multiple of
# anything, one image (half the lanes idle), split-C
SIMT_FLAT_CASES = [
    (Shape(N=9, K=40, C=20, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4"),
    (Shape(N=9, K=40, C=20, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=2,pw=2,bc=8"),
    (Shape(N=5, K=44, C=13, H=9, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=8"),
    (Shape(N=3, K=24, C=11, H=5, W=14, R=3, S=3), "flat=1,tk=4,kg=2,pw=1,bc=4"),
    (Shape(N=1, K=16, C=8, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4"),
    (Shape(N=4, K=32, C=40, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4,splits=3"),
    (Shape(N=11, K=44, C=12, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=8,pw=1,bc=4"),
    (Shape(N=6, K=36, C=9, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=1,pw=2,bc=8"),
]


@pytest.mark.parametrize("shape,tile", SIMT_FLAT_CASES, ids=lambda x: x if isinstance(x, str) else "x".join(map(str, x.as_tuple())))
def test_simt_flat_row_mode(shape, tile):
    """Flat row-mode tiles: 1e-5 against the double oracle, bit-exact on the
    integer twin, and bit-identical to the per-image row-mode tile (every
    output row is the same thread-level FFMA2 sequence, only the lane that
    runs it differs)."""
    inp, ker = make_inputs(shape, seed=33)
    got, plan = run(shape, inp, ker, "fp32_simt", tile=tile)
    t = plan.describe()["tile"]
    assert t["flat"] == 1 and t["staging"] == "tma" and t["th"] == shape.H
    assert rel_l2(got, oracle.conv_eq1(inp.numpy(), ker.numpy())) <= TOL["fp32_simt"]
    per_image = f"ver=2,tk=4,tw=14,kg={t['kg']},pw=1,tn=1,th={shape.H},bc={t['bc']},flat=0"
    if t["splits"] > 1:
        per_image += f",splits={t['splits']}"
    ref_tile, p2 = run(shape, inp, ker, "fp32_simt", tile=per_image)
    assert p2.describe()["tile"]["flat"] == 0
    assert np.array_equal(got, ref_tile)
    xi, wi = make_inputs(shape, seed=34, kind="int")
    goti, _ = run(shape, xi, wi, "fp32_simt", tile=tile)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


# flat tiles whose last slot tiles run as the remainder launch (simt_rem_tiles):
# ceil(CTAs / 148) = k with (k - 1) * 148 CTAs holding all but `rem` slot tiles
SIMT_REM_CASES = [
    # 75 slot tiles x 2 k tiles = 150 CTAs: 74 main tiles + 1 remainder tile (8 one-warp CTAs), ragged last slot tile
    (Shape(N=171, K=32, C=8, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4", 1),
    # 2 k tiles of 8 channels (kg = 2), ragged K and C: 76 tiles -> 74 + 2 remainder tiles, odd channel count in 2-channel chunks
    (Shape(N=173, K=14, C=7, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=2,pw=1,bc=4", 2),
    # H = 9 rows per image (slot tiles cross image boundaries at other places)
    (Shape(N=267, K=32, C=6, H=9, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4", 2),
    # 3 rounds: 223 tiles x 2 = 446 CTAs, k = 4 -> 222 main tiles
    (Shape(N=509, K=32, C=4, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=2", 1),
    # split-C (r02e): 38 slot tiles x 2 k tiles x 2 splits = 152 CTAs -> 37 main tiles + 1 remainder tile whose CTAs
    # take the same channel ranges (12 + 10 of C = 22: ragged last chunk) in 2-channel chunks, into the same partial slabs
    (Shape(N=86, K=32, C=22, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4,splits=2", 1),
    # 3 splits of 2 + 2 + 1 chunks, 26 slot tiles x 2 x 3 = 156 CTAs -> 24 main + 2 remainder tiles
    (Shape(N=58, K=32, C=20, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4,splits=3", 2),
    # the batched layer's 8-GPU shard: 14 x 16 x 2 = 448 CTAs, k = 4 -> 13 main tiles (2.8 CTAs per SM) + 128 remainder CTAs
    (Shape(N=32, K=256, C=256, H=14, W=14, R=3, S=3), "flat=1,tk=4,kg=4,pw=1,bc=4,splits=2", 1),
]


@pytest.mark.parametrize("shape,tile,rem", SIMT_REM_CASES, ids=lambda x: x if isinstance(x, str) else str(x) if isinstance(x, int) else "x".join(map(str, x.as_tuple())))
def test_simt_remainder_launch(shape, tile, rem):
    """The remainder launch of a flat tile (the last slot tiles as one-warp
    CTAs beside the main grid): bit-identical to the same tile without it
    (rem=0: every output is the same thread-level FMA sequence), 1e-5 against
    the double oracle, integer twin exact, twice (the second run re-packs Ker
    while nothing of the first is in flight)."""
    inp, ker = make_inputs(shape, seed=51)
    plan = conv.ConvPlan(*shape.as_tuple(), path="fp32_simt", tile=tile)
    t = plan.describe()["tile"]
    assert t["flat"] == 1 and t["rem"] == rem, t
    plain = conv.ConvPlan(*shape.as_tuple(), path="fp32_simt", tile=tile + ",rem=0")
    assert plain.describe()["tile"]["rem"] == 0
    di, dk = inp.cuda(), ker.cuda()
    ref = plain.run(di, dk).cpu().numpy()
    out = plan.new_output()
    for _ in range(2):
        out.fill_(float("nan"))
        plan.run(di, dk, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)
    assert rel_l2(ref, oracle.conv_eq1(inp.numpy(), ker.numpy())) <= TOL["fp32_simt"]
    xi, wi = make_inputs(shape, seed=52, kind="int")
    goti = plan.run(xi.cuda(), wi.cuda()).cpu().numpy()
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


@pytest.mark.parametrize("shape", [Shape(N=171, K=32, C=8, H=14, W=14, R=1, S=3), Shape(N=3, K=30, C=5, H=16, W=14, R=1, S=3),
                                   Shape(N=2, K=16, C=8, H=9, W=10, R=1, S=3), Shape(N=2, K=16, C=8, H=9, W=12, R=3, S=1)],
                         ids=lambda sh: "x".join(map(str, sh.as_tuple())))
def test_simt_non_square_taps_with_tma_aligned_rows(shape):
    """R != S with Win % 4 == 0 (r02e fuzz regression): the TMA staging has
    instances for 1x1 and 3x3 taps only; such problems planned a TMA tile whose
    launch failed with invalid argument.  They take the cp.async layout (or
    v1), and match the oracle -- 1e-5, integer twin exact."""
    plan = conv.ConvPlan(*shape.as_tuple(), path="fp32_simt")
    assert plan.describe()["tile"]["staging"] == "cp.async"
    inp, ker = make_inputs(shape, seed=61)
    got = plan.run(inp.cuda(), ker.cuda()).cpu().numpy()
    assert rel_l2(got, oracle.conv_eq1(inp.numpy(), ker.numpy())) <= TOL["fp32_simt"]
    xi, wi = make_inputs(shape, seed=62, kind="int")
    goti = plan.run(xi.cuda(), wi.cuda()).cpu().numpy()
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


@pytest.mark.parametrize("n", [32, 64])
def test_run_host_simt_split_remainder_shards(n):
    """The batched layer's 8- and 4-GPU shards (r02e: 2-way split-C flat tiles
    with the remainder launch): conv_run_host's chunks (each a sub-batch with
    its own main / remainder grids and partial slabs) give the bits of
    conv_run, which match the oracle on sampled images at 1e-5."""
    import dataclasses
    sh = dataclasses.replace(CONFIGS["batched"], N=n)
    inp, ker = make_inputs(sh, seed=43)
    plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt")
    t = plan.describe()["tile"]
    assert t["flat"] == 1 and t["splits"] == 2 and t["rem"] == 1, t
    dev_out = plan.run(inp.cuda(), ker.cuda()).cpu().numpy()
    for i in (0, n // 2 + 1, n - 1):
        assert rel_l2(dev_out[i:i + 1], oracle.conv_eq1(inp.numpy()[i:i + 1], ker.numpy())) <= TOL["fp32_simt"]
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    ih, kh = inp.pin_memory(), ker.pin_memory()
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(2):
        out_h.fill_(float("nan"))
        plan.run_host(ih, kh, out_h, dbuf)
        torch.cuda.synchronize()
        assert np.array_equal(out_h.numpy(), dev_out)


@pytest.mark.parametrize("path", ["fp32_simt", "bf16"])
def test_run_host_batched_planned_chunks(path):
    """The bench's e2e call: conv_run_host on the batched layer with the
    modeled chunk plan (FP32 SIMT: a 1/8-wave head and one-wave chunks;
    tensor paths: equal chunks) -- bit-identical to conv_run, twice."""
    sh = CONFIGS["batched"]
    inp, ker = make_inputs(sh, seed=41)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path)
    chunks = plan.describe()["host_pipeline"]["chunks"]
    assert len(chunks) >= 4 and sum(chunks) == sh.N
    dev_out = plan.run(inp.cuda(), ker.cuda()).cpu().numpy()
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    ih, kh = inp.pin_memory(), ker.pin_memory()
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(2):
        out_h.fill_(float("nan"))
        plan.run_host(ih, kh, out_h, dbuf)
        torch.cuda.synchronize()
        assert np.array_equal(out_h.numpy(), dev_out)


FUSE_SHAPES = [CONFIGS["tiny"], CONFIGS["r2"], CONFIGS["pw"], CONFIGS["det"],
               Shape(N=5, K=64, C=40, H=6, W=2, R=3, S=3), Shape(N=2, K=40, C=70, H=8, W=10, R=1, S=1),
               Shape(N=7, K=96, C=200, H=10, W=14, R=3, S=3), Shape(N=3, K=32, C=16, H=62, W=30, R=3, S=3)]


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", FUSE_SHAPES, ids=lambda s: "x".join(map(str, s.as_tuple())))
def test_fused_transform_bit_identical_to_separate(path, shape):
    """The cooperative in-kernel transform produces the same workspace values
    (same rounding) and the main kernel the same k-order, so fuse=1 equals
    fuse=0 bit for bit; repeated runs of one plan (flags cleared by the Ker
    launch each time) keep matching when the inputs change."""
    assert coop_ok(shape), shape
    for cg in (1, 2):
        fused = conv.ConvPlan(*shape.as_tuple(), path=path, tile=f"cg={cg},fuse=1")
        assert fused.describe()["tile"]["fuse"] == 1
        sep = conv.ConvPlan(*shape.as_tuple(), path=path, tile=f"cg={cg},fuse=0,splits=1")
        out = fused.new_output()
        ws = fused.new_workspace()
        for seed in (21, 22, 23):
            inp, ker = make_inputs(shape, seed=seed)
            i, k = inp.cuda(), ker.cuda()
            fused.run(i, k, out, ws)
            ref = sep.run(i, k)
            torch.cuda.synchronize()
            assert torch.equal(out, ref)
        ref64 = oracle.conv_eq1(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()))
        assert rel_l2(out.cpu().numpy(), ref64) <= 1e-5


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("pre_c", [0, 64, 128, 192, 4096])
def test_fused_transform_prologue_depths(path, pre_c):
    """The repack launch converts the first pre_c channels of wave 0's input
    (the prologue) and the kernel's chunk pipeline the rest: every split
    gives the same bits as the separate repack (two waves of tiles)."""
    sh = Shape(N=160, K=64, C=256, H=14, W=14, R=3, S=3)
    inp, ker = make_inputs(sh, seed=41)
    i, k = inp.cuda(), ker.cuda()
    ref = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=0,cg=1,splits=1").run(i, k)
    for cg in (1, 2):
        plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=f"fuse=1,cg={cg},pre_c={pre_c}")
        d = plan.describe()["tile"]
        assert d["fuse"] == 1 and d["pre_c"] == min(pre_c, d["cp"])
        out = plan.run(i, k)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_fused_transform_cuda_graph_replay(path):
    """The bench replays conv_run from a CUDA graph: the chunk flags must be
    re-cleared inside the graph (by the Ker launch), so a replay with new
    input values recomputes everything."""
    sh = Shape(N=6, K=128, C=128, H=14, W=14, R=3, S=3)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=1")
    inp, ker = make_inputs(sh, seed=31)
    i, k = inp.cuda(), ker.cuda()
    out, ws = plan.new_output(), plan.new_workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.run(i, k, out, ws)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(i, k, out, ws, stream=s)
    for seed in (32, 33):
        inp2, ker2 = make_inputs(sh, seed=seed)
        i.copy_(inp2)
        k.copy_(ker2)
        g.replay()
        torch.cuda.synchronize()
        ref = oracle.conv_eq1(ROUND[path](inp2.numpy()), ROUND[path](ker2.numpy()))
        assert rel_l2(out.cpu().numpy(), ref) <= 1e-5


# ---- stride (PAPER.md:201 footnote; Table 1's * layers) ------
STRIDED = [
    Shape.strided(1, 128, 64, 56, 56, 3, 3, 2),     # R4*
    Shape.strided(1, 128, 64, 56, 56, 1, 1, 2),     # R5*
    Shape.strided(1, 64, 3, 224, 224, 7, 7, 2),     # R1*
    Shape.strided(1, 256, 128, 28, 28, 3, 3, 2),    # R7*
    Shape.strided(2, 40, 17, 13, 11, 3, 2, 2),      # odd extents, (Hin - R) % U != 0
    Shape.strided(3, 24, 8, 16, 15, 5, 3, 3),       # stride 3
]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", STRIDED, ids=lambda s: f"{s.N}x{s.K}x{s.C}x{s.Hin}x{s.Win}x{s.R}x{s.S}s{s.U}")
def test_strided_parity(path, shape):
    """Strided Eq. 1 on every path against the strided oracle: tolerance on
    real inputs (and 1e-5 against the oracle on the path's rounded inputs),
    bit-exact on the integer twin."""
    inp, ker = make_inputs(shape, seed=61)
    got, plan = run(shape, inp, ker, path)
    d = plan.describe()["problem"]
    assert (d["U"], d["Hin"], d["Win"], d["H"], d["W"]) == (shape.U, shape.Hin, shape.Win, shape.H, shape.W)
    ref = oracle.conv_eq1_strided(inp.numpy(), ker.numpy(), shape.U)
    assert got.shape == ref.shape
    assert rel_l2(got, ref) <= TOL[path]
    ref_r = oracle.conv_eq1_strided(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), shape.U)
    assert rel_l2(got, ref_r) <= 1e-5
    xi, wi = make_inputs(shape, seed=62, kind="int")
    goti, _ = run(shape, xi, wi, path)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1_strided(xi.numpy(), wi.numpy(), shape.U))


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_strided_fused_and_cta_groups_bit_identical(path):
    """A multi-wave strided layer: the fused in-kernel transform and both
    CTA-group sizes give the same bits as the separate repack."""
    sh = Shape.strided(160, 128, 64, 28, 28, 3, 3, 2)
    inp, ker = make_inputs(sh, seed=63)
    i, k = inp.cuda(), ker.cuda()
    ref = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=0,cg=1,splits=1", **sh.plan_kwargs()).run(i, k)
    for spec in ("fuse=0,cg=2,splits=1", "fuse=1,cg=1", "fuse=1,cg=2", "fuse=1,cg=2,pre_c=0"):
        out = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs()).run(i, k)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), spec
    ref64 = oracle.conv_eq1_strided(ROUND[path](inp.numpy()[:2]), ROUND[path](ker.numpy()), 2)
    assert rel_l2(ref[:2].cpu().numpy(), ref64) <= 1e-5


# ---- dilation (PAPER.md:201 footnote: "stride/dilation ... the general case")
DILATED = [
    Shape.strided(2, 128, 64, 60, 60, 3, 3, 1, 2),     # R4-like, D = 2
    Shape.strided(1, 64, 96, 41, 41, 3, 3, 2, 2),      # stride 2 and dilation 2
    Shape.strided(2, 40, 17, 23, 19, 3, 2, 1, 3),      # odd extents, R != S, D = 3
    Shape.strided(1, 72, 32, 40, 40, 5, 5, 1, 4),      # wide dilated window (17 x 17)
    Shape.strided(3, 24, 8, 21, 22, 1, 1, 2, 5),       # 1 x 1: dilation has no effect
]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", DILATED, ids=lambda s: f"{s.N}x{s.K}x{s.C}x{s.Hin}x{s.Win}x{s.R}x{s.S}s{s.U}d{s.D}")
def test_dilated_parity(path, shape):
    """Strided + dilated Eq. 1 on every path against the dilated oracle:
    tolerance on real inputs (and 1e-5 against the oracle on the path's
    rounded inputs), bit-exact on the integer twin."""
    inp, ker = make_inputs(shape, seed=81)
    got, plan = run(shape, inp, ker, path)
    d = plan.describe()["problem"]
    assert (d["U"], d["D"], d["Hin"], d["Win"], d["H"], d["W"]) == (shape.U, shape.D, shape.Hin, shape.Win,
                                                                     shape.H, shape.W)
    ref = oracle.conv_eq1_dilated(inp.numpy(), ker.numpy(), shape.U, shape.D)
    assert got.shape == ref.shape
    assert rel_l2(got, ref) <= TOL[path]
    ref_r = oracle.conv_eq1_dilated(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), shape.U, shape.D)
    assert rel_l2(got, ref_r) <= 1e-5
    xi, wi = make_inputs(shape, seed=82, kind="int")
    goti, _ = run(shape, xi, wi, path)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1_dilated(xi.numpy(), wi.numpy(), shape.U, shape.D))


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_dilated_fused_and_cta_groups_bit_identical(path):
    """A multi-wave dilated layer: the fused in-kernel transform (its chunk
    ranges cover the D(R-1) halo rows) and both CTA-group sizes give the
    same bits as the separate repack; sampled points against the oracle."""
    sh = Shape.strided(96, 128, 64, 32, 32, 3, 3, 1, 2)
    inp, ker = make_inputs(sh, seed=83)
    i, k = inp.cuda(), ker.cuda()
    ref = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=0,cg=1,splits=1", **sh.plan_kwargs()).run(i, k)
    for spec in ("fuse=0,cg=2,splits=1", "fuse=1,cg=1", "fuse=1,cg=2", "fuse=1,cg=2,pre_c=0", "fuse=1,cg=2,bn=64"):
        out = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs()).run(i, k)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), spec
    ref64 = oracle.conv_eq1_dilated(ROUND[path](inp.numpy()[:2]), ROUND[path](ker.numpy()), 1, 2)
    assert rel_l2(ref[:2].cpu().numpy(), ref64) <= 1e-5
    rng = np.random.default_rng(84)
    x, w = ROUND[path](inp.numpy()), ROUND[path](ker.numpy())
    got = ref.cpu().numpy()
    for _ in range(64):
        p = (rng.integers(sh.N), rng.integers(sh.K), rng.integers(sh.H), rng.integers(sh.W))
        v = oracle.conv_eq1_point(x, w, *p, stride=1, dilation=2)
        assert abs(got[p] - v) <= 1e-4 * (1 + abs(v)), p


# ---- zero padding ("same"-padded layers) -----------
PADDED = [
    Shape.strided(2, 128, 64, 56, 56, 3, 3, 1, 1, 1, 1),      # R4 "same"
    Shape.strided(1, 64, 3, 224, 224, 7, 7, 2, 1, 3, 3),      # R1* as in ResNet (pad 3)
    Shape.strided(1, 128, 64, 56, 56, 3, 3, 2, 1, 1, 1),      # R4* as in ResNet (pad 1)
    Shape.strided(2, 40, 17, 13, 11, 3, 2, 1, 1, 2, 0),       # asymmetric pads, R != S
    Shape.strided(1, 24, 8, 9, 10, 3, 3, 2, 2, 3, 1),         # stride + dilation + padding
    Shape.strided(2, 16, 5, 5, 6, 3, 3, 1, 1, 4, 3),          # pad > kernel: border outputs read only zeros
    Shape.strided(3, 24, 8, 16, 15, 1, 1, 1, 1, 2, 2),        # 1x1 with padding: zero rim
]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", PADDED,
                         ids=lambda s: f"{s.N}x{s.K}x{s.C}x{s.Hin}x{s.Win}x{s.R}x{s.S}s{s.U}d{s.D}p{s.ph}_{s.pw}")
def test_padded_parity(path, shape):
    """Zero-padded Eq. 1 on every path against the padded oracle: tolerance
    on real inputs (1e-5 against the oracle on the path's rounded inputs),
    bit-exact on the integer twin (the padding contributes exact zeros)."""
    inp, ker = make_inputs(shape, seed=91)
    got, plan = run(shape, inp, ker, path)
    d = plan.describe()["problem"]
    assert (d["ph"], d["pw"], d["Hin"], d["Win"], d["H"], d["W"]) == (shape.ph, shape.pw, shape.Hin, shape.Win,
                                                                       shape.H, shape.W)
    pad = (shape.ph, shape.pw)
    ref = oracle.conv_eq1_padded(inp.numpy(), ker.numpy(), shape.U, shape.D, pad)
    assert got.shape == ref.shape
    assert rel_l2(got, ref) <= TOL[path]
    ref_r = oracle.conv_eq1_padded(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), shape.U, shape.D, pad)
    assert rel_l2(got, ref_r) <= 1e-5
    xi, wi = make_inputs(shape, seed=92, kind="int")
    goti, _ = run(shape, xi, wi, path)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1_padded(xi.numpy(), wi.numpy(), shape.U, shape.D, pad))


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_padded_fused_and_cta_groups_bit_identical(path):
    """A multi-wave "same"-padded layer: the fused in-kernel transform (its
    chunk ranges clamp the padding rows), both CTA-group sizes and the
    separate repack give the same bits; sampled points against the oracle."""
    sh = Shape.strided(96, 128, 64, 32, 32, 3, 3, 1, 1, 1, 1)
    inp, ker = make_inputs(sh, seed=93)
    i, k = inp.cuda(), ker.cuda()
    ref = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=0,cg=1,splits=1", **sh.plan_kwargs()).run(i, k)
    for spec in ("fuse=0,cg=2,splits=1", "fuse=1,cg=1", "fuse=1,cg=2", "fuse=1,cg=2,pre_c=0", "fuse=1,cg=2,bn=64"):
        out = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs()).run(i, k)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), spec
    ref64 = oracle.conv_eq1_padded(ROUND[path](inp.numpy()[:2]), ROUND[path](ker.numpy()), 1, 1, 1)
    assert rel_l2(ref[:2].cpu().numpy(), ref64) <= 1e-5
    rng = np.random.default_rng(94)
    x, w = ROUND[path](inp.numpy()), ROUND[path](ker.numpy())
    got = ref.cpu().numpy()
    for _ in range(64):
        p = (rng.integers(sh.N), rng.integers(sh.K), rng.choice([0, sh.H - 1, rng.integers(sh.H)]), rng.integers(sh.W))
        v = oracle.conv_eq1_point(x, w, *p, padding=1)
        assert abs(got[p] - v) <= 1e-4 * (1 + abs(v)), p


@pytest.mark.parametrize("path", PATHS)
def test_table1_layers_same_padded(path):
    """Table 1's conv2d layers as the networks run them, with
    "same" padding R//2 (stride 2 layers: ceil(Hin/2) outputs): whole output
    vs the padded oracle for layers <= 0.3 GFLOP; for the larger ones 256
    sampled points (border rows and columns included), checked two ways:
    against the oracle on the path's rounded inputs at 1e-5 (the fp32
    accumulation, reading R5) and against the oracle on the real
    inputs at the path's tolerance."""
    from paper_2101_09808_b200.inputs import TABLE1_ROWS
    rng = np.random.default_rng(95)
    for name, K, C, HW, R, U in TABLE1_ROWS:
        sh = Shape.strided(1, K, C, HW, HW, R, R, U, 1, R // 2, R // 2)
        inp, ker = make_inputs(sh, seed=96)
        got, _ = run(sh, inp, ker, path)
        x, w = inp.numpy(), ker.numpy()
        if sh.flops <= 3e8:
            ref = oracle.conv_eq1_padded(x, w, U, 1, R // 2)
            assert rel_l2(got, ref) <= TOL[path], name
        else:
            pts = [(0, rng.integers(K), rng.choice([0, sh.H - 1, rng.integers(sh.H)]),
                    rng.choice([0, sh.W - 1, rng.integers(sh.W)])) for _ in range(256)]
            val = np.array([got[p] for p in pts])
            xr, wr = ROUND[path](x), ROUND[path](w)
            ref_r = np.array([oracle.conv_eq1_point(xr, wr, *p, stride=U, padding=R // 2) for p in pts])
            assert rel_l2(val, ref_r) <= 1e-5, name
            ref = np.array([oracle.conv_eq1_point(x, w, *p, stride=U, padding=R // 2) for p in pts])
            assert rel_l2(val, ref) <= TOL[path], name


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("splits", [1, 3, 8])
def test_general_conv_with_split_k(path, splits):
    """Stride, dilation, asymmetric zero padding and split-K together: a
    deep-C, small-output layer (the split-K regime) against the padded
    oracle; bit-exact on the integer twin; deterministic run to run."""
    sh = Shape.strided(1, 96, 320, 19, 17, 3, 3, 2, 2, 2, 1)
    spec = f"splits={splits}"
    inp, ker = make_inputs(sh, seed=131)
    got, plan = run(sh, inp, ker, path, tile=spec)
    assert plan.describe()["tile"]["splits"] == splits
    pad = (sh.ph, sh.pw)
    ref = oracle.conv_eq1_padded(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), sh.U, sh.D, pad)
    assert got.shape == ref.shape
    assert rel_l2(got, ref) <= 1e-5
    again, _ = run(sh, inp, ker, path, tile=spec)
    assert np.array_equal(got, again)
    xi, wi = make_inputs(sh, seed=132, kind="int")
    goti, _ = run(sh, xi, wi, path, tile=spec)
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1_padded(xi.numpy(), wi.numpy(), sh.U, sh.D, pad))


# ---- tiny-C tap expansion (explicit im2col in the layout transform) ---------
EXPAND = [
    Shape(N=2, K=32, C=3, H=40, W=38, R=3, S=3),                 # Y0-like 3x3 stem
    Shape.strided(1, 64, 3, 45, 45, 7, 7, 2, 1, 3, 3),           # R1-like 7x7 stride-2 "same" stem
    Shape.strided(2, 24, 1, 19, 17, 3, 3, 1, 2, 1, 2),           # C = 1, dilation, asymmetric padding
    Shape(N=3, K=40, C=8, H=9, W=11, R=5, S=3),                  # C = 8 (16 B of bf16), R != S
    Shape.strided(1, 16, 4, 30, 30, 3, 3, 9, 1),                 # stride 9 (past the TMA traversal limit)
]


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", EXPAND, ids=lambda s: f"{s.N}x{s.K}x{s.C}x{s.Hin}x{s.Win}x{s.R}x{s.S}s{s.U}d{s.D}p{s.ph}")
def test_tap_expansion_parity(path, shape):
    """The tap-expanded 1x1 plan (forced, the AUTO choice for tiny C) against
    the padded oracle: 1e-5 on the path's rounded inputs, bit-exact on the
    integer twin; the plain plan (expand=0, where TMA allows it) agrees
    within tolerance."""
    inp, ker = make_inputs(shape, seed=161)
    got, plan = run(shape, inp, ker, path, tile="expand=1")
    assert plan.describe()["tile"]["expand"] == 1
    pad = (shape.ph, shape.pw)
    ref = oracle.conv_eq1_padded(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), shape.U, shape.D, pad)
    assert got.shape == ref.shape
    assert rel_l2(got, ref) <= 1e-5
    xi, wi = make_inputs(shape, seed=162, kind="int")
    goti, _ = run(shape, xi, wi, path, tile="expand=1")
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1_padded(xi.numpy(), wi.numpy(), shape.U, shape.D, pad))
    if shape.U <= 8:
        plain, p0 = run(shape, inp, ker, path, tile="expand=0")
        assert p0.describe()["tile"]["expand"] == 0
        assert rel_l2(plain, got) <= 1e-5


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_tap_expansion_auto_graph_and_host(path):
    """Table 1's C = 3 stems take the expansion automatically; a captured
    graph replays it (new inputs each replay) and conv_run_host (image
    chunks: each chunk expands its own images) is bit-identical."""
    from paper_2101_09808_b200.inputs import TABLE1
    sh = Shape.strided(4, 32, 3, 68, 68, 3, 3, 1)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile="halo=0", **sh.plan_kwargs())
    assert plan.describe()["tile"]["expand"] == 1
    for name in ("Y0", "R1"):
        t = TABLE1[name]
        assert conv.ConvPlan(*t.as_tuple(), path=path, **t.plan_kwargs()).describe()["tile"]["expand"] == 1
    inp, ker = make_inputs(sh, seed=163)
    i, k = inp.cuda(), ker.cuda()
    out, ws = plan.new_output(), plan.new_workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.run(i, k, out, ws)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(i, k, out, ws, stream=s)
    for seed in (164, 165):
        inp2, ker2 = make_inputs(sh, seed=seed)
        i.copy_(inp2)
        k.copy_(ker2)
        g.replay()
        torch.cuda.synchronize()
        r2 = oracle.conv_eq1(ROUND[path](inp2.numpy()), ROUND[path](ker2.numpy()))
        assert rel_l2(out.cpu().numpy(), r2) <= 1e-5
    dev_out = out.clone()
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    plan.run_host(inp2.pin_memory(), ker2.pin_memory(), out_h, dbuf)
    torch.cuda.synchronize()
    assert torch.equal(out_h, dev_out.cpu())


@pytest.mark.parametrize("path", PATHS)
def test_table1_layers(path):
    """Every conv2d layer of PAPER.md:439 Table 1 (batch 1, stride 1/2, input
    extents as listed) on each path against the (strided) oracle: the whole
    output for layers <= 0.3 GFLOP, 64 sampled points for the larger ones."""
    from paper_2101_09808_b200.inputs import TABLE1
    rng = np.random.default_rng(70)
    for name, sh in TABLE1.items():
        inp, ker = make_inputs(sh, seed=71)
        got, _ = run(sh, inp, ker, path)
        x, w = inp.numpy(), ker.numpy()
        if sh.flops <= 3e8:
            ref = oracle.conv_eq1_strided(x, w, sh.U)
            assert rel_l2(got, ref) <= TOL[path], name
        else:
            pts = [(0, rng.integers(sh.K), rng.integers(sh.H), rng.integers(sh.W)) for _ in range(64)]
            ref = np.array([oracle.conv_eq1_point(x, w, *p, stride=sh.U) for p in pts])
            g = np.array([got[p] for p in pts], dtype=np.float64)
            assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= TOL[path], name


@pytest.mark.parametrize("path", ["tf32", "bf16"])
def test_run_host_fused_chunks_bit_identical(path):
    """conv_run_host splits the batch into image chunks; with a fused plan each
    chunk is a fused sub-problem whose flags the chunk's Ker launch clears on
    the shared flag region: results equal the device run bit for bit, twice."""
    sh = Shape(N=24, K=96, C=128, H=14, W=14, R=3, S=3)
    inp, ker = make_inputs(sh, seed=81)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=1")
    assert plan.describe()["tile"]["fuse"] == 1
    dev_out = plan.run(inp.cuda(), ker.cuda())
    sep = conv.ConvPlan(*sh.as_tuple(), path=path, tile="fuse=0,splits=1").run(inp.cuda(), ker.cuda())
    torch.cuda.synchronize()
    assert torch.equal(dev_out, sep)
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(2):
        out_h.zero_()
        plan.run_host(inp.pin_memory(), ker.pin_memory(), out_h, dbuf)
        torch.cuda.synchronize()
        assert np.array_equal(out_h.numpy(), dev_out.cpu().numpy())


FUSE_EDGE = [
    Shape(N=1, K=40, C=72, H=120, W=60, R=3, S=3),      # one image, several waves, C % 64 != 0, K tail
    Shape(N=9, K=200, C=24, H=18, W=22, R=5, S=1),      # small C (sub-128-B k-blocks), R != S
    Shape.strided(12, 64, 96, 30, 30, 3, 3, 2),         # strided + fused
]


@pytest.mark.parametrize("path", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", FUSE_EDGE, ids=lambda s: f"{s.N}x{s.K}x{s.C}x{s.Hin}x{s.Win}x{s.R}x{s.S}s{s.U}")
def test_fused_edge_shapes_and_graph_replay(path, shape):
    """Fused transform on awkward shapes, replayed from a CUDA graph with new
    input values: equal to the separate repack bit for bit, and to the oracle
    on the rounded inputs."""
    assert coop_ok(Shape(shape.N, shape.K, shape.C, shape.Hin - shape.R + 1, shape.Win - shape.S + 1, shape.R, shape.S))
    kw = shape.plan_kwargs()
    plan = conv.ConvPlan(*shape.as_tuple(), path=path, tile="fuse=1", **kw)
    sep = conv.ConvPlan(*shape.as_tuple(), path=path, tile="fuse=0,splits=1", **kw)
    inp, ker = make_inputs(shape, seed=82)
    i, k = inp.cuda(), ker.cuda()
    out, ws = plan.new_output(), plan.new_workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.run(i, k, out, ws, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(i, k, out, ws, stream=s)
    for seed in (83, 84):
        inp2, ker2 = make_inputs(shape, seed=seed)
        i.copy_(inp2)
        k.copy_(ker2)
        g.replay()
        ref = sep.run(i, k)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    ref64 = oracle.conv_eq1_strided(ROUND[path](inp2.numpy()), ROUND[path](ker2.numpy()), shape.U)
    assert rel_l2(out.cpu().numpy(), ref64) <= 1e-5


@pytest.mark.parametrize("path", PATHS)
def test_p10_k_shards_and_strided_shards_bit_identical(path):
    """k-shards (N = 1, SURVEY Sec. 8(e) secondary split) and n-shards of a
    strided layer equal the slices of the 1-GPU result bit for bit: each
    rank's plan may re-tile, the k-order per output does not change (P10)."""
    from paper_2101_09808_b200.shard import local_inputs, shard
    for sh, dim, worlds in ((Shape(N=1, K=256, C=64, H=28, W=28, R=3, S=3), "k", (2, 4)),
                            (Shape.strided(8, 64, 32, 29, 29, 3, 3, 2), "n", (2, 4))):
        inp, ker = make_inputs(sh, seed=95)
        full, _ = run(sh, inp, ker, path, tile="splits=1")
        for world in worlds:
            for r in range(world):
                spec = shard(sh, world, r, dim=dim)
                li, lk = local_inputs(spec, inp, ker)
                got, _ = run(spec.local, li, lk, path, tile="splits=1")
                ref = full[spec.start:spec.stop] if dim == "n" else full[:, spec.start:spec.stop]
                assert np.array_equal(got, ref), (dim, world, r)


def _random_shapes(n, seed):
    """Seeded random general problems (stride, dilation, asymmetric padding),
    small enough for the oracle: the selector then picks whatever it picks
    (plain / tap-expanded / split plans, SIMT v1 / v2)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        R, S = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        U, D = int(rng.choice([1, 1, 2, 3])), int(rng.choice([1, 1, 2]))
        ph, pw = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        C = int(rng.choice([1, 2, 3, 5, 8, 16, 33, 64, 130]))
        K = int(rng.choice([1, 7, 16, 32, 40, 64, 100, 256]))
        N = int(rng.integers(1, 4))
        Hin, Win = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        if Hin + 2 * ph < D * (R - 1) + 1 or Win + 2 * pw < D * (S - 1) + 1:
            continue
        sh = Shape.strided(N, K, C, Hin, Win, R, S, U, D, ph, pw)
        if sh.flops > 2e8:
            continue
        out.append(sh)
    return out


@pytest.mark.parametrize("path", PATHS)
def test_random_general_shapes(path):
    """40 seeded random problems on every path: bit-exact on the integer
    twin, relL2 <= 1e-5 against the padded oracle on the path's rounded
    inputs.  Shapes the path cannot run must fail as INFEASIBLE, never with
    a wrong result."""
    ran = 0
    for i, sh in enumerate(_random_shapes(40, 2026)):
        pad = (sh.ph, sh.pw)
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path=path, **sh.plan_kwargs())
        except conv.ConvError as e:
            assert e.status == conv.CONV_ERR_INFEASIBLE, (sh, e)
            continue
        xi, wi = make_inputs(sh, seed=200 + i, kind="int")
        goti = plan.run(xi.cuda(), wi.cuda())
        torch.cuda.synchronize()
        refi = oracle.conv_eq1_padded(xi.numpy(), wi.numpy(), sh.U, sh.D, pad)
        assert np.array_equal(goti.cpu().numpy().astype(np.float64), refi), (sh, plan.describe()["tile"])
        inp, ker = make_inputs(sh, seed=300 + i)
        got = plan.run(inp.cuda(), ker.cuda())
        torch.cuda.synchronize()
        ref = oracle.conv_eq1_padded(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), sh.U, sh.D, pad)
        if np.linalg.norm(ref) > 0:
            assert rel_l2(got.cpu().numpy(), ref) <= 1e-5, (sh, plan.describe()["tile"])
        ran += 1
    assert ran >= 30


def test_concurrent_all_resident_plans_on_two_streams():
    """Plans whose main kernel needs every CTA resident at once -- the fused
    In transform (CTAs wait on chunks other CTAs convert) and split-K (a
    tile's splits wait on each other) -- launched back to back on two
    streams with no host synchronisation in between.  The library serialises
    such launches per device (tc.cu ResidentChain), so no grid waits on CTAs
    that cannot be scheduled (the watchdog would trap and poison the
    context) and every result equals its plan run alone, bit for bit."""
    sh_f = Shape(N=32, K=256, C=256, H=14, W=14, R=3, S=3)
    sh_s = Shape.strided(1, 96, 320, 19, 17, 3, 3, 2, 2, 2, 1)
    cases = [(sh_f, "bf16", "fuse=1,cg=2"), (sh_f, "tf32", "fuse=1,cg=1"), (sh_s, "bf16", "splits=8"),
             (sh_s, "tf32", "splits=3")]
    plans, args, refs = [], [], []
    for i, (sh, path, spec) in enumerate(cases):
        inp, ker = make_inputs(sh, seed=140 + i)
        p = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs())
        d = p.describe()["tile"]
        assert d["fuse"] == 1 or d["splits"] > 1
        a = (inp.cuda(), ker.cuda())
        refs.append(p.run(*a))
        torch.cuda.synchronize()
        plans.append(p)
        args.append(a)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[p.new_output() for _ in range(3)] for p in plans]
    wss = [[p.new_workspace() for _ in range(3)] for p in plans]
    for it in range(3):
        for i, p in enumerate(plans):
            p.run(*args[i], out=outs[i][it], workspace=wss[i][it], stream=streams[i % 2])
    torch.cuda.synchronize()
    for i in range(len(plans)):
        for it in range(3):
            assert torch.equal(outs[i][it], refs[i]), (cases[i], it)


@pytest.mark.parametrize("split", [6, 9])
def test_fp32_tc_split_pairs(split):
    """FP32_TC with 6 (i + j <= 2) and 9 (all) bf16 piece pairs: relL2 at the
    FP32 tolerance on real data over tile variants (CTA pair / single, split-K,
    BN), bit-exact on the integer twin, and its error no larger than a few
    times the FP32 SIMT path's on the same inputs."""
    sh = Shape(N=2, K=96, C=80, H=17, W=19, R=3, S=3)
    inp, ker = make_inputs(sh, seed=150)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    simt, _ = run(sh, inp, ker, "fp32_simt")
    e_simt = rel_l2(simt, ref)
    for spec in (f"split={split}", f"split={split},cg=1", f"split={split},cg=2,bn=64",
                 f"split={split},splits=4,cg=1"):
        try:
            got, plan = run(sh, inp, ker, "fp32_tc", tile=spec)
        except conv.ConvError as e:
            assert e.status == conv.CONV_ERR_INFEASIBLE and "splits" in spec
            continue
        d = plan.describe()
        assert d["path"] == "fp32_tc" and d["tile"]["split"] == split
        e = rel_l2(got, ref)
        assert e <= 1e-5 and e <= 4 * e_simt + 1e-7, (spec, e, e_simt)
    xi, wi = make_inputs(sh, seed=151, kind="int")
    goti, _ = run(sh, xi, wi, "fp32_tc", tile=f"split={split}")
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


def test_fp32_tc_extreme_magnitudes():
    """Inputs spanning many binades (|x| from 2^-60 to 2^60, both signs): the
    exact 3-piece split keeps every significand bit, so the result still
    matches the oracle at the FP32 tolerance (a 2-piece split or a TF32
    rounding would not)."""
    sh = Shape(N=1, K=32, C=48, H=12, W=12, R=3, S=3)
    g = torch.Generator().manual_seed(160)
    mant = torch.rand(sh.in_shape, generator=g) + 1.0
    ex = torch.randint(-60, 61, sh.in_shape, generator=g).to(torch.float32)
    sign = torch.randint(0, 2, sh.in_shape, generator=g).to(torch.float32) * 2 - 1
    inp = (sign * mant * torch.pow(2.0, ex)).contiguous()
    ker = (torch.rand(sh.ker_shape, generator=g) * 2 - 1).contiguous()
    got, _ = run(sh, inp, ker, "fp32_tc")
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert rel_l2(got, ref) <= 1e-5


HALO = [CONFIGS["tiny"], CONFIGS["r2"], CONFIGS["pw"], CONFIGS["det"],
        Shape(N=3, K=40, C=5, H=9, W=14, R=3, S=3),           # tiny C, several images, ragged K
        Shape(N=2, K=256, C=64, H=13, W=11, R=3, S=3),        # BN 256, odd extents
        Shape(N=1, K=7, C=17, H=30, W=29, R=2, S=3),          # R != S, ragged everything
        Shape(N=1, K=96, C=24, H=20, W=40, R=5, S=5)]         # 5x5 taps, halo 4 rows


@pytest.mark.parametrize("path", ["bf16", "tf32"])
@pytest.mark.parametrize("shape", HALO, ids=lambda s: "x".join(map(str, s.as_tuple())))
def test_halo_kernel_parity(path, shape):
    """The single-launch halo kernel (halo.cu: the input tile staged once per
    CTA, filter taps as shifted tcgen05 descriptors over the padded output
    grid): oracle parity on real inputs (path tolerance; 1e-5 against the
    rounded-input oracle), bit-exact on the integer twin, and bit-identical
    to the two-launch im2col kernel (same k order: taps, then channels)."""
    inp, ker = make_inputs(shape, seed=170)
    try:
        got, plan = run(shape, inp, ker, path, tile="halo=1")
    except conv.ConvError as e:
        assert e.status == conv.CONV_ERR_INFEASIBLE
        pytest.skip(f"not eligible: {e}")
    d = plan.describe()
    assert d["tile"]["halo"] == 1 and d["kernels"] == 2 and 0 < d["workspace_bytes"] <= 9 * 256 * 128 * 4
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert rel_l2(got, ref) <= TOL[path]
    ref_r = oracle.conv_eq1(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()))
    assert rel_l2(got, ref_r) <= 1e-5
    plain, _ = run(shape, inp, ker, path, tile="fuse=0,cg=1,splits=1,expand=0")
    assert np.array_equal(got, plain)
    xi, wi = make_inputs(shape, seed=171, kind="int")
    goti, _ = run(shape, xi, wi, path, tile="halo=1")
    assert np.array_equal(goti.astype(np.float64), oracle.conv_eq1(xi.numpy(), wi.numpy()))


def _guarded(t, pad, fill):
    """A copy of t placed in the middle of a larger buffer whose `pad`
    elements on each side hold `fill` (canaries)."""
    n = t.numel()
    buf = torch.full((n + 2 * pad,), fill, dtype=torch.float32, device="cuda")
    buf[pad:pad + n] = t.reshape(-1).cuda()
    return buf, buf[pad:pad + n].view(t.shape)


GUARD_CASES = [
    ("tiny", CONFIGS["tiny"], "fp32_simt", None), ("tiny", CONFIGS["tiny"], "fp32_tc", None),
    ("tiny", CONFIGS["tiny"], "tf32", None), ("tiny", CONFIGS["tiny"], "bf16", "halo=1"),
    ("r2", CONFIGS["r2"], "fp32_simt", None), ("r2", CONFIGS["r2"], "bf16", None),
    ("fused-2wave", Shape(N=160, K=256, C=256, H=14, W=14, R=3, S=3), "bf16", "fuse=1,cg=2"),
    ("fused-cg1", Shape(N=24, K=128, C=64, H=14, W=14, R=3, S=3), "tf32", "fuse=1,cg=1"),
    ("splitk-8", Shape.strided(1, 96, 320, 19, 17, 3, 3, 2, 2, 2, 1), "bf16", "splits=8"),
    ("splitk-3", Shape(N=1, K=128, C=256, H=7, W=7, R=3, S=3), "tf32", "splits=3"),
    ("simt-splitc", Shape(N=1, K=64, C=256, H=7, W=7, R=3, S=3), "fp32_simt", "splits=4"),
    ("fp32tc-promote", Shape(N=2, K=256, C=128, H=14, W=14, R=3, S=3), "fp32_tc", None),
    ("expand", Shape.strided(2, 32, 3, 34, 34, 3, 3, 1), "bf16", "expand=1"),
]


@pytest.mark.parametrize("case", GUARD_CASES, ids=lambda c: f"{c[0]}-{c[2]}")
def test_guard_bands_no_out_of_bounds_access(case):
    """compute-sanitizer is closed on this pool (profiles/r02/sanitizer_closed.log),
    so out-of-bounds accesses are checked with guard bands instead: Out and
    the workspace sit between canary regions that must be untouched after the
    run (no stray writes), In and Ker between NaN regions (a stray read that
    reached a valid output would make it NaN: the oracle comparison catches
    it), and two runs are bit-identical (no races on the cross-CTA flags /
    counters).  The multi-wave fused plan and the split-K plans are the ones
    whose CTAs wait on each other."""
    name, sh, path, tile = case
    pad = 4096
    inp, ker = make_inputs(sh, seed=180)
    _, gin = _guarded(inp, pad, float("nan"))
    _, gker = _guarded(ker, pad, float("nan"))
    plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile, **sh.plan_kwargs())
    canary = 1234.5
    obuf, gout = _guarded(torch.zeros(sh.out_shape), pad, canary)
    wsn = max(plan.workspace_bytes, 4)
    wbuf = torch.full(((wsn + 255) // 4 + 2 * pad + 64,), canary, dtype=torch.float32, device="cuda")
    off = pad + 64 - (pad + 64) % 64                               # 256-B aligned workspace start
    ws_view = wbuf[off:off + (wsn + 3) // 4]
    outs = []
    for _ in range(2):
        plan.run(gin, gker, gout, ws_view.view(torch.uint8)[:wsn] if plan.workspace_bytes else None)
        torch.cuda.synchronize()
        outs.append(gout.clone())
    assert torch.all(obuf[:pad] == canary) and torch.all(obuf[-pad:] == canary), "write before/after Out"
    assert torch.all(wbuf[:off] == canary) and torch.all(wbuf[off + (wsn + 3) // 4:] == canary), \
        "write outside the workspace"
    assert torch.equal(outs[0], outs[1]), "two runs differ"
    got = outs[0].cpu().numpy()
    assert np.all(np.isfinite(got)), "a NaN from outside In / Ker reached an output"
    pad_hw = (sh.ph, sh.pw)
    ref = oracle.conv_eq1_padded(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), sh.U, sh.D, pad_hw)
    assert rel_l2(got, ref) <= 1e-5          # vs the oracle on the path's rounded inputs


def test_fp32_tc_compact_layout_subprocess():
    """The compact FP32_TC workspace (default; CONV_SPLIT_COMPACT=1: the 3 bf16
    pieces once, pair blocks mapped to pieces in the producer) gives the same
    result bit for bit as the default 6-pair layout (same products, same
    k order) as the 6-pair layout (=0), in fresh processes (the knob is read once)."""
    import os
    import subprocess
    import sys
    code = """
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import Shape, make_inputs
sh = Shape(N=3, K=96, C=128, H=10, W=12, R=3, S=3)
inp, ker = make_inputs(sh, seed=190)
p = conv.ConvPlan(*sh.as_tuple(), path="fp32_tc")
out = p.run(inp.cuda(), ker.cuda()).cpu().numpy()
np.save(sys.argv[1], out)
print(p.workspace_bytes)
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        for v in ("0", "1"):
            f = os.path.join(d, f"o{v}.npy")
            r = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True, timeout=300,
                               env={**os.environ, "CONV_SPLIT_COMPACT": v})
            assert r.returncode == 0, r.stderr[-2000:]
            res[v] = (np.load(f), int(r.stdout.strip().splitlines()[-1]))
    assert res["1"][1] < res["0"][1]                      # the compact workspace is smaller
    assert np.array_equal(res["0"][0], res["1"][0])


def test_simt_ker_pack_forms_subprocess():
    """The FP32 SIMT Ker pack (KCRS -> [K/bko][C][R][S][bko], a permutation):
    the tiled transpose (CONV_SIMT_PACK_GATHER=0, 16-B units when C*R*S % 4
    == 0, scalar otherwise) and the per-element gather (=1) give bit-identical
    convolutions, on ragged k tiles and odd C*R*S, in fresh processes (the
    knob is read once)."""
    import os
    import subprocess
    import sys
    code = """
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import Shape, make_inputs
outs = []
for sh in (Shape(N=2, K=44, C=13, H=9, W=14, R=3, S=3), Shape(N=1, K=70, C=12, H=6, W=7, R=3, S=3),
           Shape(N=1, K=36, C=40, H=5, W=9, R=1, S=1)):
    inp, ker = make_inputs(sh, seed=77)
    p = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt")
    outs.append(p.run(inp.cuda(), ker.cuda()).cpu().numpy())
np.savez(sys.argv[1], *outs)
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    res = {}
    with tempfile.TemporaryDirectory() as d:
        for v in ("0", "1"):
            f = os.path.join(d, f"o{v}.npz")
            r = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True, timeout=300,
                               env={**os.environ, "CONV_SIMT_PACK_GATHER": v})
            assert r.returncode == 0, r.stderr[-2000:]
            z = np.load(f)
            res[v] = [z[k] for k in sorted(z.files)]
    for a, b in zip(res["0"], res["1"]):
        assert np.array_equal(a, b)
