"""CPU-only checks of the C ABI: the library loads, exports every symbol
include/conv.h declares, refuses to plan without an sm_100 device (no CPU
fallback), and its data-movement model reproduces the paper's worked numbers.
"""
import itertools
import os
import re

import pytest
import torch

from paper_2101_09808_b200 import conv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2101_09808_b200 import build
    build.build()
    return conv.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "conv.h")).read()
    return sorted(set(re.findall(r"CONV_API[^;(]*?\b(conv_\w+)\s*\(", src)))


def test_header_declares_what_binding_lists():
    assert declared_symbols() == sorted(conv.EXPORTED)


def test_exports_every_declared_symbol(lib):
    out = os.popen(f"nm -D --defined-only {conv.LIB_PATH}").read()
    exported = set(re.findall(r" T (conv_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(lib, s)


def test_version(lib):
    assert "sm_100a" in conv.version()


def test_library_has_no_cpu_fallback(lib):
    """Without an sm_100 device conv_plan_create fails loudly."""
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(conv.ConvError) as e:
        conv.ConvPlan(1, 16, 16, 8, 8, 3, 3)
    assert e.value.status in (conv.CONV_ERR_UNSUPPORTED_DEVICE, conv.CONV_ERR_INVALID_ARGUMENT)


def test_invalid_extents_rejected_before_device(lib):
    h = lib.conv_plan_create(1, 1, 1, 0, 1, 1, 1)
    assert not h
    assert "extent must be >= 1" in conv.last_error()
    h = lib.conv_plan_create(70000, 70000, 1, 1, 1, 1, 1)
    assert not h
    assert "2^31" in conv.last_error()


def test_null_plan_calls_are_safe(lib):
    lib.conv_plan_destroy(None)
    assert lib.conv_plan_workspace_bytes(None) == 0
    assert lib.conv_plan_num_kernels(None) == -1
    assert lib.conv_run(None, None, None, None, None, None) == conv.CONV_ERR_INVALID_ARGUMENT


# ---- the selector's model: worked numbers -----------------

def test_eq5_worked_example(lib):
    """Eq. 5 at N=(n1,k4,c2,r1,s1,h4,w4), T=(1,2,2,1,1,2,2):
    substituting into the printed formula gives
    2*[4 + 1*2*(2*2*8 + 1*2*2*4)] = 200 = Out 128 + In 64 + Ker 8."""
    Nx = dict(n=1, k=4, c=2, r=1, s=1, h=4, w=4)
    T = dict(n=1, k=2, c=2, r=1, s=1, h=2, w=2)
    dv_in, dv_ker, dv_out = conv.model_dv(["k", "c", "r", "s", "n", "h", "w"], Nx, T)
    assert (dv_in, dv_ker, dv_out) == (64.0, 8.0, 128.0)


def eq5(Nx, T):
    """Eq. 5 exactly as printed."""
    n, k, c, r, s, h, w = (Nx[x] for x in "nkcrshw")
    tn, tk, tc, tr, ts, th, tw = (T[x] for x in "nkcrshw")
    return (k / tk) * (c / tc) * (r / tr) * (s / ts) * (
        tk * tc * tr * ts + (n / tn) * (h / th) * (2 * (w / tw) * tn * tk * th * tw + tn * tc * (th + tr - 1) * (w + ts - 1)))


def test_eq5_class_members_equal_printed_formula(lib):
    """Every permutation in the class <{kt,ct,rt,st},{nt,ht},wt> (4!*2! = 48
    members) gives Eq. 5's value at random divisible tiles."""
    import random
    rng = random.Random(0)
    for _ in range(20):
        Nx, T = {}, {}
        for x in "nkcrshw":
            t = rng.choice([1, 2, 3])
            T[x] = t
            Nx[x] = t * rng.choice([1, 2, 4])
        expected = eq5(Nx, T)
        for outer in itertools.permutations("kcrs"):
            for mid in itertools.permutations("nh"):
                tot = sum(conv.model_dv(list(outer) + list(mid) + ["w"], Nx, T))
                assert abs(tot - expected) <= 1e-9 * expected


def test_eq3_matmul(lib):
    """Eq. 3: N=4, T=2 => 64*(1/2+1/2+2/4) = 96."""
    Nx = dict(i=4, j=4, k=4)
    T = dict(i=2, j=2, k=2)
    assert conv.model_dv_matmul(["i", "j", "k"], Nx, T) == 96.0
    for Ni, Nj, Nk, Ti, Tj in [(8, 6, 10, 2, 3), (16, 16, 4, 4, 8)]:
        got = conv.model_dv_matmul(["i", "j", "k"], dict(i=Ni, j=Nj, k=Nk), dict(i=Ti, j=Tj, k=2))
        assert abs(got - Ni * Nj * Nk * (1 / Ti + 1 / Tj + 2 / Nk)) < 1e-9


def test_footprints(lib):
    """Eq. 4 LHS: T=(n1,k2,c2,r1,s1,h2,w2) -> 8 + 4 + 8 = 20;
    In footprint with T=(n1,c3,h2,w2,r3,s3) is 1*3*4*4 = 48."""
    assert conv.model_footprint(dict(n=1, k=2, c=2, r=1, s=1, h=2, w=2)) == 20.0
    fp = conv.model_footprint(dict(n=1, k=1, c=3, r=3, s=3, h=2, w=2))
    assert fp == 48 + 1 * 3 * 3 * 3 + 1 * 1 * 2 * 2


def test_single_tile_permutation_invariance(lib):
    """T = N: every permutation moves each tensor exactly once (Out twice)."""
    Nx = dict(n=2, k=3, c=4, r=3, s=2, h=5, w=6)
    exp = (2 * 4 * (5 + 3 - 1) * (6 + 2 - 1), 3 * 4 * 3 * 2, 2 * 2 * 3 * 5 * 6)
    for perm in list(itertools.permutations("nkcrshw"))[::97]:
        assert conv.model_dv(list(perm), Nx, Nx) == exp


def test_model_rejects_bad_input(lib):
    with pytest.raises(ValueError):
        conv.model_dv(list("nkcrshw"), dict(n=1, k=1, c=1, r=1, s=1, h=1, w=1), dict(n=2, k=1, c=1, r=1, s=1, h=1, w=1))
    with pytest.raises(KeyError):
        conv.model_dv(list("nkcrshx"), dict(n=1, k=1, c=1, r=1, s=1, h=1, w=1), dict(n=1, k=1, c=1, r=1, s=1, h=1, w=1))


# ---- the selector on a described B200 (offline plans, no device) -------------

def _offline(shape, path, tile=None):
    return conv.ConvPlan(*shape.as_tuple(), path=path, tile=tile, offline_device=conv.B200)


def test_simt_remainder_launch_plan(lib):
    """Host logic of the flat tile's remainder launch (simt_rem_tiles): on 148
    SMs the batched layer's 112 slot tiles x 16 k tiles = 1792 CTAs are 12.1
    per SM, so 111 tiles (1776 CTAs = 12 per SM) stay in the main grid and one
    runs as 64 one-warp CTAs; 253 images (111 slot tiles) need none; the tile
    key rem=0 turns it off; a remainder that would need more than one warp
    per SM is not taken."""
    import dataclasses
    from paper_2101_09808_b200.inputs import CONFIGS, Shape
    flat = "flat=1,tk=4,kg=4,pw=1,bc=4"
    sh = CONFIGS["batched"]
    d = _offline(sh, "fp32_simt").describe()
    assert d["tile"]["flat"] == 1 and d["tile"]["rem"] == 1, d["tile"]
    assert _offline(sh, "fp32_simt", flat + ",rem=0").describe()["tile"]["rem"] == 0
    assert _offline(dataclasses.replace(sh, N=253), "fp32_simt", flat).describe()["tile"]["rem"] == 0
    # 128 images: 56 slot tiles x 16 = 896 CTAs, k = 7, 55 main tiles (880 <= 888), 1 remainder tile
    assert _offline(dataclasses.replace(sh, N=128), "fp32_simt", flat).describe()["tile"]["rem"] == 1
    # 240 images: 105 tiles, k = 12, 101 main tiles -> 4 remainder tiles = 256 warps > 148: not taken
    assert _offline(dataclasses.replace(sh, N=240), "fp32_simt", flat).describe()["tile"]["rem"] == 0
    # fewer CTAs than SMs: nothing to take off
    assert _offline(Shape(N=8, K=32, C=8, H=14, W=14, R=3, S=3), "fp32_simt", flat).describe()["tile"]["rem"] == 0
    # 1x3 taps: the TMA staging (and with it flat tiles and the remainder launch) has 1x1 / 3x3 instances only
    sh13 = Shape(N=171, K=32, C=8, H=14, W=14, R=1, S=3)
    assert _offline(sh13, "fp32_simt").describe()["tile"]["staging"] == "cp.async"
    with pytest.raises(conv.ConvError):
        _offline(sh13, "fp32_simt", flat)
    assert _offline(Shape(N=171, K=32, C=8, H=14, W=14, R=3, S=3), "fp32_simt", flat).describe()["tile"]["rem"] == 1
    # split-C: a slot tile is k tiles x splits CTAs (N = 32: 14 x 16 x 2 = 448, k = 4, 13 main tiles, 128 remainder CTAs);
    # 4 splits would need 256 remainder CTAs: not taken
    assert _offline(dataclasses.replace(sh, N=32), "fp32_simt", flat + ",splits=2").describe()["tile"]["rem"] == 1
    assert _offline(dataclasses.replace(sh, N=32), "fp32_simt", flat + ",splits=4").describe()["tile"]["rem"] == 0
    # conv_run_host runs its chunks with the finer kg = 4 flat tile (61-image one-wave chunks) while
    # the device plan is the kg = 8 tile; a forced kg keeps the plan's tile
    hp = d["host_pipeline"]
    assert d["tile"]["kg"] == 8 and hp["simt_kg"] == 4 and sum(hp["chunks"]) == sh.N and max(hp["chunks"]) == 61, hp
    hp8 = _offline(sh, "fp32_simt", "flat=1,tk=4,kg=8,pw=1,bc=4").describe()["host_pipeline"]
    assert hp8["simt_kg"] == 8 and max(hp8["chunks"]) == 84, hp8
    # the modeled time with the remainder launch is below the one without
    with_rem = _offline(sh, "fp32_simt", flat).describe()["model"]["model_us"]
    without = _offline(sh, "fp32_simt", flat + ",rem=0").describe()["model"]["model_us"]
    assert with_rem < without


@pytest.mark.parametrize("path", ["fp32_simt", "tf32", "bf16"])
def test_selector_respects_capacity(lib, path):
    """Every emitted tile satisfies the per-level capacity constraints (Eq. 4
    per level): shared memory per CTA <= opt-in, TMEM 2*BN <= 512."""
    import dataclasses
    from paper_2101_09808_b200.inputs import CONFIGS, Shape
    shapes = list(CONFIGS.values()) + [Shape(1, 5, 3, 7, 9, 3, 3), Shape(2, 300, 700, 9, 10, 1, 1),
                                       Shape(1, 64, 4096, 3, 3, 3, 3), Shape(1, 8, 8, 2, 3000, 1, 5)]
    for sh in shapes:
        d = _offline(sh, path).describe()
        assert d["path"] == path
        assert d["model"]["smem_bytes"] <= conv.B200["smem_optin"]
        if path != "fp32_simt":
            assert 2 * d["tile"]["bn"] <= 512 and d["tile"]["cg"] in (1, 2)
            assert d["tile"]["cp"] >= sh.C and (d["tile"]["cp"] * (2 if path == "bf16" else 4)) % 32 == 0
        else:
            t = d["tile"]
            lanes = t["threads"] // 32 // t["kg"] * 32           # output-row slots per k group
            assert t["threads"] <= 512
            if t["flat"]:
                # flat row mode: whole images (th = H, TW = W), 32*pw consecutive
                # (image, row) slots per CTA, tn = the images such a run can span
                assert t["th"] == sh.H and t["tw"] == sh.W and t["staging"] == "tma"
                assert t["tn"] == min(sh.N, (lanes + sh.H - 2) // sh.H + 1)
            else:
                assert t["tn"] * t["th"] * sh.W <= lanes * t["tw"]


def test_selector_forced_tiles(lib):
    from paper_2101_09808_b200.inputs import CONFIGS
    sh = CONFIGS["batched"]
    for cg in (1, 2):
        for bn in (32, 128, 256):
            d = _offline(sh, "bf16", tile=f"bn={bn},cg={cg}").describe()
            assert (d["tile"]["bn"], d["tile"]["cg"]) == (bn, cg)
    with pytest.raises(conv.ConvError) as e:
        _offline(sh, "bf16", tile="bn=48")
    assert e.value.status == conv.CONV_ERR_INFEASIBLE
    with pytest.raises(conv.ConvError) as e:
        _offline(sh, "bf16", tile="bogus=1")
    assert e.value.status == conv.CONV_ERR_INVALID_ARGUMENT


def test_selector_model_levels_consistent(lib):
    """The reported model time is at least every level's bandwidth-scaled
    cost (Sec. 5 min-max: cost = max over levels)."""
    from paper_2101_09808_b200.inputs import CONFIGS
    for sh in CONFIGS.values():
        for path in ("tf32", "bf16", "fp32_simt"):
            m = _offline(sh, path).describe()["model"]
            lv = m["levels"]
            assert m["model_us"] >= lv["l2_smem"]["us"] * 0.999
            assert m["model_us"] >= lv["compute"]["flops_issued_us"] * 0.999
            assert lv["l2_smem"]["us"] == pytest.approx(lv["l2_smem"]["dv_bytes"] / lv["l2_smem"]["bw"] * 1e6, rel=1e-3, abs=1e-3)


def test_offline_plan_cannot_run(lib):
    from paper_2101_09808_b200.inputs import CONFIGS
    p = _offline(CONFIGS["tiny"], "tf32")
    assert lib.conv_run(p._h, 16, 16, 16, 256, None) == conv.CONV_ERR_UNSUPPORTED_DEVICE


def test_tensor_l2_volume_matches_im2col_replay(lib):
    """DV_{L2->SMEM} of the tensor path = (A im2col replay + B re-reads) from
    the Sec. 3.2 evaluator = ceil(M/BM)*BM*R*S*Cp*e + ceil(M/BM)*K*R*S*Cp*e."""
    from paper_2101_09808_b200.inputs import CONFIGS
    sh = CONFIGS["batched"]
    for cg in (1, 2):
        d = _offline(sh, "bf16", tile=f"bn=256,cg={cg}").describe()
        bm = 128 * cg
        mt = -(-sh.N * sh.H * sh.W // bm)
        exp = mt * bm * 9 * 256 * 2 + mt * 256 * 9 * 256 * 2
        assert d["model"]["levels"]["l2_smem"]["dv_bytes"] == pytest.approx(exp, rel=1e-9)


def test_strided_plans_offline(lib):
    """conv_plan_create_strided(_offline): output extents (Hin-R)/U + 1 (floor),
    describe() reports U and the input extents; SIMT picks v1 for U > 1 (v2
    needs U = 1); bad strides / tiny inputs are rejected before any device."""
    sh = dict(sms=148, smem_optin=232448, l2_bytes=132120576)
    for (Hin, R, U) in ((56, 3, 2), (224, 7, 2), (13, 3, 2), (16, 5, 3)):
        H = (Hin - R) // U + 1
        p = conv.ConvPlan(1, 64, 32, H, H, R, R, stride=U, in_hw=(Hin, Hin), offline_device=sh)
        d = p.describe()["problem"]
        assert (d["U"], d["Hin"], d["Win"], d["H"], d["W"]) == (U, Hin, Hin, H, H)
        ps = conv.ConvPlan(1, 64, 32, H, H, R, R, stride=U, in_hw=(Hin, Hin), offline_device=sh, path="fp32_simt")
        assert ps.describe()["tile"]["ver"] == 1
    assert not lib.conv_plan_create_strided(1, 1, 1, 8, 8, 3, 3, 0)
    assert "extent must be >= 1" in conv.last_error()
    assert not lib.conv_plan_create_strided(1, 1, 1, 2, 8, 3, 3, 1)
    assert "smaller than the kernel" in conv.last_error()
    with pytest.raises(conv.ConvError) as e:   # TMA im2col traversal stride <= 8
        conv.ConvPlan(1, 8, 64, 3, 3, 3, 3, stride=9, in_hw=(21, 21), offline_device=sh, path="bf16")
    assert e.value.status == conv.CONV_ERR_INFEASIBLE
    # a tiny-C layer runs its tap-expanded 1x1 equivalent: any stride
    d = conv.ConvPlan(1, 8, 8, 3, 3, 3, 3, stride=9, in_hw=(21, 21), offline_device=sh, path="bf16").describe()
    assert d["tile"]["expand"] == 1
    with pytest.raises(ValueError):   # H, W inconsistent with the input extents
        conv.ConvPlan(1, 8, 8, 5, 5, 3, 3, stride=2, in_hw=(21, 21), offline_device=sh)


def test_dilated_plans_offline(lib):
    """conv_plan_create_dilated (PAPER.md:201 footnote: stride/dilation):
    describe() reports D and the output extents (Hin - D(R-1) - 1)/U + 1;
    SIMT falls back to v1 (v2 needs U = D = 1); D = 1 is the strided plan;
    bad dilations, inputs smaller than the dilated kernel and dilated kernels
    past the TMA im2col box (D(R-1) > 128) are rejected."""
    sh = dict(sms=148, smem_optin=232448, l2_bytes=132120576)
    for (Hin, R, U, D) in ((56, 3, 1, 2), (57, 3, 2, 2), (40, 5, 1, 3), (30, 1, 1, 4)):
        H = (Hin - D * (R - 1) - 1) // U + 1
        p = conv.ConvPlan(1, 64, 32, H, H, R, R, stride=U, dilation=D, in_hw=(Hin, Hin), offline_device=sh)
        d = p.describe()["problem"]
        assert (d["U"], d["D"], d["Hin"], d["Win"], d["H"], d["W"]) == (U, D, Hin, Hin, H, H)
        ps = conv.ConvPlan(1, 64, 32, H, H, R, R, stride=U, dilation=D, in_hw=(Hin, Hin), offline_device=sh,
                           path="fp32_simt")
        assert ps.describe()["tile"]["ver"] == 1
    a = conv.ConvPlan(2, 64, 32, 13, 13, 3, 3, stride=2, in_hw=(28, 28), offline_device=sh).describe()
    b = conv.ConvPlan(2, 64, 32, 13, 13, 3, 3, stride=2, dilation=1, in_hw=(28, 28), offline_device=sh).describe()
    assert a == b
    assert not lib.conv_plan_create_dilated(1, 1, 1, 8, 8, 3, 3, 1, 0)
    assert "extent must be >= 1" in conv.last_error()
    assert not lib.conv_plan_create_dilated(1, 1, 1, 4, 8, 3, 3, 1, 2)   # dilated kernel is 5x5
    assert "smaller than the kernel" in conv.last_error()
    with pytest.raises(conv.ConvError) as e:   # D(R-1) = 129 > 128
        conv.ConvPlan(1, 8, 64, 2, 2, 2, 2, dilation=129, in_hw=(131, 131), offline_device=sh, path="bf16")
    assert e.value.status == conv.CONV_ERR_INFEASIBLE


def test_padded_plans_offline(lib):
    """conv_plan_create_padded ("same"-padded layers):
    describe() reports ph/pw and H = (Hin + 2ph - D(R-1) - 1)/U + 1; SIMT
    uses v1 (v2 has no padding); pad 0 is the dilated plan; negative pads,
    padded inputs smaller than the dilated kernel and pads past the TMA box
    are rejected with the right status."""
    sh = dict(sms=148, smem_optin=232448, l2_bytes=132120576)
    for (Hin, R, U, D, ph, pw) in ((56, 3, 1, 1, 1, 1), (224, 7, 2, 1, 3, 3), (14, 3, 2, 2, 2, 1), (5, 3, 1, 1, 4, 0)):
        H = (Hin + 2 * ph - D * (R - 1) - 1) // U + 1
        W = (Hin + 2 * pw - D * (R - 1) - 1) // U + 1
        p = conv.ConvPlan(1, 64, 32, H, W, R, R, stride=U, dilation=D, padding=(ph, pw), in_hw=(Hin, Hin),
                          offline_device=sh)
        d = p.describe()["problem"]
        assert (d["U"], d["D"], d["ph"], d["pw"], d["Hin"], d["H"], d["W"]) == (U, D, ph, pw, Hin, H, W)
        ps = conv.ConvPlan(1, 64, 32, H, W, R, R, stride=U, dilation=D, padding=(ph, pw), in_hw=(Hin, Hin),
                           offline_device=sh, path="fp32_simt")
        assert ps.describe()["tile"]["ver"] == 1
    a = conv.ConvPlan(2, 64, 32, 13, 13, 3, 3, stride=2, dilation=2, in_hw=(30, 30), offline_device=sh).describe()
    b = conv.ConvPlan(2, 64, 32, 13, 13, 3, 3, stride=2, dilation=2, padding=0, in_hw=(30, 30),
                      offline_device=sh).describe()
    assert a == b
    assert not lib.conv_plan_create_padded(1, 1, 1, 8, 8, 3, 3, 1, 1, -1, 0)
    assert "padding must be >= 0" in conv.last_error()
    assert lib.conv_last_status() == conv.CONV_ERR_INVALID_ARGUMENT
    assert not lib.conv_plan_create_padded(1, 1, 1, 1, 1, 5, 5, 1, 1, 1, 1)   # 3x3 padded input, 5x5 kernel
    assert "smaller than the kernel" in conv.last_error()
    with pytest.raises(conv.ConvError) as e:   # lower corner -129
        conv.ConvPlan(1, 8, 64, 3 + 258 - 2, 3, 3, 3, padding=(129, 0), in_hw=(3, 5), offline_device=sh, path="bf16")
    assert e.value.status == conv.CONV_ERR_INFEASIBLE
    # tiny C: the tap expansion computes the padded taps directly (no TMA box)
    d = conv.ConvPlan(1, 8, 8, 3 + 258 - 2, 3, 3, 3, padding=(129, 0), in_hw=(3, 5), offline_device=sh,
                      path="bf16").describe()
    assert d["tile"]["expand"] == 1


def test_production_build(lib):
    """The in-tree library is a production build: the kernel timeline
    instrumentation (CONV_BUILD_TRACE=1, scripts/trace_tc.py) is compiled
    out -- it cost ~1.8 % on the headline."""
    v = lib.conv_version().decode()
    assert v.startswith("0.1.0 sm_100a") and "+trace" not in v


def test_simt_register_table_matches_library(lib):
    """The SIMT model's registers per thread (csrc/simt_regs.inc) are those
    ptxas gave every kernel instance of the built library (cuobjdump), and
    every instance the dispatch can launch is listed."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "gen_simt_regs", os.path.join(os.path.dirname(os.path.dirname(__file__)), "scripts", "gen_simt_regs.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    if not os.path.exists(gen.CUOBJDUMP):
        pytest.skip("cuobjdump not available")
    rows = gen.table()
    assert open(gen.INC).read() == gen.render(rows), "run scripts/gen_simt_regs.py after changing simt.cu"
    keys = {r[:6] for r in rows}
    for tk, tw in itertools.product((4, 8), range(1, 9)):               # v1: dispatch_simt
        for sc in (0, 1):
            assert (1, tk, tw, 0, 0, sc) in keys
    v2 = [(tk, tw) for tk in (4, 8) for tw in (4, 8)] + [(4, 14), (4, 7)]  # v2: dispatch_simt2
    for (tk, tw), (kr, ks), sc in itertools.product(v2, ((1, 1), (3, 3), (0, 1), (0, 3)), (0, 1)):
        assert (2, tk, tw, kr, ks, sc) in keys


def test_tap_expansion_and_split_c_offline(lib):
    """Selector features on a described B200 (no device): the C = 3 stems of
    Table 1 take the tiny-C tap expansion (workspace = the expanded 1x1
    problem's NHWC In' + Ker'), deep-C small-output layers take split-K
    (tensor) / split-C (SIMT, one more kernel), forced fused / split-K plans
    never expand, and the batched headline layer is neither expanded nor
    split."""
    from paper_2101_09808_b200.inputs import CONFIGS, TABLE1
    y0 = TABLE1["Y0"]
    d = conv.ConvPlan(*y0.as_tuple(), path="bf16", offline_device=conv.B200, **y0.plan_kwargs()).describe()
    t = d["tile"]
    assert t["expand"] == 1 and t["fuse"] == 0 and t["splits"] == 1
    cp = t["cp"]
    assert cp >= y0.R * y0.S * y0.C and cp % 8 == 0
    in_ws = y0.N * y0.H * y0.W * cp * 2
    ker_ws = y0.K * cp * 2
    al = lambda x: (x + 255) // 256 * 256
    assert d["workspace_bytes"] == al(in_ws) + al(ker_ws)
    r1 = TABLE1["R1"]
    assert conv.ConvPlan(*r1.as_tuple(), path="tf32", offline_device=conv.B200,
                         **r1.plan_kwargs()).describe()["tile"]["expand"] == 1
    # forcing the fused transform or split-K keeps the plain path (a small
    # tiny-C layer: one wave, a TMA-legal NCHW plane)
    from paper_2101_09808_b200.inputs import Shape
    small = Shape(N=1, K=32, C=3, H=8, W=8, R=3, S=3)
    ts = conv.ConvPlan(*small.as_tuple(), path="bf16", offline_device=conv.B200).describe()["tile"]
    assert ts["expand"] == 1 or ts["halo"] == 1      # tap expansion or the single-launch halo kernel (modeled)
    assert conv.ConvPlan(*small.as_tuple(), path="bf16", offline_device=conv.B200,
                         tile="halo=0").describe()["tile"]["expand"] == 1
    for spec, key, val in (("fuse=1", "fuse", 1), ("splits=2", "splits", 2)):
        dd = conv.ConvPlan(*small.as_tuple(), path="bf16", tile=spec, offline_device=conv.B200).describe()
        assert dd["tile"]["expand"] == 0 and dd["tile"][key] == val
    m9 = TABLE1["M9"]
    assert conv.ConvPlan(*m9.as_tuple(), path="bf16", offline_device=conv.B200,
                         **m9.plan_kwargs()).describe()["tile"]["splits"] > 1
    ps = conv.ConvPlan(*m9.as_tuple(), path="fp32_simt", offline_device=conv.B200, **m9.plan_kwargs())
    assert ps.describe()["tile"]["splits"] > 1 and ps.num_kernels == 3
    b = CONFIGS["batched"]
    for path in ("bf16", "tf32", "fp32_simt"):
        tb = conv.ConvPlan(*b.as_tuple(), path=path, offline_device=conv.B200).describe()["tile"]
        assert tb.get("splits", 1) == 1 and tb.get("expand", 0) == 0


# ---- measured peaks (K5 probes) ------------------------------------------------

def test_peaks_inc_matches_measured_json():
    """csrc/peaks_measured.inc (the selector's constants) is the one
    scripts/measure_peaks.py generated from profiles/peaks_measured.json."""
    import json
    doc = json.load(open(os.path.join(ROOT, "profiles", "peaks_measured.json")))
    inc = open(os.path.join(ROOT, "paper_2101_09808_b200", "csrc", "peaks_measured.inc")).read()
    vals = {m.group(1): float(m.group(2)) for m in re.finditer(r"#define (CONV_\w+) ([0-9.e]+)", inc)}
    sel = doc["selected"]
    assert vals["CONV_PEAK_FP32"] == sel["peak_fp32_tflops"] * 1e12
    assert vals["CONV_PEAK_TF32"] == sel["peak_tf32_tflops"] * 1e12
    assert vals["CONV_BW_L2_SMEM"] == sel["bw_l2_smem_tbs"] * 1e12
    assert sel["peak_fp32_tflops"] == doc["probes"]["ffma_fp32"]["value"]
    assert sel["peak_tf32_tflops"] == doc["probes"]["cublas_tf32"]["value"]
    # each probe reached a plausible fraction of the B200's nominal rates
    assert 50 < sel["peak_fp32_tflops"] < 80            # 148 SM x 128 lanes x 2 x <= 1.965 GHz = 74.4
    assert 500 < sel["peak_tf32_tflops"] < 1200         # nominal dense tf32 1.1 PF
    assert 5 < sel["bw_l2_smem_tbs"] < 40


def test_probe_library_exports():
    from paper_2101_09808_b200 import build
    build.build()
    src = open(os.path.join(ROOT, "include", "conv_probes.h")).read()
    declared = set(re.findall(r"CONV_PROBE_API[^;(]*?\b(probe_\w+)\s*\(", src))
    out = os.popen(f"nm -D --defined-only {build.PROBES_LIB}").read()
    exported = set(re.findall(r" T (probe_\w+)", out))
    assert declared and declared <= exported


def test_simt_staging_choice_offline(lib):
    """FP32 SIMT v2 staging (simt2_layout): the TMA box + bulk Ker copy
    wherever In rows are 16-B multiples (Win % 4 == 0) and the box fits TMA's
    256-element dims; the per-thread cp.async layout otherwise, and always for
    v1 (strided) tiles.  The batched layer's plan is the r02d headline tile
    (flat row mode: 32 consecutive (image, row) slots per CTA, boxes of 4
    images, 8 k groups, the last slot tile as the remainder launch); its
    128- and 64-image shards take flat tiles with a remainder launch too."""
    import dataclasses
    from paper_2101_09808_b200.inputs import CONFIGS, TABLE1
    d = _offline(CONFIGS["batched"], "fp32_simt").describe()["tile"]
    assert (d["ver"], d["tk"], d["tw"], d["kg"], d["tn"], d["th"], d["bc"], d["flat"], d["rem"], d["staging"]) == \
        (2, 4, 14, 8, 4, 14, 6, 1, 1, "tma")       # r02e: 6-channel chunks on the kg = 8 flat tile
    d = _offline(dataclasses.replace(CONFIGS["batched"], N=128), "fp32_simt").describe()["tile"]
    assert (d["ver"], d["tk"], d["tw"], d["kg"], d["th"], d["bc"], d["flat"], d["rem"], d["staging"]) == \
        (2, 4, 14, 8, 14, 6, 1, 1, "tma")
    d = _offline(dataclasses.replace(CONFIGS["batched"], N=64), "fp32_simt").describe()["tile"]
    # r02e: the 64- and 32-image shards take a 2-way split-C flat tile with the remainder launch
    assert (d["ver"], d["tk"], d["tw"], d["kg"], d["th"], d["splits"], d["flat"], d["rem"], d["staging"]) == \
        (2, 4, 14, 8, 14, 2, 1, 1, "tma")
    d = _offline(dataclasses.replace(CONFIGS["batched"], N=32), "fp32_simt").describe()["tile"]
    assert (d["ver"], d["tk"], d["tw"], d["kg"], d["th"], d["splits"], d["flat"], d["rem"], d["staging"]) == \
        (2, 4, 14, 4, 14, 2, 1, 1, "tma")
    for name in ("r2", "det", "tiny"):                       # Win = 58, 138, 10
        assert _offline(CONFIGS[name], "fp32_simt").describe()["tile"]["staging"] == "cp.async"
    sh = TABLE1["Y2"]                                        # Win = 272: a row wider than a TMA box
    assert _offline(sh, "fp32_simt").describe()["tile"]["staging"] == "cp.async"
    sh = TABLE1["M2"]                                        # stride 2: v1
    t = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", offline_device=conv.B200, **sh.plan_kwargs()).describe()["tile"]
    assert t["ver"] == 1 and t["staging"] == "cp.async"
