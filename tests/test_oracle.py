"""Pins for the CPU oracle, CPU only.

Each test pins ``oracle.conv_eq1`` (Eq. 1, Listing 2 order
PAPER.md:150-158) to something other than itself: hand-worked values
(tests/golden), closed forms, an independent algorithm (integral images),
textbook/library routines (float64 matmul, torch conv2d) and brute force.
A dropped term, a wrong sign or index, a flipped kernel or a transposed
operand fails at least one of them (see the docstrings).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2101_09808_b200.inputs import CONFIGS, Shape, make_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["eq1_hand_2x2.json", "eq1_hand_2ch.json"])
def test_hand_worked_golden(name):
    """Hand-worked Eq. 1 values (catches kernel flip, c/k transposition)."""
    g = _golden(name)
    inp = np.array(g["In"], dtype=np.float32)
    ker = np.array(g["Ker"], dtype=np.float32)
    out = oracle.conv_eq1(inp, ker)
    np.testing.assert_array_equal(out, np.array(g["Out"], dtype=np.float64))


def test_p1_identity_1x1():
    """P1: K=C, R=S=1, Ker=delta_kc => Out == In exactly."""
    sh = Shape(N=2, K=5, C=5, H=7, W=9, R=1, S=1)
    inp, _ = make_inputs(sh, seed=3)
    ker = np.eye(5, dtype=np.float32).reshape(5, 5, 1, 1)
    out = oracle.conv_eq1(inp.numpy(), ker)
    np.testing.assert_array_equal(out, inp.numpy().astype(np.float64))


@pytest.mark.parametrize("r0,s0", [(r, s) for r in range(2) for s in range(3)])
def test_p2_shifted_delta(r0, s0):
    """P2: Ker = delta_kc delta_{r r0} delta_{s s0} => Out[n,k,h,w] =
    In[n,k,h+r0,w+s0].  R != S and H != W, so a flipped kernel, swapped r/s
    or h/w, or an off-by-one at the last row/column fails."""
    sh = Shape(N=2, K=3, C=3, H=5, W=6, R=2, S=3)
    inp, _ = make_inputs(sh, seed=4)
    ker = np.zeros(sh.ker_shape, dtype=np.float32)
    for k in range(3):
        ker[k, k, r0, s0] = 1.0
    out = oracle.conv_eq1(inp.numpy(), ker)
    exp = inp.numpy()[:, :, r0:r0 + sh.H, s0:s0 + sh.W].astype(np.float64)
    np.testing.assert_array_equal(out, exp)


def test_p3_all_ones_input():
    """P3: In == 1 => Out[n,k,:,:] = sum_{c,r,s} Ker[k,c,r,s] (per-k constant)."""
    sh = Shape(N=2, K=4, C=3, H=4, W=5, R=3, S=2)
    _, ker = make_inputs(sh, seed=5)
    inp = np.ones(sh.in_shape, dtype=np.float32)
    out = oracle.conv_eq1(inp, ker.numpy())
    for k in range(sh.K):
        exp = math.fsum(ker.numpy()[k].astype(np.float64).ravel().tolist())
        np.testing.assert_allclose(out[:, k], exp, rtol=1e-14, atol=1e-14)


def test_p4_all_ones_kernel_box_sum():
    """P4: Ker == 1 => Out = R x S x C box sum of In, identical for all k.
    Expected values come from integral images (summed-area tables) -- a
    different algorithm from the loop nest."""
    sh = Shape(N=2, K=3, C=4, H=6, W=5, R=3, S=2)
    inp, _ = make_inputs(sh, seed=6, kind="int")
    x = inp.numpy().astype(np.float64).sum(axis=1)          # [N, Hin, Win]
    sat = np.zeros((sh.N, sh.Hin + 1, sh.Win + 1))
    sat[:, 1:, 1:] = x.cumsum(1).cumsum(2)
    box = (sat[:, sh.R:, sh.S:] - sat[:, :-sh.R, sh.S:]
           - sat[:, sh.R:, :-sh.S] + sat[:, :-sh.R, :-sh.S])
    out = oracle.conv_eq1(inp.numpy(), np.ones(sh.ker_shape, dtype=np.float32))
    for k in range(sh.K):
        np.testing.assert_array_equal(out[:, k], box)


def test_p5_linearity_exact_on_integers():
    """P5: conv(a*In1 + b*In2, Ker) = a*conv(In1) + b*conv(In2) and likewise
    in Ker; exact on small-integer data with small-integer a, b."""
    sh = Shape(N=2, K=3, C=4, H=5, W=4, R=2, S=3)
    i1, k1 = make_inputs(sh, seed=7, kind="int")
    i2, k2 = make_inputs(sh, seed=8, kind="int")
    a, b = 3.0, -2.0
    i1, i2, k1, k2 = (t.numpy() for t in (i1, i2, k1, k2))
    lhs = oracle.conv_eq1((a * i1 + b * i2).astype(np.float32), k1)
    rhs = a * oracle.conv_eq1(i1, k1) + b * oracle.conv_eq1(i2, k1)
    np.testing.assert_array_equal(lhs, rhs)
    lhs = oracle.conv_eq1(i1, (a * k1 + b * k2).astype(np.float32))
    rhs = a * oracle.conv_eq1(i1, k1) + b * oracle.conv_eq1(i1, k2)
    np.testing.assert_array_equal(lhs, rhs)


def test_p6_integer_twin_exact_integers():
    """P6: integer-twin inputs give integer outputs with |Out| <= 4*C*R*S,
    equal to torch's float64 conv2d bit-for-bit."""
    sh = CONFIGS["tiny"]
    inp, ker = make_inputs(sh, seed=1, kind="int")
    out = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert np.all(out == np.round(out))
    assert np.abs(out).max() <= 4 * sh.C * sh.R * sh.S
    ref = torch.nn.functional.conv2d(inp.double(), ker.double()).numpy()
    np.testing.assert_array_equal(out, ref)


def test_p7_pointwise_is_a_gemm():
    """P7: R=S=1 => Out[n] = Ker[:,:,0,0] @ In[n].reshape(C, H*W) (float64
    matmul, a textbook routine; pw config shape)."""
    sh = Shape(N=2, K=32, C=16, H=9, W=11, R=1, S=1)
    inp, ker = make_inputs(sh, seed=9)
    out = oracle.conv_eq1(inp.numpy(), ker.numpy())
    k2 = ker.numpy()[:, :, 0, 0].astype(np.float64)
    for n in range(sh.N):
        exp = k2 @ inp.numpy()[n].reshape(sh.C, -1).astype(np.float64)
        np.testing.assert_allclose(out[n].reshape(sh.K, -1), exp, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", ["tiny", "r2"])
def test_p8_torch_conv2d_float64(name):
    """P8: torch.nn.functional.conv2d (cross-correlation) in float64 on the
    CPU, test-only library cross-check."""
    sh = CONFIGS[name]
    inp, ker = make_inputs(sh, seed=0)
    out = oracle.conv_eq1(inp.numpy(), ker.numpy())
    ref = torch.nn.functional.conv2d(inp.double(), ker.double()).numpy()
    err = np.abs(out - ref).max()
    assert err <= 1e-12 * max(1.0, np.abs(ref).max()), err


def test_p8_odd_shape():
    sh = Shape(N=2, K=5, C=3, H=7, W=9, R=3, S=2)
    inp, ker = make_inputs(sh, seed=2)
    out = oracle.conv_eq1(inp.numpy(), ker.numpy())
    ref = torch.nn.functional.conv2d(inp.double(), ker.double()).numpy()
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13)


def test_p9_brute_force_points():
    """P9: random output points equal the correctly rounded (fsum) sum of
    their C*R*S exact products, within the double-summation bound."""
    sh = CONFIGS["r2"]
    inp, ker = make_inputs(sh, seed=0)
    x, w = inp.numpy(), ker.numpy()
    out = oracle.conv_eq1(x, w)
    rng = np.random.default_rng(0)
    crs = sh.C * sh.R * sh.S
    for _ in range(200):
        n, k = rng.integers(sh.N), rng.integers(sh.K)
        h, ww = rng.integers(sh.H), rng.integers(sh.W)
        exact = oracle.conv_eq1_point(x, w, n, k, h, ww)
        absum = float(np.abs(x[n, :, h:h + sh.R, ww:ww + sh.S].astype(np.float64)
                             * w[k].astype(np.float64)).sum())
        assert abs(out[n, k, h, ww] - exact) <= crs * 2.0 ** -53 * absum + 1e-300


def test_point_matches_closed_form():
    """conv_eq1_point on the P2 shifted-delta kernel returns In exactly."""
    sh = Shape(N=1, K=2, C=2, H=3, W=4, R=2, S=3)
    inp, _ = make_inputs(sh, seed=11)
    ker = np.zeros(sh.ker_shape, dtype=np.float32)
    ker[1, 0, 1, 2] = 1.0
    x = inp.numpy()
    for h in range(sh.H):
        for w in range(sh.W):
            assert oracle.conv_eq1_point(x, ker, 0, 1, h, w) == float(x[0, 0, h + 1, w + 2])


def test_thread_count_invariance():
    """Planes are summed serially, so 1 and many threads agree bit-for-bit."""
    sh = Shape(N=2, K=6, C=5, H=7, W=6, R=3, S=3)
    inp, ker = make_inputs(sh, seed=12)
    a = oracle.conv_eq1(inp.numpy(), ker.numpy(), nthreads=1)
    b = oracle.conv_eq1(inp.numpy(), ker.numpy(), nthreads=8)
    assert np.array_equal(a, b)


def test_rejects_bad_shapes():
    with pytest.raises(ValueError):
        oracle.conv_eq1(np.zeros((1, 2, 3, 3), np.float32), np.zeros((1, 3, 1, 1), np.float32))
    with pytest.raises(ValueError):
        oracle.conv_eq1(np.zeros((1, 1, 2, 2), np.float32), np.zeros((1, 1, 3, 3), np.float32))


# ---- rounding helpers (reading R5) --------------------------------

def test_bf16_rne_matches_torch_cast():
    """round_bf16_rne == torch's CPU fp32->bf16 cast (round-to-nearest-even)."""
    g = torch.Generator().manual_seed(0)
    x = torch.cat([torch.rand(100000, generator=g) * 2 - 1,
                   torch.randn(100000, generator=g) * 1e3,
                   torch.tensor([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 0.0, -0.0])])
    ref = x.to(torch.bfloat16).to(torch.float32).numpy()
    got = oracle.round_bf16_rne(x.numpy())
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_tf32_rna_ties_and_bound():
    """TF32 keeps 10 mantissa bits; ulp(1) = 2^-10.  Ties round away from 0."""
    f = np.float32
    cases = {
        1.0 + 2 ** -11: 1.0 + 2 ** -10,            # exact tie -> away from zero
        -(1.0 + 2 ** -11): -(1.0 + 2 ** -10),
        1.0 + 2 ** -12: 1.0,                       # below half ulp -> down
        1.0 + 3 * 2 ** -11: 1.0 + 2 * 2 ** -10,    # tie at odd -> away (up)
        1.0 + 2 ** -10: 1.0 + 2 ** -10,            # representable -> unchanged
    }
    for x, exp in cases.items():
        assert oracle.round_tf32_rna(np.array([x], f))[0] == f(exp)
    g = np.random.default_rng(1)
    x = (g.random(100000, dtype=np.float32) * 2 - 1) * f(37.0)
    r = oracle.round_tf32_rna(x)
    assert np.all((r.view(np.uint32) & 0x1FFF) == 0)
    ulp = np.ldexp(1.0, np.frexp(np.abs(x).astype(np.float64))[1] - 11)
    assert np.all(np.abs(r.astype(np.float64) - x) <= ulp / 2)


# ---- strided Eq. 1 (PAPER.md:201 footnote; Table 1 stride-2 layers)

def test_strided_hand_worked_golden():
    """Hand-worked stride-2 values (tests/golden/eq1_stride2_hand.json):
    catches U*(h+r) instead of U*h+r, a stride on one axis only, and reading
    past the last full window."""
    g = _golden("eq1_stride2_hand.json")
    out = oracle.conv_eq1_strided(np.array(g["In"], dtype=np.float32), np.array(g["Ker"], dtype=np.float32),
                                  g["stride"])
    np.testing.assert_array_equal(out, np.array(g["Out"], dtype=np.float64))


def test_strided_unit_stride_is_eq1():
    """U = 1 reduces to the (pinned) stride-1 oracle, bit for bit."""
    sh = Shape(N=2, K=4, C=3, H=6, W=7, R=3, S=2)
    inp, ker = make_inputs(sh, seed=51)
    np.testing.assert_array_equal(oracle.conv_eq1_strided(inp.numpy(), ker.numpy(), 1),
                                  oracle.conv_eq1(inp.numpy(), ker.numpy()))


@pytest.mark.parametrize("U", [2, 3])
def test_strided_is_subsampled_unit_stride(U):
    """Out_U[h, w] = Out_1[U h, U w] exactly (same products, same summation
    order); input extents with (Hin - R) % U != 0 check the floor."""
    inp = torch.rand(2, 3, 12, 11, generator=torch.Generator().manual_seed(52)) * 2 - 1
    ker = torch.rand(5, 3, 3, 2, generator=torch.Generator().manual_seed(53)) * 2 - 1
    full = oracle.conv_eq1(inp.numpy(), ker.numpy())
    got = oracle.conv_eq1_strided(inp.numpy(), ker.numpy(), U)
    assert got.shape == (2, 5, (12 - 3) // U + 1, (11 - 2) // U + 1)
    np.testing.assert_array_equal(got, full[:, :, ::U, ::U])


@pytest.mark.parametrize("U", [2, 3])
def test_strided_vs_torch_conv2d(U):
    """Library cross-check: torch conv2d (float64, stride U, no padding)."""
    inp = torch.rand(2, 4, 15, 13, generator=torch.Generator().manual_seed(54)) * 2 - 1
    ker = torch.rand(3, 4, 3, 3, generator=torch.Generator().manual_seed(55)) * 2 - 1
    got = oracle.conv_eq1_strided(inp.numpy(), ker.numpy(), U)
    ref = torch.nn.functional.conv2d(inp.double(), ker.double(), stride=U).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)
    xi = torch.randint(-2, 3, (1, 4, 15, 13), generator=torch.Generator().manual_seed(56)).float()
    wi = torch.randint(-2, 3, (3, 4, 3, 3), generator=torch.Generator().manual_seed(57)).float()
    np.testing.assert_array_equal(oracle.conv_eq1_strided(xi.numpy(), wi.numpy(), U),
                                  torch.nn.functional.conv2d(xi.double(), wi.double(), stride=U).numpy())


def test_strided_points_brute_force():
    """Sampled outputs of the strided oracle vs the correctly rounded sum."""
    inp = torch.rand(2, 8, 21, 17, generator=torch.Generator().manual_seed(58)) * 2 - 1
    ker = torch.rand(6, 8, 7, 7, generator=torch.Generator().manual_seed(59)) * 2 - 1
    x, w = inp.numpy(), ker.numpy()
    out = oracle.conv_eq1_strided(x, w, 2)
    rng = np.random.default_rng(60)
    for _ in range(50):
        p = (rng.integers(2), rng.integers(6), rng.integers(out.shape[2]), rng.integers(out.shape[3]))
        assert abs(out[p] - oracle.conv_eq1_point(x, w, *p, stride=2)) <= 1e-13 * (1 + abs(out[p]))


# ---- dilation (PAPER.md:201 footnote: "stride/dilation ... the general case")

def test_dilated_unit_is_strided():
    """D = 1 reduces to the (pinned) strided oracle, bit for bit."""
    inp = torch.rand(2, 3, 13, 12, generator=torch.Generator().manual_seed(101)) * 2 - 1
    ker = torch.rand(4, 3, 3, 2, generator=torch.Generator().manual_seed(102)) * 2 - 1
    for U in (1, 2):
        np.testing.assert_array_equal(oracle.conv_eq1_dilated(inp.numpy(), ker.numpy(), U, 1),
                                      oracle.conv_eq1_strided(inp.numpy(), ker.numpy(), U))


@pytest.mark.parametrize("U,D", [(1, 2), (2, 2), (1, 3), (2, 3)])
def test_dilated_is_zero_inserted_kernel(U, D):
    """Dilation D = the strided oracle with the kernel spread over a
    (D(R-1)+1) x (D(S-1)+1) grid of zeros: the extra terms are exact zeros,
    so the double sums are identical bit for bit (catches D*r vs r, a
    dilation on one axis only, a wrong output extent)."""
    inp = torch.rand(2, 3, 17, 15, generator=torch.Generator().manual_seed(103)) * 2 - 1
    ker = torch.rand(4, 3, 3, 2, generator=torch.Generator().manual_seed(104)) * 2 - 1
    k = ker.numpy()
    big = np.zeros((4, 3, D * 2 + 1, D * 1 + 1), dtype=np.float32)
    big[:, :, ::D, ::D] = k
    got = oracle.conv_eq1_dilated(inp.numpy(), k, U, D)
    np.testing.assert_array_equal(got, oracle.conv_eq1_strided(inp.numpy(), big, U))


@pytest.mark.parametrize("U,D", [(1, 2), (2, 3)])
def test_dilated_vs_torch_and_points(U, D):
    """Library cross-check (torch conv2d f64 with stride and dilation) and
    correctly rounded brute-force points."""
    inp = torch.rand(2, 4, 19, 16, generator=torch.Generator().manual_seed(105)) * 2 - 1
    ker = torch.rand(3, 4, 3, 3, generator=torch.Generator().manual_seed(106)) * 2 - 1
    got = oracle.conv_eq1_dilated(inp.numpy(), ker.numpy(), U, D)
    ref = torch.nn.functional.conv2d(inp.double(), ker.double(), stride=U, dilation=D).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)
    rng = np.random.default_rng(107)
    for _ in range(30):
        p = (rng.integers(2), rng.integers(3), rng.integers(got.shape[2]), rng.integers(got.shape[3]))
        v = oracle.conv_eq1_point(inp.numpy(), ker.numpy(), *p, stride=U, dilation=D)
        assert abs(got[p] - v) <= 1e-13 * (1 + abs(v))


# ---- zero padding (DESIGN reading R3) --------------

def test_padded_zero_pad_is_dilated():
    """Padding 0 reduces to the (pinned) dilated oracle, bit for bit."""
    inp = torch.rand(2, 3, 14, 13, generator=torch.Generator().manual_seed(111)) * 2 - 1
    ker = torch.rand(4, 3, 3, 2, generator=torch.Generator().manual_seed(112)) * 2 - 1
    for U, D in ((1, 1), (2, 1), (1, 2), (2, 3)):
        np.testing.assert_array_equal(oracle.conv_eq1_padded(inp.numpy(), ker.numpy(), U, D, 0),
                                      oracle.conv_eq1_dilated(inp.numpy(), ker.numpy(), U, D))


@pytest.mark.parametrize("U,D,pad", [(1, 1, 1), (1, 1, (2, 0)), (2, 1, 3), (1, 2, 2), (2, 2, (1, 3))])
def test_padded_vs_torch_and_points(U, D, pad):
    """Library cross-check (torch conv2d f64 with padding, stride, dilation)
    and correctly rounded brute-force points (with explicit tap bounds)."""
    inp = torch.rand(2, 4, 15, 12, generator=torch.Generator().manual_seed(113)) * 2 - 1
    ker = torch.rand(3, 4, 3, 5, generator=torch.Generator().manual_seed(114)) * 2 - 1
    got = oracle.conv_eq1_padded(inp.numpy(), ker.numpy(), U, D, pad)
    p2 = (pad, pad) if isinstance(pad, int) else pad
    ref = torch.nn.functional.conv2d(inp.double(), ker.double(), stride=U, dilation=D, padding=p2).numpy()
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)
    rng = np.random.default_rng(115)
    corners = [(0, 0, 0, 0), (1, 2, got.shape[2] - 1, got.shape[3] - 1), (0, 1, 0, got.shape[3] - 1)]
    pts = corners + [(rng.integers(2), rng.integers(3), rng.integers(got.shape[2]), rng.integers(got.shape[3]))
                     for _ in range(30)]
    for p in pts:
        v = oracle.conv_eq1_point(inp.numpy(), ker.numpy(), *p, stride=U, dilation=D, padding=pad)
        assert abs(got[p] - v) <= 1e-13 * (1 + abs(v)), p


def test_padded_interior_is_unpadded_output():
    """Stride 1: Out_pad[n,k,h+ph,w+pw] = Out_valid[n,k,h,w] bit for bit
    (same products, same order); the padded output is (Hin+2ph-R+1) wide."""
    inp = torch.rand(2, 3, 11, 10, generator=torch.Generator().manual_seed(116)) * 2 - 1
    ker = torch.rand(4, 3, 3, 3, generator=torch.Generator().manual_seed(117)) * 2 - 1
    full = oracle.conv_eq1_padded(inp.numpy(), ker.numpy(), 1, 1, (2, 1))
    valid = oracle.conv_eq1(inp.numpy(), ker.numpy())
    assert full.shape == (2, 4, 11 + 4 - 2, 10 + 2 - 2)
    np.testing.assert_array_equal(full[:, :, 2:2 + valid.shape[2], 1:1 + valid.shape[3]], valid)


def test_padded_all_ones_closed_form():
    """In = 1, Ker = 1: Out[h,w] = C * (#taps r with 0 <= U h + D r - ph < Hin)
    * (#taps s likewise) -- an independent count of the in-range taps."""
    N, C, Hin, Win, R, S, U, D, ph, pw = 1, 5, 9, 8, 3, 4, 2, 2, 3, 2
    got = oracle.conv_eq1_padded(np.ones((N, C, Hin, Win), np.float32), np.ones((2, C, R, S), np.float32),
                                 U, D, (ph, pw))
    for h in range(got.shape[2]):
        for w in range(got.shape[3]):
            nr = sum(1 for r in range(R) if 0 <= U * h + D * r - ph < Hin)
            ns = sum(1 for s in range(S) if 0 <= U * w + D * s - pw < Win)
            assert got[0, 1, h, w] == C * nr * ns, (h, w)


def test_bf16_three_piece_split_is_exact():
    """DESIGN.md reading R15 (the FP32_TC path): x0 = bf16(x), x1 = bf16(x -
    x0), x2 = bf16(x - x0 - x1) reproduces every binary32 x exactly
    (x0 + x1 + x2 == x, each remainder exact in fp32, x2 representable in
    bf16), every piece product x_i * y_j is exact in fp32 (8 x 8 bits), and
    the three pairs with i + j > 2 that the 6-pair variant drops are below
    3 * 2^-24 |x * y| (products inside binary32's normal range; outside it
    any fp32 arithmetic over/underflows).  Pinned with the oracle's bf16
    rounding (RNE)."""
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(-1, 1, 20000), rng.standard_normal(5000) * 1e30,
                        rng.standard_normal(5000) * 1e-30]).astype(np.float32)
    y = rng.permutation(x)

    def split(v):
        v0 = oracle.round_bf16_rne(v)
        r1 = (v - v0).astype(np.float32)
        v1 = oracle.round_bf16_rne(r1)
        r2 = (r1 - v1).astype(np.float32)
        v2 = oracle.round_bf16_rne(r2)
        assert np.array_equal(v2, r2)                            # the last remainder is a bf16
        assert np.array_equal(v0.astype(np.float64) + v1 + v2, v.astype(np.float64))
        return v0, v1, v2

    xs, ys = split(x), split(y)
    exact = x.astype(np.float64) * y.astype(np.float64)
    for i in range(3):
        for j in range(3):
            with np.errstate(over="ignore", under="ignore"):
                pf = (xs[i] * ys[j]).astype(np.float32)          # fp32 product of two pieces
            p64 = xs[i].astype(np.float64) * ys[j]
            # exact wherever the product is in binary32's normal range (as
            # for any fp32 arithmetic, products outside it over/underflow)
            ok = (np.abs(p64) >= 2.0 ** -126) & (np.abs(p64) < 2.0 ** 127)
            assert ok.mean() > 0.5
            assert np.array_equal(pf[ok].astype(np.float64), p64[ok])
    dropped = sum(xs[i].astype(np.float64) * ys[j] for i, j in ((1, 2), (2, 1), (2, 2)))
    nz = exact != 0
    assert np.all(np.abs(dropped[nz]) <= 3 * 2.0 ** -24 * np.abs(exact[nz]))
    six = sum(xs[i].astype(np.float64) * ys[j] for i, j in ((0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0)))
    assert np.array_equal(six + dropped, exact)
