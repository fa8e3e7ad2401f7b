"""Seeded synthetic inputs shared by the tests, the bench and the oracle.

This module holds NO arithmetic of the method; it
only draws tensors.  Everything is generated on the CPU with a
``torch.Generator`` so that the oracle, every GPU and every shard see the same
bits, independent of device.

* ``kind="real"``: In, then Ker, i.i.d. uniform[-1, 1) as
  ``torch.rand(shape) * 2 - 1`` (fp32), the value distribution BASELINE.json's
  configs state.
* ``kind="int"``: the integer twin, values in {-2,...,2}
  (``torch.randint(-2, 3, shape)`` cast to fp32).  Every value is exact in
  bf16/tf32 and every partial sum (|.| <= 4*C*R*S < 2^24) is exact in fp32, so
  all paths must reproduce Eq. 1 bit-for-bit.

Layouts follow PAPER.md:425 (NCHW In/Out, KCRS Ker).  H, W are OUTPUT extents
(reading R1); In is [N, C, H+R-1, W+S-1].
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Shape:
    """H, W are OUTPUT extents.  U is the stride, D the dilation
    (PAPER.md:201 footnote; Table 1's * layers) and ph/pw the zero padding
    (SURVEY NEXT-2); hin/win are explicit input extents of a general layer
    (0: the minimal (H-1)*U + D*(R-1) + 1 - 2ph).  Use ``Shape.strided`` to
    build one from input extents as Table 1 lists them."""
    N: int
    K: int
    C: int
    H: int
    W: int
    R: int
    S: int
    U: int = 1
    hin: int = 0
    win: int = 0
    D: int = 1
    ph: int = 0
    pw: int = 0

    @classmethod
    def strided(cls, N, K, C, Hin, Win, R, S, U, D=1, ph=0, pw=0) -> "Shape":
        Re, Se = D * (R - 1) + 1, D * (S - 1) + 1
        return cls(N, K, C, (Hin + 2 * ph - Re) // U + 1, (Win + 2 * pw - Se) // U + 1, R, S, U, Hin, Win, D, ph, pw)

    @property
    def Hin(self) -> int:
        return self.hin or (self.H - 1) * self.U + self.D * (self.R - 1) + 1 - 2 * self.ph

    @property
    def Win(self) -> int:
        return self.win or (self.W - 1) * self.U + self.D * (self.S - 1) + 1 - 2 * self.pw

    def plan_kwargs(self) -> dict:
        """Keyword arguments of ConvPlan for this shape (stride, dilation, padding, input extents)."""
        if self.U == 1 and self.D == 1 and self.ph == 0 and self.pw == 0 and not self.hin and not self.win:
            return {}
        kw = {"stride": self.U, "in_hw": (self.Hin, self.Win)}
        if self.D != 1:
            kw["dilation"] = self.D
        if self.ph or self.pw:
            kw["padding"] = (self.ph, self.pw)
        return kw

    @property
    def in_shape(self):
        return (self.N, self.C, self.Hin, self.Win)

    @property
    def ker_shape(self):
        return (self.K, self.C, self.R, self.S)

    @property
    def out_shape(self):
        return (self.N, self.K, self.H, self.W)

    @property
    def flops(self) -> int:
        """2*N*K*H*W*C*R*S (BASELINE.json metric; H, W output extents)."""
        return 2 * self.N * self.K * self.H * self.W * self.C * self.R * self.S

    @property
    def compulsory_bytes(self) -> int:
        """fp32 bytes of In + Ker + Out, each touched once."""
        n_in = self.N * self.C * self.Hin * self.Win
        n_ker = self.K * self.C * self.R * self.S
        n_out = self.N * self.K * self.H * self.W
        return 4 * (n_in + n_ker + n_out)

    def as_tuple(self):
        return (self.N, self.K, self.C, self.H, self.W, self.R, self.S)


# BASELINE.json "configs", in order.  Names are used by tests and bench.
CONFIGS = {
    "tiny": Shape(N=1, K=16, C=16, H=8, W=8, R=3, S=3),
    "r2": Shape(N=1, K=64, C=64, H=56, W=56, R=3, S=3),
    "pw": Shape(N=1, K=256, C=64, H=56, W=56, R=1, S=1),
    "det": Shape(N=1, K=64, C=32, H=136, W=136, R=3, S=3),
    "batched": Shape(N=256, K=256, C=256, H=14, W=14, R=3, S=3),
}


# PAPER.md:439-477, Table 1: the 32 conv2d layers of Yolo-9000, ResNet-18 and
# MobileNet, batch 1, H/W = INPUT extents, stride 2 for the layers marked *.
# (name, K, C, H/W, R/S, stride).  The MobileNet rows are run as the dense
# convolutions Table 1 lists (reading R7).
TABLE1_ROWS = [
    ("Y0", 32, 3, 544, 3, 1), ("Y2", 64, 32, 272, 3, 1), ("Y4", 128, 64, 136, 3, 1),
    ("Y5", 64, 128, 136, 1, 1), ("Y8", 256, 128, 68, 3, 1), ("Y9", 128, 256, 68, 1, 1),
    ("Y12", 512, 256, 34, 3, 1), ("Y13", 256, 512, 34, 1, 1), ("Y18", 1024, 512, 17, 3, 1),
    ("Y19", 512, 1024, 17, 1, 1), ("Y23", 28269, 1024, 17, 1, 1),
    ("R1", 64, 3, 224, 7, 2), ("R2", 64, 64, 56, 3, 1), ("R3", 64, 64, 56, 1, 1),
    ("R4", 128, 64, 56, 3, 2), ("R5", 128, 64, 56, 1, 2), ("R6", 128, 128, 28, 3, 1),
    ("R7", 256, 128, 28, 3, 2), ("R8", 256, 128, 28, 3, 1), ("R9", 256, 256, 14, 3, 1),
    ("R10", 512, 256, 14, 3, 2), ("R11", 512, 256, 14, 1, 2), ("R12", 512, 512, 7, 3, 1),
    ("M1", 32, 32, 112, 3, 1), ("M2", 64, 64, 112, 3, 2), ("M3", 128, 128, 56, 3, 1),
    ("M4", 128, 128, 56, 3, 2), ("M5", 256, 256, 28, 3, 1), ("M6", 256, 256, 28, 3, 2),
    ("M7", 512, 512, 14, 3, 1), ("M8", 512, 512, 14, 3, 2), ("M9", 1024, 1024, 7, 3, 1),
]
TABLE1 = {name: Shape.strided(1, K, C, HW, HW, R, R, U) for name, K, C, HW, R, U in TABLE1_ROWS}


def make_inputs(shape: Shape, seed: int = 0, kind: str = "real"):
    """Return (In, Ker) as contiguous CPU fp32 tensors, In drawn first."""
    g = torch.Generator().manual_seed(int(seed))
    if kind == "real":
        inp = torch.rand(shape.in_shape, generator=g, dtype=torch.float32) * 2 - 1
        ker = torch.rand(shape.ker_shape, generator=g, dtype=torch.float32) * 2 - 1
    elif kind == "int":
        inp = torch.randint(-2, 3, shape.in_shape, generator=g).to(torch.float32)
        ker = torch.randint(-2, 3, shape.ker_shape, generator=g).to(torch.float32)
    else:
        raise ValueError(f"unknown input kind {kind!r}")
    return inp.contiguous(), ker.contiguous()
