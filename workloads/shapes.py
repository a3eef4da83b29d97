"""Conv shape tables for the paper's workloads (ResNet-50, MobileNet-v2, Inception-v3).

The paper evaluates these models (Table 2) but lists no layer
shapes; the tables below follow the torchvision definitions (SURVEY.md
Appendix A).  Pure data: no arithmetic of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class ConvShape:
    name: str
    C: int          # input channels
    K: int          # output channels
    H: int          # input height
    W: int          # input width
    R: int = 1
    S: int = 1
    stride: tuple = (1, 1)
    pad: tuple = (0, 0, 0, 0)   # top, left, bottom, right
    groups: int = 1
    relu: bool = True
    act6: bool = False          # ReLU6 (MobileNet) via output-domain act_max
    src: str = ""               # name of the layer whose output feeds this one ("" = fresh buffer)

    @property
    def P(self) -> int:
        return (self.H + self.pad[0] + self.pad[2] - (self.R - 1) - 1) // self.stride[0] + 1

    @property
    def Q(self) -> int:
        return (self.W + self.pad[1] + self.pad[3] - (self.S - 1) - 1) // self.stride[1] + 1

    def macs(self, n: int = 1) -> int:
        return n * self.P * self.Q * self.K * (self.C // self.groups) * self.R * self.S


def _c(name, C, K, H, R=1, s=1, p=None, relu=True, src="", groups=1, act6=False, W=None, S=None):
    if S is None:
        S = R
    if W is None:
        W = H
    if p is None:
        p = ((R - 1) // 2, (S - 1) // 2, (R - 1) // 2, (S - 1) // 2)
    elif isinstance(p, int):
        p = (p, p, p, p)
    return ConvShape(name, C, K, H, W, R, S, (s, s), p, groups, relu, act6, src)


def resnet50_convs() -> list[ConvShape]:
    """The 53 convolutions of ResNet-50 v1.5 at 224x224 (stride on the 3x3)."""
    L = [_c("conv1", 3, 64, 224, 7, 2, 3)]
    cin, H = 64, 56
    prev = ""          # stem output passes through maxpool (glue, not on the path) -> fresh buffer
    for li, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)], 1):
        out = width * 4
        for b in range(blocks):
            s = stride if b == 0 else 1
            pre = f"layer{li}.{b}"
            L.append(_c(f"{pre}.conv1", cin, width, H, 1, 1, 0, src=prev))
            L.append(_c(f"{pre}.conv2", width, width, H, 3, s, 1, src=f"{pre}.conv1"))
            H2 = (H + 2 - 3) // s + 1
            L.append(_c(f"{pre}.conv3", width, out, H2, 1, 1, 0, relu=False, src=f"{pre}.conv2"))
            if b == 0:
                L.append(_c(f"{pre}.downsample", cin, out, H, 1, s, 0, relu=False, src=prev))
            prev = f"{pre}.conv3"
            cin, H = out, H2
    assert len(L) == 53
    return L


def resnet50_fc() -> tuple[int, int]:
    """(in_features, out_features) of the final dense layer."""
    return 2048, 1000


def resnet50_unique() -> list[ConvShape]:
    """Unique conv shapes of ResNet-50 (the C2 layer sweep)."""
    seen, out = set(), []
    for c in resnet50_convs():
        key = (c.C, c.K, c.H, c.R, c.stride)
        if key not in seen:
            seen.add(key)
            out.append(c)
    return out


def mobilenet_v2_convs() -> list[ConvShape]:
    """MobileNet-v2 (width 1.0, 224x224): stem, 17 inverted residual blocks, last 1x1."""
    L = [_c("stem", 3, 32, 224, 3, 2, 1, act6=True)]
    cin, H, prev = 32, 112, "stem"
    cfg = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
    bi = 0
    for t, c, n, s in cfg:
        for i in range(n):
            st = s if i == 0 else 1
            hid = cin * t
            pre = f"block{bi}"
            if t != 1:
                L.append(_c(f"{pre}.expand", cin, hid, H, 1, 1, 0, act6=True, src=prev))
                prev = f"{pre}.expand"
            L.append(_c(f"{pre}.dw", hid, hid, H, 3, st, 1, groups=hid, act6=True, src=prev))
            H2 = (H + 2 - 3) // st + 1
            L.append(_c(f"{pre}.project", hid, c, H2, 1, 1, 0, relu=False, src=f"{pre}.dw"))
            prev, cin, H = f"{pre}.project", c, H2
            bi += 1
    L.append(_c("last", 320, 1280, 7, 1, 1, 0, act6=True, src=prev))
    return L


def inception_v3_convs() -> list[ConvShape]:
    """Inception-v3 (299x299) convolutions, torchvision layout (94 convs)."""
    L = []

    def add(name, C, K, H, R, S=None, s=1, p=None, W=None):
        L.append(_c(name, C, K, H, R, s, p, S=S, W=W))

    add("Conv2d_1a_3x3", 3, 32, 299, 3, s=2, p=0)
    add("Conv2d_2a_3x3", 32, 32, 149, 3, p=0)
    add("Conv2d_2b_3x3", 32, 64, 147, 3, p=1)
    add("Conv2d_3b_1x1", 64, 80, 73, 1, p=0)
    add("Conv2d_4a_3x3", 80, 192, 73, 3, p=0)

    def mixed_a(n, cin, pool_features, H=35):
        add(f"{n}.branch1x1", cin, 64, H, 1)
        add(f"{n}.branch5x5_1", cin, 48, H, 1)
        add(f"{n}.branch5x5_2", 48, 64, H, 5)
        add(f"{n}.branch3x3dbl_1", cin, 64, H, 1)
        add(f"{n}.branch3x3dbl_2", 64, 96, H, 3)
        add(f"{n}.branch3x3dbl_3", 96, 96, H, 3)
        add(f"{n}.branch_pool", cin, pool_features, H, 1)

    mixed_a("Mixed_5b", 192, 32)
    mixed_a("Mixed_5c", 256, 64)
    mixed_a("Mixed_5d", 288, 64)
    # Mixed_6a (reduction)
    add("Mixed_6a.branch3x3", 288, 384, 35, 3, s=2, p=0)
    add("Mixed_6a.branch3x3dbl_1", 288, 64, 35, 1)
    add("Mixed_6a.branch3x3dbl_2", 64, 96, 35, 3)
    add("Mixed_6a.branch3x3dbl_3", 96, 96, 35, 3, s=2, p=0)

    def mixed_c(n, c7, H=17):
        cin = 768
        add(f"{n}.branch1x1", cin, 192, H, 1)
        add(f"{n}.branch7x7_1", cin, c7, H, 1)
        add(f"{n}.branch7x7_2", c7, c7, H, 1, S=7, p=(0, 3, 0, 3))
        add(f"{n}.branch7x7_3", c7, 192, H, 7, S=1, p=(3, 0, 3, 0))
        add(f"{n}.branch7x7dbl_1", cin, c7, H, 1)
        add(f"{n}.branch7x7dbl_2", c7, c7, H, 7, S=1, p=(3, 0, 3, 0))
        add(f"{n}.branch7x7dbl_3", c7, c7, H, 1, S=7, p=(0, 3, 0, 3))
        add(f"{n}.branch7x7dbl_4", c7, c7, H, 7, S=1, p=(3, 0, 3, 0))
        add(f"{n}.branch7x7dbl_5", c7, 192, H, 1, S=7, p=(0, 3, 0, 3))
        add(f"{n}.branch_pool", cin, 192, H, 1)

    mixed_c("Mixed_6b", 128)
    mixed_c("Mixed_6c", 160)
    mixed_c("Mixed_6d", 160)
    mixed_c("Mixed_6e", 192)
    # Mixed_7a (reduction)
    add("Mixed_7a.branch3x3_1", 768, 192, 17, 1)
    add("Mixed_7a.branch3x3_2", 192, 320, 17, 3, s=2, p=0)
    add("Mixed_7a.branch7x7x3_1", 768, 192, 17, 1)
    add("Mixed_7a.branch7x7x3_2", 192, 192, 17, 1, S=7, p=(0, 3, 0, 3))
    add("Mixed_7a.branch7x7x3_3", 192, 192, 17, 7, S=1, p=(3, 0, 3, 0))
    add("Mixed_7a.branch7x7x3_4", 192, 192, 17, 3, s=2, p=0)

    def mixed_e(n, cin, H=8):
        add(f"{n}.branch1x1", cin, 320, H, 1)
        add(f"{n}.branch3x3_1", cin, 384, H, 1)
        add(f"{n}.branch3x3_2a", 384, 384, H, 1, S=3, p=(0, 1, 0, 1))
        add(f"{n}.branch3x3_2b", 384, 384, H, 3, S=1, p=(1, 0, 1, 0))
        add(f"{n}.branch3x3dbl_1", cin, 448, H, 1)
        add(f"{n}.branch3x3dbl_2", 448, 384, H, 3)
        add(f"{n}.branch3x3dbl_3a", 384, 384, H, 1, S=3, p=(0, 1, 0, 1))
        add(f"{n}.branch3x3dbl_3b", 384, 384, H, 3, S=1, p=(1, 0, 1, 0))
        add(f"{n}.branch_pool", cin, 192, H, 1)

    mixed_e("Mixed_7b", 1280)
    mixed_e("Mixed_7c", 2048)
    assert len(L) == 94, len(L)
    return L
