"""Operator graphs of the paper's whole-model workloads, synthetic weights.

Architectures follow SURVEY.md §8(d) (public model definitions, treated as proposals):
  candy       fast-neural-style TransformerNet (artifact model P:741-743) at 224^2:
              reflect-pad + conv, InstanceNorm(affine), ReLU, 5 residual blocks,
              nearest x2 upsample + conv, 9x9 output conv.
  segformer   SegFormer-B0 (artifact model P:743) at 512^2: MiT-b0 encoder
              (C = 32/64/160/256, heads 1/2/5/8, sr 8/4/2/1, depth 2/2/2/2, MLP x4,
              LN eps 1e-6, overlapping patch embeddings, Mix-FFN with 3x3 depthwise conv)
              + all-MLP decoder (256 channels, 150 classes).  Token layout [1, HW, C];
              the decoder's 1x1 convolutions are written as MatMuls on tokens and its
              upsampling is nearest (the public model uses bilinear).
BatchNorms are folded into the preceding conv at build time.
"""
from __future__ import annotations

import math

from .graphs import GraphBuilder


class _M:
    """Small helper around GraphBuilder that names weights automatically."""

    def __init__(self, dtype):
        self.b = GraphBuilder(dtype)
        self.n = 0

    def w(self, shape, std=None, mean=0.0, suffix=""):
        self.n += 1
        fan_in = 1
        for d in shape[1:] if len(shape) > 1 else shape:
            fan_in *= d
        if std is None:
            std = 1.0 / math.sqrt(max(1, fan_in))
        return self.b.input(f"w{self.n}{suffix}", shape, mean=mean, std=std)

    def op(self, *a, **k):
        return self.b.op(*a, **k)


# ---------------------------------------------------------------------------------- Candy
def candy(size: int = 224, dtype: str = "bf16", blocks: int = 5, batch: int = 1):
    m = _M(dtype)
    x = m.b.input("x", [batch, 3, size, size])

    def conv_layer(h, cin, cout, k, stride):
        p = k // 2
        h = m.op("Pad", h, pads=[[0, 0], [0, 0], [p, p], [p, p]], mode="reflect")
        w = m.w([cout, cin, k, k], std=math.sqrt(2.0 / (cin * k * k)))
        bias = m.w([cout], std=0.02)
        return m.op("Conv", h, w, bias, stride=[stride, stride], pads=[0, 0], groups=1)

    def inorm(h, c):
        g = m.w([c], mean=1.0, std=0.1)
        be = m.w([c], std=0.1)
        return m.op("InstanceNorm", h, g, be, eps=1e-5)

    h = m.op("Relu", inorm(conv_layer(x, 3, 32, 9, 1), 32))
    h = m.op("Relu", inorm(conv_layer(h, 32, 64, 3, 2), 64))
    h = m.op("Relu", inorm(conv_layer(h, 64, 128, 3, 2), 128))
    for _ in range(blocks):
        r = h
        t = m.op("Relu", inorm(conv_layer(h, 128, 128, 3, 1), 128))
        t = inorm(conv_layer(t, 128, 128, 3, 1), 128)
        h = m.op("Add", t, r)
    h = m.op("Upsample2x", h)
    h = m.op("Relu", inorm(conv_layer(h, 128, 64, 3, 1), 64))
    h = m.op("Upsample2x", h)
    h = m.op("Relu", inorm(conv_layer(h, 64, 32, 3, 1), 32))
    h = conv_layer(h, 32, 3, 9, 1)
    m.b.output(h)
    return m.b.build()


# ------------------------------------------------------------------------------ SegFormer
def segformer(size: int = 512, dtype: str = "bf16", dims=(32, 64, 160, 256), heads=(1, 2, 5, 8),
              srs=(8, 4, 2, 1), depths=(2, 2, 2, 2), mlp=4, decoder=256, classes=150, batch: int = 1):
    m = _M(dtype)
    nb = batch
    x = m.b.input("x", [nb, 3, size, size])
    eps = 1e-6

    def ln(t, c):
        g = m.w([c], mean=1.0, std=0.1)
        be = m.w([c], std=0.1)
        return m.op("LayerNorm", t, g, be, axis=-1, eps=eps)

    def linear(t, cin, cout):
        w = m.w([cin, cout])
        b = m.w([cout], std=0.02)
        return m.op("Add", m.op("MatMul", t, w), b)

    def to_tokens(t, c, h, w):          # [N,C,H,W] -> [N,HW,C]
        t = m.op("Reshape", t, shape=[nb, c, h * w])
        return m.op("Transpose", t, perm=[0, 2, 1])

    def to_nchw(t, c, h, w):            # [N,HW,C] -> [N,C,H,W]
        t = m.op("Transpose", t, perm=[0, 2, 1])
        return m.op("Reshape", t, shape=[nb, c, h, w])

    feats = []
    cur, cin, hw = x, 3, size
    for s, (c, nh, sr, depth) in enumerate(zip(dims, heads, srs, depths)):
        k, st = (7, 4) if s == 0 else (3, 2)
        w = m.w([c, cin, k, k])
        b = m.w([c], std=0.02)
        t = m.op("Conv", cur, w, b, stride=[st, st], pads=[k // 2, k // 2], groups=1)
        hw = hw // st
        n = hw * hw
        t = ln(to_tokens(t, c, hw, hw), c)
        d = c // nh
        for _ in range(depth):
            # efficient self-attention with spatial reduction
            y = ln(t, c)
            q = linear(y, c, c)
            if sr > 1:
                kvx = to_nchw(y, c, hw, hw)
                wr = m.w([c, c, sr, sr])
                br = m.w([c], std=0.02)
                kvx = m.op("Conv", kvx, wr, br, stride=[sr, sr], pads=[0, 0], groups=1)
                nr = (hw // sr) ** 2
                kvx = ln(to_tokens(kvx, c, hw // sr, hw // sr), c)
            else:
                kvx, nr = y, n
            kv = linear(kvx, c, 2 * c)
            qh = m.op("Transpose", m.op("Reshape", q, shape=[nb, n, nh, d]), perm=[0, 2, 1, 3])
            kk = m.op("Slice", kv, axis=2, start=0, end=c)
            vv = m.op("Slice", kv, axis=2, start=c, end=2 * c)
            kt = m.op("Transpose", m.op("Reshape", kk, shape=[nb, nr, nh, d]), perm=[0, 2, 3, 1])
            vh = m.op("Transpose", m.op("Reshape", vv, shape=[nb, nr, nh, d]), perm=[0, 2, 1, 3])
            sc = m.op("DivC", m.op("MatMul", qh, kt), c=math.sqrt(d))
            p = m.op("Softmax", sc, axis=3)
            o = m.op("MatMul", p, vh)
            o = m.op("Reshape", m.op("Transpose", o, perm=[0, 2, 1, 3]), shape=[nb, n, c])
            t = m.op("Add", t, linear(o, c, c))
            # Mix-FFN: fc1 -> 3x3 depthwise conv -> GELU -> fc2
            y = ln(t, c)
            y = linear(y, c, mlp * c)
            y = to_nchw(y, mlp * c, hw, hw)
            wd = m.w([mlp * c, 1, 3, 3], std=1.0 / 3.0)
            bd = m.w([mlp * c], std=0.02)
            y = m.op("Conv", y, wd, bd, stride=[1, 1], pads=[1, 1], groups=mlp * c)
            y = m.op("GELU", to_tokens(y, mlp * c, hw, hw))
            t = m.op("Add", t, linear(y, mlp * c, c))
        t = ln(t, c)
        feats.append((t, c, hw))
        cur, cin = to_nchw(t, c, hw, hw), c
    # all-MLP decoder: project every stage to `decoder` channels, upsample to 1/4, fuse
    top = feats[0][2]
    ups = []
    for (t, c, hw) in reversed(feats):
        u = linear(t, c, decoder)                                 # [N, hw*hw, D]
        f = top // hw
        if f > 1:                                                 # nearest x f in NHWC tokens
            u = m.op("Reshape", u, shape=[nb, hw, hw, decoder])
            u = m.op("Broadcast", u, axis=2, size=f)
            u = m.op("Broadcast", u, axis=4, size=f)
            u = m.op("Reshape", u, shape=[nb, top * top, decoder])
        ups.append(u)
    u = m.op("Concat", *ups, axis=2)                              # [1, top^2, 4D]
    u = m.op("Relu", linear(u, 4 * decoder, decoder))             # linear_fuse (+folded BN) + ReLU
    u = linear(u, decoder, classes)                               # linear_pred
    m.b.output(u)
    return m.b.build()


# --------------------------------------------------------------------------- EfficientViT
def efficientvit(size: int = 224, dtype: str = "bf16", widths=(16, 32, 64, 128, 256), depths=(1, 2, 3, 3, 4),
                 dim: int = 16, expand: int = 4, eps: float = 1e-15, batch: int = 1):
    """EfficientViT-B1 backbone: conv stem + DSConv, MBConv
    stages, then EfficientViT blocks (LiteMLA ReLU linear attention with 5x5 multi-scale
    aggregation + MBConv).  Hardswish activations, BN folded.  Pointwise (1x1) convs are
    MatMuls over [C, HW] (tcgen05 GEMMs); depthwise / strided convs stay Conv.  At batch
    N > 1 a pointwise conv is the token-major MatMul [N, HW, Cin] x W^T (see _pw)."""
    m = _M(dtype)
    nb = batch
    x = m.b.input("x", [nb, 3, size, size])

    def conv(h, cin, cout, k, stride=1, groups=1, bias=True):
        w = m.w([cout, cin // groups, k, k])
        args = [h, w] + ([m.w([cout], std=0.02)] if bias else [])
        return m.op("Conv", *args, stride=[stride, stride], pads=[k // 2, k // 2], groups=groups)

    def pw(h, cin, cout, hw, bias=True):             # 1x1 conv as MatMul on [C, HW]
        if nb > 1:
            return _pw(m, h, nb, cin, cout, hw, bias)
        t = m.op("Reshape", h, shape=[cin, hw * hw])
        t = m.op("MatMul", m.w([cout, cin]), t)
        if bias:
            t = m.op("Add", t, m.w([cout, 1], std=0.02))
        return m.op("Reshape", t, shape=[1, cout, hw, hw])

    def mbconv(h, cin, cout, hw, stride, act_last=False):
        mid = cin * expand
        t = m.op("HardSwish", pw(h, cin, mid, hw))
        t = m.op("HardSwish", conv(t, mid, mid, 3, stride, groups=mid))
        hw2 = hw // stride
        t = pw(t, mid, cout, hw2)
        return (m.op("HardSwish", t) if act_last else t), hw2

    def lite_mla(h, c, hw):
        heads = c // dim
        n = hw * hw
        qkv = pw(h, c, 3 * c, hw, bias=False)                                        # [1,3c,hw,hw]
        agg = conv(qkv, 3 * c, 3 * c, 5, groups=3 * c, bias=False)                   # 5x5 depthwise
        agg = conv(agg, 3 * c, 3 * c, 1, groups=3 * heads, bias=False)               # grouped 1x1
        ms = m.op("Concat", qkv, agg, axis=1)                                        # [1,6c,hw,hw]
        ms = m.op("Reshape", ms, shape=[nb, 2 * heads, 3 * dim, n])
        ms = m.op("Transpose", ms, perm=[0, 1, 3, 2])                                # [1,2h,n,3d]
        q = m.op("Relu", m.op("Slice", ms, axis=3, start=0, end=dim))
        k = m.op("Relu", m.op("Slice", ms, axis=3, start=dim, end=2 * dim))
        v = m.op("Slice", ms, axis=3, start=2 * dim, end=3 * dim)
        v = m.op("Pad", v, pads=[[0, 0], [0, 0], [0, 0], [0, 1]], mode="constant", value=1.0)
        kt = m.op("Transpose", k, perm=[0, 1, 3, 2])                                 # [1,2h,d,n]
        kv = m.op("MatMul", kt, v)                                                   # [1,2h,d,d+1]
        o = m.op("MatMul", q, kv)                                                    # [1,2h,n,d+1]
        num = m.op("Slice", o, axis=3, start=0, end=dim)
        den = m.op("AddC", m.op("Slice", o, axis=3, start=dim, end=dim + 1), c=eps)
        den = m.op("Reshape", den, shape=[nb, 2 * heads, n])
        o = m.op("Div", num, m.op("Broadcast", den, axis=3, size=dim))
        o = m.op("Transpose", o, perm=[0, 1, 3, 2])                                  # [1,2h,d,n]
        o = m.op("Reshape", o, shape=[nb, 2 * c, hw, hw])
        return pw(o, 2 * c, c, hw)

    h = m.op("HardSwish", conv(x, 3, widths[0], 3, 2))
    hw = size // 2
    for _ in range(depths[0]):                                                       # DSConv + residual
        t = m.op("HardSwish", conv(h, widths[0], widths[0], 3, groups=widths[0]))
        h = m.op("Add", h, pw(t, widths[0], widths[0], hw))
    cin = widths[0]
    for w, d in zip(widths[1:3], depths[1:3]):
        for i in range(d):
            t, hw2 = mbconv(h, cin, w, hw, 2 if i == 0 else 1)
            h = t if i == 0 else m.op("Add", h, t)
            hw, cin = hw2, w
    for w, d in zip(widths[3:], depths[3:]):
        h, hw = mbconv(h, cin, w, hw, 2)
        cin = w
        for _ in range(d):
            h = m.op("Add", h, lite_mla(h, w, hw))
            t, _ = mbconv(h, w, w, hw, 1)
            h = m.op("Add", h, t)
    m.b.output(h)
    return m.b.build()


# ----------------------------------------------------------------------------- YOLOX-Nano
def yolox_nano(size: int = 416, dtype: str = "bf16", width: float = 0.25, classes: int = 80, batch: int = 1):
    """YOLOX-Nano: Focus, depthwise CSPDarknet (depth 0.33,
    width 0.25), SPP 5/9/13, PAFPN, decoupled heads; SiLU, BN folded.  Output
    [1, 3549, 85] at 416^2 = cat(reg, sigmoid(obj), sigmoid(cls)) per anchor point (the box
    decode with grids / strides is not part of the graph).  1x1 convs are MatMuls over
    [C, HW]; depthwise and 3x3 convs stay Conv.  At batch N > 1 a pointwise conv is the
    token-major MatMul [N, HW, Cin] x W^T (see _pw) and the output is [N, 3549, 85]."""
    m = _M(dtype)
    nb = batch
    x = m.b.input("x", [nb, 3, size, size])
    c0 = int(64 * width)

    def silu(h):
        return m.op("SiLU", h)

    def pw(h, cin, cout, hw):                       # BaseConv 1x1 + SiLU as a MatMul
        if nb > 1:
            return silu(_pw(m, h, nb, cin, cout, hw, True))
        t = m.op("Reshape", h, shape=[cin, hw * hw])
        t = m.op("Add", m.op("MatMul", m.w([cout, cin]), t), m.w([cout, 1], std=0.02))
        return silu(m.op("Reshape", t, shape=[1, cout, hw, hw]))

    def conv(h, cin, cout, k, stride, groups=1):
        t = m.op("Conv", h, m.w([cout, cin // groups, k, k]), m.w([cout], std=0.02),
                 stride=[stride, stride], pads=[k // 2, k // 2], groups=groups)
        return silu(t)

    def dwconv(h, cin, cout, hw, stride=1):         # depthwise 3x3 + pointwise 1x1
        t = conv(h, cin, cin, 3, stride, groups=cin)
        return pw(t, cin, cout, hw // stride), hw // stride

    def csp(h, cin, cout, hw, n, shortcut=True):
        hid = cout // 2
        x1 = pw(h, cin, hid, hw)
        for _ in range(n):
            y = pw(x1, hid, hid, hw)
            y, _ = dwconv(y, hid, hid, hw)
            x1 = m.op("Add", y, x1) if shortcut else y
        x2 = pw(h, cin, hid, hw)
        return pw(m.op("Concat", x1, x2, axis=1), 2 * hid, cout, hw)

    # Focus: space-to-depth, channel order (w-parity, h-parity, c)
    hw = size // 2
    f = m.op("Reshape", x, shape=[nb, 3, hw, 2, hw, 2])
    f = m.op("Transpose", f, perm=[0, 5, 3, 1, 2, 4])
    f = m.op("Reshape", f, shape=[nb, 12, hw, hw])
    h = conv(f, 12, c0, 3, 1)
    h, hw = dwconv(h, c0, 2 * c0, hw, 2)
    h = csp(h, 2 * c0, 2 * c0, hw, 1)
    h, hw = dwconv(h, 2 * c0, 4 * c0, hw, 2)
    x2 = csp(h, 4 * c0, 4 * c0, hw, 1)                                      # 52^2, 64
    h, hw1 = dwconv(x2, 4 * c0, 8 * c0, hw, 2)
    x1 = csp(h, 8 * c0, 8 * c0, hw1, 1)                                     # 26^2, 128
    h, hw0 = dwconv(x1, 8 * c0, 16 * c0, hw1, 2)
    sp = pw(h, 16 * c0, 8 * c0, hw0)                                        # SPP
    pools = [m.op("MaxPool", sp, k=k, stride=1, pad=k // 2) for k in (5, 9, 13)]
    h = pw(m.op("Concat", sp, *pools, axis=1), 32 * c0, 16 * c0, hw0)
    x0 = csp(h, 16 * c0, 16 * c0, hw0, 1, shortcut=False)                  # 13^2, 256
    # PAFPN
    fpn0 = pw(x0, 16 * c0, 8 * c0, hw0)
    u = m.op("Concat", m.op("Upsample2x", fpn0), x1, axis=1)
    u = csp(u, 16 * c0, 8 * c0, hw1, 1, shortcut=False)
    fpn1 = pw(u, 8 * c0, 4 * c0, hw1)
    u = m.op("Concat", m.op("Upsample2x", fpn1), x2, axis=1)
    pan2 = csp(u, 8 * c0, 4 * c0, hw, 1, shortcut=False)                   # 52^2, 64
    d, _ = dwconv(pan2, 4 * c0, 4 * c0, hw, 2)
    pan1 = csp(m.op("Concat", d, fpn1, axis=1), 8 * c0, 8 * c0, hw1, 1, shortcut=False)
    d, _ = dwconv(pan1, 8 * c0, 8 * c0, hw1, 2)
    pan0 = csp(m.op("Concat", d, fpn0, axis=1), 16 * c0, 16 * c0, hw0, 1, shortcut=False)
    # decoupled heads
    hid = int(256 * width)
    outs = []
    for feat, cin, s in ((pan2, 4 * c0, hw), (pan1, 8 * c0, hw1), (pan0, 16 * c0, hw0)):
        st = pw(feat, cin, hid, s)
        c, _ = dwconv(st, hid, hid, s)
        c, _ = dwconv(c, hid, hid, s)
        r, _ = dwconv(st, hid, hid, s)
        r, _ = dwconv(r, hid, hid, s)

        if nb > 1:
            def pred(t, cout):                                                   # [N, s*s, cout]
                return _pw(m, t, nb, hid, cout, s, True, tokens_out=True)
            o = m.op("Concat", pred(r, 4), m.op("Sigmoid", pred(r, 1)), m.op("Sigmoid", pred(c, classes)), axis=2)
            outs.append(o)                                                       # [N, s*s, 85]
            continue

        def pred(t, cout):
            t2 = m.op("Reshape", t, shape=[hid, s * s])
            return m.op("Add", m.op("MatMul", m.w([cout, hid]), t2), m.w([cout, 1], std=0.02))   # [cout, s*s]
        o = m.op("Concat", pred(r, 4), m.op("Sigmoid", pred(r, 1)), m.op("Sigmoid", pred(c, classes)), axis=0)
        outs.append(o)                                                                           # [85, s*s]
    if nb > 1:
        m.b.output(m.op("Concat", *outs, axis=1))                                                # [N, 3549, 85]
        return m.b.build()
    o = m.op("Concat", *outs, axis=1)                                                            # [85, 3549]
    o = m.op("Transpose", o, perm=[1, 0])
    m.b.output(m.op("Reshape", o, shape=[1, o_n(size), 5 + classes]))
    return m.b.build()


def _pw(m, h, nb, cin, cout, hw, bias, tokens_out=False):
    """Batched pointwise (1x1) convolution on [N, Cin, H, W] as a token-major MatMul:
    [N, HW, Cin] x W^T[Cin, Cout] (+ bias) -> [N, Cout, H, W] (or the [N, HW, Cout] tokens).
    MatMul broadcasts a 2-D B over the batch (ONNX semantics); the transposes are layout
    primitives the GEMM template folds into its operand views / store addresses."""
    t = m.op("Reshape", h, shape=[nb, cin, hw * hw])
    t = m.op("Transpose", t, perm=[0, 2, 1])
    t = m.op("MatMul", t, m.w([cin, cout], std=1.0 / math.sqrt(cin), suffix="T"))   # W^T of the batch-1 graph
    if bias:
        t = m.op("Add", t, m.w([cout], std=0.02))
    if tokens_out:
        return t
    t = m.op("Transpose", t, perm=[0, 2, 1])
    return m.op("Reshape", t, shape=[nb, cout, hw, hw])


def o_n(size):
    return sum((size // s) ** 2 for s in (8, 16, 32))


MODELS = {"candy": candy, "segformer": segformer, "efficientvit": efficientvit, "yolox": yolox_nano,
          # the paper's EfficientViT resolution (reading A22), 1024:1 K^T V at stage 3
          "efficientvit2048": lambda batch=1: efficientvit(size=2048, batch=batch)}
