"""Model sources in the reference's own text format (``.rly``) plus seeded weights.

The reference (MicroRelay) has no model zoo: its only model interchange is the
text format (``parser.cpp`` / ``printer.cpp``).  This module
writes the *unfused* CNNs of BASELINE.json's configs as ``def @main(...)``
programs in that format, with

* conv/dense weights and biases as ``@main`` parameters (so the reference's
  ``fold`` leaves them alone and the backend hoists their prologues to
  weight-load time),
* folded batch-norm as ``multiply(conv, gamma'[C,1,1])`` with gamma' a metadata
  constant -- ``ScaleFolder::const_of`` only folds constants
  (``rewrites.cpp:117-126``),
* pooling as the extension operator ``max_pool2d(x, %win)`` whose window
  argument is a shape-only ``[C, C, KH, KW]`` parameter typed by the
  reference's existing ``Conv2D`` relation,
* a symbolic batch dimension ``?n`` so one fused module serves every batch
  shard (``test_infer.cpp:90-102``).

Weights come from ``numpy.random.Generator(PCG64(seed))``: He-normal
N(0, sqrt(2/fan_in)) for conv/dense, N(0, 0.05) for biases, U[0.5, 1.5) for
gamma' (SURVEY.md 8(d) "Weights and seeds").  The same host buffers go to the
CPU oracle and to the GPU.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Tuple

import numpy as np


def fmt_f32(v: float) -> str:
    """%.9g of a float32, always with a float marker (the parser reads a bare
    integer token as an int32 scalar, parser.cpp:631)."""
    s = "%.9g" % float(np.float32(v))
    if not any(ch in s for ch in ".eEn"):
        s += ".0"
    return s


@dataclasses.dataclass
class Param:
    name: str
    shape: Tuple  # first dim may be "?n"
    kind: str  # "input" | "conv_w" | "dense_w" | "bias" | "window"


@dataclasses.dataclass
class ModelSource:
    name: str
    text: str
    params: List[Param]
    input_shape: Tuple[int, ...]  # per-sample (C, H, W)
    num_classes: int

    def param_shapes(self, batch: int) -> Dict[str, Tuple[int, ...]]:
        out = {}
        for p in self.params:
            out[p.name] = tuple(batch if d == "?n" else d for d in p.shape)
        return out


class _Builder:
    def __init__(self, seed: int):
        self.rng = np.random.Generator(np.random.PCG64(seed))
        self.params: List[Param] = []
        self.lines: List[str] = []
        self.meta: List[str] = []
        self.counter = 0

    def fresh(self, prefix="v"):
        self.counter += 1
        return "%s%d" % (prefix, self.counter)

    def param(self, name, shape, kind):
        self.params.append(Param(name, tuple(shape), kind))
        return "%" + name

    def let(self, expr):
        v = self.fresh()
        self.lines.append("  let %%%s = %s;" % (v, expr))
        return "%" + v

    def meta_const(self, values: np.ndarray, shape):
        vals = ", ".join(fmt_f32(x) for x in np.asarray(values, np.float32).reshape(-1))
        shp = "(" + ", ".join(str(d) for d in shape) + ")"
        self.meta.append("  const[%d] = const([%s], %s, float32);" % (len(self.meta), vals, shp))
        return "meta[Constant][%d]" % (len(self.meta) - 1)

    # layers ---------------------------------------------------------------
    def conv_bn(self, x, cin, cout, k, stride, pad, tag, relu=True, bn=True, act=None):
        w = self.param("w_" + tag, (cout, cin, k, k), "conv_w")
        y = self.let("conv2d(%s, %s, strides=(%d, %d), padding=(%d, %d))" % (x, w, stride, stride, pad, pad))
        if bn:
            gamma = self.rng.uniform(0.5, 1.5, size=(cout,)).astype(np.float32)
            y = self.let("multiply(%s, %s)" % (y, self.meta_const(gamma, (cout, 1, 1))))
        b = self.param("b_" + tag, (cout,), "bias")
        y = self.let("bias_add(%s, %s)" % (y, b))
        if act is not None:
            return self.act(y, act)
        if relu:
            y = self.let("relu(%s)" % y)
        return y

    def max_pool(self, x, c, k, stride, pad, tag):
        win = self.param("win_" + tag, (c, c, k, k), "window")
        return self.let("max_pool2d(%s, %s, strides=(%d, %d), padding=(%d, %d))" % (x, win, stride, stride, pad, pad))

    def dense(self, x, cin, cout, tag, relu=False):
        w = self.param("w_" + tag, (cout, cin), "dense_w")
        y = self.let("dense(%s, %s)" % (x, w))
        b = self.param("b_" + tag, (cout,), "bias")
        y = self.let("bias_add(%s, %s)" % (y, b))
        if relu:
            y = self.let("relu(%s)" % y)
        return y

    def depthwise_bn(self, x, c, k, stride, pad, tag, act="relu6"):
        """depthwise_conv2d (extension op, registered on the reference's
        OpRegistry by oracle/ref_harness.cpp) + folded BN (channel multiply
        left in the epilogue: fold-scale folds only conv2d) + bias + relu6."""
        win = self.param("win_" + tag, (c, c, k, k), "window")
        w = self.param("w_" + tag, (c, 1, k, k), "dw_w")
        y = self.let("depthwise_conv2d(%s, %s, %s, strides=(%d, %d), padding=(%d, %d))"
                     % (x, win, w, stride, stride, pad, pad))
        gamma = self.rng.uniform(0.5, 1.5, size=(c,)).astype(np.float32)
        y = self.let("multiply(%s, %s)" % (y, self.meta_const(gamma, (c, 1, 1))))
        b = self.param("b_" + tag, (c,), "bias")
        y = self.let("bias_add(%s, %s)" % (y, b))
        return self.act(y, act)

    def act(self, y, act):
        if act == "relu":
            return self.let("relu(%s)" % y)
        if act == "relu6":
            return self.let("clip(%s, a_min=0.0, a_max=6.0)" % y)
        return y

    def finish(self, name, result, input_shape, num_classes):
        sig = []
        for p in self.params:
            dims = ", ".join(str(d) for d in p.shape)
            sig.append("%%%s: Tensor[(%s), float32]" % (p.name, dims))
        body = "\n".join(self.lines)
        text = "def @main(%s) {\n%s\n  %s\n}\n" % (", ".join(sig), body, result)
        if self.meta:
            text += "metadata {\n" + "\n".join(self.meta) + "\n}\n"
        return ModelSource(name, text, list(self.params), tuple(input_shape), num_classes)


def resnet18(image: int = 224, num_classes: int = 1000, seed: int = 1,
             widths=(64, 128, 256, 512)) -> ModelSource:
    """ResNet-18 v1 (BasicBlock x [2,2,2,2]) with folded BN, NCHW."""
    b = _Builder(seed)
    x = b.param("x", ("?n", 3, image, image), "input")
    y = b.conv_bn(x, 3, widths[0], 7, 2, 3, "stem")
    y = b.max_pool(y, widths[0], 3, 2, 1, "pool")
    hw = (image + 2 * 3 - 7) // 2 + 1
    hw = (hw + 2 - 3) // 2 + 1
    cin = widths[0]
    for li, cout in enumerate(widths):
        for bi in range(2):
            stride = 2 if (li > 0 and bi == 0) else 1
            tag = "l%db%d" % (li + 1, bi)
            a = b.conv_bn(y, cin, cout, 3, stride, 1, tag + "c1")
            a = b.conv_bn(a, cout, cout, 3, 1, 1, tag + "c2", relu=False)
            if stride != 1 or cin != cout:
                sc = b.conv_bn(y, cin, cout, 1, stride, 0, tag + "ds", relu=False)
            else:
                sc = y
            y = b.let("relu(%s)" % b.let("add(%s, %s)" % (a, sc)))
            cin = cout
        if li > 0:
            hw = (hw + 2 - 3) // 2 + 1
    g = b.let("sum(%s, axis=(2, 3))" % y)
    g = b.let("multiply(%s, const %s)" % (g, fmt_f32(1.0 / (hw * hw))))
    out = b.dense(g, cin, num_classes, "fc")
    return b.finish("resnet18", out, (3, image, image), num_classes)


def mobilenet_v1(image: int = 224, num_classes: int = 1000, seed: int = 1, alpha: float = 1.0) -> ModelSource:
    """MobileNet-v1: 3x3/s2 stem, 13 x {depthwise
    3x3 + BN + relu6, pointwise 1x1 + BN + relu6}, global average (sum x 1/HW)
    + dense."""
    b = _Builder(seed)
    c = lambda v: max(8, int(v * alpha))  # noqa: E731
    x = b.param("x", ("?n", 3, image, image), "input")
    y = b.conv_bn(x, 3, c(32), 3, 2, 1, "stem", act="relu6")
    hw = (image + 2 - 3) // 2 + 1
    cin = c(32)
    cfg = [(64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2)] + [(512, 1)] * 5 + [(1024, 2), (1024, 1)]
    for i, (cout, st) in enumerate(cfg):
        y = b.depthwise_bn(y, cin, 3, st, 1, "dw%d" % i)
        y = b.conv_bn(y, cin, c(cout), 1, 1, 0, "pw%d" % i, act="relu6")
        hw = (hw + 2 - 3) // st + 1
        cin = c(cout)
    g = b.let("sum(%s, axis=(2, 3))" % y)
    g = b.let("multiply(%s, const %s)" % (g, fmt_f32(1.0 / (hw * hw))))
    out = b.dense(g, cin, num_classes, "fc")
    return b.finish("mobilenet_v1", out, (3, image, image), num_classes)


def vgg16(image: int = 224, num_classes: int = 1000, seed: int = 1, batch: int = 1,
          widths=(64, 128, 256, 512, 512), fc: int = 4096) -> ModelSource:
    """VGG-16 (config C4): 13 x conv3x3 + bias + relu, 5 x max_pool 2x2/s2,
    flatten (reshape: static batch) + dense 4096 + relu, dense 4096 + relu,
    dense classes."""
    bld = _Builder(seed)
    x = bld.param("x", (batch, 3, image, image), "input")
    y, cin, hw = x, 3, image
    reps = (2, 2, 3, 3, 3)
    for si, (cout, r) in enumerate(zip(widths, reps)):
        for j in range(r):
            y = bld.conv_bn(y, cin, cout, 3, 1, 1, "c%d_%d" % (si + 1, j + 1), bn=False)
            cin = cout
        y = bld.max_pool(y, cin, 2, 2, 0, "p%d" % (si + 1))
        hw //= 2
    flat = cin * hw * hw
    y = bld.let("reshape(%s, newshape=(%d, %d))" % (y, batch, flat))
    y = bld.dense(y, flat, fc, "fc6", relu=True)
    y = bld.dense(y, fc, fc, "fc7", relu=True)
    out = bld.dense(y, fc, num_classes, "fc8")
    src = bld.finish("vgg16", out, (3, image, image), num_classes)
    return src


def dqn(num_actions: int = 18, seed: int = 1, batch: int = 1) -> ModelSource:
    """Nature DQN (config C4): x [N,4,84,84] scaled by 1/255, conv 8x8/s4
    4->32, conv 4x4/s2 32->64, conv 3x3/s1 64->64 (bias + relu each), flatten
    (static batch) + dense 512 + relu, dense actions."""
    bld = _Builder(seed)
    x = bld.param("x", (batch, 4, 84, 84), "input")
    y = bld.let("multiply(%s, const %s)" % (x, fmt_f32(1.0 / 255.0)))
    y = bld.conv_bn(y, 4, 32, 8, 4, 0, "c1", bn=False)
    y = bld.conv_bn(y, 32, 64, 4, 2, 0, "c2", bn=False)
    y = bld.conv_bn(y, 64, 64, 3, 1, 0, "c3", bn=False)
    y = bld.let("reshape(%s, newshape=(%d, %d))" % (y, batch, 64 * 7 * 7))
    y = bld.dense(y, 3136, 512, "fc1", relu=True)
    out = bld.dense(y, 512, num_actions, "fc2")
    return bld.finish("dqn", out, (4, 84, 84), num_actions)


MODELS = {"resnet18": resnet18, "mobilenet_v1": mobilenet_v1, "vgg16": vgg16, "dqn": dqn}


def branchy(image: int = 32, num_classes: int = 10, seed: int = 1, width: int = 32) -> ModelSource:
    """A small Inception-style net whose blocks hold PARALLEL convs over one
    input with the same in-channels, kernel and attributes -- the pattern the
    reference's combine-conv pass (rewrites.cpp:276-401) merges into one conv
    over concatenated weights + a split:
      stem 3x3 -> {1x1 a, 1x1 b, 1x1 c (half width)} -> 3x3 on a and b -> add
      -> {3x3 p, 3x3 r} -> add -> relu -> global sums -> two dense heads -> add.
    combine-conv only merges convs that bind back to back (none of them used
    before the last one binds, rewrites.cpp:306-323) and whose weights have a
    known shape (let-bound constants: use bind_weights), so the parallel convs
    are emitted first and carry no folded batch-norm."""
    b = _Builder(seed)
    x = b.param("x", ("?n", 3, image, image), "input")
    y = b.conv_bn(x, 3, width, 3, 1, 1, "stem")

    def parallel(src, specs):
        convs = []
        for tag, cout, k, pad in specs:  # the convs bind back to back
            w = b.param("w_" + tag, (cout, width, k, k), "conv_w")
            convs.append(b.let("conv2d(%s, %s, strides=(1, 1), padding=(%d, %d))" % (src, w, pad, pad)))
        outs = []
        for (tag, cout, k, pad), cv in zip(specs, convs):
            bb = b.param("b_" + tag, (cout,), "bias")
            outs.append(b.let("bias_add(%s, %s)" % (cv, bb)))
        return outs

    a, c, d = parallel(y, [("b1a", width, 1, 0), ("b1b", width, 1, 0), ("b1c", width // 2, 1, 0)])
    a, c, d = (b.let("relu(%s)" % v) for v in (a, c, d))
    a = b.conv_bn(a, width, width, 3, 1, 1, "b1a2", relu=False)
    c = b.conv_bn(c, width, width, 3, 1, 1, "b1b2", relu=False)
    z = b.let("relu(%s)" % b.let("add(%s, %s)" % (a, c)))
    p, r = parallel(z, [("b2p", width, 3, 1), ("b2r", width, 3, 1)])
    z = b.let("relu(%s)" % b.let("add(%s, %s)" % (p, r)))
    g = b.let("sum(%s, axis=(2, 3))" % z)
    g = b.let("multiply(%s, const %s)" % (g, fmt_f32(1.0 / (image * image))))
    gd = b.let("sum(%s, axis=(2, 3))" % d)
    gd = b.let("multiply(%s, const %s)" % (gd, fmt_f32(1.0 / (image * image))))
    h = b.let("add(%s, %s)" % (b.dense(g, width, num_classes, "fc"), b.dense(gd, width // 2, num_classes, "fcd")))
    return b.finish("branchy", h, (3, image, image), num_classes)


def make_weights(src: ModelSource, seed: int = 1) -> Dict[str, np.ndarray]:
    """Seeded random-init weights for every non-input parameter (host fp32)."""
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    out = {}
    for p in src.params:
        if p.kind == "input":
            continue
        shape = tuple(int(d) for d in p.shape)
        if p.kind in ("conv_w", "dense_w", "dw_w"):
            fan_in = int(np.prod(shape[1:]))
            out[p.name] = (rng.standard_normal(shape) * np.sqrt(2.0 / fan_in)).astype(np.float32)
        elif p.kind == "bias":
            out[p.name] = (rng.standard_normal(shape) * 0.05).astype(np.float32)
        elif p.kind == "window":
            out[p.name] = np.zeros(shape, np.float32)  # shape-only argument
        else:
            raise ValueError(p.kind)
    return out


def make_inputs(src: ModelSource, batch: int, seed: int = 0) -> np.ndarray:
    """Synthetic images x ~ U[0,1), NCHW float32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.random((batch,) + tuple(src.input_shape), dtype=np.float32)
    if src.name == "dqn":  # Atari frames: integer pixel values in [0, 255]
        x = np.floor(x * 256.0).astype(np.float32)
    return x


def make_inputs_diverse(src: ModelSource, batch: int, seed: int = 0, start: int = 0, rows=None) -> np.ndarray:
    """Synthetic images whose rows differ in kind, not just in noise, so that
    batch-indexing or row-permutation bugs change the logits and the top-1
    classes spread (U[0,1) images of a random-init net all share one arg-max).

    Image i draws its own generator (seed, i), so row i is the same at every
    batch size and any seeded subset of a large batch can be regenerated
    alone.  Kind = i % 8: 0 U[0,1); 1 affine U[0,1)*s+o (signed); 2 N(0, sigma);
    3 ramp along h or w plus noise; 4 checkerboard of random period/amplitude;
    5 per-channel constant colour plus small noise; 6 per-channel sinusoid;
    7 sparse bright blobs on zero (exercises the input clip).  DQN frames are
    then mapped to integer pixels in [0, 255].  Rows start .. start+batch-1,
    or the explicit global row indices `rows` (a seeded subset of a large batch)."""
    rows = list(range(start, start + batch)) if rows is None else [int(r) for r in rows]
    batch = len(rows)
    c, h, w = src.input_shape
    x = np.empty((batch, c, h, w), np.float32)
    hh, ww = np.meshgrid(np.arange(h, dtype=np.float32), np.arange(w, dtype=np.float32), indexing="ij")
    for j, i in enumerate(rows):
        r = np.random.Generator(np.random.PCG64([seed, i]))
        kind = i % 8
        if kind == 0:
            img = r.random((c, h, w), dtype=np.float32)
        elif kind == 1:
            img = r.random((c, h, w), dtype=np.float32) * r.uniform(0.2, 3.0) + r.uniform(-1.0, 1.0)
        elif kind == 2:
            img = r.standard_normal((c, h, w), dtype=np.float32) * r.uniform(0.3, 2.0)
        elif kind == 3:
            ramp = hh / h if r.random() < 0.5 else ww / w
            img = ramp[None] * r.uniform(-2, 2, (c, 1, 1)) + 0.1 * r.standard_normal((c, h, w))
        elif kind == 4:
            p = int(r.integers(2, 17))
            cb = ((hh // p + ww // p) % 2)[None]
            img = cb * r.uniform(-2, 2, (c, 1, 1)) + r.uniform(-0.5, 0.5, (c, 1, 1))
        elif kind == 5:
            img = r.uniform(-1.5, 1.5, (c, 1, 1)) + 0.05 * r.standard_normal((c, h, w))
        elif kind == 6:
            f = r.uniform(0.02, 0.4, (c, 2))
            ph = r.uniform(0, 6.3, (c, 1, 1))
            img = np.sin(f[:, :1, None] * hh[None] + f[:, 1:, None] * ww[None] + ph) * r.uniform(0.5, 2.5)
        else:
            img = np.zeros((c, h, w), np.float32)
            for _ in range(int(r.integers(3, 12))):
                y0, x0 = int(r.integers(0, h)), int(r.integers(0, w))
                rad = int(r.integers(2, max(3, h // 6)))
                img[:, max(0, y0 - rad):y0 + rad, max(0, x0 - rad):x0 + rad] += r.uniform(-40, 40, (c, 1, 1))
        x[j] = img
    if src.name.startswith("dqn"):
        lo, hi = x.min(axis=(1, 2, 3), keepdims=True), x.max(axis=(1, 2, 3), keepdims=True)
        x = np.floor((x - lo) / np.maximum(hi - lo, 1e-6) * 255.999).astype(np.float32)
    return x


def bind_weights(src: ModelSource, weights: Dict[str, np.ndarray],
                 kinds=("conv_w", "dense_w", "bias", "dw_w")) -> ModelSource:
    """Model interchange: the same network with its
    weights embedded in the module's metadata pool (`let %w = meta[Constant][i]`,
    printed like printer.cpp:173-194) instead of passed as @main parameters.
    The reference's `fold` pass then hoists every weight prologue (folded-BN
    multiply, the weight realize chain) into the constants at compile time."""
    head, rest = src.text.split(") {\n", 1)
    body, tail = rest.split("\n}\n", 1)
    meta_lines = []
    if tail.startswith("metadata {\n"):
        meta_lines = tail[len("metadata {\n"):].rsplit("\n}", 1)[0].split("\n")
    keep, lets = [], []
    for p in src.params:
        if p.kind not in kinds:
            keep.append(p)
            continue
        vals = ", ".join(fmt_f32(v) for v in np.asarray(weights[p.name], np.float32).reshape(-1))
        shp = "(" + ", ".join(str(d) for d in p.shape) + ")"
        meta_lines.append("  const[%d] = const([%s], %s, float32);" % (len(meta_lines), vals, shp))
        lets.append("  let %%%s = meta[Constant][%d];" % (p.name, len(meta_lines) - 1))
    sig = ", ".join("%%%s: Tensor[(%s), float32]" % (p.name, ", ".join(str(d) for d in p.shape)) for p in keep)
    text = "def @main(%s) {\n%s\n%s\n}\nmetadata {\n%s\n}\n" % (sig, "\n".join(lets), body, "\n".join(meta_lines))
    return ModelSource(src.name + "_const", text, keep, src.input_shape, src.num_classes)
