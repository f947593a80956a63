"""The CPU oracle (oracle/mr_oracle.c via oracle/port.py) pinned against
(1) the SPEC.md / SURVEY.md 8(c) known answers and (2) the reference
interpreter's own outputs: the committed golden fixtures, and live runs of
the unmodified reference (oracle/_ref/mr_ref) where it is built."""
import os

import numpy as np
import pytest

from oracle import port

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def realize(x, c1=128.0, lo=-128.0, hi=127.0, dtype="int8"):
    """The realize chain Q (quantize.cpp:181-201): cast(clip(round(x * c1)))."""
    t = port.OPS["multiply"](np.asarray(x, np.float32), np.float32(c1))
    t = port.OPS["round"](t)
    t = port.op_clip(t, lo, hi)
    return port.op_cast(t, dtype).vals


# ---- known answers -------


def test_simq_known_answers():
    x = np.asarray([0.0, 0.30, 10.0], np.float32)
    y = port.op_simulated_quantize(x, bits=8, sign=1, scale=1.0)
    assert y.tolist() == [0.0, 0.296875, 0.9921875]


def test_realize_known_answers():
    assert realize([0.30, 10.0, -10.0]).tolist() == [38, 127, -128]


def test_realize_round_half_even():
    assert realize([0.5 / 128, 1.5 / 128, 2.5 / 128, -0.5 / 128]).tolist() == [0, 2, 2, 0]


def test_realize_equals_simulate():
    rng = np.random.default_rng(3)
    x = rng.normal(0, 0.5, 4096).astype(np.float32)
    codes = realize(x)
    deq = port.OPS["multiply"](port.op_cast(port.IntTensor(codes, "int8"), "float32"), np.float32(1 / 128))
    simq = port.op_simulated_quantize(x, 8, 1, 1.0)
    # equal as numbers; the only bit difference is the sign of zero (an
    # int8 code has no -0, simulated_quantize keeps nearbyintf's -0)
    assert np.array_equal(deq, simq)
    diff = bits(deq) != bits(simq)
    assert np.all(simq[diff] == 0)


def test_cast_truncates_and_wraps():
    y = port.op_cast(np.asarray([1.9, -1.9, 200.0, -200.0, 255.0, 1e20, np.nan], np.float32), "int8").vals
    assert y.tolist() == [1, -1, -56, 56, -1, -1, 0]
    assert port.op_cast(np.asarray([300.0, -1.0], np.float32), "uint8").vals.tolist() == [44, 255]


def test_conv_1x1_ones_is_channel_sum():
    x = np.asarray([[1, 2, 3, 4], [10, 20, 30, 40], [100, 200, 300, 400]], np.float32).reshape(1, 3, 2, 2)
    y = port.op_conv2d(x, np.ones((1, 3, 1, 1), np.float32))
    assert y.ravel().tolist() == [111, 222, 333, 444]


def test_dense_identity():
    x = np.random.default_rng(0).normal(size=(3, 5)).astype(np.float32)
    assert np.array_equal(port.op_dense(x, np.eye(5, dtype=np.float32)), x)


def test_relu_negative_zero_and_nan():
    y = port.OPS["relu"](np.asarray([-0.0, np.nan, -1.0, 2.0], np.float32))
    assert bits(y).tolist() == bits(np.asarray([0.0, 0.0, 0.0, 2.0], np.float32)).tolist()


def test_round_ties_to_even():
    assert port.OPS["round"](np.asarray([0.5, 1.5, 2.5, -0.5], np.float32)).tolist() == [0, 2, 2, -0.0]


def test_conv_accumulation_order_is_sequential():
    # (1e8 + 1) - 1e8 in float: sequential ic order loses the 1, a tree would not
    x = np.asarray([1e8, 1.0, -1e8], np.float32).reshape(1, 3, 1, 1)
    y = port.op_conv2d(x, np.ones((1, 3, 1, 1), np.float32))
    assert y.ravel().tolist() == [0.0]


def test_max_pool_skips_padding():
    x = -np.arange(1, 17, dtype=np.float32).reshape(1, 1, 4, 4)
    y = port.op_max_pool2d(x, np.zeros((1, 1, 3, 3)), strides=(2, 2), padding=(1, 1))
    # padded taps are skipped (never a 0 from the border)
    assert y.ravel().tolist() == [-1.0, -2.0, -5.0, -6.0]


def test_sum_seeded_row_major():
    x = np.random.default_rng(1).normal(size=(2, 3, 4, 5)).astype(np.float32)
    y = port.op_sum(x, axis=(2, 3))
    ref = np.zeros((2, 3), np.float32)
    for n in range(2):
        for c in range(3):
            acc = np.float32(x[n, c, 0, 0])
            for v in x[n, c].ravel()[1:]:
                acc = np.float32(acc + v)
            ref[n, c] = acc
    assert np.array_equal(bits(y), bits(ref))


def test_binary_broadcast_rounds_once():
    a = np.asarray([1.0000001, 3.0], np.float32)
    b = np.asarray([[0.1], [1e-8]], np.float32)
    y = port.OPS["multiply"](a, b)
    assert y.shape == (2, 2)
    assert np.array_equal(bits(y), bits((a.astype(np.float64) * b.astype(np.float64)).astype(np.float32)))


# ---- the restatement against the reference's own outputs ----------------------


def _golden_case(name, batch, prec):
    import paper_1904_08368_b200 as mrb
    from paper_1904_08368_b200 import modelzoo
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, batch, seed=0)
    return text, x, [w[p.name] for p in src.params if p.kind != "input"]


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_port_matches_reference_golden_tiny(prec):
    text, x, wl = _golden_case("resnet18_tiny", 4, prec)
    g = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))
    assert np.array_equal(bits(port.run_weights(text, x, wl)), bits(g[prec]))


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_port_matches_reference_golden_resnet18(prec):
    text, x, wl = _golden_case("resnet18", 2, prec)
    g = np.load(os.path.join(GOLD, "resnet18_b2.npz"))
    assert np.array_equal(bits(port.run_weights(text, x, wl)), bits(g[prec]))


SMALL = """def @main(%x: Tensor[(?n, 3, 9, 7), float32], %w: Tensor[(5, 3, 3, 3), float32], %b: Tensor[(5), float32], %r: Tensor[(?n, 5, 5, 4), float32]) {
  let %f0 = fn(%x, %w, %b, %r) [Primitive=true] {
    let %q0 = multiply(%x, const 16.0);
    let %q1 = round(%q0);
    let %q2 = clip(%q1, a_max=127.0, a_min=-128.0);
    let %q3 = cast(%q2, dtype="int8");
    let %q4 = cast(%q3, dtype="float32");
    let %q5 = multiply(%q4, const 0.0625);
    let %a = conv2d(%q5, %w, padding=(1, 1), strides=(2, 2));
    let %c = bias_add(%a, %b);
    let %d = add(%c, %r);
    relu(%d)
  };
  let %v = %f0(%x, %w, %b, %r);
  %v
}
"""


def test_port_matches_live_reference_small_module():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref/mr_ref not built (needs /root/reference)")
    rng = np.random.default_rng(7)
    for trial in range(3):  # batch 1: the harness runs one interp() call per image
        x = rng.normal(0, 2, (1, 3, 9, 7)).astype(np.float32)
        x[0, 0, 0, :3] = [-0.0, 0.5 / 16, 1.5 / 16]  # negative zero and RNE ties
        w = rng.normal(0, 0.3, (5, 3, 3, 3)).astype(np.float32)
        b = rng.normal(0, 0.1, 5).astype(np.float32)
        r = rng.normal(0, 1, (1, 5, 5, 4)).astype(np.float32)
        mine = port.run_module(SMALL, [x, w, b, r])
        theirs = ref.run(SMALL, x, [w, b, r]).out  # first @main param = the data input
        assert np.array_equal(bits(mine), bits(theirs)), trial


@pytest.mark.parametrize("name,prec", [("mobilenet_v1", "int8"), ("mobilenet_v1", "fp32"), ("dqn", "int8"),
                                       ("dqn", "fp32"), ("vgg16", "fp32")])
def test_port_matches_reference_golden_other_models(name, prec):
    """depthwise_conv2d (MobileNet), the flatten reshape + large dense heads
    (VGG-16, DQN): the port against the reference's own outputs."""
    path = os.path.join(GOLD, "%s_b2.npz" % name)
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    text, x, wl = _golden_case(name, 2, prec)
    assert np.array_equal(bits(port.run_weights(text, x, wl)), bits(np.load(path)[prec]))


@pytest.mark.parametrize("name,batch,prec", [("resnet18_tiny", 4, "int8"), ("resnet18_tiny", 4, "fp32"),
                                             ("dqn", 2, "int8"), ("dqn", 2, "fp32")])
def test_port_layout_pass_modules(name, batch, prec):
    """The layout=NHWC pass output (transposes + NHWC conv2d) evaluates to the
    reference's NCHW results bit for bit (oracle/build_models: same k)."""
    import paper_1904_08368_b200 as mrb
    from paper_1904_08368_b200 import modelzoo
    text, meta, src = mrb.load_model(name + "_nhwc", prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, batch, seed=0)
    y = port.run_weights(text, x, [w[p.name] for p in src.params if p.kind != "input"])
    assert np.array_equal(bits(y), bits(np.load(os.path.join(GOLD, "%s_b%d.npz" % (name, batch)))[prec]))


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_port_matches_reference_weights_in_metadata(prec):
    """Model interchange: weights embedded in the
    module (modelzoo.bind_weights, folded by the reference's passes; the
    printer inlines small tensors as const(...) and pools the rest in the
    metadata section) evaluate bit-identically to the reference's run."""
    import paper_1904_08368_b200 as mrb
    from paper_1904_08368_b200 import modelzoo
    text, meta, src = mrb.load_model("resnet18_small_const", prec)
    assert [p.kind for p in src.params] == ["input", "window"]
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, 4, seed=0)
    y = port.run_module(text, [x] + [w[p.name] for p in src.params if p.kind != "input"])
    gold = np.load(os.path.join(GOLD, "resnet18_small_const_b4.npz"))
    assert np.array_equal(bits(y), bits(gold[prec]))
