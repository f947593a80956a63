"""GPU parity: the B200 executor against the reference interpreter.

Bar (BASELINE.json north_star): int8 realized modules bit-exact; float modules
in the strict fp32 mode bit-exact (same arithmetic order as kernels.cpp); the
bf16 mode within max|d|/max|ref| <= 1e-2 on the logits plus top-1 agreement.
References: tests/golden/*.npz written by tests/golden/make_golden.py from
oracle/_ref/mr_ref (the unmodified reference's interp()).
"""
import os

import numpy as np
import pytest

import paper_1904_08368_b200 as mrb
from paper_1904_08368_b200 import modelzoo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BF16_TOL = 1e-2  # normwise: max|gpu - ref| / max|ref| on logits


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def setup(name, prec, batch, **kw):
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    ex = mrb.Executor(text, batch=batch, **kw)
    ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
    return ex, src


def normwise(y, r):
    return float(np.max(np.abs(y - r)) / np.max(np.abs(r)))


@pytest.mark.gpu
@pytest.mark.parametrize("force_simt", [False, True])
def test_tiny_int8_bitexact(gpu, force_simt):
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))
    ex, src = setup("resnet18_tiny", "int8", 4, force_simt=force_simt)
    x = modelzoo.make_inputs(src, 4, seed=0)
    y = ex.run_host(x)
    mism = int(np.sum(bits(y) != bits(gold["int8"])))
    assert mism == 0, "%d/%d logits differ (max |d| %g)" % (mism, y.size, np.max(np.abs(y - gold["int8"])))
    for g in ex.describe()["groups"]:
        if "Q[" in g["desc"] and g["kernel"] != "max_pool":
            assert g["exact"].startswith("proven"), g


@pytest.mark.gpu
def test_tiny_fp32_strict_bitexact(gpu):
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))
    ex, src = setup("resnet18_tiny", "fp32", 4, float_mode=mrb.MR_FLOAT_FP32_STRICT)
    x = modelzoo.make_inputs(src, 4, seed=0)
    y = ex.run_host(x)
    assert np.array_equal(bits(y), bits(gold["fp32"])), np.max(np.abs(y - gold["fp32"]))


@pytest.mark.gpu
@pytest.mark.parametrize("force_simt", [False, True])
def test_tiny_bf16_tolerance(gpu, force_simt):
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))
    ex, src = setup("resnet18_tiny", "fp32", 4, force_simt=force_simt)
    x = modelzoo.make_inputs(src, 4, seed=0)
    y = ex.run_host(x)
    assert normwise(y, gold["fp32"]) <= BF16_TOL
    assert np.array_equal(np.argmax(y, 1), np.argmax(gold["fp32"], 1))


@pytest.mark.gpu
def test_resnet18_int8_bitexact_full_size(gpu):
    gold = np.load(os.path.join(GOLD, "resnet18_b2.npz"))
    ex, src = setup("resnet18", "int8", 2)
    x = modelzoo.make_inputs(src, 2, seed=0)
    y = ex.run_host(x)
    assert np.array_equal(bits(y), bits(gold["int8"])), int(np.sum(bits(y) != bits(gold["int8"])))


@pytest.mark.gpu
def test_resnet18_bf16_full_size(gpu):
    gold = np.load(os.path.join(GOLD, "resnet18_b2.npz"))
    ex, src = setup("resnet18", "fp32", 2)
    x = modelzoo.make_inputs(src, 2, seed=0)
    y = ex.run_host(x)
    assert normwise(y, gold["fp32"]) <= BF16_TOL
    assert np.array_equal(np.argmax(y, 1), np.argmax(gold["fp32"], 1))


@pytest.mark.gpu
def test_submit_host_pipeline_matches_blocking(gpu):
    """mr_exec_submit_host (double-buffered async H2D) returns exactly what the
    blocking call returns, batch by batch, including across stage reuse."""
    import torch
    ex, src = setup("resnet18_tiny", "int8", 4)
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))
    xs = [modelzoo.make_inputs(src, 4, seed=s) for s in range(5)]
    want = [ex.run_host(x) for x in xs]
    assert np.array_equal(bits(want[0]), bits(gold["int8"]))
    pins = [torch.from_numpy(x).pin_memory().numpy() for x in xs]
    outs = [torch.empty(ex.output_shape, dtype=torch.float32).pin_memory().numpy() for _ in xs]
    for _ in range(2):
        for x, o in zip(pins, outs):
            ex.submit_host(x, o)
        ex.sync()
        for o, w in zip(outs, want):
            assert np.array_equal(bits(o), bits(w))


# ---- BASELINE.json configs[2..3]: MobileNet-v1 (depthwise), VGG-16, DQN (flatten heads) ----
OTHER = [("mobilenet_v1", "int8"), ("mobilenet_v1", "fp32"), ("dqn", "int8"), ("dqn", "fp32"), ("vgg16", "fp32")]


@pytest.mark.gpu
@pytest.mark.parametrize("name,prec", OTHER)
def test_other_models(gpu, name, prec):
    """int8 modules bit-exact; float modules in bf16 mode within the normwise
    tolerance + top-1 agreement, against the reference interpreter (b2)."""
    gold = np.load(os.path.join(GOLD, "%s_b2.npz" % name))
    ex, src = setup(name, prec, 2)
    y = ex.run_host(modelzoo.make_inputs(src, 2, seed=0))
    if prec == "int8":
        assert np.array_equal(bits(y), bits(gold["int8"])), int(np.sum(bits(y) != bits(gold["int8"])))
    else:
        assert normwise(y, gold["fp32"]) <= BF16_TOL, normwise(y, gold["fp32"])
        assert np.array_equal(np.argmax(y, 1), np.argmax(gold["fp32"], 1))


@pytest.mark.gpu
def test_dqn_fp32_strict_bitexact(gpu):
    gold = np.load(os.path.join(GOLD, "dqn_b2.npz"))
    ex, src = setup("dqn", "fp32", 2, float_mode=mrb.MR_FLOAT_FP32_STRICT)
    y = ex.run_host(modelzoo.make_inputs(src, 2, seed=0))
    assert np.array_equal(bits(y), bits(gold["fp32"])), np.max(np.abs(y - gold["fp32"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["resnet18_tiny", "resnet18", "mobilenet_v1", "dqn"])
def test_gpu_calibration_matches_reference(gpu, name):
    """mr_calibrate picks the same global scale as the
    reference's quant_calibrate (quantize.cpp:138-177) on the same weights and
    calibration images (models/<name>.json, written by oracle/build_models.py)."""
    import time
    text, meta, src = mrb.load_model(name, "int8")
    cal = meta["calibration"]
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, cal["images"], seed=cal["inputs_seed"])
    t0 = time.time()
    k, trials = mrb.calibrate(text, [w[p.name] for p in src.params if p.kind != "input"], [x])
    print(name, "k", k, "trials", trials, "gpu seconds %.3f" % (time.time() - t0),
          "reference seconds", cal["seconds"])
    assert k == cal["k"]
    assert trials == k + 17  # every k below overflowed


@pytest.mark.gpu
def test_gpu_calibration_fails_like_reference(gpu):
    """A range where every scale overflows fails with CalibrationFailed."""
    text, meta, src = mrb.load_model("resnet18_tiny", "int8")
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, 1, seed=0)
    with pytest.raises(mrb.BackendError) as e:
        mrb.calibrate(text, [w[p.name] for p in src.params if p.kind != "input"], [x], k_min=-16, k_max=-10)
    assert e.value.code == 15  # MR_ERR_CALIBRATION_FAILED (DiagCode::CalibrationFailed + 1)


@pytest.mark.gpu
@pytest.mark.parametrize("name,batch,prec,fm", [("resnet18_tiny", 4, "int8", 0), ("resnet18_tiny", 4, "fp32", 1),
                                                ("dqn", 2, "int8", 0)])
def test_layout_pass_modules_bitexact(gpu, name, batch, prec, fm):
    """The layout=NHWC pass output runs through the same
    executor and matches the reference bit for bit."""
    gold = np.load(os.path.join(GOLD, "%s_b%d.npz" % (name, batch)))
    ex, src = setup(name + "_nhwc", prec, batch, float_mode=fm)
    y = ex.run_host(modelzoo.make_inputs(src, batch, seed=0))
    assert np.array_equal(bits(y), bits(gold[prec])), int(np.sum(bits(y) != bits(gold[prec])))


@pytest.mark.gpu
def test_resnet18_fp32_strict_full_size(gpu):
    """fp32 in the reference's exact accumulation order (kernels.cpp:684-701), full size."""
    gold = np.load(os.path.join(GOLD, "resnet18_b2.npz"))
    ex, src = setup("resnet18", "fp32", 2, float_mode=mrb.MR_FLOAT_FP32_STRICT)
    y = ex.run_host(modelzoo.make_inputs(src, 2, seed=0))
    assert np.array_equal(bits(y), bits(gold["fp32"])), int(np.sum(bits(y) != bits(gold["fp32"])))


# The benchmarked-batch checks (b256 every row, bf16 top-1 >= 99 % against the
# reference's fp32 rows, C5 at batch 4096) live in tests/test_gpu_b256.py.


@pytest.mark.gpu
@pytest.mark.parametrize("prec,fm", [("int8", 0), ("fp32", 1)])
def test_weights_in_metadata_bitexact(gpu, prec, fm):
    """Model interchange: a module with its weights in
    the metadata pool runs with only the data input and the pool window bound;
    int8 and fp32-strict match the reference bit for bit."""
    gold = np.load(os.path.join(GOLD, "resnet18_small_const_b4.npz"))
    ex, src = setup("resnet18_small_const", prec, 4, float_mode=fm)
    y = ex.run_host(modelzoo.make_inputs(src, 4, seed=0))
    assert np.array_equal(bits(y), bits(gold[prec])), int(np.sum(bits(y) != bits(gold[prec])))


@pytest.mark.gpu
def test_device_run_graph_and_profile_paths_agree(gpu):
    """mr_exec_run on device buffers (CUDA-graph replay, one graph per input
    address), the per-launch profile path and the host path return the same
    bits; a second input buffer gets its own graph and the first still works."""
    import torch
    ex, src = setup("resnet18_tiny", "int8", 4)
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))["int8"]
    x = modelzoo.make_inputs(src, 4, seed=0)
    xd = torch.from_numpy(x).cuda()
    xd2 = xd.clone()
    out = torch.empty(ex.output_shape, dtype=torch.float32, device="cuda")
    for buf in (xd, xd2, xd):
        out.zero_()
        ex.run_device(buf.data_ptr(), buf.shape, out.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(bits(out.cpu().numpy()), bits(gold))
    ms = ex.profile_device(xd.data_ptr(), xd.shape, out.data_ptr())
    torch.cuda.synchronize()
    d = ex.describe()
    assert len(ms) == len(d["launches"]) and all(t > 0 for t in ms)
    assert np.array_equal(bits(out.cpu().numpy()), bits(gold))
    assert sum(L["kernels"] for L in d["launches"]) == ex.launch_count()


@pytest.mark.gpu
def test_int8_input_quantization_edge_values(gpu):
    """The realize chain at the input (multiply, rint, clip, cast to int8) on
    ties, the clip boundaries, -0, huge values, infinities and NaN: the whole
    int8 network matches the oracle (pinned to the reference) bit for bit."""
    from oracle import port
    ex, src = setup("resnet18_tiny", "int8", 4)
    text, meta, _ = mrb.load_model("resnet18_tiny", "int8")
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, 4, seed=3)
    c1 = 2.0  # the module's input site scale (x * 2.0, see models/resnet18_tiny_int8.fused.rly)
    assert "multiply(%x, const 2.0)" in text
    edge = np.array([0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 63.5, 64.0, 127.5, -127.5, -128.5, -129.5, 126.5,
                     -0.0, 1e30, -1e30, np.inf, -np.inf, np.nan, 3.4e38, -3.4e38, 1e-40, 0.4999999], np.float32) / c1
    flat = x.reshape(-1)
    rng = np.random.default_rng(5)
    idx = rng.choice(flat.size, size=4000, replace=False)
    flat[idx] = np.resize(edge, idx.size)
    y = ex.run_host(x)
    want = port.run_weights(text, x, [w[p.name] for p in src.params if p.kind != "input"])
    assert np.array_equal(bits(y), bits(want)), int(np.sum(bits(y) != bits(want)))


@pytest.mark.gpu
@pytest.mark.parametrize("name,prec,fm", [("dqn_b256", "int8", 0), ("vgg16_b256", "fp32", 1)])
def test_config_c4_at_batch256_matches_small_batch_golden(gpu, name, prec, fm):
    """BASELINE config C4 modules compiled at the benchmark batch (static
    reshape heads): images 0-1 of a batch-256 run equal the reference's batch-2
    goldens bit for bit (per-sample independence; int8, and fp32-strict)."""
    base = name.split("_b256")[0]
    gold = np.load(os.path.join(GOLD, "%s_b2.npz" % base))[prec]
    ex, src = setup(name, prec, 256, float_mode=fm)
    x = modelzoo.make_inputs(src, 256, seed=0)
    x2 = modelzoo.make_inputs(src, 2, seed=0)
    assert np.array_equal(x[:2], x2)
    y = ex.run_host(x)
    assert np.array_equal(bits(y[:2]), bits(gold)), int(np.sum(bits(y[:2]) != bits(gold)))


@pytest.mark.gpu
@pytest.mark.parametrize("name,batch,gold_b,prec", [("resnet18", 1, 2, "int8"), ("resnet18", 3, 2, "int8"),
                                                     ("resnet18_tiny", 1, 4, "int8"), ("resnet18_tiny", 5, 4, "int8"),
                                                     ("resnet18_tiny", 9, 4, "int8"), ("resnet18_tiny", 7, 4, "fp32")])
def test_ragged_batches_match_golden_rows(gpu, name, batch, gold_b, prec):
    """Batch sizes that fill no tile (1, 3, 5, 7, 9): the rows the golden covers
    match it bit for bit (int8; fp32-strict), the tail tiles are masked."""
    gold = np.load(os.path.join(GOLD, "%s_b%d.npz" % (name, gold_b)))[prec]
    ex, src = setup(name, prec, batch, float_mode=mrb.MR_FLOAT_FP32_STRICT if prec == "fp32" else 0)
    x = modelzoo.make_inputs(src, max(batch, gold_b), seed=0)
    assert np.array_equal(x[:gold_b], modelzoo.make_inputs(src, gold_b, seed=0))
    y = ex.run_host(np.ascontiguousarray(x[:batch]))
    k = min(batch, gold_b)
    assert np.array_equal(bits(y[:k]), bits(gold[:k])), int(np.sum(bits(y[:k]) != bits(gold[:k])))


@pytest.mark.gpu
@pytest.mark.parametrize("prec,fm", [("int8", 0), ("fp32", 1), ("fp32", 0)])
@pytest.mark.parametrize("gold_name,batch,diverse", [("branchy_b4.npz", 4, False), ("branchy_div_b64.npz", 64, True)])
def test_combine_conv_module_matches_reference(gpu, prec, fm, gold_name, batch, diverse):
    """the reference's combine-conv output (concat-weight
    convs + Opaque split groups, models/branchy_*.fused.rly) runs through the
    executor with the combined convs sliced per output-channel block: int8 and
    fp32-strict bit-exact, bf16 in tolerance, against reference-generated goldens."""
    gold = np.load(os.path.join(GOLD, gold_name))[prec]
    ex, src = setup("branchy", prec, batch, float_mode=fm)
    x = modelzoo.make_inputs_diverse(src, batch, seed=0) if diverse else modelzoo.make_inputs(src, batch, seed=0)
    y = ex.run_host(x)
    if prec == "int8" or fm == mrb.MR_FLOAT_FP32_STRICT:
        assert np.array_equal(bits(y), bits(gold)), int(np.sum(bits(y) != bits(gold)))
    else:
        assert normwise(y, gold) <= BF16_TOL


@pytest.mark.gpu
def test_unproven_int8_group_is_refused(gpu):
    """SURVEY F4 / ADVICE: int8 exactness needs every partial sum below 2^24 quanta.
    Weights scaled so every code saturates at +-127 on K = 4608 break the bound
    (127 * 4608 * 128 > 2^24): set_weights must refuse with MR_ERR_INEXACT_INT8 (104)
    instead of running a group whose result could differ from interp()."""
    text, meta, src = mrb.load_model("resnet18", "int8")
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    big = {k: (v * 1e4 if v.ndim == 4 and v.shape[1] == 512 else v) for k, v in w.items()}
    ex = mrb.Executor(text, batch=2)
    with pytest.raises(mrb.BackendError) as e:
        ex.set_weights([big[p.name] for p in src.params if p.kind != "input"])
    assert e.value.code == mrb.MR_ERR_INEXACT_INT8
    assert "2^24" in str(e.value)


@pytest.mark.gpu
def test_run_device_writes_caller_output_and_rejects_host_pointer(gpu):
    """mr_exec_run: the final launch writes the caller's device buffer (one graph
    per input/output address set; two outputs hold the same bits), and a host
    pointer as output fails cleanly with MR_ERR_INVALID_ARGUMENT."""
    import torch
    ex, src = setup("resnet18_tiny", "int8", 4)
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))["int8"]
    xd = torch.from_numpy(modelzoo.make_inputs(src, 4, seed=0)).cuda()
    outs = [torch.full(ex.output_shape, float("nan"), device="cuda") for _ in range(2)]
    for o in outs + outs:
        ex.run_device(xd.data_ptr(), xd.shape, o.data_ptr())
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(bits(o.cpu().numpy()), bits(gold))
    host = np.empty(ex.output_shape, np.float32)
    with pytest.raises(mrb.BackendError) as e:
        ex.run_device(xd.data_ptr(), xd.shape, host.ctypes.data)
    assert e.value.code == 102
