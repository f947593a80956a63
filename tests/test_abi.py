"""CPU checks of the drop-in boundary (include/mrb200.h): the sm_100a library
loads, exports every declared symbol, and the host-only half of
mr_exec_create (parse + lower, mr_module_lower) behaves like the reference's
compile step.  No compute call is made without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1904_08368_b200 as mrb


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mrb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mr_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = mrb.lib()
    syms = declared_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(mrb.EXPORTS) == syms


def test_library_is_sm100a_only():
    info = mrb.lib().mr_build_info().decode()
    assert "sm_100a" in info
    out = os.popen("cuobjdump --list-elf %s 2>/dev/null" % mrb.LIB_PATH).read()
    if out:
        archs = set(re.findall(r"sm_\d+a?", out))
        assert archs == {"sm_100a"}, archs


def test_default_options():
    o = mrb.Options()
    mrb.lib().mr_exec_default_options(ctypes.byref(o))
    assert (o.device, o.batch, o.n_data_inputs, o.float_mode, o.use_cuda_graph, o.force_simt) == (0, 1, 1, 0, 1, 0)


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_lower_resnet18_22_groups(prec):
    text, meta, src = mrb.load_model("resnet18", prec)
    d = mrb.lower(text, batch=256)
    g = d["groups"]
    assert len(g) == 22  # stem, pool, 4 + 5 + 5 + 5, head
    assert [x["anchor"] for x in g].count("conv2d") == 20
    assert [x["anchor"] for x in g].count("max_pool2d") == 1
    assert g[-1]["anchor"] == "dense" and d["result_shape"] == [256, 1000]
    assert d["int8"] == (prec == "int8")
    stem = g[0]
    assert stem["kernel"] == [7, 7] and stem["strides"] == [2, 2] and stem["padding"] == [3, 3]
    assert stem["out_shape"] == [256, 64, 112, 112]
    # Gb-last ends in sum(axis=(2, 3)) (EpiKind::SumHW = 8)
    assert g[-2]["epilogue"][-1] == 8 and g[-2]["out_shape"] == [256, 512]
    if prec == "int8":
        assert all(x["weight_quant"] for x in g if x["anchor"] != "max_pool2d")


def test_lower_batch_binds_symbolic_dim():
    text, meta, src = mrb.load_model("resnet18_tiny", "int8")
    for b in (1, 3, 64):
        assert mrb.lower(text, batch=b)["result_shape"] == [b, 10]


def test_lower_syntax_error_status():
    with pytest.raises(mrb.BackendError) as e:
        mrb.lower("def @main(%x: Tensor[(1, 3), float32]) { let %a = ; %a }", 1)
    assert e.value.code == 6  # MR_ERR_SYNTAX (DiagCode::Syntax + 1)


UNSUPPORTED = """def @main(%x: Tensor[(?n, 4, 8, 8), float32]) {
  let %f = fn(%x) [Primitive=true] {
    exp(%x)
  };
  let %v = %f(%x);
  %v
}
"""


def test_lower_unsupported_group_fails_at_compile_time():
    with pytest.raises(mrb.BackendError) as e:
        mrb.lower(UNSUPPORTED, 2)
    assert e.value.code in (2, 100)  # unknown operator / MR_ERR_UNSUPPORTED_GROUP
    assert "%f" in str(e.value) or "exp" in str(e.value)


def test_lower_rejects_bad_batch():
    text, _, _ = mrb.load_model("resnet18_tiny", "int8")
    with pytest.raises(mrb.BackendError) as e:
        mrb.lower(text, 0)
    assert e.value.code == 102


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_executor_fails_loudly_without_gpu():
    """No CPU fallback: creating an executor without a device is an error."""
    text, _, _ = mrb.load_model("resnet18_tiny", "int8")
    with pytest.raises(mrb.BackendError) as e:
        mrb.Executor(text, batch=2)
    assert e.value.code == 101  # MR_ERR_CUDA


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1904_08368_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp", ".cuh", ".h")) or f == "Makefile":
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                bad = re.findall(r"from oracle|import oracle|libmr_oracle|mr_oracle\.h|\bmro_\w+|\bmr_ref\b|oracle/_ref", src)
                assert not bad, (f, bad)


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_lower_layout_pass_module(prec):
    """the layout=NHWC pass output lowers to the same 22 groups."""
    text, _, _ = mrb.load_model("resnet18_tiny_nhwc", prec)
    d = mrb.lower(text, 4)
    assert len(d["groups"]) == 22 and d["result_shape"] == [4, 10]


def test_combine_conv_is_identity_on_baseline_models():
    """the reference's combine-conv pass finds no
    same-geometry parallel conv2d pairs in the BASELINE models, so its output
    lowers to the same groups as the plain pipeline (the concat / split form it
    produces where it does fire: test_combine_conv_concat_split_lowers)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref/mr_ref not built (needs /root/reference)")
    from paper_1904_08368_b200 import modelzoo
    for src in (modelzoo.resnet18(image=32, num_classes=10, widths=(32, 32, 64, 64)), modelzoo.dqn(batch=2),
                modelzoo.mobilenet_v1(image=32)):
        plain = ref.compile(src.text, "fold-scale,fold,dce,fuse", 0)
        comb = ref.compile(src.text, "fold-scale,fold,dce,combine-conv,fuse", 0)
        a, b = mrb.lower(plain, 2), mrb.lower(comb, 2)
        assert [g["desc"] for g in a["groups"]] == [g["desc"] for g in b["groups"]]


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_combine_conv_concat_split_lowers(prec):
    """SURVEY.md 8(f) rank 4, combine-conv where it fires (modelzoo.branchy:
    three 1x1 convs and two 3x3 convs sharing inputs).  The reference's output
    holds weight tuples, concat-weight conv groups, Opaque split groups and
    projections, with the member convs' bias/relu left in the consumers
    (rewrites.cpp:365-385, registry.cpp:695-696); the lowering slices each
    combined conv per output-channel block and re-fuses the consumers' leading
    elementwise ops, so no split / concat / tuple survives and every group is
    an ordinary conv or dense with its epilogue (combine.cpp)."""
    text, _, _ = mrb.load_model("branchy", prec)
    assert "split(" in text and "concat(" in text  # the reference did combine
    d = mrb.lower(text, 4)
    descs = [g["desc"] for g in d["groups"]]
    assert len(d["groups"]) == 10 and d["result_shape"] == [4, 10]
    assert not any("split" in x or "concat" in x for x in descs)
    assert sum(g["anchor"] == "conv2d" for g in d["groups"]) == 8  # stem + 3 + 2 slices + the two 3x3 consumers
    assert any(x.endswith("bias -> add -> relu -> sum") for x in descs)  # the anchorless add group, re-fused


@pytest.mark.parametrize("prec", ["int8", "fp32"])
def test_lower_weights_in_metadata(prec):
    """Weights embedded as @main-level constants lower
    to the same 22 groups; the constants become hidden parameters the executor
    uploads itself, so only the data input and the pool window stay @main
    arguments."""
    text, meta, src = mrb.load_model("resnet18_small_const", prec)
    d = mrb.lower(text, 4)
    assert len(d["groups"]) == 22 and d["result_shape"] == [4, 10]
    assert d["n_params"] > 2  # x, win_pool + the embedded weights
    if prec == "int8":
        assert all(x["weight_quant"] for x in d["groups"] if x["anchor"] != "max_pool2d")
