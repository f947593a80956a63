"""Group level of the boundary (include/mrb200.h mr_group_*):
one Primitive closure application (interp.cpp:86-101) compiled and launched on
its own, checked group by group against the oracle's per-group trace
(oracle/port.py run_module(trace=...), pinned to the reference in
test_oracle.py)."""
import ctypes
import re

import numpy as np
import pytest

import paper_1904_08368_b200 as mrb
from paper_1904_08368_b200 import modelzoo


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _compile_status(text, name, batch=2):
    L = mrb.lib()
    o = mrb.Options()
    L.mr_exec_default_options(ctypes.byref(o))
    o.batch = batch
    h = ctypes.c_void_p()
    st = L.mr_group_compile(text.encode(), name.encode(), ctypes.byref(o), ctypes.byref(h))
    if st == 0:
        L.mr_group_destroy(h)
    return st


def test_group_compile_unknown_group_is_unbound_variable():
    text, _, _ = mrb.load_model("resnet18_tiny", "int8")
    assert _compile_status(text, "%nosuchgroup") == 1  # MR_ERR_UNBOUND_VARIABLE (DiagCode::UnboundVariable + 1)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
@pytest.mark.parametrize("name,prec", [("resnet18_tiny", "int8"), ("resnet18_tiny", "fp32"), ("mobilenet_v1", "int8"),
                                       ("dqn", "int8"), ("dqn", "fp32"), ("vgg16", "fp32")])
def test_every_group_extracts_and_lowers(name, prec):
    """Every group of the module extracts and lowers on the host (any
    MR_ERR_UNSUPPORTED_GROUP would surface here); the device step then fails
    loudly with MR_ERR_CUDA -- there is no CPU fallback."""
    text, _, _ = mrb.load_model(name, prec)
    groups = re.findall(r"let (%fused\d+) = fn", text)
    assert groups
    for gname in groups:
        assert _compile_status(text, gname) == 101, gname
    bound = re.findall(r"let (%\w+) = %fused\d+\(", text)
    assert _compile_status(text, bound[0]) == 101  # by the value the call binds


def oracle_trace(name, prec, batch):
    from oracle import port
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, batch, seed=0)
    trace = []
    port.run_module(text, [x] + [w[p.name] for p in src.params if p.kind != "input"], trace=trace)
    return text, trace


@pytest.mark.gpu
@pytest.mark.parametrize("name,prec,batch", [("resnet18_tiny", "int8", 2), ("resnet18_tiny", "fp32", 2),
                                             ("mobilenet_v1", "int8", 2), ("dqn", "int8", 2),
                                             ("resnet18_small_const", "int8", 2)])
def test_every_group_bitexact_through_group_api(gpu, name, prec, batch):
    """Each group of the module, launched alone on the oracle's own operands,
    reproduces the oracle's result for that group bit for bit (int8 realized
    groups; float groups in the strict fp32 mode)."""
    import torch
    text, trace = oracle_trace(name, prec, batch)
    assert len(trace) >= 3
    fm = mrb.MR_FLOAT_FP32_STRICT if prec == "fp32" else mrb.MR_FLOAT_BF16
    for fn, args, ref in trace:
        g = mrb.Group(text, fn, batch=batch, float_mode=fm)
        assert g.n_operands == len(args)
        assert g.output_shape == tuple(ref.shape), (fn, g.output_shape, ref.shape)
        dev = [torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda() for a in args]
        out = torch.empty(ref.shape, dtype=torch.float32, device="cuda")
        g.launch([(t.data_ptr(), tuple(t.shape)) for t in dev], out.data_ptr())
        torch.cuda.synchronize()
        y = out.cpu().numpy()
        mism = int(np.sum(y.view(np.uint32) != np.ascontiguousarray(ref, np.float32).view(np.uint32)))
        assert mism == 0, "%s: %d/%d differ (max |d| %g)" % (fn, mism, y.size, np.max(np.abs(y - ref)))


@pytest.mark.gpu
def test_group_launch_restages_weights_on_new_address(gpu):
    """Weight operands are staged by address: a new weight tensor changes the
    result; the same address reuses the staged prologue."""
    import torch
    text, trace = oracle_trace("resnet18_tiny", "int8", 2)
    fn, args, ref = trace[2]  # a layer-1 conv group
    g = mrb.Group(text, fn, batch=2)
    dev = [torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda() for a in args]
    ops = [(t.data_ptr(), tuple(t.shape)) for t in dev]
    out = torch.empty(ref.shape, dtype=torch.float32, device="cuda")
    g.launch(ops, out.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    # replace the 4-D weight operand with its negation at a new address
    wi = next(i for i, a in enumerate(args) if a.ndim == 4 and a.shape[0] != 2)  # OIHW, O != batch
    neg = -dev[wi]
    ops2 = list(ops)
    ops2[wi] = (neg.data_ptr(), tuple(neg.shape))
    out2 = torch.empty_like(out)
    g.launch(ops2, out2.data_ptr())
    torch.cuda.synchronize()
    assert not np.array_equal(out2.cpu().numpy(), ref)
    g.launch(ops, out2.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), ref)


@pytest.mark.gpu
def test_group_launch_arity_error(gpu):
    text, trace = oracle_trace("resnet18_tiny", "int8", 2)
    fn, args, ref = trace[0]
    g = mrb.Group(text, fn, batch=2)
    with pytest.raises(mrb.BackendError) as e:
        g.launch([], 0)
    assert e.value.code == 13  # MR_ERR_ARITY_MISMATCH
