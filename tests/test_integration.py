"""The reference-side binding, compiled for real: the hook a
MicroRelay maintainer adds next to interp() -- integration/b200_backend.cpp --
built against the UNMODIFIED reference headers and library
(oracle/_ref/libmicrorelay_core.a) plus libmrb200.so, driven by
integration/ref_b200_run.cpp, the reference CLI's `run` with the hook in place
of interp().  The module is parsed by the reference's parser; the hook prints
it (print_module) and hands it to the C ABI.
"""
import os
import subprocess
import tempfile

import numpy as np
import pytest

import paper_1904_08368_b200 as mrb
from paper_1904_08368_b200 import modelzoo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ref_b200_run")
GOLD = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/proj/core/src"


def _need_exe():
    if os.path.isdir(REF_SRC):  # build container: (re)build the binding from the reference
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "integration")])
    if not os.path.exists(EXE):
        pytest.skip("ref_b200_run not built (needs /root/reference at build time)")


def _run(mode, name, prec, x, extra=(), args=None):
    from oracle import ref
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    with tempfile.TemporaryDirectory() as d:
        f, a, o = (os.path.join(d, n) for n in ("m.rly", "a.bin", "o.bin"))
        open(f, "w").write(text)
        ref.write_tensors(a, args if args is not None else [x] + ref.weight_list(src, w))
        p = subprocess.run([EXE, mode, f, a, o] + list(extra), capture_output=True, text=True, timeout=600)
        out = ref.read_tensors(o)[0].copy() if p.returncode == 0 else None
        return p, out


def test_binding_builds_and_links_against_the_reference():
    _need_exe()
    p = subprocess.run([EXE], capture_output=True, text=True)
    assert p.returncode == 2 and "usage" in p.stderr


def test_binding_interp_mode_is_the_reference():
    """Same binary, interp() path: the reference itself reproduces the golden."""
    _need_exe()
    gold = np.load(os.path.join(GOLD, "resnet18_tiny_b4.npz"))
    _, _, src = mrb.load_model("resnet18_tiny", "int8")
    p, y = _run("interp", "resnet18_tiny", "int8", modelzoo.make_inputs(src, 4, seed=0))
    assert p.returncode == 0, p.stderr
    assert np.array_equal(y.view(np.uint32), gold["int8"].view(np.uint32))


def test_binding_b200_mode_fails_as_a_diagnostic_without_gpu():
    """No CPU fallback: the hook raises the reference's Diagnostic (DiagCode
    Internal for MR_ERR_CUDA) and the CLI exits with its diagnostic status."""
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("checks the no-GPU failure mode")
    _need_exe()
    _, _, src = mrb.load_model("resnet18_tiny", "int8")
    p, _ = _run("b200", "resnet18_tiny", "int8", modelzoo.make_inputs(src, 4, seed=0))
    assert p.returncode == 3 and "b200:" in p.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["b200", "session"])
@pytest.mark.parametrize("name,prec,batch", [("resnet18_tiny", "int8", 4), ("resnet18", "int8", 2)])
def test_binding_runs_the_executor_bitexact(gpu, mode, name, prec, batch):
    _need_exe()
    gold = np.load(os.path.join(GOLD, "%s_b%d.npz" % (name, batch)))
    _, _, src = mrb.load_model(name, prec)
    p, y = _run(mode, name, prec, modelzoo.make_inputs(src, batch, seed=0))
    assert p.returncode == 0, p.stderr
    assert np.array_equal(y.view(np.uint32), gold[prec].view(np.uint32))


@pytest.mark.gpu
def test_binding_group_hook_bitexact(gpu):
    """Interpreter::apply's hook: every group of the tiny int8 module through
    B200Group.apply on the oracle's per-group operands, bit for bit."""
    _need_exe()
    from oracle import port
    text, meta, src = mrb.load_model("resnet18_tiny", "int8")
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, 2, seed=0)
    trace = []
    port.run_module(text, [x] + [w[p.name] for p in src.params if p.kind != "input"], trace=trace)
    for fn, args, want in trace:
        p, y = _run("group", "resnet18_tiny", "int8", None, extra=[fn, "2"],
                    args=[np.ascontiguousarray(a, np.float32) for a in args])
        assert p.returncode == 0, (fn, p.stderr)
        assert np.array_equal(y.view(np.uint32), np.ascontiguousarray(want, np.float32).view(np.uint32)), fn
