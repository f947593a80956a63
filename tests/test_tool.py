"""The C++ host program over the C ABI (paper_1904_08368_b200/tools/mrb200_run.cpp):
the reference CLI's `run` (tools/microrelay.cpp:100-131) for fused modules,
driving include/mrb200.h from C++ without Python in the loop."""
import os
import subprocess

import numpy as np
import pytest

import paper_1904_08368_b200 as mrb
from paper_1904_08368_b200 import modelzoo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_1904_08368_b200", "_lib", "mrb200_run")
GOLD = os.path.join(ROOT, "tests", "golden")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _args(tmp_path, name, prec, batch):
    from oracle import ref  # tensor file format shared with the reference harness
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    x = modelzoo.make_inputs(src, batch, seed=0)
    mod = tmp_path / "m.rly"
    mod.write_text(text)
    args = tmp_path / "args.bin"
    ref.write_tensors(str(args), [x] + [w[p.name] for p in src.params if p.kind != "input"])
    return str(mod), str(args), str(tmp_path / "out.bin")


def test_tool_built_and_usage():
    assert os.access(TOOL, os.X_OK)
    r = subprocess.run([TOOL], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr and "sm_100a" in r.stderr


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_tool_fails_loudly_without_gpu(tmp_path):
    mod, args, out = _args(tmp_path, "resnet18_tiny", "int8", 2)
    r = subprocess.run([TOOL, mod, args, out], capture_output=True, text=True)
    assert r.returncode == 101, r.stderr  # MR_ERR_CUDA: no CPU fallback


@pytest.mark.gpu
@pytest.mark.parametrize("name,prec,strict", [("resnet18_tiny", "int8", False), ("resnet18_tiny", "fp32", True),
                                              ("resnet18_small_const", "int8", False)])
def test_tool_bitexact(gpu, tmp_path, name, prec, strict):
    from oracle import ref
    mod, args, out = _args(tmp_path, name, prec, 4)
    cmd = [TOOL, mod, args, out] + (["--fp32-strict"] if strict else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    y = ref.read_tensors(out)[0]
    gold = np.load(os.path.join(GOLD, "%s_b4.npz" % name))[prec]
    assert np.array_equal(y.view(np.uint32), np.ascontiguousarray(gold, np.float32).view(np.uint32))
