"""Driver for oracle/_ref/mr_ref -- TEST INFRASTRUCTURE ONLY.

Runs the unmodified reference compiler + interpreter (ref_harness.cpp over
the library built from /root/reference by oracle/Makefile) as a subprocess.
Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this module; the product never does.
"""
from __future__ import annotations

import os
import struct
import subprocess
import tempfile
from typing import Dict, List, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
EXE = os.path.join(_HERE, "_ref", "mr_ref")


class RefError(RuntimeError):
    pass


def available() -> bool:
    return os.path.exists(EXE)


def write_tensors(path: str, arrays: Sequence[np.ndarray]) -> None:
    """int32 count; per tensor int32 ndim, int64 dims, float32 data."""
    with open(path, "wb") as f:
        f.write(struct.pack("<i", len(arrays)))
        for a in arrays:
            a = np.ascontiguousarray(a, dtype=np.float32)
            f.write(struct.pack("<i", a.ndim))
            f.write(np.asarray(a.shape, dtype="<i8").tobytes())
            f.write(a.tobytes())


def read_tensors(path: str) -> List[np.ndarray]:
    out = []
    with open(path, "rb") as f:
        (n,) = struct.unpack("<i", f.read(4))
        for _ in range(n):
            (nd,) = struct.unpack("<i", f.read(4))
            dims = np.frombuffer(f.read(8 * nd), dtype="<i8")
            cnt = int(np.prod(dims)) if nd else 1
            out.append(np.frombuffer(f.read(4 * cnt), dtype="<f4").reshape(tuple(int(d) for d in dims)))
    return out


def _call(args: List[str], timeout=None) -> subprocess.CompletedProcess:
    if not available():
        raise RefError("reference harness not built: %s (make -C oracle)" % EXE)
    p = subprocess.run([EXE] + args, capture_output=True, text=True, timeout=timeout)
    if p.returncode != 0:
        raise RefError(p.stderr.strip() or ("mr_ref exit %d" % p.returncode))
    return p


def compile(text: str, passes: str, quant_k: int = 0) -> str:
    """run_pipeline(passes), `quantize` realized at global scale 2^quant_k."""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "model.rly")
        open(src, "w").write(text)
        return _call(["compile", src, passes, str(int(quant_k))]).stdout


def compile_calibrated(text: str, passes: str, args: Sequence[np.ndarray], timeout=None) -> str:
    """The stock run_pipeline, quant_calibrate on one calibration sample."""
    with tempfile.TemporaryDirectory() as d:
        src, a = os.path.join(d, "model.rly"), os.path.join(d, "args.bin")
        open(src, "w").write(text)
        write_tensors(a, args)
        return _call(["calibrated", src, passes, a], timeout=timeout).stdout


def calibrate(text: str, pre_passes: str, args: Sequence[np.ndarray], timeout=None) -> int:
    with tempfile.TemporaryDirectory() as d:
        src, a = os.path.join(d, "model.rly"), os.path.join(d, "args.bin")
        open(src, "w").write(text)
        write_tensors(a, args)
        return int(_call(["calibrate", src, pre_passes, a], timeout=timeout).stdout.strip())


class RunResult:
    def __init__(self, out: np.ndarray, seconds: List[float]):
        self.out = out
        self.seconds = seconds


def run(fused_text: str, images: np.ndarray, weights: Sequence[np.ndarray], timeout=None,
        workdir: str = None, whole_batch: bool = False) -> RunResult:
    """interp(@main) once per image (batch-1 calls) -> stacked float32 output;
    whole_batch: one call over the batch (static-batch modules: reshape heads)."""
    with tempfile.TemporaryDirectory(dir=workdir) as d:
        src = os.path.join(d, "fused.rly")
        wf, xf, of = (os.path.join(d, n) for n in ("w.bin", "x.bin", "out.bin"))
        open(src, "w").write(fused_text)
        write_tensors(wf, weights)
        write_tensors(xf, [images])
        p = _call(["runall" if whole_batch else "run", src, wf, xf, of], timeout=timeout)
        secs = [float(l.split()[-1]) for l in p.stderr.splitlines() if l.startswith(("image ", "batch "))]
        return RunResult(read_tensors(of)[0].copy(), secs)


def weight_list(src, weights: Dict[str, np.ndarray]) -> List[np.ndarray]:
    """@main arguments after the input, in declaration order."""
    return [weights[p.name] for p in src.params if p.kind != "input"]
