"""B200-native backend for Relay's fused-group execution path (arXiv 1904.08368).

The reference (MicroRelay, /root/reference) runs a fused module -- the output
of ``run_pipeline(..., "fuse")`` and optionally the quantization ``Realize``
pass -- with ``interp(m, "main", args)`` (``interp.hpp:50-51``), evaluating each
``[Primitive=true]`` group op by op.  This package is the drop-in for that
call on B200: ``Executor(fused_text, batch=...)`` lowers every group to one
hand-written sm_100a kernel launch behind the C ABI in ``include/mrb200.h``
(``_lib/libmrb200.so``), and ``Executor.run`` replaces ``interp``.

There is no CPU fallback: importing works without a GPU (for the CPU test
suite), but every compute call goes through the CUDA library and raises
``BackendError`` if it is missing.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MRB200_LIB") or os.path.join(_HERE, "_lib", "libmrb200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "mrb200.h")

MR_FLOAT_BF16 = 0
MR_FLOAT_FP32_STRICT = 1
MR_FLOAT_TF32 = 2
MR_FLOAT = 2
MR_ERR_UNSUPPORTED_GROUP = 100
MR_ERR_INEXACT_INT8 = 104

# every symbol include/mrb200.h declares
EXPORTS = [
    "mr_exec_default_options", "mr_exec_create", "mr_exec_set_weights", "mr_exec_run",
    "mr_exec_run_host", "mr_exec_submit_host", "mr_exec_sync", "mr_exec_output_shape", "mr_exec_describe", "mr_exec_launch_count",
    "mr_exec_profile", "mr_exec_destroy", "mr_last_error_message", "mr_module_lower", "mr_calibrate", "mr_build_info",
    "mr_group_compile", "mr_group_signature", "mr_group_launch", "mr_group_reload", "mr_group_destroy",
]


class BackendError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("mrb200 status %d: %s" % (code, msg))
        self.code = code


class Tensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("ndim", ctypes.c_int32), ("shape", ctypes.c_int64 * 8),
                ("type_code", ctypes.c_int32), ("bits", ctypes.c_int32)]


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("batch", ctypes.c_int64), ("n_data_inputs", ctypes.c_int32),
                ("float_mode", ctypes.c_int32), ("use_cuda_graph", ctypes.c_int32),
                ("force_simt", ctypes.c_int32)]


_lib = None


def lib():
    """Loads _lib/libmrb200.so (fails loudly if the extension was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BackendError(-1, "CUDA extension not built: %s (run __graft_entry__.build())" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        L.mr_exec_default_options.argtypes = [ctypes.POINTER(Options)]
        L.mr_exec_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(Options), ctypes.POINTER(ctypes.c_void_p)]
        L.mr_exec_set_weights.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(Tensor)]
        L.mr_exec_run.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor), ctypes.POINTER(Tensor), ctypes.c_void_p]
        L.mr_exec_run_host.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor), ctypes.POINTER(Tensor),
                                       ctypes.c_void_p]
        L.mr_exec_submit_host.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor), ctypes.POINTER(Tensor),
                                          ctypes.c_void_p]
        L.mr_exec_sync.argtypes = [ctypes.c_void_p]
        L.mr_exec_output_shape.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor)]
        L.mr_exec_describe.argtypes = [ctypes.c_void_p]
        L.mr_exec_describe.restype = ctypes.c_char_p
        L.mr_exec_launch_count.argtypes = [ctypes.c_void_p]
        L.mr_exec_launch_count.restype = ctypes.c_int32
        L.mr_exec_profile.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor), ctypes.POINTER(Tensor),
                                      ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int32]
        L.mr_exec_profile.restype = ctypes.c_int32
        L.mr_exec_destroy.argtypes = [ctypes.c_void_p]
        L.mr_last_error_message.restype = ctypes.c_char_p
        L.mr_build_info.restype = ctypes.c_char_p
        L.mr_calibrate.argtypes = [ctypes.c_char_p, ctypes.POINTER(Options), ctypes.c_int32, ctypes.POINTER(Tensor),
                                   ctypes.c_int32, ctypes.POINTER(Tensor), ctypes.c_int32, ctypes.c_int32,
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        L.mr_module_lower.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int32,
                                      ctypes.POINTER(ctypes.c_char_p)]
        L.mr_group_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(Options),
                                       ctypes.POINTER(ctypes.c_void_p)]
        L.mr_group_signature.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(Tensor)]
        L.mr_group_launch.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor), ctypes.c_int32, ctypes.POINTER(Tensor),
                                      ctypes.c_void_p]
        L.mr_group_reload.argtypes = [ctypes.c_void_p]
        L.mr_group_destroy.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise BackendError(status, lib().mr_last_error_message().decode())


def _tensor(ptr: int, shape: Sequence[int]) -> Tensor:
    t = Tensor()
    t.data = ptr
    t.ndim = len(shape)
    for i, d in enumerate(shape):
        t.shape[i] = int(d)
    t.type_code = MR_FLOAT
    t.bits = 32
    return t


def lower(fused_text: str, batch: int = 1, n_data_inputs: int = 1) -> dict:
    """Host-only parse + lowering of a fused module (no device needed):
    the group list mr_exec_create would compile, or BackendError with the
    same status (MR_ERR_SYNTAX = 6, MR_ERR_UNSUPPORTED_GROUP = 100 ...)."""
    out = ctypes.c_char_p()
    _check(lib().mr_module_lower(fused_text.encode(), int(batch), int(n_data_inputs), ctypes.byref(out)))
    return json.loads(out.value.decode())


def calibrate(fused_int8_text: str, weights: Sequence[np.ndarray], batches: Sequence[np.ndarray],
              k_min: int = -16, k_max: int = 16, device: int = 0):
    """GPU calibration sweep (mr_calibrate): the global scale exponent k the
    reference's quant_calibrate would pick for these weights and calibration
    batches.  Returns (k, trials)."""
    batches = [np.ascontiguousarray(b, np.float32) for b in batches]
    ws = [np.ascontiguousarray(w, np.float32) for w in weights]
    opts = Options()
    lib().mr_exec_default_options(ctypes.byref(opts))
    opts.device = device
    opts.batch = int(batches[0].shape[0])
    wt = (Tensor * max(1, len(ws)))(*[_tensor(w.ctypes.data, w.shape) for w in ws])
    xt = (Tensor * len(batches))(*[_tensor(b.ctypes.data, b.shape) for b in batches])
    k, trials = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib().mr_calibrate(fused_int8_text.encode(), ctypes.byref(opts), len(ws), wt, len(batches), xt,
                              int(k_min), int(k_max), ctypes.byref(k), ctypes.byref(trials)))
    return int(k.value), int(trials.value)


class Executor:
    """interp() replacement for one fused module at a fixed batch.

    fused_text   print_module output of run_pipeline(..., "fuse") (optionally
                 with "quantize"), i.e. models/*.fused.rly
    batch        binds @main's symbolic batch dim ?n
    float_mode   MR_FLOAT_BF16 (default), MR_FLOAT_TF32 or MR_FLOAT_FP32_STRICT
                 for the float parts of the module; int8 realized groups are
                 always bit-exact int8 x int8 -> int32
    """

    def __init__(self, fused_text: str, batch: int = 1, device: int = 0, float_mode: int = MR_FLOAT_BF16,
                 use_cuda_graph: bool = True, force_simt: bool = False):
        L = lib()
        opts = Options()
        L.mr_exec_default_options(ctypes.byref(opts))
        opts.device = device
        opts.batch = batch
        opts.float_mode = float_mode
        opts.use_cuda_graph = 1 if use_cuda_graph else 0
        opts.force_simt = 1 if force_simt else 0
        h = ctypes.c_void_p()
        _check(L.mr_exec_create(fused_text.encode(), ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        self.batch = batch
        shp = Tensor()
        _check(L.mr_exec_output_shape(self._h, ctypes.byref(shp)))
        self.output_shape = tuple(shp.shape[i] for i in range(shp.ndim))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mr_exec_destroy(h)
            self._h = None

    def describe(self) -> dict:
        return json.loads(lib().mr_exec_describe(self._h).decode())

    def launch_count(self) -> int:
        return int(lib().mr_exec_launch_count(self._h))

    def set_weights(self, weights: Sequence[np.ndarray]):
        """Non-data @main arguments, host float32, in parameter order."""
        arrs = [np.ascontiguousarray(w, dtype=np.float32) for w in weights]
        ts = (Tensor * len(arrs))(*[_tensor(a.ctypes.data, a.shape) for a in arrs])
        _check(lib().mr_exec_set_weights(self._h, len(arrs), ts))
        self._keep = arrs

    def run_device(self, x_ptr: int, x_shape: Sequence[int], out_ptr: int, stream: int = 0):
        """Device pointers (e.g. torch .data_ptr()); stream-ordered, no sync."""
        tin = _tensor(x_ptr, x_shape)
        tout = _tensor(out_ptr, self.output_shape)
        _check(lib().mr_exec_run(self._h, ctypes.byref(tin), ctypes.byref(tout), ctypes.c_void_p(stream)))

    def run_host(self, x: np.ndarray, stream: int = 0) -> np.ndarray:
        """End to end from host memory (H2D, run, D2H, sync)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(self.output_shape, np.float32)
        return self.run_host_into(x, out, stream)

    def run_host_into(self, x: np.ndarray, out: np.ndarray, stream: int = 0) -> np.ndarray:
        tin = _tensor(x.ctypes.data, x.shape)
        tout = _tensor(out.ctypes.data, out.shape)
        _check(lib().mr_exec_run_host(self._h, ctypes.byref(tin), ctypes.byref(tout), ctypes.c_void_p(stream)))
        return out

    def submit_host(self, x: np.ndarray, out: np.ndarray, stream: int = 0) -> None:
        """Asynchronous end to end (mr_exec_submit_host): H2D of x (pinned for
        overlap) on an internal copy stream, run, D2H into out; no wait.
        Keep x and out alive and untouched until sync()."""
        tin = _tensor(x.ctypes.data, x.shape)
        tout = _tensor(out.ctypes.data, out.shape)
        _check(lib().mr_exec_submit_host(self._h, ctypes.byref(tin), ctypes.byref(tout), ctypes.c_void_p(stream)))

    def sync(self) -> None:
        _check(lib().mr_exec_sync(self._h))

    def profile_device(self, x_ptr: int, x_shape: Sequence[int], out_ptr: int, stream: int = 0) -> List[float]:
        tin = _tensor(x_ptr, x_shape)
        tout = _tensor(out_ptr, self.output_shape)
        cap = 4096
        ms = (ctypes.c_float * cap)()
        n = lib().mr_exec_profile(self._h, ctypes.byref(tin), ctypes.byref(tout), ctypes.c_void_p(stream), ms, cap)
        if n < 0:
            raise BackendError(-1, lib().mr_last_error_message().decode())
        return [ms[i] for i in range(n)]


class Group:
    """One Primitive closure application (mr_group_*; interp.cpp:86-101):
    group `name` (%fusedN or the value its call binds) of a fused module,
    compiled alone.  launch() takes the call's arguments in order as DEVICE
    float32 tensors (pointer, shape) and writes the result to a device buffer."""

    def __init__(self, fused_text: str, name: str, batch: int = 1, device: int = 0,
                 float_mode: int = MR_FLOAT_BF16, use_cuda_graph: bool = True, force_simt: bool = False):
        L = lib()
        opts = Options()
        L.mr_exec_default_options(ctypes.byref(opts))
        opts.device, opts.batch, opts.float_mode = device, batch, float_mode
        opts.use_cuda_graph = 1 if use_cuda_graph else 0
        opts.force_simt = 1 if force_simt else 0
        h = ctypes.c_void_p()
        _check(L.mr_group_compile(fused_text.encode(), name.encode(), ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        n, shp = ctypes.c_int32(0), Tensor()
        _check(L.mr_group_signature(self._h, ctypes.byref(n), ctypes.byref(shp)))
        self.n_operands = int(n.value)
        self.output_shape = tuple(shp.shape[i] for i in range(shp.ndim))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mr_group_destroy(h)
            self._h = None

    def launch(self, operands: Sequence[tuple], out_ptr: int, stream: int = 0) -> None:
        ts = (Tensor * max(1, len(operands)))(*[_tensor(p, s) for p, s in operands])
        tout = _tensor(out_ptr, self.output_shape)
        _check(lib().mr_group_launch(self._h, ts, len(operands), ctypes.byref(tout), ctypes.c_void_p(stream)))

    def reload(self) -> None:
        lib().mr_group_reload(self._h)


def build_info() -> str:
    return lib().mr_build_info().decode()


def model_path(name: str) -> str:
    return os.path.join(os.path.dirname(_HERE), "models", name)


def load_model(name: str, precision: str):
    """(fused text, meta json, source) for models/<name>_<precision>.fused.rly."""
    from . import modelzoo
    root = os.path.dirname(_HERE)
    meta = json.load(open(os.path.join(root, "models", name + ".json")))
    text = open(os.path.join(root, "models", "%s_%s.fused.rly" % (name, precision))).read()
    builder = getattr(modelzoo, meta["builder"])
    kw = {k: tuple(v) if isinstance(v, list) else v for k, v in meta["builder_kwargs"].items()}
    src = builder(**kw)
    if meta.get("bind_weights"):  # weights live in the module's metadata pool
        src = modelzoo.bind_weights(src, modelzoo.make_weights(src, seed=meta["weights_seed"]))
    return text, meta, src
