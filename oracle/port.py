"""oracle/port.py -- TEST INFRASTRUCTURE ONLY: the CPU restatement ("port")
of the reference's evaluation of a fused module.

It parses the text form the reference prints after FuseOps
(printer.cpp; the subset SURVEY.md 8(b) names: `def @main` with typed
params, `let` chains, `fn(...) [Primitive=true] { ... }` groups, op calls
with attributes, `const` scalars and `meta[Constant][i]`) and evaluates it
the way the reference interpreter does (interp.cpp:218-222: each let bound
once, each Primitive function applied to its arguments), with every operator
executed by the C restatement in mr_oracle.c (kernels.cpp semantics).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module; the product never does.

Parity pinned: tests/test_oracle.py checks run_module() bit-for-bit against
tests/golden/*.npz, which the UNMODIFIED reference interpreter produced
(tests/golden/make_golden.py over oracle/_ref/mr_ref).
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "_ref", "libmr_oracle.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise RuntimeError("oracle not built: %s (make -C oracle oracle)" % SO)
        L = ctypes.CDLL(SO)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.mro_set_threads.argtypes = [I]
        L.mro_binary_f32.argtypes = [I, P, P, P, P, P, P, I]
        for f in ("mro_relu_f32", "mro_round_f32"):
            getattr(L, f).argtypes = [P, P, I64]
        L.mro_clip_f32.argtypes = [P, P, I64, ctypes.c_double, ctypes.c_double]
        L.mro_cast_f32_to_int.argtypes = [P, P, I64, I, I]
        L.mro_cast_int_to_f32.argtypes = [P, P, I64]
        L.mro_conv2d_f32.argtypes = [P, P, P] + [I64] * 11
        L.mro_dense_f32.argtypes = [P, P, P, I64, I64, I64]
        L.mro_bias_add_f32.argtypes = [P, P, P, P, I, I]
        L.mro_sum_f32.argtypes = [P, P, P, I, P]
        L.mro_max_pool2d_f32.argtypes = [P, P] + [I64] * 10
        L.mro_simq_f32.argtypes = [P, P, I64, ctypes.c_double, I, I]
        L.mro_dwconv2d_f32.argtypes = [P, P, P] + [I64] * 10
        L.mro_set_threads(os.cpu_count() or 1)
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().mro_set_threads(int(n))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---- values -----------------------------------------------------------------
# float32 tensors are np.float32 arrays; integer tensors (cast targets) are
# IntTensor(np.int64 values, dtype name), as TensorLiteral::ints() holds them.


class IntTensor:
    def __init__(self, vals: np.ndarray, dtype: str):
        self.vals = vals
        self.dtype = dtype


_INT_BITS = {"int8": (8, 1), "uint8": (8, 0), "int16": (16, 1), "int32": (32, 1), "int64": (64, 1)}


# ---- operators (kernels.cpp) ---------------------------------------------------


def _f32(a) -> np.ndarray:
    if isinstance(a, IntTensor):
        raise TypeError("float32 operator applied to %s" % a.dtype)
    return np.ascontiguousarray(a, dtype=np.float32)


def _binary(op: int, a, b) -> np.ndarray:
    a, b = _f32(a), _f32(b)
    out_shape = np.broadcast_shapes(a.shape, b.shape)
    nd = len(out_shape)

    def strides(x):
        sh = (1,) * (nd - x.ndim) + x.shape
        st, acc = [0] * nd, 1
        for d in range(nd - 1, -1, -1):
            st[d] = 0 if sh[d] == 1 and out_shape[d] != 1 else acc
            acc *= sh[d]
        return np.asarray(st, np.int64)

    out = np.empty(out_shape, np.float32)
    sa, sb, od = strides(a), strides(b), np.asarray(out_shape, np.int64)
    lib().mro_binary_f32(op, _p(a), _p(sa), _p(b), _p(sb), _p(out), _p(od), nd)
    return out


def _unary(fn: str, x) -> np.ndarray:
    x = _f32(x)
    y = np.empty_like(x)
    getattr(lib(), fn)(_p(x), _p(y), x.size)
    return y


def op_clip(x, a_min, a_max):
    x = _f32(x)
    y = np.empty_like(x)
    lib().mro_clip_f32(_p(x), _p(y), x.size, float(a_min), float(a_max))
    return y


def op_cast(x, dtype: str):
    if dtype == "float32":
        if isinstance(x, IntTensor):
            y = np.empty(x.vals.shape, np.float32)
            v = np.ascontiguousarray(x.vals, np.int64)
            lib().mro_cast_int_to_f32(_p(v), _p(y), v.size)
            return y
        return _f32(x).copy()
    bits, signed = _INT_BITS[dtype]
    if isinstance(x, IntTensor):
        raise NotImplementedError("int -> int cast is not on the fused path")
    x = _f32(x)
    y = np.empty(x.shape, np.int64)
    lib().mro_cast_f32_to_int(_p(x), _p(y), x.size, bits, signed)
    return IntTensor(y, dtype)


def op_conv2d(x, w, strides=(1, 1), padding=(0, 0), layout="NCHW"):
    if layout == "NHWC":
        # kernels.cpp:640-716 walks the same (n, oc, oh, ow, ic, kh, kw) loops for
        # NHWC/HWIO, only the indexing differs: same sums, same order
        y = op_conv2d(np.ascontiguousarray(np.transpose(_f32(x), (0, 3, 1, 2))),
                      np.ascontiguousarray(np.transpose(_f32(w), (3, 2, 0, 1))), strides, padding)
        return np.ascontiguousarray(np.transpose(y, (0, 2, 3, 1)))
    if layout != "NCHW":
        raise NotImplementedError("oracle conv2d: NCHW / NHWC only")
    x, w = _f32(x), _f32(w)
    N, C, H, W = x.shape
    OC, IC, KH, KW = w.shape
    if IC != C:
        raise ValueError("conv2d: channel mismatch")
    sh, sw = strides
    ph, pw = padding
    OH, OW = (H - KH + 2 * ph) // sh + 1, (W - KW + 2 * pw) // sw + 1
    y = np.empty((N, OC, OH, OW), np.float32)
    lib().mro_conv2d_f32(_p(x), _p(w), _p(y), N, C, H, W, OC, KH, KW, sh, sw, ph, pw)
    return y


def op_max_pool2d(x, win, strides=(1, 1), padding=(0, 0)):
    x = _f32(x)
    N, C, H, W = x.shape
    KH, KW = np.shape(win)[2], np.shape(win)[3]
    sh, sw = strides
    ph, pw = padding
    OH, OW = (H - KH + 2 * ph) // sh + 1, (W - KW + 2 * pw) // sw + 1
    y = np.empty((N, C, OH, OW), np.float32)
    lib().mro_max_pool2d_f32(_p(x), _p(y), N, C, H, W, KH, KW, sh, sw, ph, pw)
    return y


def op_depthwise_conv2d(x, win, w, strides=(1, 1), padding=(0, 0)):
    x, w = _f32(x), _f32(w)
    N, C, H, W = x.shape
    KH, KW = w.shape[2], w.shape[3]
    sh, sw = strides
    ph, pw = padding
    OH, OW = (H - KH + 2 * ph) // sh + 1, (W - KW + 2 * pw) // sw + 1
    y = np.empty((N, C, OH, OW), np.float32)
    lib().mro_dwconv2d_f32(_p(x), _p(w), _p(y), N, C, H, W, KH, KW, sh, sw, ph, pw)
    return y


def op_transpose(x, axes):
    """kernels.cpp:399-431: a fresh tensor with permuted axes (values unchanged)."""
    if isinstance(x, IntTensor):
        return IntTensor(np.ascontiguousarray(np.transpose(x.vals, tuple(axes))), x.dtype)
    return np.ascontiguousarray(np.transpose(_f32(x), tuple(int(a) for a in axes)))


def op_reshape(x, newshape):
    """kernels.cpp:390-397: a view (same row-major data, new shape)."""
    if isinstance(x, IntTensor):
        return IntTensor(x.vals.reshape(tuple(newshape)), x.dtype)
    return _f32(x).reshape(tuple(int(d) for d in newshape))


def op_dense(x, w):
    x, w = _f32(x), _f32(w)
    n, k = x.shape
    m = w.shape[0]
    y = np.empty((n, m), np.float32)
    lib().mro_dense_f32(_p(x), _p(w), _p(y), n, k, m)
    return y


def op_bias_add(x, b, axis=1):
    x, b = _f32(x), _f32(b)
    y = np.empty_like(x)
    dims = np.asarray(x.shape, np.int64)
    lib().mro_bias_add_f32(_p(x), _p(b), _p(y), _p(dims), x.ndim, int(axis))
    return y


def op_sum(x, axis=None, keepdims=False):
    x = _f32(x)
    axes = list(range(x.ndim)) if axis is None else [int(a) for a in (axis if isinstance(axis, (tuple, list)) else [axis])]
    red = np.zeros(x.ndim, np.int32)
    red[axes] = 1
    out_shape = tuple((1 if red[d] else x.shape[d]) for d in range(x.ndim) if keepdims or not red[d])
    y = np.empty(out_shape, np.float32)
    dims = np.asarray(x.shape, np.int64)
    lib().mro_sum_f32(_p(x), _p(y), _p(dims), x.ndim, _p(red))
    return y


def op_simulated_quantize(x, bits=8, sign=1, scale=None, **_):
    if scale is None:
        raise ValueError("simulated_quantize has no calibrated scale")
    x = _f32(x)
    y = np.empty_like(x)
    lib().mro_simq_f32(_p(x), _p(y), x.size, float(scale), int(bits), int(sign))
    return y


OPS = {
    "simulated_quantize": op_simulated_quantize,
    "add": lambda a, b: _binary(0, a, b),
    "subtract": lambda a, b: _binary(1, a, b),
    "multiply": lambda a, b: _binary(2, a, b),
    "divide": lambda a, b: _binary(3, a, b),
    "relu": lambda x: _unary("mro_relu_f32", x),
    "round": lambda x: _unary("mro_round_f32", x),
    "clip": op_clip,
    "cast": op_cast,
    "conv2d": op_conv2d,
    "nn.conv2d": op_conv2d,
    "max_pool2d": op_max_pool2d,
    "depthwise_conv2d": op_depthwise_conv2d,
    "reshape": op_reshape,
    "transpose": op_transpose,
    "dense": op_dense,
    "nn.dense": op_dense,
    "bias_add": op_bias_add,
    "nn.bias_add": op_bias_add,
    "sum": op_sum,
}

# ---- parser (the printed fused-module subset) --------------------------------

_TOK = re.compile(r"""
    (?P<ws>\s+|//[^\n]*)
  | (?P<var>%[A-Za-z_][A-Za-z0-9_.]*)
  | (?P<gvar>@[A-Za-z_][A-Za-z0-9_]*)
  | (?P<num>[-+]?(?:\d+\.\d*|\.\d+|\d+)(?:[eE][-+]?\d+)?f?)
  | (?P<str>"[^"]*")
  | (?P<ident>[A-Za-z_?][A-Za-z0-9_.]*)
  | (?P<punct>[()\[\]{},;=:])
""", re.X)


def tokenize(text: str) -> List[tuple]:
    out, i = [], 0
    while i < len(text):
        m = _TOK.match(text, i)
        if not m:
            raise SyntaxError("oracle parser: bad character %r at %d" % (text[i], i))
        i = m.end()
        if m.lastgroup != "ws":
            out.append((m.lastgroup, m.group()))
    out.append(("eof", ""))
    return out


class _P:
    def __init__(self, toks):
        self.t, self.i = toks, 0

    def peek(self, k=0):
        return self.t[self.i + k]

    def next(self):
        tok = self.t[self.i]
        self.i += 1
        return tok

    def expect(self, v):
        tok = self.next()
        if tok[1] != v:
            raise SyntaxError("oracle parser: expected %r, got %r" % (v, tok[1]))
        return tok

    def accept(self, v):
        if self.peek()[1] == v:
            self.i += 1
            return True
        return False


# AST: ("var", name) | ("const", ndarray) | ("meta", i) | ("call", op, [args], attrs)
#      | ("fn", [params], body) | ("apply", callee_expr, [args]) | ("let", name, value, body)


def _parse_value(p: _P):
    """attribute values: numbers, strings, identifiers, tuples."""
    kind, v = p.peek()
    if v == "(" or v == "[":
        close = ")" if v == "(" else "]"
        p.next()
        items = []
        while not p.accept(close):
            items.append(_parse_value(p))
            p.accept(",")
        return tuple(items)
    p.next()
    if kind == "num":
        v = v.rstrip("f")
        return float(v) if any(c in v for c in ".eE") else int(v)
    if kind == "str":
        return v[1:-1]
    if v in ("True", "true"):
        return True
    if v in ("False", "false"):
        return False
    return v


def _parse_type(p: _P):
    # Tensor[(d0, d1, ...), dtype]  -- only skipped (shapes come from the inputs)
    depth = 0
    while True:
        _, v = p.next()
        if v == "[":
            depth += 1
        elif v == "]":
            depth -= 1
            if depth == 0:
                return


def _parse_expr(p: _P):
    kind, v = p.peek()
    if v == "let":
        p.next()
        name = p.next()[1]
        p.expect("=")
        val = _parse_expr(p)
        p.expect(";")
        body = _parse_expr(p)
        return ("let", name, val, body)
    if v == "fn":
        p.next()
        p.expect("(")
        params = []
        while not p.accept(")"):
            params.append(p.next()[1])
            if p.accept(":"):
                _parse_type(p)
            p.accept(",")
        if p.accept("["):  # [Primitive=true]
            while not p.accept("]"):
                p.next()
        p.expect("{")
        body = _parse_expr(p)
        p.expect("}")
        e = ("fn", params, body)
    elif kind == "var":
        p.next()
        e = ("var", v)
    elif v == "const":
        p.next()
        if p.accept("("):  # tensor literal const(values, (dims), dtype) (printer.cpp:173-194)
            vals = _parse_value(p)
            p.expect(",")
            shape = _parse_value(p)
            p.expect(",")
            p.next()  # dtype
            p.expect(")")
            e = ("const", np.asarray(vals, np.float32).reshape(shape))
        else:
            num = _parse_value(p)
            e = ("const", np.asarray(num, np.float32))
    elif v == "meta":
        p.next()
        p.expect("[")
        p.next()
        p.expect("]")
        p.expect("[")
        idx = int(p.next()[1])
        p.expect("]")
        e = ("meta", idx)
    elif kind == "ident":
        p.next()
        p.expect("(")
        args, attrs = [], {}
        while not p.accept(")"):
            if p.peek()[0] == "ident" and p.peek(1)[1] == "=":
                k = p.next()[1]
                p.next()
                attrs[k] = _parse_value(p)
            else:
                args.append(_parse_expr(p))
            p.accept(",")
        return ("call", v, args, attrs)
    elif v == "(":
        p.next()
        e = _parse_expr(p)
        p.expect(")")
    else:
        raise SyntaxError("oracle parser: unexpected %r" % v)
    while p.peek()[1] == "(":  # application
        p.next()
        args = []
        while not p.accept(")"):
            args.append(_parse_expr(p))
            p.accept(",")
        e = ("apply", e, args)
    return e


class Module:
    def __init__(self, params: List[str], body, meta: List[np.ndarray]):
        self.params, self.body, self.meta = params, body, meta


def parse_module(text: str) -> Module:
    meta_text = ""
    k = text.find("\nmetadata")
    if k >= 0:
        text, meta_text = text[:k], text[k:]
    p = _P(tokenize(text))
    p.expect("def")
    p.next()  # @main
    p.expect("(")
    params = []
    while not p.accept(")"):
        params.append(p.next()[1])
        if p.accept(":"):
            _parse_type(p)
        p.accept(",")
    if p.accept("->"):
        _parse_type(p)
    p.expect("{")
    body = _parse_expr(p)
    p.expect("}")
    meta = []
    if meta_text:
        q = _P(tokenize(meta_text))
        q.expect("metadata")
        q.expect("{")
        while not q.accept("}"):
            q.next()  # const
            q.expect("[")
            i = int(q.next()[1])
            q.expect("]")
            q.expect("=")
            q.expect("const")
            q.expect("(")
            vals = _parse_value(q)
            q.expect(",")
            shape = _parse_value(q)
            q.expect(",")
            q.next()  # dtype
            q.expect(")")
            q.accept(";")
            while len(meta) <= i:
                meta.append(None)
            meta[i] = np.asarray(vals, np.float32).reshape(shape)
    return Module(params, body, meta)


# ---- evaluation (interp.cpp) -----------------------------------------------------


class _Closure:
    def __init__(self, params, body, env):
        self.params, self.body, self.env = params, body, env


def _eval(e, env: Dict[str, object], mod: Module):
    while e[0] == "let":  # iterative let chains (deep modules)
        env = dict(env)
        env[e[1]] = _eval(e[2], env, mod)
        e = e[3]
    tag = e[0]
    if tag == "var":
        return env[e[1]]
    if tag == "const":
        return e[1]
    if tag == "meta":
        return mod.meta[e[1]]
    if tag == "fn":
        return _Closure(e[1], e[2], env)
    if tag == "call":
        args = [_eval(a, env, mod) for a in e[2]]
        try:
            f = OPS[e[1]]
        except KeyError:
            raise NotImplementedError("oracle: operator %s is not on the fused path" % e[1])
        return f(*args, **e[3])
    if tag == "apply":
        fn = _eval(e[1], env, mod)
        args = [_eval(a, env, mod) for a in e[2]]
        inner = dict(fn.env)
        inner.update(zip(fn.params, args))
        out = _eval(fn.body, inner, mod)
        trace = getattr(mod, "trace", None)
        if trace is not None and e[1][0] == "var":  # per-group record for the group-level tests
            trace.append((e[1][1], args, out.vals if isinstance(out, IntTensor) else out))
        return out
    raise ValueError(tag)


def run_module(text_or_module, args: Sequence[np.ndarray], trace: list = None) -> np.ndarray:
    """Evaluates @main on `args` (float32 arrays in parameter order).  With
    `trace` (a list), appends (function name, arguments, result) for every
    closure application -- one entry per Primitive group of a fused module."""
    mod = parse_module(text_or_module) if isinstance(text_or_module, str) else text_or_module
    mod.trace = trace
    if len(args) != len(mod.params):
        raise ValueError("run_module: %d arguments for %d parameters" % (len(args), len(mod.params)))
    env = {name: np.ascontiguousarray(a, np.float32) for name, a in zip(mod.params, args)}
    out = _eval(mod.body, env, mod)
    if isinstance(out, IntTensor):
        out = out.vals
    return out


def run_weights(text: str, x: np.ndarray, weights: Sequence[np.ndarray]) -> np.ndarray:
    """Convenience: first parameter is the data input, the rest the weights
    in @main parameter order (modelzoo.ModelSource order)."""
    return run_module(text, [x] + list(weights))
