"""Per-group parity: truncate a fused module at each group's output and compare
the executor with the reference interpreter on every intermediate
("bitwise same_as on logits and on every group output in
debug mode").  The truncation only edits @main's result variable, so both
sides execute the identical prefix of the reference's own fused program.

    python tests/group_bisect.py resnet18_tiny int8 [batch]
"""
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def group_outputs(text):
    """@main-level let variables bound to a group call, in order."""
    return re.findall(r"^  let %(\w+) = %fused\d+\(", text, flags=re.M)


def truncate(text, var):
    """Return @main's text with its result replaced by %var."""
    head, sep, meta = text.partition("\nmetadata {")
    m = list(re.finditer(r"\n  %(\w+)\n}\n?", head))
    if not m:
        raise ValueError("cannot find @main's result")
    last = m[-1]
    head = head[: last.start()] + "\n  %" + var + "\n}\n" + head[last.end():]
    return head + (sep + meta if sep else "")


def compare(name, prec, batch=2, float_mode=None, force_simt=False, stop_at_first=True):
    import paper_1904_08368_b200 as mrb
    from paper_1904_08368_b200 import modelzoo
    from oracle import ref

    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    wl = [w[p.name] for p in src.params if p.kind != "input"]
    x = modelzoo.make_inputs(src, batch, seed=0)
    results = []
    for var in group_outputs(text):
        t = truncate(text, var)
        r = ref.run(t, x, wl).out
        kw = {} if float_mode is None else {"float_mode": float_mode}
        ex = mrb.Executor(t, batch=batch, force_simt=force_simt, **kw)
        ex.set_weights(wl)
        y = ex.run_host(x)
        bad = int(np.sum(y.view(np.uint32) != r.view(np.uint32)))
        results.append((var, bad, float(np.max(np.abs(y - r))) if y.size else 0.0, y.size))
        print("%-8s mismatches %d  max|d| %g  (of %d)" % results[-1], flush=True)
        if bad and stop_at_first:
            idx = np.argwhere(y.view(np.uint32) != r.view(np.uint32))[:5]
            for i in idx:
                print("   at", tuple(i), "gpu", y[tuple(i)], "ref", r[tuple(i)])
            break
    return results


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "resnet18_tiny"
    prec = sys.argv[2] if len(sys.argv) > 2 else "int8"
    batch = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    compare(name, prec, batch)
