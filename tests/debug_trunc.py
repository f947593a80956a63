"""Debug helper: run a fused module truncated at one group output on the GPU,
print the executor's plan and the mismatch pattern against the reference."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402
from oracle import port  # noqa: E402
from group_bisect import truncate  # noqa: E402

name, prec, var, batch = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
text, meta, src = mrb.load_model(name, prec)
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
wl = [w[p.name] for p in src.params if p.kind != "input"]
x = modelzoo.make_inputs(src, batch, seed=0)
t = truncate(text, var)
r = port.run_weights(t, x, wl)
ex = mrb.Executor(t, batch=batch)
ex.set_weights(wl)
y = ex.run_host(x)
d = ex.describe()
for g in d["groups"]:
    print(g["name"], g["kernel"], g["plan"])
for L in d["launches"]:
    print("  launch", L["name"], L["kernel"])
bad = y.view(np.uint32) != r.view(np.uint32)
print("mismatch", int(bad.sum()), "of", y.size)
if y.ndim == 4:
    print("bad per channel", bad.sum(axis=(0, 2, 3)).tolist())
    print("bad per row", bad.sum(axis=(0, 1, 3)).tolist())
    print("bad per col", bad.sum(axis=(0, 1, 2)).tolist())
    print("bad per image", bad.sum(axis=(1, 2, 3)).tolist())
    print("gpu zeros", int((y == 0).sum()), "ref zeros", int((r == 0).sum()))
