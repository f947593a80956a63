"""Debug helper: run models/<name>_<prec> once (no CUDA graph), compare with
the golden output, print the plan.  python tests/run_model.py NAME PREC [BATCH]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

name, prec = sys.argv[1], sys.argv[2]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 2
text, meta, src = mrb.load_model(name, prec)
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
try:
    ex = mrb.Executor(text, batch=batch, use_cuda_graph=False)
except mrb.BackendError as e:
    print("CREATE FAILED", e)
    d = mrb.lower(text, batch)
    for g in d["groups"]:
        print("  ", g["name"], g["anchor"], g["epilogue"], g["desc"][:100])
    sys.exit(1)
for g in ex.describe()["groups"]:
    print("  ", g["name"], g["kernel"], g["exact"], g["plan"][:90])
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
y = ex.run_host(modelzoo.make_inputs(src, batch, seed=0))
gp = os.path.join(ROOT, "tests", "golden", "%s_b%d.npz" % (name, batch))
if os.path.exists(gp):
    g = np.load(gp)[prec]
    print("mismatch", int(np.sum(y.view(np.uint32) != g.view(np.uint32))), "of", y.size,
          "normwise", float(np.max(np.abs(y - g)) / np.max(np.abs(g))))
