"""One int8 (or bf16) ResNet-18 batch through the executor without a CUDA
graph, for ncu launch lists / kernel captures:
    python tests/profile_run.py [int8|fp32] [batch] [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "int8"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
text, meta, src = mrb.load_model("resnet18", prec)
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
ex = mrb.Executor(text, batch=batch, use_cuda_graph=False)
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
x = modelzoo.make_inputs(src, batch, seed=0)
for _ in range(runs):
    y = ex.run_host(x)
print("ok", y.shape, float(np.abs(y).sum()))
for g in ex.describe()["groups"]:
    print(g["name"], g["kernel"], g["plan"])
