"""One batch of a model through the executor without a CUDA graph (ncu captures):
    python tests/profile_model.py MODEL [int8|fp32] [batch] [runs] [float_mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

name = sys.argv[1]
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 256
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
fm = int(sys.argv[5]) if len(sys.argv) > 5 else mrb.MR_FLOAT_BF16
text, meta, src = mrb.load_model(name, prec)
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
ex = mrb.Executor(text, batch=batch, use_cuda_graph=False, float_mode=fm)
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
x = modelzoo.make_inputs(src, batch, seed=0)
for _ in range(runs):
    y = ex.run_host(x)
print("ok", y.shape)
