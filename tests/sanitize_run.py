"""One small int8 + bf16 inference for compute-sanitizer (tcgen05 conv, stem
fused with max_pool, the tcgen05 dense head, sum, input conversion), no CUDA
graph so every kernel is a plain launch:
    compute-sanitizer --tool {memcheck|racecheck|synccheck} python tests/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ok = True
for name, batch, prec in (("resnet18_tiny", 4, "int8"), ("resnet18", 2, "int8"), ("branchy", 4, "int8")):
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    ex = mrb.Executor(text, batch=batch, use_cuda_graph=False)
    ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
    y = ex.run_host(modelzoo.make_inputs(src, batch, seed=0))
    g = np.load(os.path.join(GOLD, "%s_b%d.npz" % (name, batch)))[prec]
    same = np.array_equal(y.view(np.uint32), g.view(np.uint32))
    ok = ok and same
    print(name, prec, "bit-exact" if same else "MISMATCH", ex.launch_count(), "kernels")
text, meta, src = mrb.load_model("resnet18_tiny", "fp32")
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
ex = mrb.Executor(text, batch=4, use_cuda_graph=False)
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
y = ex.run_host(modelzoo.make_inputs(src, 4, seed=0))
print("resnet18_tiny bf16 ran", y.shape)
sys.exit(0 if ok else 1)
