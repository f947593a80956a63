"""One batch of models/<name>_<prec> without a CUDA graph, for ncu captures:
    python tests/profile_model.py NAME PREC BATCH"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

name, prec, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
text, meta, src = mrb.load_model(name, prec)
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
ex = mrb.Executor(text, batch=batch, use_cuda_graph=False)
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
print(ex.run_host(modelzoo.make_inputs(src, batch, seed=0)).shape)
