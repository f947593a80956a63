"""Debug helper: one tiny int8 ResNet-18 batch without a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet18_tiny"
text, meta, src = mrb.load_model(name, "int8")
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
ex = mrb.Executor(text, batch=4, use_cuda_graph=False)
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
print(ex.run_host(modelzoo.make_inputs(src, 4, seed=0))[0, :4])
