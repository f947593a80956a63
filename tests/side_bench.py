"""Side measurement for the other BASELINE configs (not the contract line):
    python tests/side_bench.py MODEL BATCH PREC [steps]
Device-resident throughput of models/<MODEL>_<PREC>.fused.rly through the
executor (CUDA-graph replay, CUDA events), e.g. vgg16_b256 fp32 (bf16 mode),
dqn_b256 int8 / fp32, mobilenet_v1 fp32.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

name, batch, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 50
fmode = sys.argv[5] if len(sys.argv) > 5 else "bf16"  # float modules: bf16 | tf32
text, meta, src = mrb.load_model(name, prec)
w = modelzoo.make_weights(src, seed=meta["weights_seed"])
ex = mrb.Executor(text, batch=batch, **({"float_mode": mrb.MR_FLOAT_TF32} if fmode == "tf32" else {}))
ex.set_weights([w[p.name] for p in src.params if p.kind != "input"])
x = torch.from_numpy(modelzoo.make_inputs(src, batch, seed=0)).cuda()
out = torch.empty(ex.output_shape, dtype=torch.float32, device="cuda")
sh = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    ex.run_device(x.data_ptr(), x.shape, out.data_ptr(), sh)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    ex.run_device(x.data_ptr(), x.shape, out.data_ptr(), sh)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
line = {"model": name, "precision": "int8" if prec == "int8" else fmode, "batch": batch,
        "ms_per_step": ms, "images_per_s": batch / ms * 1e3, "launches": ex.launch_count()}
if os.environ.get("SIDE_PER_LAUNCH"):
    per = ex.profile_device(x.data_ptr(), x.shape, out.data_ptr(), sh)
    torch.cuda.synchronize()
    d = ex.describe()
    line["per_launch"] = [(L["name"], L["kernel"], round(t, 4), round(L["flops"] / 1e9, 1)) for L, t in zip(d["launches"], per)]
print(json.dumps(line))
