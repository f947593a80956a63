import sys, json, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1904_08368_b200 as mrb
from paper_1904_08368_b200 import modelzoo
for name, prec, batch in [("resnet18_tiny", "int8", 4), ("resnet18_tiny", "fp32", 4), ("resnet18", "int8", 2), ("resnet18", "fp32", 2)]:
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    wl = [w[p.name] for p in src.params if p.kind != "input"]
    x = modelzoo.make_inputs(src, batch, seed=0)
    outs = {}
    for simt in (True, False):
        ex = mrb.Executor(text, batch=batch, force_simt=simt)
        ex.set_weights(wl)
        outs[simt] = ex.run_host(x)
        if not simt:
            for g in ex.describe()["groups"][:4]: print("  ", g["name"], g["kernel"], g["plan"])
    a, b = outs[True], outs[False]
    print(name, prec, "TC vs SIMT: bitwise mismatches", int(np.sum(a.view(np.uint32) != b.view(np.uint32))), "max|d|", float(np.max(np.abs(a-b))), "rel", float(np.max(np.abs(a-b))/np.max(np.abs(a))), flush=True)
