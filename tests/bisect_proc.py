"""Per-group bisect, one process per truncated module (an illegal access
poisons the CUDA context): compares every group output with the CPU oracle.
    python tests/bisect_proc.py NAME PREC [BATCH] [float_mode]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def child(name, prec, batch, var, fm):
    import paper_1904_08368_b200 as mrb
    from paper_1904_08368_b200 import modelzoo
    from oracle import port
    from group_bisect import truncate
    text, meta, src = mrb.load_model(name, prec)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    wl = [w[p.name] for p in src.params if p.kind != "input"]
    x = modelzoo.make_inputs(src, batch, seed=0)
    t = truncate(text, var)
    r = port.run_weights(t, x, wl)
    ex = mrb.Executor(t, batch=batch, use_cuda_graph=False, float_mode=fm)
    ex.set_weights(wl)
    y = ex.run_host(x)
    bad = int(np.sum(y.view(np.uint32) != r.view(np.uint32)))
    nw = float(np.max(np.abs(y - r)) / max(np.max(np.abs(r)), 1e-30))
    kern = [g["kernel"] for g in ex.describe()["groups"]]
    print("RESULT %s bad=%d/%d normwise=%.3g kernels=%s" % (var, bad, y.size, nw, kern[-1]), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5], int(sys.argv[6]))
        sys.exit(0)
    from group_bisect import group_outputs
    import paper_1904_08368_b200 as mrb
    name, prec = sys.argv[1], sys.argv[2]
    batch = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    fm = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    text, _, _ = mrb.load_model(name, prec)
    for var in group_outputs(text):
        p = subprocess.run([sys.executable, __file__, "--child", name, prec, str(batch), var, str(fm)],
                           capture_output=True, text=True, timeout=600)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        print(line[0] if line else "FAIL %s rc=%d %s" % (var, p.returncode, p.stderr.strip().splitlines()[-1][:200]),
              flush=True)
        if not line:
            break
