"""Generates tests/golden/*.npz from the REFERENCE interpreter (oracle/_ref/mr_ref).

Run in the build container (needs oracle/_ref built from /root/reference):
    python tests/golden/make_golden.py
Each fixture holds the reference's interp() output of a models/*.fused.rly
module on seeded inputs (modelzoo.make_inputs) and seeded weights
(modelzoo.make_weights), plus a checksum of the inputs so a numpy change in
the generators is detected instead of silently compared.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
import paper_1904_08368_b200 as mrb  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def make(name, batch):
    res = {}
    for prec in ("int8", "fp32"):
        if not os.path.exists(os.path.join(ROOT, "models", "%s_%s.fused.rly" % (name, prec))):
            continue
        text, meta, src = mrb.load_model(name, prec)
        w = modelzoo.make_weights(src, seed=meta["weights_seed"])
        x = modelzoo.make_inputs(src, batch, seed=0)
        static = "batch" in meta["builder_kwargs"]  # static-batch module (reshape head)
        r = ref.run(text, x, ref.weight_list(src, w), whole_batch=static)
        res[prec] = r.out
        res[prec + "_seconds"] = np.asarray(r.seconds)
    res["x_sha256"] = np.asarray(sha(x))
    res["w_sha256"] = np.asarray(sha(np.concatenate([v.ravel() for v in w.values()])))
    np.savez(os.path.join(OUT, "%s_b%d.npz" % (name, batch)), **res)
    print(name, batch, {k: v.shape for k, v in res.items()})


if __name__ == "__main__":
    todo = {"resnet18_tiny": 4, "resnet18": 2, "mobilenet_v1": 2, "dqn": 2, "vgg16": 2, "resnet18_small_const": 4}
    for name in sys.argv[1:] or list(todo):
        make(name, todo[name])
