"""Generates tests/golden/*.npz from the REFERENCE interpreter (oracle/_ref/mr_ref).

Run in the build container (needs oracle/_ref built from /root/reference):
    python tests/golden/make_golden.py
Each fixture holds the reference's interp() output of a models/*.fused.rly
module on seeded inputs (modelzoo.make_inputs) and seeded weights
(modelzoo.make_weights), plus a checksum of the inputs so a numpy change in
the generators is detected instead of silently compared.
"""
import concurrent.futures as cf
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
    res["w_sha256"] = np.asarray(sha(np.concatenate([v.ravel() for v in w.values()] or [np.zeros(0, np.float32)])))
    np.savez(os.path.join(OUT, "%s_b%d.npz" % (name, batch)), **res)
    print(name, batch, {k: v.shape for k, v in res.items()})


def c5_rows(total=4096, n=256, seed=5):
    """The seeded subset of config C5's batch-4096 rows checked against the
    reference (all 4096 images or a seeded subset of >= 256)."""
    return np.sort(np.random.Generator(np.random.PCG64(seed)).choice(total, n, replace=False))


def make_diverse(name, batch, jobs=None, precs=("int8", "fp32"), rows=None, tag=None):
    """`<name>_div_b<batch>.npz`: the reference's logits of `batch` DIVERSE images
    (modelzoo.make_inputs_diverse, seed 0), for the GPU tests at the benchmarked
    batch.  Batch-1 modules run as independent batch-1
    interp() calls spread over `jobs` processes (per-sample independence,
    SURVEY.md 8(e)); static-batch modules run whole-batch, one process per
    precision."""
    jobs = jobs or os.cpu_count()
    res = {}
    src0 = None
    for prec in precs:
        text, meta, src = mrb.load_model(name, prec)
        src0 = src
        w = modelzoo.make_weights(src, seed=meta["weights_seed"])
        x = modelzoo.make_inputs_diverse(src, batch, seed=0, rows=rows)
        wl = ref.weight_list(src, w)
        static = "batch" in meta["builder_kwargs"]
        if static:
            res[prec] = cf.ThreadPoolExecutor(1).submit(ref.run, text, x, wl, None, None, True)
            continue
        chunks = np.array_split(np.arange(batch), jobs)
        with cf.ThreadPoolExecutor(jobs) as pool:
            futs = [pool.submit(ref.run, text, x[c], wl) for c in chunks if len(c)]
            outs = [f.result() for f in futs]
        res[prec] = np.concatenate([o.out for o in outs])
        res[prec + "_seconds"] = np.asarray(sum((o.seconds for o in outs), []))
        print(name, prec, "done", flush=True)
    for prec in precs:
        if isinstance(res[prec], cf.Future):
            r = res[prec].result()
            res[prec] = r.out
            res[prec + "_seconds"] = np.asarray(r.seconds)
    res["x_sha256"] = np.asarray(sha(x))
    res["w_sha256"] = np.asarray(sha(np.concatenate([v.ravel() for v in w.values()] or [np.zeros(0, np.float32)])))
    if rows is not None:
        res["rows"] = np.asarray(rows, np.int64)
    np.savez(os.path.join(OUT, tag or "%s_div_b%d.npz" % (name, batch)), **res)
    for prec in precs:
        top = res[prec].reshape(batch, -1).argmax(1)
        print(name, prec, "distinct top-1:", len(set(top.tolist())), flush=True)


if __name__ == "__main__":
    todo = {"resnet18_tiny": 4, "resnet18": 2, "mobilenet_v1": 2, "dqn": 2, "vgg16": 2, "resnet18_small_const": 4,
            "branchy": 4}
    diverse = {"resnet18": 256, "mobilenet_v1": 256, "dqn_b256": 256, "resnet18_tiny": 64, "branchy": 64}
    args = sys.argv[1:]
    if args and args[0] == "c5":  # ResNet-18 int8, seeded 256-row subset of the batch-4096 config
        make_diverse("resnet18", 256, precs=("int8",), rows=c5_rows(), tag="resnet18_div_c5sub256.npz")
    elif args and args[0] == "diverse":
        for name in args[1:] or list(diverse):
            make_diverse(name, diverse[name])
    else:
        for name in args or list(todo):
            make(name, todo[name])
