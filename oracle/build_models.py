"""Compile the model zoo with the REFERENCE compiler -> models/*.rly.

Oracle tooling (runs in the build container, where /root/reference and
oracle/_ref/mr_ref exist).  For every model it writes

  models/<name>.src.rly           the unfused source (modelzoo.py)
  models/<name>_fp32.fused.rly    run_pipeline("fold-scale,fold,dce,fuse")
  models/<name>_int8.fused.rly    run_pipeline("fold-scale,fold,dce,quantize,fuse")
  models/<name>.json              calibrated k + seeds + pass lists

The int8 module uses the global scale 2^k that the reference's own
quant_calibrate (quantize.cpp:138-177) picks on ONE calibration image
(modelzoo.make_inputs(seed=0)[0]) with the seeded weights; the fixed-k
compile is checked equal to the stock calibrated run_pipeline on small
models by tests/test_oracle_ref.py.

The fused modules are the drop-in artifact the backend consumes: the exact
text the reference's printer (printer.cpp) emits for its fused program.

usage: python oracle/build_models.py [name ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, _ROOT)

from oracle import ref  # noqa: E402
from paper_1904_08368_b200 import modelzoo  # noqa: E402

PRE = "fold-scale,fold,dce"
FP32 = PRE + ",fuse"
INT8 = PRE + ",quantize,fuse"

CONFIGS = {
    # name: (builder, kwargs)
    "resnet18": (modelzoo.resnet18, {}),
    "resnet18_tiny": (modelzoo.resnet18, dict(image=32, num_classes=10, widths=(32, 32, 64, 64))),
    # BASELINE.json configs[2..3] (parity cases): MobileNet-v1 224, VGG-16 224, Nature DQN.
    # VGG-16 and DQN flatten with a static-batch reshape: compiled at batch 2.
    "mobilenet_v1": (modelzoo.mobilenet_v1, {}),
    "vgg16": (modelzoo.vgg16, dict(batch=2)),
    "dqn": (modelzoo.dqn, dict(batch=2)),
    # model interchange: weights embedded in the metadata
    # pool (modelzoo.bind_weights), folded by the reference's own passes
    "resnet18_small_const": (modelzoo.resnet18, dict(image=32, num_classes=10, widths=(16, 16, 32, 32))),
    # BASELINE config C4 at its benchmark batch (static-batch reshape heads): throughput
    # modules only (tests/side_bench.py); the int8 DQN reuses dqn's calibrated k
    "vgg16_b256": (modelzoo.vgg16, dict(batch=256)),
    "dqn_b256": (modelzoo.dqn, dict(batch=256)),
    # the reference's combine-conv pass on a net with parallel
    # same-geometry convs (concat-weight conv + the Opaque split group in the output)
    "branchy": (modelzoo.branchy, {}),
}
K_FROM = {"dqn_b256": "dqn"}
BIND = {"resnet18_small_const", "branchy"}
# pass lists with combine-conv before fuse (and before quantize for int8)
COMBINE = {"branchy"}
# float-only (BASELINE lists them as bf16 configs; an int8 calibration sweep of
# the 224x224 VGG-16 in the reference interpreter takes about an hour)
NO_INT8 = {"vgg16", "vgg16_b256"}


def build(name: str, out_dir: str) -> dict:
    fn, kw = CONFIGS[name]
    src = fn(**kw)
    w = modelzoo.make_weights(src, seed=1)
    if name in BIND:
        src = modelzoo.bind_weights(src, w)
        w = {p.name: w[p.name] for p in src.params if p.kind != "input"}
    batch = kw.get("batch", 1)  # static-batch modules calibrate on their own batch
    x = modelzoo.make_inputs(src, batch, seed=0)
    t0 = time.time()
    if name in K_FROM:
        k = json.load(open(os.path.join(out_dir, K_FROM[name] + ".json")))["calibration"]["k"]
    else:
        k = None if name in NO_INT8 else ref.calibrate(src.text, PRE, [x] + ref.weight_list(src, w))
    t_cal = time.time() - t0
    fp32_passes = FP32.replace(",fuse", ",combine-conv,fuse") if name in COMBINE else FP32
    int8_passes = INT8.replace(",quantize", ",combine-conv,quantize") if name in COMBINE else INT8
    fused_fp32 = ref.compile(src.text, fp32_passes, 0)
    fused_int8 = None if k is None else ref.compile(src.text, int8_passes, k)
    open(os.path.join(out_dir, name + ".src.rly"), "w").write(src.text)
    open(os.path.join(out_dir, name + "_fp32.fused.rly"), "w").write(fused_fp32)
    if fused_int8 is not None:
        open(os.path.join(out_dir, name + "_int8.fused.rly"), "w").write(fused_int8)
    meta = {
        "name": name,
        "builder": fn.__name__,
        "bind_weights": name in BIND,
        "builder_kwargs": {k2: list(v) if isinstance(v, tuple) else v for k2, v in kw.items()},
        "weights_seed": 1,
        "calibration": None if k is None else (
            {"k": k, "scale": 2.0 ** k, "k_from": K_FROM[name]} if name in K_FROM else
            {"inputs_seed": 0, "images": batch, "k": k, "scale": 2.0 ** k, "seconds": round(t_cal, 1), "pre_passes": PRE}),
        "passes": {"fp32": fp32_passes, "int8": None if k is None else int8_passes},
        "groups": {"fp32": fused_fp32.count("[Primitive=true]"),
                   "int8": None if fused_int8 is None else fused_int8.count("[Primitive=true]")},
    }
    json.dump(meta, open(os.path.join(out_dir, name + ".json"), "w"), indent=1)
    return meta


if __name__ == "__main__":
    names = sys.argv[1:] or list(CONFIGS)
    out = os.path.join(_ROOT, "models")
    os.makedirs(out, exist_ok=True)
    for n in names:
        print(json.dumps(build(n, out)), flush=True)
