"""Refreshes the measured numbers quoted in DESIGN.md (the ResNet-18 per-launch
table) and README.md from profiles/<tag>_bench*.json, written by
tests/final_profiles.sh + tests/summarize_profiles.py.
    python tests/update_docs_numbers.py [tag]"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"


def prof(name):
    return json.load(open(os.path.join(ROOT, "profiles", "%s_%s.json" % (tag, name))))


d = prof("bench")
c5, mb, vgg, dqn = prof("bench_c5"), prof("bench_mbv1"), prof("bench_vgg"), prof("bench_dqn")
rows = ["Per launch, from `profiles/%s_bench.json` `per_launch` (CUDA events around each launch of a" % tag,
        "non-graph replay, scaled so the launches add up to the CUDA-graph step; `ms_event` there is the",
        "raw event time). int8 peak = the tcgen05 `kind::i8` microbenchmark.", "",
        "| launch | kernel | alg. MB | GOP | ms | roofline ms | bound | frac |", "|---|---|---|---|---|---|---|---|"]
tot = roof = 0.0
for L in d["per_launch"]:
    rows.append("| %s | %s | %.1f | %.2f | %.4f | %.4f | %s | %.2f |" % (
        L["launch"], L["kernel"], L["bytes"] / 1e6, L["ops"] / 1e9, L["ms"], L["roof_ms"], L["bound"], L["frac"]))
    tot += L["ms"]
    roof += L["roof_ms"]
rows += ["", "Step: %.3f ms in the CUDA graph (%.1f k img/s int8; bf16 %.1f k img/s) against a %.3f ms"
         " per-group roofline sum: %d %% of roofline. Batch 4096 (C5, one GPU, `--global-batch 4096`):"
         " %.2f ms per step, %.1f k img/s. End to end through `mr_exec_submit_host` (pinned host"
         " buffers, H2D + run + D2H every step): %.1f k img/s (PCIe-bound: 154 MB of fp32 input per step at the 55.3 GB/s host-to-device rate `tests/h2d_rate.py` measures with 1, 2 or 4 copy streams)."
         " Clocks: median %s MHz of %s, reasons %s." % (
             d["ms_per_step"], d["value"] / 1e3, d["bf16"]["value"] / 1e3, roof, round(100 * roof / d["ms_per_step"]),
             c5["ms_per_step"], c5["value"] / 1e3, d["e2e"]["value"] / 1e3, d["clocks"]["sm_mhz"],
             d["clocks"]["sm_max_mhz"], d["clocks"]["reasons"]),
         "",
         "| Config (batch 256, one B200) | int8 img/s | bf16 img/s |", "|---|---|---|",
         "| C2 ResNet-18 | %.1f k | %.1f k |" % (d["value"] / 1e3, d["bf16"]["value"] / 1e3),
         "| C3 MobileNet-v1 | %.1f k | %.1f k |" % (mb["value"] / 1e3, mb["bf16"]["value"] / 1e3),
         "| C4 VGG-16 | — (float config) | %.1f k |" % (vgg["value"] / 1e3),
         "| C4 Nature DQN | %.1f k | %.1f k |" % (dqn["value"] / 1e3, dqn["bf16"]["value"] / 1e3)]
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
a, b = s.index("<!-- per-launch:begin -->"), s.index("<!-- per-launch:end -->")
s = s[:a] + "<!-- per-launch:begin -->\n" + "\n".join(rows) + "\n" + s[b:]
open(p, "w").write(s)
p = os.path.join(ROOT, "README.md")
s = open(p).read()
a, b = s.index("<!-- status:begin -->"), s.index("<!-- status:end -->")
status = ("Round-%s status (one B200, batch 256): ResNet-18 int8 %.0fk images/s on device, bit-exact with the "
          "reference on every row; %.0fk images/s end to end from pinned host memory (PCIe-bound: 154 MB of fp32 "
          "input per step); bf16 %.0fk images/s; batch 4096 (C5) %.0fk images/s. The reference CPU interpreter "
          "runs %.1f images/s on %d cores. MobileNet-v1 %.0fk int8 / %.0fk bf16, VGG-16 %.0fk bf16, Nature DQN "
          "%.0fk int8 images/s. bf16 and tf32 agree with the reference's fp32 top-1 on >= 99%% of 256 diverse "
          "images (tf32 normwise error ~5e-4); the layout=NHWC and combine-conv pass outputs and modules with "
          "embedded weights run bit-exact (int8); every group also runs alone through `mr_group_*`; the GPU "
          "calibration sweep picks the reference's scale. Details and per-launch rooflines: DESIGN.md."
          % (tag[1:], d["value"] / 1e3, d["e2e"]["value"] / 1e3, d["bf16"]["value"] / 1e3, c5["value"] / 1e3,
             d["cpu_baseline"]["value"] if d.get("cpu_baseline") else float("nan"),
             d["cpu_baseline"]["cores"] if d.get("cpu_baseline") else 0, mb["value"] / 1e3, mb["bf16"]["value"] / 1e3,
             vgg["value"] / 1e3, dqn["value"] / 1e3))
s = s[:a] + "<!-- status:begin -->\n" + status + "\n" + s[b:]
open(p, "w").write(s)
print(d["value"], d["bf16"]["value"], c5["value"], mb["value"], mb["bf16"]["value"], vgg["value"], dqn["value"])
