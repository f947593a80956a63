"""Refreshes the measured numbers quoted in DESIGN.md (per-launch table, step
summary, side configs) and README.md from profiles/r01_bench.json and the
gpurun_out/ side benches written by tests/final_profiles.sh."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


d = json.load(open(os.path.join(ROOT, "profiles", "r01_bench.json")))
big = last(os.path.join(ROOT, "gpurun_out", "bench_b4096.json"))
mb = last(os.path.join(ROOT, "gpurun_out", "bench_mbv1.json"))
rows = ["| launch | kernel | alg. MB | GOP | ms | roofline ms | bound | frac |", "|---|---|---|---|---|---|---|---|"]
tot = roof = 0.0
for L in d["per_launch"]:
    rows.append("| %s | %s | %.1f | %.2f | %.4f | %.4f | %s | %.2f |" % (
        L["launch"], L["kernel"], L["bytes"] / 1e6, L["ops"] / 1e9, L["ms"], L["roof_ms"], L["bound"], L["frac"]))
    tot += L["ms"]
    roof += L["roof_ms"]
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
ia = s.index("| launch | kernel | alg. MB | GOP | ms | roofline ms | bound | frac |")
ib = s.index("Other BASELINE configs at batch 256")
s = s[:ia] + "\n".join(rows) + """

Sum %.3f ms profiled (non-graph, event-separated) vs %.3f ms roofline sum: the step runs
at %d %% of its per-group roofline; in the CUDA graph the step is %.3f ms (%.1f k img/s;
bf16 %.1f k img/s). Batch 4096 on one GPU (config C5): %.1f ms per step, %.1f k img/s.

""" % (tot, roof, round(100 * roof / tot), d["ms_per_step"], d["value"] / 1e3, d["bf16"]["value"] / 1e3,
       big["ms_per_step"], big["value"] / 1e3) + s[ib:]
s = re.sub(r"\| C3 MobileNet-v1 \| [\d.]+ k \| [\d.]+ k \|",
           "| C3 MobileNet-v1 | %.1f k | %.1f k |" % (mb["value"] / 1e3, mb["bf16"]["value"] / 1e3), s)
open(p, "w").write(s)
p = os.path.join(ROOT, "README.md")
s = open(p).read()
s = re.sub(r"int8 \d+k images/s on device", "int8 %dk images/s on device" % round(d["value"] / 1e3), s)
s = re.sub(r"bf16 \d+k images/s; at batch 4096 on one GPU, \d+k images/s int8",
           "bf16 %dk images/s; at batch 4096 on one GPU, %dk images/s int8" % (round(d["bf16"]["value"] / 1e3),
                                                                               round(big["value"] / 1e3)), s)
s = re.sub(r"MobileNet-v1 \(\d+k int8 / \d+k bf16 images/s\)",
           "MobileNet-v1 (%dk int8 / %dk bf16 images/s)" % (round(mb["value"] / 1e3), round(mb["bf16"]["value"] / 1e3)), s)
open(p, "w").write(s)
print(d["value"], d["bf16"]["value"], big["value"], mb["value"], mb["bf16"]["value"])
