"""Print a bench line's step times and depthwise per-launch event times (A/B helper).
    python tests/show_dw.py BENCH_JSON"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("int8 %.4f ms  bf16 %.4f ms" % (d["ms_per_step"], d["bf16"]["ms_per_step"]))
for key, pl in (("int8", d["per_launch"]), ("bf16", d["bf16"]["per_launch"])):
    print(key, " ".join("%s:%.4f" % (x["launch"], x["ms_event"]) for x in pl if x["kernel"] == "dwconv"))
