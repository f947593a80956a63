"""Summarise an ncu --set full report's SASS page: hottest instruction
windows by executed instructions and stall samples (profiling helper).
    python tests/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX LAUNCH_SKIP [WINDOW]"""
import csv
import io
import subprocess
import sys

rep, kre, skip = sys.argv[1], sys.argv[2], int(sys.argv[3])
win = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
I = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) > I["Instructions Executed"] and r[0].startswith("0x")]


def g(r, k):
    v = r[I[k]].strip()
    return int(v) if v and v != "-" else 0


tot = sum(g(r, "Instructions Executed") for r in data)
samp = sum(g(r, "Warp Stall Sampling (All Samples)") for r in data)
print(rows[0][0][:150], "\ntotal warp-instructions", tot, "stall samples", samp, "sass lines", len(data))
for i in range(0, len(data), win):
    s = sum(g(r, "Instructions Executed") for r in data[i:i + win])
    ss = sum(g(r, "Warp Stall Sampling (All Samples)") for r in data[i:i + win])
    if s > tot * 0.02 or ss > samp * 0.02:
        top = max(data[i:i + win], key=lambda r: g(r, "Instructions Executed"))
        print("%5d %5.1f%% inst %5.1f%% stall | %s" % (i, 100.0 * s / tot, 100.0 * ss / max(samp, 1), top[1].strip()[:70]))
