"""Turns the raw outputs of tests/final_profiles.sh (gpurun_out/) into the
committed profiles/ artifacts: r01_bench.json (the bench line), traffic.json
(+ the traffic CSVs), r01_launches.csv/.md (ncu launch list summary) and
r01_conv_tc_full.md (ncu --set full summary of the first conv launches).
    python tests/summarize_profiles.py [round-tag]"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    bench = last_json(os.path.join(OUT, "bench_final.json"))
    json.dump(bench, open(os.path.join(PROF, tag + "_bench.json"), "w"))
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tests", "ncu_traffic.py"),
                           "int8=" + os.path.join(OUT, "traffic_int8.csv"), "bf16=" + os.path.join(OUT, "traffic_fp32.csv")],
                          stdout=subprocess.DEVNULL)
    shutil.copy(os.path.join(OUT, "traffic_int8.csv"), os.path.join(PROF, tag + "_traffic_int8.csv"))
    shutil.copy(os.path.join(OUT, "traffic_fp32.csv"), os.path.join(PROF, tag + "_traffic_bf16.csv"))

    # launch list
    rows = [r for r in csv.reader(open(os.path.join(OUT, "launches_bench.csv"))) if len(r) > 5]
    h = rows[0]
    I = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[1:] if r[I["Metric Name"]] == "gpu__time_duration.sum"]
    with open(os.path.join(PROF, tag + "_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "duration_ns"])
        for r in data:
            w.writerow([r[I["ID"]], r[I["Kernel Name"]][:90], r[I["Grid Size"]], r[I["Block Size"]], r[I["Metric Value"]]])
    fam = collections.OrderedDict()
    for r in data:
        k = r[I["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1]
        c, t = fam.get(k, (0, 0.0))
        fam[k] = (c + 1, t + float(r[I["Metric Value"]]))
    conv_i8 = sum(t for k, (c, t) in fam.items() if k.startswith("k_conv_tc<1"))
    other_i8 = sum(t for k, (c, t) in fam.items()
                   if k.startswith(("k_input_s2d_ct<3, 3, 16", "k_dense_ks<0", "k_to_nchw")))
    other_i8 += sum(t for k, (c, t) in fam.items() if k.startswith("k_sum_hw")) / 2
    lines = ["# ncu launch list, round %s (final build)" % tag[1:], "",
             "Command (after the same command exited 0 without ncu, tests/final_profiles.sh):",
             "`ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --no-cuda-graph "
             "--steps 2 --warmup 1 --no-cpu-baseline`",
             "(the bench replays its launch list without the CUDA graph here so every launch is listed: %d launches"
             " over the warm-up, timed, end-to-end and per-launch profile passes of both pipelines, plus the"
             " one-time weight preparation). Per-launch times are cold-cache and serialised. Full list: `%s_launches.csv`."
             % (len(data), tag), "", "| kernel | launches | total us |", "|---|---|---|"]
    for k, (c, t) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        lines.append("| %s | %d | %.0f |" % (k, c, t / 1e3))
    lines += ["", "int8 step: the tcgen05 conv kernel is %.0f us of %.0f us = **%.1f %%** (sum_hw counted half: it serves "
              "both pipelines), next to bench.py's live `roofline.share_of_step` (%.3f)."
              % (conv_i8 / 1e3, (conv_i8 + other_i8) / 1e3, 100 * conv_i8 / (conv_i8 + other_i8),
                 bench["roofline"]["share_of_step"])]
    open(os.path.join(PROF, tag + "_launches.md"), "w").write("\n".join(lines) + "\n")

    # --set full summary
    raw = subprocess.run(["ncu", "-i", os.path.join(OUT, "conv_full.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        h, units, ks = rr[0], rr[1], rr[2:]
        J = {k: i for i, k in enumerate(h)}
        want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
                ("dram__bytes_write.sum", "DRAM write"),
                ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
                ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
                ("lts__t_sector_hit_rate.pct", "L2 hit rate %"), ("launch__registers_per_thread", "registers/thread"),
                ("launch__grid_size", "grid"), ("launch__block_size", "block"),
                ("smsp__sass_inst_executed_op_utcmma.sum", "tcgen05.mma instructions"),
                ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
                ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue")]
        names = ["stem+maxpool (fused21+20, TC_STEM_POOL)", "layer1 Ga (fused19: conv+bias+relu+requant)",
                 "layer1 Gb (fused18: conv+bias+residual+relu, fp32 + int8 codes)"]
        out = ["# ncu --set full, round %s (final build): first three tcgen05 conv launches of one int8 ResNet-18 b256 step"
               % tag[1:], "",
               "Command: `ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -c 3 python "
               "tests/profile_run.py int8 256 1`",
               "(tests/final_profiles.sh; per-launch, cold-cache, serialised replay: absolute times differ from the "
               "in-graph bench, shares agree).", "", "| metric | " + " | ".join(names) + " |", "|---|---|---|---|"]
        for key, label in want:
            if key in J:
                out.append("| %s (%s) | %s |" % (label, units[J[key]], " | ".join(k[J[key]] for k in ks[:3])))
        open(os.path.join(PROF, tag + "_conv_tc_full.md"), "w").write("\n".join(out) + "\n")
    print("profiles/ updated:", bench["value"], bench["ms_per_step"])


if __name__ == "__main__":
    main()
