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
                   if k.startswith(("k_input_s2d_ct<3, 3, 16", "k_dense_tc<1", "k_to_nchw")))
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

    # --set full summaries: every captured launch, one row each
    def full_table(rep, title, cmd, md):
        if rep.endswith(".csv"):
            if not os.path.exists(rep):
                return
            raw = open(rep).read()
        else:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        if len(rr) <= 2:
            return
        h, units, ks = rr[0], rr[1], rr[2:]
        J = {k: i for i, k in enumerate(h)}
        want = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "DRAM rd MB"),
                ("dram__bytes_write.sum", "DRAM wr MB"),
                ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
                ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
                ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue %"),
                ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("launch__registers_per_thread", "regs")]
        out = ["# " + title, "", "Command: `%s`" % cmd,
               "(per-launch, cold-cache, serialised replay under ncu: absolute times differ from the in-graph "
               "bench, shares agree; DRAM MB in the units ncu reports).", "",
               "| # | kernel | " + " | ".join(l for _, l in want) + " |", "|---|---|" + "---|" * len(want)]
        kn = J.get("Kernel Name")
        for i, k in enumerate(ks):
            name = k[kn].split("(")[0].replace("void ", "").split("::")[-1][:48] if kn is not None else "?"
            vals = []
            for key, _ in want:
                v = k[J[key]] if key in J else ""
                try:
                    v = "%.1f" % float(v.replace(",", ""))
                except ValueError:
                    pass
                vals.append(v)
            out.append("| %d | %s | %s |" % (i, name, " | ".join(vals)))
        open(os.path.join(PROF, md), "w").write("\n".join(out) + "\n")

    full_table(os.path.join(OUT, "conv_full_raw.csv"),
               "ncu --set full, round %s: every tcgen05 conv launch of one int8 ResNet-18 b256 step "
               "(input conversion, stem+pool, 19 convs, the fused sum + tcgen05 dense head)" % tag[1:],
               "ncu --set full --clock-control none -k regex:\"k_conv_tc|k_dense_tc|k_sum_hw|k_input\" "
               "-c 25 python tests/profile_run.py int8 256 1", tag + "_conv_tc_full.md")
    full_table(os.path.join(OUT, "dw_full_raw.csv"),
               "ncu --set full, round %s: the 13 depthwise launches of one MobileNet-v1 bf16 b256 step" % tag[1:],
               "ncu --set full --clock-control none -k regex:k_dw3x3 -c 13 python tests/profile_model.py mobilenet_v1 fp32 256 1",
               tag + "_dw_full.md")
    for side in ("bench_c5", "bench_mbv1", "bench_vgg", "bench_dqn"):
        f = os.path.join(OUT, side + ".json")
        if os.path.exists(f):
            try:
                json.dump(last_json(f), open(os.path.join(PROF, "%s_%s.json" % (tag, side)), "w"))
            except Exception:
                pass
    print("profiles/ updated:", bench["value"], bench["ms_per_step"])


if __name__ == "__main__":
    main()
