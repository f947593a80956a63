"""Builds profiles/traffic.json from ncu CSV logs of one executor step
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv --log-file X python tests/profile_run.py PREC 256 1`): DRAM bytes per
kernel family per step, keyed like bench.py's roofline families.

    python tests/ncu_traffic.py int8=gpurun_out/traffic_int8.csv bf16=gpurun_out/traffic_fp32.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def family(kname, prec):
    if "k_conv_tc" in kname:
        return "conv_i8_tcgen05" if prec == "int8" else "conv_bf16_tcgen05"
    for key, fam in (("k_input", "input_convert"), ("k_dense_ks", "dense_i8" if prec == "int8" else "dense_bf16"),
                     ("k_dense<", "dense_i8" if prec == "int8" else "dense_bf16"),
                     ("k_sum_hw", "sum_hw"), ("k_to_nchw", "result_to_nchw"), ("k_maxpool", "max_pool")):
        if key in kname:
            return fam
    return None


def parse(path, prec):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    I = {k: i for i, k in enumerate(h)}
    per = {}
    for r in rows[1:]:
        if r[I["Metric Name"]] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        v = float(r[I["Metric Value"]].replace(",", ""))
        unit = r[I["Metric Unit"]]
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        key = (r[I["ID"]], r[I["Kernel Name"]])
        per[key] = per.get(key, 0.0) + v
    fams = {}
    for (kid, kname), b in per.items():
        f = family(kname, prec)
        if f:
            fams.setdefault(f, {"bytes_per_step": 0.0, "launches": 0})
            fams[f]["bytes_per_step"] += b
            fams[f]["launches"] += 1
    return fams


if __name__ == "__main__":
    out = {"source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, one executor step "
                     "(tests/profile_run.py, no CUDA graph), per kernel family"}
    for arg in sys.argv[1:]:
        prec, path = arg.split("=", 1)
        out[prec] = parse(path, prec)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))
