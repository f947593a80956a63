"""Benchmark: ResNet-18 fused inference (int8 realized, bf16 float) images/s on B200.

Contract (see the task's bench.py section):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--global-batch B] [--model NAME]
One step = one pass of the fused ResNet-18 (22 Primitive groups, reference
compiler output models/resnet18_int8.fused.rly) over a batch of 256 synthetic
224x224 images per GPU (BASELINE.json configs[1]).  N>1 runs one process per
GPU: under torchrun as launched by the driver, or -- when WORLD_SIZE is unset --
bench.py re-launches itself under torch.distributed.run with N ranks.  Each rank
runs its own batch shard with no collective on the data path:
256 per GPU by default ("scaling": "weak"), or --global-batch B split B/N per
GPU by paper_1904_08368_b200.shard (config C5: --global-batch 4096,
"scaling": "strong"; the shards' logits are gathered to rank 0 in row order
after the timed region).  Timing is on the device (CUDA events around K
CUDA-graph replays, barrier + synchronize on both sides), max over ranks.
`e2e` is the same metric through the public API from pinned host buffers
(H2D input + run + D2H logits every step).  `roofline` is the dominant
kernel's live CUDA-event duration vs its algorithmic bytes/ops.
`cpu_baseline` / --impl reference time the reference interpreter
(oracle/_ref/mr_ref, the unmodified MicroRelay interp()) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-18 images/sec (int8 & bf16) at 1/2/4/8 B200 vs CPU ref; % roofline"
UNIT = "images/s"
BATCH_PER_GPU = 256


def peaks():
    """HBM and bf16 from the driver's MEASURED_PEAKS.json; the int8 tensor peak
    (no cuBLAS int8 figure there) from our tcgen05 kind::i8 microbenchmark
    (tests/tc_peak.cu -> profiles/tc_peak.json, N=256), else 2x bf16."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        pk = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
              "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    else:
        pk = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    tp = os.path.join(ROOT, "profiles", "tc_peak.json")
    if os.path.exists(tp):
        pk["i8_tops"] = json.load(open(tp))["i8_tops"]["256"]
        pk["i8_source"] = "tcgen05 kind::i8 microbenchmark, N=256 (profiles/tc_peak.json)"
    else:
        pk["i8_tops"] = 2.0 * pk["bf16_tflops"]
        pk["i8_source"] = "2x measured bf16 (estimate)"
    return pk


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons polled through NVML every
    10 ms on a background thread DURING the timed region (nvidia-smi's
    fastest loop is too coarse for a sub-second region).  __enter__ returns
    only after the first sample, so the region is covered from its start."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.sm, self.max_sm, self.mask = [], 0, 0
        self.stop = threading.Event()
        self.t = None
        self.err = None

    def _handle(self, nv):
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.device)
            bus = "%08X:%02X:%02X.0" % (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.device)

    def _run(self, nv, h, first):
        while True:
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                try:
                    self.mask |= nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    self.mask |= nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            except Exception as e:
                self.err = str(e)
            first.set()
            if self.stop.wait(0.01):
                return

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            first = threading.Event()
            self.t = threading.Thread(target=self._run, args=(nv, h, first), daemon=True)
            self.t.start()
            first.wait(5)
        except Exception as e:
            self.err = str(e)
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        reasons = sorted(n for bit, n in self.REASONS.items() if self.mask & bit)
        out = {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm or None,
               "reasons": reasons, "samples": len(self.sm), "source": "nvml 10 ms poll"}
        if self.err:
            out["error"] = self.err
        return out


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def max_over_ranks(v: float, world: int):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


MODEL = "resnet18"  # --model: another BASELINE config as a side measurement (not the contract line)


def load(precision):
    import paper_1904_08368_b200 as mrb
    from paper_1904_08368_b200 import modelzoo
    text, meta, src = mrb.load_model(MODEL, precision)
    w = modelzoo.make_weights(src, seed=meta["weights_seed"])
    wl = [w[p.name] for p in src.params if p.kind != "input"]
    return mrb, modelzoo, text, meta, src, wl


def time_ours(precision, batch, steps, warmup, rank, world, local, graph=True, shard=None):
    """Device-resident throughput + e2e + per-launch profile for one precision.
    batch = this rank's images per step; shard = (start, stop) global rows of a
    --global-batch run (inputs: modelzoo.make_inputs_diverse rows start..stop-1,
    so the reassembled logits are the same whatever N is)."""
    import torch
    mrb, modelzoo, text, meta, src, wl = load(precision)
    ex = mrb.Executor(text, batch=batch, device=local, use_cuda_graph=graph)
    ex.set_weights(wl)
    if shard is not None:
        x_host = modelzoo.make_inputs_diverse(src, shard[1] - shard[0], seed=0, start=shard[0])
    else:
        x_host = modelzoo.make_inputs(src, batch, seed=rank)
    x_dev = torch.from_numpy(x_host).to(f"cuda:{local}")
    out = torch.empty(ex.output_shape, dtype=torch.float32, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    launches = ex.launch_count()
    for _ in range(warmup):
        ex.run_device(x_dev.data_ptr(), x_dev.shape, out.data_ptr(), sh)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        e0.record(stream)
        for _ in range(steps):
            ex.run_device(x_dev.data_ptr(), x_dev.shape, out.data_ptr(), sh)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    ms_step = ms / steps
    total = shard[2] if shard is not None else batch * world  # images per step over all ranks
    value = total * steps / (ms / 1e3)
    logits = out.cpu().numpy().copy()

    # e2e through the public API from pinned host memory: every step uploads its
    # input (H2D), runs, and reads back its logits (D2H).  Streaming form
    # (mr_exec_submit_host): step i+1's upload overlaps step i's kernels.
    x_pin = torch.from_numpy(x_host).pin_memory()
    y_pin = torch.empty(ex.output_shape, dtype=torch.float32).pin_memory()
    xn, yn = x_pin.numpy(), y_pin.numpy()
    for _ in range(max(1, warmup)):
        ex.submit_host(xn, yn, sh)
    ex.sync()
    torch.cuda.synchronize()
    barrier(world)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e2.record(stream)
    for _ in range(steps):
        ex.submit_host(xn, yn, sh)
    e3.record(stream)
    ex.sync()
    torch.cuda.synchronize()
    wall_e2e = time.perf_counter() - t0
    barrier(world)
    ms_e2e = max_over_ranks(e2.elapsed_time(e3), world)
    # the same through the blocking call (H2D, run, D2H, synchronize per step)
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nsync = max(1, steps // 4)
    e4.record(stream)
    for _ in range(nsync):
        ex.run_host_into(xn, yn, sh)
    e5.record(stream)
    torch.cuda.synchronize()
    ms_sync = max_over_ranks(e4.elapsed_time(e5), world)
    e2e = {"value": total * steps / (ms_e2e / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(x_host.nbytes), "d2h_bytes_per_step": int(np.prod(ex.output_shape) * 4),
           "ms_per_step": ms_e2e / steps, "api": "mr_exec_submit_host x K + mr_exec_sync (pinned host buffers)",
           "wall_ms_per_step": 1e3 * wall_e2e / steps,
           "blocking_call": {"value": batch * world * nsync / (ms_sync / 1e3), "ms_per_step": ms_sync / nsync,
                             "api": "mr_exec_run_host per step"}}

    # per-launch device times (CUDA events between launches on the same stream)
    desc = ex.describe()
    per = np.zeros(len(desc["launches"]))
    reps = max(3, min(steps, 10))
    for _ in range(reps):
        t = ex.profile_device(x_dev.data_ptr(), x_dev.shape, out.data_ptr(), sh)
        per += np.asarray(t[: len(per)])
    per /= reps
    return dict(value=value, ms_step=ms_step, e2e=e2e, clocks=clk.summary(), launches=launches,
                desc=desc, per_launch_ms=per.tolist(), meta=meta, logits=logits)


# SURVEY.md 8(d) / Appendix A grading basis: ResNet-18's per-group roofline at the
# reference's unfused group structure (every distinct tensor once at its storage
# dtype; int8 peak 4.5 POPS, bf16 1,646.9 TF/s, HBM 6,445 GB/s): 0.861 ms (int8)
# and 0.748 ms (bf16) per 256 images, i.e. per image:
SURVEY_ROOF_US_PER_IMAGE = {("resnet18", "int8"): 861.0 / 256, ("resnet18", "bf16"): 748.0 / 256}


def roofline(res, precision, pk, model=None, batch=None):
    """Dominant kernel (largest share of the step) vs its algorithmic bytes/ops."""
    desc, per = res["desc"], graph_scaled(res)
    # aggregate by kernel family
    fam = {}
    for L, ms in zip(desc["launches"], per):
        # "conv_i8_tcgen05+max_pool" (the fused stem) is the same kernel family
        f = fam.setdefault(L["kernel"].split("+")[0], {"ms": 0.0, "bytes": 0.0, "flops": 0.0, "n": 0})
        f["ms"] += ms
        f["bytes"] += L["bytes"]
        f["flops"] += L["flops"]
        f["n"] += 1
    top = max(fam.items(), key=lambda kv: kv[1]["ms"])
    name, f = top
    hbm = pk["hbm_gbs"]
    tc = pk["i8_tops"] if precision == "int8" else pk["bf16_tflops"]
    t_mem = f["bytes"] / (hbm * 1e9)
    t_tc = f["flops"] / (tc * 1e12)
    bound = "hbm" if t_mem >= t_tc else "tensor"
    secs = f["ms"] / 1e3
    if bound == "hbm":
        achieved, peak, unit = f["bytes"] / secs / 1e9, hbm, "GB/s"
    else:
        achieved, peak, unit = f["flops"] / secs / 1e12, tc, "TFLOP/s" if precision != "int8" else "TOP/s"
    total_ms = sum(per)
    traffic = traffic_step = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        t = json.load(open(tf)).get(precision, {}).get(name)
        if t is not None:  # ncu DRAM bytes of the family: per launch (like `achieved`) and per step
            traffic_step = t["bytes_per_step"]
            traffic = traffic_step / max(1, t.get("launches", f["n"]))
    # whole-step roofline: sum over launches of max(bytes/BW, flops/peak)
    t_roof = sum(max(L["bytes"] / (hbm * 1e9), L["flops"] / (tc * 1e12)) for L in desc["launches"])
    return {"kernel": name, "launches": f["n"], "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": traffic, "share_of_step": f["ms"] / total_ms,
            "peak_source": pk["source"] + ("" if precision != "int8" else "; int8 tensor peak: " + pk["i8_source"]),
            "traffic_per_step": traffic_step,
            "algorithmic": {"bytes": f["bytes"], "ops": f["flops"], "avg_ms": f["ms"] / f["n"],
                            "bytes_per_launch": f["bytes"] / f["n"], "ops_per_launch": f["flops"] / f["n"]},
            "step_roofline_ms": t_roof * 1e3, "step_profiled_ms": sum(res["per_launch_ms"]),
            "step_graph_ms": res["ms_step"], "step_frac": (t_roof * 1e3) / res["ms_step"],
            "timing": "per-launch CUDA-event times of a non-graph replay, scaled by (graph ms/step) / (sum of "
                      "the per-launch times) so the launches add up to the measured CUDA-graph step",
            "survey_basis": survey_basis(res, precision, model, batch)}


def survey_basis(res, precision, model, batch):
    """The step against SURVEY Appendix A's per-group roofline (the reference's
    unfused groups: our cross-group fusions move fewer bytes than that basis,
    the `step_roofline_ms` above is our own plan's)."""
    us = SURVEY_ROOF_US_PER_IMAGE.get((model, precision))
    if us is None or not batch:
        return None
    t = us * batch / 1e3
    return {"step_roofline_ms": t, "frac": t / res["ms_step"], "source": "SURVEY.md 8(d) / Appendix A"}


def graph_scaled(res):
    """Per-launch ms rescaled so they sum to the CUDA-graph ms/step: the event-
    separated non-graph replay adds a launch gap per kernel (and loses the
    programmatic-dependent-launch overlap), so its absolute times overstate
    every launch; the shares are what it measures."""
    per = np.asarray(res["per_launch_ms"], np.float64)
    return (per * (res["ms_step"] / per.sum())).tolist() if per.sum() > 0 else per.tolist()


def per_launch_table(res, precision, pk):
    """Every launch of one step: algorithmic bytes / ops, live device time and
    its own roofline fraction (max of the HBM and tensor-pipe bounds)."""
    hbm = pk["hbm_gbs"] * 1e9
    tc = (pk["i8_tops"] if precision == "int8" else pk["bf16_tflops"]) * 1e12
    out = []
    for L, ms, raw in zip(res["desc"]["launches"], graph_scaled(res), res["per_launch_ms"]):
        t_roof = max(L["bytes"] / hbm, L["flops"] / tc)
        out.append({"launch": L["name"], "kernel": L["kernel"], "bytes": L["bytes"], "ops": L["flops"],
                    "ms": round(ms, 4), "ms_event": round(raw, 4), "roof_ms": round(t_roof * 1e3, 4),
                    "bound": "hbm" if L["bytes"] / hbm >= L["flops"] / tc else "tensor",
                    "frac": round(t_roof * 1e3 / ms, 3) if ms > 0 else None})
    return out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference(precision, procs, steps=1, warm=1, per_step=2, timeout=1800):
    """Reference interp() (oracle/_ref/mr_ref, the unmodified MicroRelay build)
    on the host cores, following BASELINE.md's CPU plan: `procs` worker
    processes, each runs `warm` untimed warm-up image(s), then `steps` steps of
    `per_step` images (one step = per_step * procs images, 2*P by default).  A
    step's time is the max over workers of their per-image interp() seconds
    for that step (the workers run concurrently), so the warm-up is excluded."""
    from oracle import ref
    mrb, modelzoo, text, meta, src, wl = load(precision)
    per_proc = warm + steps * per_step
    x = modelzoo.make_inputs(src, procs * per_proc, seed=0)
    tmp = tempfile.mkdtemp(prefix="mrref_")
    fused = os.path.join(tmp, "fused.rly")
    open(fused, "w").write(text)
    wf = os.path.join(tmp, "w.bin")
    ref.write_tensors(wf, wl)
    ps = []
    t0 = time.time()
    for i in range(procs):
        xf = os.path.join(tmp, "x%d.bin" % i)
        ref.write_tensors(xf, [x[i * per_proc:(i + 1) * per_proc]])
        ps.append(subprocess.Popen([ref.EXE, "run", fused, wf, xf, os.path.join(tmp, "o%d.bin" % i)],
                                   stdout=subprocess.DEVNULL, stderr=subprocess.PIPE, text=True))
    secs = []
    for p in ps:
        _, err = p.communicate(timeout=timeout)
        if p.returncode != 0:
            raise RuntimeError("mr_ref failed: " + err[-500:])
        secs.append([float(l.split()[2]) for l in err.splitlines() if l.startswith("image ")])
    wall = time.time() - t0
    step_s = [max(sum(s[warm + k * per_step: warm + (k + 1) * per_step]) for s in secs) for k in range(steps)]
    timed = [v for s in secs for v in s[warm:]]
    value = per_step * procs * steps / sum(step_s)
    name = {"resnet18": "ResNet-18", "mobilenet_v1": "MobileNet-v1", "dqn": "DQN"}.get(MODEL, MODEL)
    return {"value": value, "unit": UNIT, "cores": procs, "kind": "reference",
            "sample": "%s %s: %d worker processes x (%d warm-up + %d x %d timed) batch-1 interp() calls; step = %d "
                      "images; mean %.2f s/image/core" % (name, precision, procs, warm, steps, per_step,
                                                          per_step * procs, float(np.mean(timed)) if timed else -1),
            "cpu_model": cpu_model(), "ms_per_step": 1e3 * sum(step_s) / steps, "steps": steps, "warmup": warm,
            "wall_s": wall}


def host_cores():
    """Host threads for the CPU reference (capped: each interp() worker holds
    a few hundred MB of materialized intermediates)."""
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    return max(1, min(n, 64))


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(n):
    """`--gpus N` without torchrun: start N ranks of this very command under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


PRETTY = {"resnet18": "ResNet-18 (fused, 22 Primitive groups)", "mobilenet_v1": "MobileNet-v1 (fused, 28 groups)",
          "vgg16_b256": "VGG-16 (fused, static batch 256)", "dqn_b256": "Nature DQN (fused, static batch 256)",
          "resnet18_tiny": "ResNet-18 tiny (32x32)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH_PER_GPU, help="images per GPU per step (weak scaling)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="total images per step split over the N GPUs (config C5: 4096; strong scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bf16", action="store_true")
    ap.add_argument("--model", default="resnet18",
                    help="models/<name>: resnet18 (the contract workload) or another BASELINE config "
                         "(mobilenet_v1, vgg16_b256, dqn_b256) as a side measurement")
    ap.add_argument("--no-cuda-graph", action="store_true",
                    help="replay the launch list without a CUDA graph (for ncu launch lists: ncu cannot replay "
                         "the captured graph)")
    ap.add_argument("--dry-run", action="store_true",
                    help="start the ranks and plan the shards, no GPU work (the CPU test of the multi-rank path)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(args.gpus))
    rank, world, local = dist_env()
    warmup = max(args.warmup, 3)
    global MODEL
    MODEL = args.model
    from paper_1904_08368_b200 import shard as shd
    has_int8 = os.path.exists(os.path.join(ROOT, "models", "%s_int8.fused.rly" % MODEL))
    prec = "int8" if has_int8 else "fp32"
    strong = args.global_batch > 0
    gbatch = args.global_batch if strong else args.batch * world
    a, b = shd.shard_range(gbatch, rank, world) if strong else (rank * args.batch, (rank + 1) * args.batch)
    batch = b - a
    meta = json.load(open(os.path.join(ROOT, "models", MODEL + ".json")))
    k = (meta.get("calibration") or {}).get("k")
    config = {"workload": "%s_%s_b%d" % (MODEL, "int8" if has_int8 else "bf16", gbatch),
              "model": PRETTY.get(MODEL, MODEL), "batch_per_gpu": batch if not strong else shd.shard_sizes(gbatch, world),
              "global_batch": gbatch, "parallelism": "batch shards, no collectives (dp%d)" % world,
              "module": "models/%s_%s.fused.rly (reference run_pipeline %s%s)"
                        % (MODEL, prec, meta["passes"][prec], "; k=%d" % k if has_int8 else ""),
              "inputs": ("modelzoo.make_inputs_diverse rows [g*B/N, (g+1)*B/N) of one global batch" if strong
                         else "modelzoo.make_inputs U[0,1), seed = rank"),
              "l2": "inputs larger than L2: the fp32 input batch + the activations of one step exceed 126 MB; no flush"}

    if args.dry_run:  # the multi-rank plumbing only (CPU test): ranks, shards, gather to rank 0
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
            parts = [None] * world
            dist.all_gather_object(parts, {"rank": rank, "world": world, "shard": [a, b]})
            dist.destroy_process_group()
        else:
            parts = [{"rank": 0, "world": 1, "shard": [a, b]}]
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": parts, "config": config}), flush=True)
        return

    if args.impl == "reference":
        if rank != 0:
            return
        cores = host_cores()
        steps, wu = max(1, min(args.steps, 2)), 1  # bounded sample: 1 warm-up image, then 2*P images per step
        r = cpu_reference(prec, cores, steps=steps, warm=wu)
        v = r["value"]
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": steps, "warmup": wu, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "f32 (fake-quant int8)" if has_int8 else "f32", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                                 "sample": r["sample"] + "; each step = one such sample", "cpu_model": r["cpu_model"]},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "note": "steps/warmup bounded so the CPU arm ends in about a minute (requested --steps %d --warmup %d)"
                        % (args.steps, args.warmup)}
        print(json.dumps(line), flush=True)
        return

    if world != args.gpus:
        print("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world), file=sys.stderr)
        sys.exit(2)
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(local)
    pk = peaks()
    shard = (a, b, gbatch) if strong else None
    res = time_ours(prec, batch, args.steps, warmup, rank, world, local, not args.no_cuda_graph, shard)
    roof = roofline(res, "int8" if has_int8 else "bf16", pk, MODEL, batch)
    gathered = None
    if strong and world > 1:  # result collection after the timed region: the shards' logits in row order
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, (a, res["logits"]))
        gathered = np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])])
    elif strong:
        gathered = res["logits"]
    bf16 = None
    if has_int8 and not args.no_bf16:
        rb = time_ours("fp32", batch, args.steps, warmup, rank, world, local, not args.no_cuda_graph, shard)
        bf16 = {"value": rb["value"], "unit": UNIT, "ms_per_step": rb["ms_step"], "e2e": rb["e2e"],
                "roofline": roofline(rb, "bf16", pk, MODEL, batch), "gpu_launches": rb["launches"] * args.steps,
                "module": "models/%s_fp32.fused.rly (bf16 operands, fp32 accumulate)" % MODEL,
                "per_launch": per_launch_table(rb, "bf16", pk)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(prec, host_cores(), steps=1, warm=1)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "failed: %s" % e}
    if rank == 0:
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": warmup, "ms_per_step": res["ms_step"], "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "int8 (int32 accumulate; fp32 epilogue/residual)" if has_int8 else "bf16 (fp32 accumulate)",
                "data": "synthetic", "config": config, "e2e": res["e2e"], "gpu_launches": res["launches"] * args.steps,
                "clocks": res["clocks"], "roofline": roof, "cpu_baseline": cpu, "bf16": bf16,
                "per_group_ms": {L["name"] + ":" + L["kernel"]: round(ms, 4)
                                 for L, ms in zip(res["desc"]["launches"], graph_scaled(res))},
                "per_launch": per_launch_table(res, "int8" if has_int8 else "bf16", pk),
                "plans": {g["name"]: g["kernel"] + (": " + g["plan"] if g["plan"] else "") for g in res["desc"]["groups"]}}
        if gathered is not None:
            import hashlib
            line["rows"] = {"shape": list(gathered.shape),
                            "sha256": hashlib.sha256(np.ascontiguousarray(gathered).tobytes()).hexdigest(),
                            "note": "logits of all shards gathered in row order after the timed region"}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
