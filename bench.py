#!/usr/bin/env python
"""Benchmark of the out-of-core ResNet-50 training step (BASELINE.json metric).

Default workload (N=1): BASELINE.json config 2 -- ResNet-50 v1.5, batch 640 at
224x224 (the paper's 50 GB case) under a 16 GiB device-memory budget,
feature maps swapped over the host link / recomputed per the PoocH plan. The
timed step is one full training iteration (forward, backward with swap-in /
recompute, [allreduce], momentum SGD) -- the whole hot path of SURVEY.md 8(a).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--batch B] [--budget-gib G] [--workload cfg2|cfg3|cfg4]

--workload cfg4 runs BASELINE config 4 instead: the 3D U-Net (conv3d-BN-ReLU, widths
256/512/1024/1024) at batch 1 on a 256^3 volume, whose 207 GB of maps exceed HBM; its
in-core comparison is the same net at half the edge (the per-voxel rate).

Under torchrun (N>1) every rank runs its own out-of-core executor on its own
shard (weak scaling) with an NCCL gradient allreduce; the step time is the max
over ranks of the CUDA-event time. Rank 0 prints ONE JSON line.

--impl reference times the CPU oracle (oracle/, fp64 NumPy) on the box's host
cores on a bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "ResNet-50 images/s at >HBM batch, 1/2/4/8 B200; overhead vs in-core; swap GB/s"
METRIC_3D = "3D U-Net volumes/s at a >HBM footprint (batch 1, 256^3); overhead vs in-core per voxel; swap GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--edge", type=int, default=None, help="cfg4: volume edge (default 256)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--budget-gib", type=float, default=None)
    ap.add_argument("--li-cap", type=int, default=12)
    ap.add_argument("--no-incore", action="store_true", help="skip the in-core comparison run")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--profile-iters", type=int, default=3)
    ap.add_argument("--ablation", action="store_true",
                    help="also run the paper's strategies (Sec. 5.1-5.2) on the same executor and report each")
    ap.add_argument("--ncu-step", action="store_true",
                    help="profile/plan, 1 warm-up step, then exactly one step inside cudaProfilerStart/Stop "
                         "(for ncu --profile-from-start off); prints nothing")
    ap.add_argument("--fuse", type=int, default=0, choices=[0, 1],
                    help="1: BN-ReLU applied on the consuming conv's operand load (SURVEY 8(f) f2; "
                         "ResNet-50 105 -> 73 maps)")
    ap.add_argument("--dump-profile", default=None,
                    help="write the measured profile (+ plan classes) as JSON to this path (offline planning)")
    ap.add_argument("--precision", type=int, default=1, choices=[0, 1],
                    help="contractions: 1 = 3xTF32 (default, fp32-faithful), 0 = single TF32")
    return ap.parse_args()


class Workload:
    def __init__(self, net, batch, budget, name, in_hw, classes, width=32):
        self.net, self.batch, self.budget, self.name = net, batch, budget, name
        self.in_hw, self.classes, self.width = in_hw, classes, width
        self.three = net == "unet3d"
        self.unit = "volumes/s" if self.three else "images/s"
        self.metric = METRIC_3D if self.three else METRIC

    fuse = False   # BN-ReLU prologue fusion, set from --fuse

    def context(self, device=0, in_hw=None):
        from paper_1907_05013_b200.executor import Context
        return Context.builtin(self.net, self.batch, in_hw=in_hw or self.in_hw, classes=self.classes,
                               width=self.width, device=device, fuse=self.fuse)


def workload(args):
    if args.workload == "cfg2":
        batch = args.batch or 640
        budget = int((args.budget_gib or 16.0) * (1 << 30))
        name = "cfg2: ResNet-50 v1.5 batch %d 224^2, device budget %.0f GiB (paper's 50 GB case)" % (
            batch, budget / (1 << 30))
        return Workload("resnet50", batch, budget, name, 224, 1000)
    if args.workload == "cfg3":
        batch = args.batch or 2560
        name = "cfg3: ResNet-50 v1.5 batch %d 224^2, all free HBM" % batch
        return Workload("resnet50", batch, None, name, 224, 1000)
    e = args.edge or 256
    budget = int(args.budget_gib * (1 << 30)) if args.budget_gib else None
    # (the 3D U-Net has no fusable BN-ReLU: fusion is 2D only)
    name = "cfg4: 3D U-Net (widths 256/512/1024/1024) batch 1, %d^3 volume, %s" % (
        e, "all free HBM" if budget is None else "device budget %.0f GiB" % (budget / (1 << 30)))
    return Workload("unet3d", 1, budget, name, e, 2, 256)


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, idx=0):
        self.samples = []
        self.stop = threading.Event()
        self.idx = idx

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self.run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons}


def peaks():
    p = {"hbm_gbs": 6536.0, "bf16_tflops": 1651.0, "bf16_tflops_sustained": 1385.7, "src": "MEASURED_PEAKS.json"}
    try:
        p.update(json.load(open(os.path.join(HERE, "MEASURED_PEAKS.json"))))
    except Exception:
        p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
             "src": "fallback (B200_PROFILING.md)"}
    # TF32 = bf16 x the guide's nominal ratio (1.1 / 2.25 PFLOP/s dense)
    p["tf32_tflops_sustained"] = p["bf16_tflops_sustained"] * (1.1 / 2.25)
    return p


# ------------------------------------------------------------------ CPU oracle sample
def cpu_sample(target_s=15.0, batch=1):
    """The oracle as it stands: fp64 NumPy ResNet-50 fwd+bwd at 224^2 on host cores."""
    import numpy as np
    import synthdata
    from oracle import nets
    cores = len(os.sched_getaffinity(0))
    net = nets.resnet50()
    params = nets.init_params(net, seed=2)
    x = synthdata.images(batch, 224, 224, 3, seed=0)
    t = synthdata.labels(batch, 1000, seed=1)
    n_img, t0 = 0, time.time()
    while True:
        nets.forward_backward(net, params, x, t)
        n_img += batch
        if time.time() - t0 > target_s:
            break
    dt = time.time() - t0
    return {"value": n_img / dt, "unit": "images/s", "cores": cores, "kind": "oracle",
            "sample": "%d fp64 ResNet-50 v1.5 fwd+bwd step(s) at batch %d, 224^2 (NumPy, BLAS threads = cores)" % (
                n_img // batch, batch)}


def cpu_sample_3d(target_s=15.0, edge=16, width=32):
    """The oracle as it stands on the 3D U-Net (fp64 NumPy) at a bounded size: per-voxel rate."""
    import numpy as np
    import synthdata
    from oracle import nets
    cores = len(os.sched_getaffinity(0))
    net = nets.unet3d(in_d=edge, width=width, classes=2)
    params = nets.init_params(net, seed=2)
    g = synthdata.rng(0)
    x = g.standard_normal((1, edge, edge, edge, 1))
    t = g.integers(0, 2, (1, edge, edge, edge))
    n, t0 = 0, time.time()
    while True:
        nets.forward_backward(net, params, x, t)
        n += 1
        if time.time() - t0 > target_s:
            break
    dt = time.time() - t0
    return {"value": n * edge ** 3 / dt, "unit": "voxels/s", "cores": cores, "kind": "oracle",
            "sample": "%d fp64 3D U-Net fwd+bwd step(s) at %d^3, width %d (NumPy, BLAS threads = cores)" % (
                n, edge, width)}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = workload(args).name
    per = []
    cs = None
    for i in range(args.warmup + args.steps):
        s = cpu_sample(target_s=0.0, batch=1)
        if i >= args.warmup:
            per.append(s["value"])
        cs = s
    v = statistics.median(per)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name + " -- oracle sample: 1 image per step"},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": cs["cores"], "kind": "oracle",
                             "sample": "1 fp64 ResNet-50 fwd+bwd image per step, 224^2"},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def our_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1907_05013_b200.executor import Context
    import synthdata

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev_idx = local
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W = workload(args)
    W.fuse = bool(args.fuse) and not W.three
    if W.fuse:
        W.name += ", BN-ReLU prologue fusion (f2)"
    batch, budget, wname = W.batch, W.budget, W.name
    ctx = W.context(device=dev_idx)
    ctx.set_precision(args.precision)
    free, total = torch.cuda.mem_get_info()
    if budget is None:
        budget = int(free - (3 << 30))
    budget = budget // 256 * 256
    if world > 1:  # one budget for all ranks (free HBM can differ by a few MB): identical plans
        t = torch.tensor([budget], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        budget = int(t.item())
    maps_total = sum(ctx_map_bytes(ctx))
    host_bytes = int(min(maps_total * 1.02 + (64 << 20), 0.6 * os.sysconf("SC_PAGE_SIZE") *
                         os.sysconf("SC_PHYS_PAGES") / max(1, world)))
    host_bytes = host_bytes // 4096 * 4096
    dev = torch.empty(budget, dtype=torch.uint8, device="cuda")
    from paper_1907_05013_b200.executor import PinnedHost
    while True:  # the host may cap page-locked memory: halve until registration succeeds
        try:
            host = PinnedHost(host_bytes)
            break
        except RuntimeError:
            if host_bytes < (8 << 30):
                raise
            host_bytes = host_bytes // 2 // 4096 * 4096
    streams = [torch.cuda.Stream() for _ in range(3)]
    ctx.set_budget(dev, budget, host, host_bytes)
    ctx.set_streams(*streams)
    if world > 1:
        from paper_1907_05013_b200.dp import broadcast_unique_id
        ctx.set_comm(broadcast_unique_id(rank, device="cuda"), rank, world)
    # parameters and the synthetic batch (seed 0 + rank / 1 + rank; identical weights)
    g = synthdata.rng(2)
    for i, (name, numel) in enumerate(ctx.params()):
        if name.endswith(".w"):
            fan = numel // int(name_out_channels(ctx, name))
            ctx.set_param(i, synthdata.he_normal((numel,), fan, g))
        elif ".gamma" in name:
            ctx.set_param(i, np.ones(numel, np.float32))
        else:
            ctx.set_param(i, np.zeros(numel, np.float32))
    xp, lp = ctx.input_slot()
    x_host, l_host = synth_batch(W, rank)
    base = dev.data_ptr()
    x_dev = dev[xp - base: xp - base + x_host.numel() * 4].view(torch.float32)
    l_dev = dev[lp - base: lp - base + l_host.numel() * 4].view(torch.int32)
    x_dev.copy_(x_host)
    l_dev.copy_(l_host)
    torch.cuda.synchronize()

    # ---- profile (Sec. 4.2) + plan (Sec. 4.4); max over ranks so every rank runs one plan
    t0 = time.time()
    prof = ctx.profile(args.profile_iters)
    prof_s = time.time() - t0
    if world > 1:
        from paper_1907_05013_b200.dp import agree_profile
        agreed = agree_profile(prof, device="cuda")
        ctx.set_profile(agreed["fwd"], agreed["bwd"], agreed["rec"], agreed["d2h"], agreed["h2d"], agreed["tail"])
    cls, rep = ctx.plan("pooch", li_cap=args.li_cap)
    counts = {"keep": cls.count(0), "swap": cls.count(1), "recompute": cls.count(2)}
    if args.dump_profile and rank == 0:
        with open(args.dump_profile, "w") as f:
            json.dump({"workload": wname, "batch": batch, "budget": budget, "profile": prof, "classes": cls,
                       "report": {k: (v if isinstance(v, (int, float)) else str(v)) for k, v in rep.items()}}, f)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    lo = ctx.loss_slot() - base
    loss_dev = dev[lo: lo + 4].view(torch.float32)

    def timed(n_steps, e2e=False):
        s = streams[0]
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        loss_h = torch.empty(1, dtype=torch.float32).pin_memory()
        e0.record(s)
        for _ in range(n_steps):
            if e2e:
                with torch.cuda.stream(s):
                    x_dev.copy_(x_host, non_blocking=True)
                    l_dev.copy_(l_host, non_blocking=True)
            ctx.train_step(0.01, sync_loss=False)
            if e2e:
                with torch.cuda.stream(s):
                    loss_h.copy_(loss_dev, non_blocking=True)
        e1.record(s)
        barrier()
        ms = e0.elapsed_time(e1) / n_steps
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64).cuda()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    if args.ncu_step:
        ctx.train_step(0.01, sync_loss=False)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        ctx.train_step(0.01, sync_loss=False)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return
    for _ in range(args.warmup):
        ctx.train_step(0.01, sync_loss=False)
    torch.cuda.synchronize()
    with Clocks(dev_idx) as clk:
        ms = timed(args.steps)
    ms_e2e = timed(max(2, args.steps // 2), e2e=True)
    # instrumented step: per kernel family times (CUDA events on the launching streams)
    ctx.set_timing(True)
    ctx.train_step(0.01, sync_loss=True)
    fam = ctx.family_stats()
    segs = ctx.timing_segments()
    tim = ctx.last_timing()
    ctx.set_timing(False)
    launches = kernel_launches(ctx, args.steps)

    ablation = None
    if args.ablation:
        ablation = {}
        # the paper's strategies (Sec. 5.1-5.2) on the same executor; "pooch_paper" is PoocH
        # without the executor's local refinement (DESIGN.md Reading 42), "pooch" with it
        for strat in ("swap_all_naive", "swap_all", "swap_opt", "superneurons", "pooch_paper", "pooch"):
            try:
                if strat == "pooch_paper":
                    os.environ["POOCH_PLAN_NO_REFINE"] = "1"
                c2, r2 = ctx.plan("pooch" if strat == "pooch_paper" else strat, li_cap=args.li_cap)
            except Exception as e:  # infeasible plans are a result (superneurons OOM)
                ablation[strat] = {"feasible": False, "why": str(e)[:160]}
                continue
            finally:
                os.environ.pop("POOCH_PLAN_NO_REFINE", None)
            ctx.train_step(0.01, sync_loss=False)
            ms_s = timed(2)
            ablation[strat] = {"feasible": True, "ms_per_step": ms_s, "images_per_s": batch * world * 1000.0 / ms_s,
                               "simulated_ms": r2["makespan_ns"] / 1e6,
                               "counts": [c2.count(0), c2.count(1), c2.count(2)]}
        ctx.plan("pooch", li_cap=args.li_cap)

    # ---- in-core comparison (the same kernels, every map kept) where it fits
    # (after the out-of-core context and its arena are released: the in-core run needs the HBM)
    incore = None
    if not args.no_incore and world == 1:
        params_host = [ctx.get_param(i, 0) for i in range(len(ctx.params()))]
        ctx.close()
        dev = x_dev = l_dev = loss_dev = None  # noqa: F841 (drop the arena before the in-core run)
        torch.cuda.empty_cache()
        incore = incore_run(params_host, batch, streams, args)

    value = batch * world * 1000.0 / ms
    pk = peaks()
    roof = roofline(fam, pk, segs, args.precision)
    line = {
        "metric": W.metric, "value": value, "unit": W.unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (%s tensor-core contractions, fp32 accumulate/storage)" % ("3xtf32" if args.precision else "tf32"),
        "data": "synthetic (x ~ N(0,1), labels U[0,%d), He-normal weights; seeded)" % W.classes,
        "config": {"workload": wname, "global_batch": batch * world, "seq_len": None,
                   "parallelism": "dp%d" % world, "budget_bytes_per_gpu": budget,
                   "host_arena_bytes": host_bytes, "l2": "inputs > L2 (maps are GBs)",
                   "plan_counts": counts, "planner_ms": rep["wall_ms"], "planner_sims": rep["n_sims"],
                   "profile_s": prof_s, "simulated_ms_per_step": rep["makespan_ns"] / 1e6,
                   "arena_high_water_bytes": rep["arena_bytes"], "L_O": rep["lo_size"], "L_I": rep["li_size"]},
        "clocks": clk.summary(),
        "e2e": {"value": batch * world * 1000.0 / ms_e2e, "unit": W.unit,
                "h2d_bytes_per_step": int(x_host.numel() * 4 + l_host.numel() * 4), "d2h_bytes_per_step": 4},
        "gpu_launches": launches,
        "roofline": roof,
        "swap": swap_stats(fam, prof),
        "families": families_table(fam, peaks(), segs, args.precision),
    }
    if ablation is not None:
        line["ablation"] = ablation
    if W.three:
        line["voxels_per_s"] = value * W.in_hw ** 3
    if incore is not None:
        line["incore"] = incore
        if W.three and incore.get("voxels_per_s"):
            line["overhead_vs_incore"] = 1.0 - line["voxels_per_s"] / incore["voxels_per_s"]
        elif incore.get("images_per_s"):
            line["overhead_vs_incore"] = 1.0 - value / incore["images_per_s"]
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_sample_3d(15.0) if W.three else cpu_sample(15.0, batch=1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pad4(x):
    import numpy as np
    out = np.zeros(x.shape[:3] + (4,), np.float32)
    out[..., :3] = x
    return out


def synth_batch(W, rank):
    """Pinned host copies of the synthetic input and labels (seed 0 + rank / 1 + rank)."""
    import numpy as np
    import torch
    import synthdata
    if W.three:
        e = W.in_hw
        x = np.zeros((e * e * e, 32), np.float32)          # 1 channel padded to 32
        x[:, 0] = synthdata.rng(0 + rank).standard_normal(e * e * e, dtype=np.float32)
        lab = synthdata.rng(1 + rank).integers(0, W.classes, e * e * e).astype(np.int32)
        return torch.from_numpy(x.reshape(-1)).pin_memory(), torch.from_numpy(lab).pin_memory()
    x = torch.from_numpy(np.ascontiguousarray(pad4(synthdata.images(W.batch, 224, 224, 3, seed=0 + rank))))
    return x.reshape(-1).pin_memory(), torch.from_numpy(synthdata.labels(W.batch, 1000, seed=1 + rank)).pin_memory()


def ctx_map_bytes(ctx):
    return [ctx.batch * l.cout * max(l.dout, 1) * l.hout * l.wout * 4 for l in ctx.layers]


def name_out_channels(ctx, pname):
    task = pname.rsplit(".", 1)[0]
    for l in ctx.layers:
        name = l.name.decode()
        if name == task or (l.kind == 9 and name.split("+", 1)[1] == task):   # 9: BNRELU_CONV "<bn>+<conv>"
            return l.cout if l.kind in (0, 9) else ((l.cout + 3) // 4 * 4)
    raise KeyError(pname)


def kernel_launches(ctx, steps):
    import ctypes as C
    from paper_1907_05013_b200._lib import lib
    v = C.c_int64()
    if hasattr(lib, "pooch_kernel_launches"):
        lib.pooch_kernel_launches(ctx.h, C.byref(v))
        return int(v.value) * steps
    return None


def tensor_peak(pk, precision):
    """Contraction roof in algorithmic FLOP/s for the precision the kernels compute in: TF32
    (bf16 sustained x the guide's nominal 1.1/2.25 ratio), or 3xTF32 = TF32 / 3 (three TF32
    MMAs per fp32 product)."""
    return pk["tf32_tflops_sustained"] * 1e12 / (3.0 if precision else 1.0)


def seg_roof(segs, pk, precision):
    """Per family: sum of launch times, of per-launch roofline times max(F / P_tensor, B / BW),
    and of the time in launches whose binding roof is the tensor pipe."""
    P, BW = tensor_peak(pk, precision), pk["hbm_gbs"] * 1e9
    out = {}
    for f, ms, fl, by in segs:
        if f in ("other", "stall", "swap_out", "swap_in", "allreduce") or ms <= 0:
            continue
        e = out.setdefault(f, {"t": 0.0, "bound": 0.0, "t_tensor": 0.0, "flops": 0.0, "bytes": 0.0})
        t = ms / 1e3
        tt, tb = fl / P, by / BW
        e["t"] += t
        e["bound"] += max(tt, tb)
        e["t_tensor"] += t if tt >= tb and fl > 0 else 0.0
        e["flops"] += fl
        e["bytes"] += by
    return out


def roofline(fam, pk, segs=None, precision=1):
    """Dominant kernel family of the instrumented step vs its roof:
    achieved / peak on the family's binding roof, plus the per-launch roofline fraction
    (sum of max(F / P_tensor, B / BW) over its launches / their measured time)."""
    sr = seg_roof(segs or [], pk, precision)
    if not sr:
        return None
    k, e = max(sr.items(), key=lambda kv: kv[1]["t"])
    tensor = e["t_tensor"] >= 0.5 * e["t"]
    P = tensor_peak(pk, precision)
    src = pk["src"] + " bf16 sustained x (1.1/2.25) nominal tf32 ratio" + (" / 3 (3xTF32)" if precision else "")
    launches = fam[k]["launches"] if k in fam else None
    if tensor:
        ach = e["flops"] / e["t"] / 1e12
        return {"kernel": k, "bound": "tensor", "achieved": ach, "peak": P / 1e12, "unit": "TFLOP/s",
                "frac": ach / (P / 1e12), "roofline_time_frac": e["bound"] / e["t"], "traffic": traffic_for(k),
                "launches": launches, "peak_src": src}
    ach = e["bytes"] / e["t"] / 1e9
    return {"kernel": k, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": ach / pk["hbm_gbs"], "roofline_time_frac": e["bound"] / e["t"], "traffic": traffic_for(k),
            "launches": launches, "peak_src": pk["src"]}


def families_table(fam, pk, segs=None, precision=1):
    """Per kernel family of the instrumented step: time, launches, achieved algorithmic
    GB/s and TFLOP/s, the binding roof (the one most of the family's launch time is bound
    by) with its fraction, and the per-launch roofline fraction."""
    out = {}
    sr = seg_roof(segs or [], pk, precision)
    P, bw = tensor_peak(pk, precision), pk["hbm_gbs"] * 1e9
    for k, v in fam.items():
        if v["ms"] <= 0:
            continue
        t = v["ms"] / 1e3
        e = {"ms": round(v["ms"], 3), "launches": v["launches"]}
        if v["bytes"] > 0:
            e["gbs"] = round(v["bytes"] / t / 1e9, 1)
        if v["flops"] > 0:
            e["tflops"] = round(v["flops"] / t / 1e12, 2)
        if k in sr:
            r = sr[k]
            tensor = r["t_tensor"] >= 0.5 * r["t"]
            e["bound"] = "tensor" if tensor else "hbm"
            e["frac"] = round((r["flops"] / r["t"] / P) if tensor else (r["bytes"] / r["t"] / bw), 4)
            e["roofline_time_frac"] = round(r["bound"] / r["t"], 4)
        out[k] = e
    return out


def traffic_for(family):
    try:
        d = json.load(open(os.path.join(HERE, "profiles", "ncu_traffic.json")))
        e = d.get(family)
        return None if e is None else e["dram_bytes_per_launch"]
    except Exception:
        return None


def swap_stats(fam, prof):
    out = {"probe_d2h_gbs": prof["d2h_gbs"], "probe_h2d_gbs": prof["h2d_gbs"], "probe_duplex_gbs": prof["duplex_gbs"]}
    for k in ("swap_out", "swap_in"):
        v = fam[k]
        out[k + "_gbs"] = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else None
        out[k + "_bytes"] = v["bytes"]
    return out


def incore_run(params_host, batch, streams, args):
    """Same kernels with every map kept: needs the full footprint in HBM. For the 3D U-Net
    (cfg4, which cannot fit) the same net at half the volume edge gives the per-voxel rate."""
    import torch
    W = workload(args)
    W.fuse = bool(args.fuse) and not W.three
    try:
        edge = W.in_hw // 2 if W.three else None
        ctx = W.context(in_hw=edge)
        ctx.set_precision(args.precision)
        need = int(ctx.resident_bytes() + sum(ctx_map_bytes(ctx)) * 1.4)
        free_now, _ = torch.cuda.mem_get_info()
        if need > free_now - (2 << 30):
            return {"images_per_s": None, "note": "in-core does not fit (%d GB needed)" % (need >> 30)}
        big = torch.empty(need // 256 * 256, dtype=torch.uint8, device="cuda")
        ctx.set_budget(big, big.numel(), None, 0)
        ctx.set_streams(*streams)
        for i, (name, numel) in enumerate(ctx.params()):
            ctx.set_param(i, params_host[i])
        if W.three:  # its own input of the smaller volume
            Wi = Workload(W.net, 1, None, W.name, edge, W.classes, W.width)
            xh, lh = synth_batch(Wi, 0)
            base = big.data_ptr()
            xp, lp = ctx.input_slot()
            big[xp - base: xp - base + xh.numel() * 4].view(torch.float32).copy_(xh)
            big[lp - base: lp - base + lh.numel() * 4].view(torch.int32).copy_(lh)
        ctx.profile(1)
        ctx.plan("incore")
        for _ in range(2):
            ctx.train_step(0.01, sync_loss=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = max(2, args.steps)
        e0.record(streams[0])
        for _ in range(n):
            ctx.train_step(0.01, sync_loss=False)
        e1.record(streams[0])
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        ctx.set_timing(True)
        ctx.train_step(0.01, sync_loss=False)
        torch.cuda.synchronize()
        fam = families_table(ctx.family_stats(), peaks(), ctx.timing_segments(), args.precision)
        ctx.set_timing(False)
        ctx.close()
        del big
        torch.cuda.empty_cache()
        out = {"images_per_s": batch * 1000.0 / ms, "ms_per_step": ms, "families": fam}
        if W.three:
            out = {"volume_edge": edge, "voxels_per_s": edge ** 3 * 1000.0 / ms, "ms_per_step": ms, "families": fam}
        return out
    except Exception as e:  # report, never fake
        return {"images_per_s": None, "note": "in-core run failed: %s" % e}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    our_arm(args)


if __name__ == "__main__":
    main()
