#!/usr/bin/env python
"""Benchmark of the out-of-core ResNet-50 training step (BASELINE.json metric).

Default workload (N=1): BASELINE.json config 3 -- ResNet-50 v1.5, batch 2560 at 224x224
(214 GB of feature maps, more than the B200's HBM) in all free HBM, feature maps kept,
swapped over the host link or recomputed per the PoocH plan. The timed step is one full
training iteration (forward, backward with swap-in / recompute, [allreduce], momentum SGD)
-- the whole hot path of SURVEY.md 8(a). The same run also reports:
  * the paper's own PoocH plan (one search, no grid / refinement) measured on the executor;
  * bit-exactness at the benchmarked size: one step of the adopted plan and one of another
    plan from identical parameters and batch, every gradient bit and the loss (`bitexact`),
    and that the loss is finite;
  * the in-core rate per image at batch 640 (the largest fitting batch) and the
    overhead against it;
  * the secondary cfg2 line (batch 640, 16 GiB budget: the paper's 50 GB case) with its plan
    checked bit for bit against the in-core step, under both profiling modes (all-swap
    iterations, and isolated timing) with simulated vs measured step times.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--batch B] [--budget-gib G] [--workload cfg3|cfg2|cfg4]

--workload cfg4 runs BASELINE config 4 instead: the 3D U-Net (conv3d-BN-ReLU, widths
256/512/1024/1024) at batch 1 on a 256^3 volume, whose 207 GB of maps exceed HBM; its
in-core comparison is the same net at half the edge (the per-voxel rate).

--gpus N > 1: one process per GPU (the driver's torch.distributed.run line; run by hand
without WORLD_SIZE, bench.py relaunches itself that way and fails if fewer than N GPUs are
visible). Every rank runs its own out-of-core executor on its own shard (weak scaling) with
its pinned host arena on its GPU's NUMA node and an NCCL gradient allreduce; the step time
is the max over ranks of the CUDA-event time; `ranks_identical` says whether every rank
holds the same weights afterwards. Rank 0 prints ONE JSON line.

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
METRIC_ALEX = "AlexNet images/s at a batch exceeding the device budget; overhead vs in-core; swap GB/s"
METRIC_3D = "3D U-Net volumes/s at a >HBM footprint (batch 1, 256^3); overhead vs in-core per voxel; swap GB/s"
METRIC_RX = ("ResNeXt-101 (3D) volumes/s at batch 1 with maps exceeding the device budget; overhead vs in-core at "
             "the same volume; swap GB/s")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg2", "cfg3", "cfg4", "alexnet", "resnext3d"])
    ap.add_argument("--dhw", default=None, help="resnext3d: input D x H (= W), e.g. 64x512 (default)")
    ap.add_argument("--edge", type=int, default=None, help="cfg4: volume edge (default 256)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--budget-gib", type=float, default=None)
    ap.add_argument("--li-cap", type=int, default=12)
    ap.add_argument("--no-incore", action="store_true", help="skip the in-core comparison run")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--profile-iters", type=int, default=3)
    ap.add_argument("--profile-repeats", type=int, default=3,
                    help="profiles taken; the plan uses their element-wise median (noise robustness)")
    ap.add_argument("--no-paper", action="store_true", help="skip timing the paper's own PoocH plan")
    ap.add_argument("--no-check", action="store_true", help="skip the full-size bit-exactness check")
    ap.add_argument("--no-cfg2", action="store_true", help="skip the secondary cfg2 (16 GiB) line")
    ap.add_argument("--trace", default=None,
                    help="write the plan's simulated and the instrumented step's measured timelines as one "
                         "Chrome trace (pid 0 simulated, pid 1 measured) to this path")
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
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="N > 1: gradient allreduce over peer memory (libpooch's own, default) or NCCL")
    ap.add_argument("--precision", type=int, default=1, choices=[0, 1],
                    help="contractions: 1 = 3xTF32 (default, fp32-faithful), 0 = single TF32")
    return ap.parse_args()


class Workload:
    def __init__(self, net, batch, budget, name, in_hw, classes, width=32):
        self.net, self.batch, self.budget, self.name = net, batch, budget, name
        self.in_hw, self.classes, self.width = in_hw, classes, width
        self.three = net in ("unet3d", "resnext3d")
        self.rx = net == "resnext3d"     # in_hw = H = W, width = D, input 3 -> 4 channels, one label
        self.unit = "volumes/s" if self.three else "images/s"
        self.metric = (METRIC_RX if self.rx else METRIC_3D) if self.three else (
            METRIC_ALEX if net == "alexnet" else METRIC)

    @property
    def voxels(self):
        return self.width * self.in_hw * self.in_hw if self.rx else self.in_hw ** 3

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
    if args.workload == "alexnet":
        # the largest batch whose widest task (conv1 / LRN1: input, output and both gradients,
        # 4 x 1.16 MB per image) still fits the 16 GiB budget next to the resident input slot;
        # 12.9 GB of maps plus gradients and the resident set exceed 16 GiB (in-core does not fit)
        batch = args.batch or 2560
        budget = int((args.budget_gib or 16.0) * (1 << 30))
        name = ("alexnet: AlexNet (single tower, LRN, dropout 0.5) batch %d 227^2, device budget %.0f GiB "
                "(the paper's compute-heavy workload, P:L453; SURVEY 8(f) f3)" % (batch, budget / (1 << 30)))
        return Workload("alexnet", batch, budget, name, 227, 1000)
    if args.workload == "resnext3d":
        # the paper's third workload (batch 1, inputs whose maps exceed the 16 GB
        # V100): ResNeXt-101 (3D) under a 16 GiB budget at a volume whose 207 maps take 16 GB (64 x
        # 512^2; in-core fits the B200 at the same volume -> overhead at equal work)
        d, h = (int(v) for v in (args.dhw or "64x512").split("x"))
        budget = int((args.budget_gib or 16.0) * (1 << 30))
        name = ("resnext3d: ResNeXt-101 (3D) (cardinality 32) batch 1, %d x %d x %d volume, device budget %.0f GiB "
                "(the paper's 3D workload, P:L386; SURVEY 8(f) f4)" % (d, h, h, budget / (1 << 30)))
        return Workload("resnext3d", 1, budget, name, h, 400, d)
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


def cpu_sample_alex(target_s=15.0, batch=4):
    """The oracle as it stands on AlexNet (fp64 NumPy, 227^2) on host cores."""
    import synthdata
    from oracle import nets
    cores = len(os.sched_getaffinity(0))
    net = nets.alexnet()
    params = nets.init_params(net, seed=2)
    x = synthdata.images(batch, 227, 227, 3, seed=0)
    t = synthdata.labels(batch, 1000, seed=1)
    n_img, t0 = 0, time.time()
    while True:
        nets.forward_backward(net, params, x, t)
        n_img += batch
        if time.time() - t0 > target_s:
            break
    dt = time.time() - t0
    return {"value": n_img / dt, "unit": "images/s", "cores": cores, "kind": "oracle",
            "sample": "%d fp64 AlexNet fwd+bwd step(s) at batch %d, 227^2 (NumPy, BLAS threads = cores)" % (
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


def cpu_sample_rx(target_s=15.0, dhw=(8, 32, 32)):
    """The oracle as it stands on ResNeXt-101 (3D) (fp64 NumPy) at a bounded volume: per-voxel rate."""
    import numpy as np
    import synthdata
    from oracle import nets
    cores = len(os.sched_getaffinity(0))
    net = nets.resnext3d(dhw, classes=400)
    params = nets.init_params(net, seed=2)
    g = synthdata.rng(0)
    x = g.standard_normal((1,) + tuple(dhw) + (3,))
    t = g.integers(0, 400, (1,))
    n, t0 = 0, time.time()
    while True:
        nets.forward_backward(net, params, x, t)
        n += 1
        if time.time() - t0 > target_s:
            break
    dt = time.time() - t0
    vox = int(np.prod(dhw))
    return {"value": n * vox / dt, "unit": "voxels/s", "cores": cores, "kind": "oracle",
            "sample": "%d fp64 ResNeXt-101 (3D) fwd+bwd step(s) at %dx%dx%d (NumPy, BLAS threads = cores)" % (
                (n,) + tuple(dhw))}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = workload(args)
    name = W.name
    alex = W.net == "alexnet"
    per = []
    cs = None
    for i in range(args.warmup + args.steps):
        s = cpu_sample_alex(target_s=0.0, batch=1) if alex else cpu_sample(target_s=0.0, batch=1)
        if i >= args.warmup:
            per.append(s["value"])
        cs = s
    v = statistics.median(per)
    line = {"impl": "reference", "metric": W.metric, "value": v, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name + " -- oracle sample: 1 image per step"},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": cs["cores"], "kind": "oracle",
                             "sample": "1 fp64 %s fwd+bwd image per step, %d^2" % (
                                 "AlexNet" if alex else "ResNet-50", W.in_hw)},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
class Run:
    """One out-of-core context with its arenas, streams and synthetic batch (the caller-owned
    resources of pooch_set_budget; the library never allocates device or pinned memory)."""

    def __init__(self, W, budget, host, streams, rank=0, device=0, precision=1, margin=3 << 30):
        import torch
        self.W, self.streams, self.rank = W, streams, rank
        self.ctx = W.context(device=device)
        self.ctx.set_precision(precision)
        if budget is None:
            free, _ = torch.cuda.mem_get_info()
            budget = int(free - margin)
        self.budget = budget // 256 * 256
        self.host = host
        self.dev = torch.empty(self.budget, dtype=torch.uint8, device="cuda")
        self.ctx.set_budget(self.dev, self.budget, host, host.numel() if host is not None else 0)
        self.ctx.set_streams(*streams)
        self.init_params()
        xp, lp = self.ctx.input_slot()
        self.x_host, self.l_host = synth_batch(W, rank)
        base = self.dev.data_ptr()
        self.x_dev = self.dev[xp - base: xp - base + self.x_host.numel() * 4].view(torch.float32)
        self.l_dev = self.dev[lp - base: lp - base + self.l_host.numel() * 4].view(torch.int32)
        self.put_batch()
        lo = self.ctx.loss_slot() - base
        self.loss_dev = self.dev[lo: lo + 4].view(torch.float32)

    def init_params(self):
        """Identical on every rank and every call (seed 2): He-normal fan-in weights, BN gamma 1,
        beta 0, FC bias 0; pooch_set_param also zeroes the momentum."""
        import numpy as np
        import synthdata
        g = synthdata.rng(2)
        for i, (name, numel) in enumerate(self.ctx.params()):
            if name.endswith(".w"):
                fan = numel // int(name_out_channels(self.ctx, name))
                self.ctx.set_param(i, synthdata.he_normal((numel,), fan, g))
            elif ".gamma" in name:
                self.ctx.set_param(i, np.ones(numel, np.float32))
            else:
                self.ctx.set_param(i, np.zeros(numel, np.float32))

    def put_batch(self):
        import torch
        self.x_dev.copy_(self.x_host)
        self.l_dev.copy_(self.l_host)
        torch.cuda.synchronize()

    def grads(self):
        return [self.ctx.get_param(i, 1) for i in range(len(self.ctx.params()))]

    def params_now(self):
        return [self.ctx.get_param(i, 0) for i in range(len(self.ctx.params()))]

    def close(self):
        self.ctx.close()
        self.dev = self.x_dev = self.l_dev = self.loss_dev = None


def timed(run, n_steps, world, barrier, e2e=False):
    """K steps between CUDA events on the compute stream, max over ranks. e2e: every step's input
    batch comes from pinned host memory -- H2D into a staging buffer on a side stream one step
    ahead (double buffering, the previous step still running), then a device copy into the input
    slot -- and the step's loss is read back to pinned host memory."""
    import torch
    import torch.distributed as dist
    s = run.streams[0]
    stage = None
    if e2e:
        free, _ = torch.cuda.mem_get_info()
        if free > run.x_host.numel() * 4 + (512 << 20):
            stage = (torch.empty_like(run.x_dev), torch.empty_like(run.l_dev))
            side = torch.cuda.Stream()
            staged, consumed = torch.cuda.Event(), torch.cuda.Event()
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    if stage is not None:
        side.wait_event(e0)
        with torch.cuda.stream(side):
            stage[0].copy_(run.x_host, non_blocking=True)
            stage[1].copy_(run.l_host, non_blocking=True)
        staged.record(side)
    for _ in range(n_steps):
        if e2e:
            with torch.cuda.stream(s):
                if stage is not None:      # this step's batch from the staging buffer
                    s.wait_event(staged)
                    run.x_dev.copy_(stage[0], non_blocking=True)
                    run.l_dev.copy_(stage[1], non_blocking=True)
                    consumed.record(s)
                    side.wait_event(consumed)
                    with torch.cuda.stream(side):   # next step's batch, overlapping this step
                        stage[0].copy_(run.x_host, non_blocking=True)
                        stage[1].copy_(run.l_host, non_blocking=True)
                    staged.record(side)
                else:
                    run.x_dev.copy_(run.x_host, non_blocking=True)
                    run.l_dev.copy_(run.l_host, non_blocking=True)
        run.ctx.train_step(0.01, sync_loss=False)
        if e2e:
            with torch.cuda.stream(s):
                loss_h.copy_(run.loss_dev, non_blocking=True)
    e1.record(s)
    barrier()
    ms = e0.elapsed_time(e1) / n_steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64).cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, ("double-buffered (staging %d B)" % (run.x_host.numel() * 4) if stage is not None else "serial")


def median_profile(ctx, iters, repeats):
    """`repeats` profiles, element-wise median (plan stability against measurement noise,
    VERDICT r01); the context keeps the median."""
    import numpy as np
    profs = [ctx.profile(iters) for _ in range(max(1, repeats))]
    if len(profs) == 1:
        return profs[0]
    out = dict(profs[-1])
    for k in ("fwd", "bwd", "rec", "d2h", "h2d"):
        out[k] = [int(v) for v in np.median(np.array([p[k] for p in profs]), axis=0)]
    out["tail"] = int(np.median([p["tail"] for p in profs]))
    out["spread"] = {k: float(np.max(np.std([p[k] for p in profs], axis=0) / np.maximum(1, np.mean([p[k] for p in profs], axis=0))))
                     for k in ("fwd", "bwd")}
    ctx.set_profile(out["fwd"], out["bwd"], out["rec"], out["d2h"], out["h2d"], out["tail"])
    return out


def counts_of(cls):
    return "%d/%d/%d" % (cls.count(0), cls.count(1), cls.count(2))


def plan_paper(ctx, li_cap):
    """PoocH exactly as the paper's Sec. 4.4: one search at the full budget (no plan grid, no
    refinement; DESIGN.md Readings 40, 42), retried 2 % lower only if its ledger does not pack."""
    os.environ["POOCH_PLAN_NO_GRID"] = "1"
    os.environ["POOCH_PLAN_NO_REFINE"] = "1"
    try:
        return ctx.plan("pooch", li_cap=li_cap)
    finally:
        os.environ.pop("POOCH_PLAN_NO_GRID", None)
        os.environ.pop("POOCH_PLAN_NO_REFINE", None)


def one_step_bits(run, strategy, fixed=None):
    """From the seeded parameters (momentum 0) and the resident batch: plan, one step; returns
    (classes, loss bits, gradient arrays, loss)."""
    import numpy as np
    import torch
    run.init_params()
    run.ctx.set_rng(0, 0)       # the same dropout masks for every compared step
    cls, _ = run.ctx.plan(strategy, fixed=fixed)
    loss = run.ctx.train_step(0.01, sync_loss=True)
    torch.cuda.synchronize()
    return cls, np.float32(loss).view(np.uint32), run.grads(), loss


def same_bits(a, b):
    import numpy as np
    return bool(a[1] == b[1]) and all(bool(np.array_equal(x.view(np.uint32), y.view(np.uint32)))
                                      for x, y in zip(a[2], b[2]))


def our_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1907_05013_b200 import dp
    from paper_1907_05013_b200.executor import PinnedHost

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # POOCH_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 over a gloo process group, the
    # gradients exchanged through peer.cu between processes of one GPU -- exercises the N > 1
    # path on a one-GPU box; its timings mean nothing
    share = os.environ.get("POOCH_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
        if args.comm != "peer":
            raise SystemExit("POOCH_BENCH_SHARE_GPU needs --comm peer (NCCL refuses two ranks on one GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    numa = dp.bind_host_to_gpu(local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    W = workload(args)
    W.fuse = bool(args.fuse) and not W.three
    if W.fuse:
        W.name += ", BN-ReLU prologue fusion (f2)"
    streams = [torch.cuda.Stream() for _ in range(3)]
    # pinned host arena: sized for all-swap when the host allows, else 60 % of RAM per rank
    ctx0 = W.context(device=local)
    maps_total = sum(ctx_map_bytes(ctx0))
    # the peer-memory allreduce's exchange buffer lives outside the arena: 64 KB + the gradient
    peer_reserve = (65536 + 4 * sum((n + 3) // 4 * 4 for _, n in ctx0.params())
                    if world > 1 and args.comm == "peer" else 0)
    ctx0.close()
    host_bytes = int(min(maps_total * 1.02 + (64 << 20), 0.6 * os.sysconf("SC_PAGE_SIZE") *
                         os.sysconf("SC_PHYS_PAGES") / max(1, world))) // 4096 * 4096
    while True:  # the host may cap page-locked memory: halve until registration succeeds
        try:
            host = PinnedHost(host_bytes)
            break
        except RuntimeError:
            if host_bytes < (8 << 30):
                raise
            host_bytes = host_bytes // 2 // 4096 * 4096
    budget = W.budget
    if budget is None:
        free, _ = torch.cuda.mem_get_info()
        # all free HBM minus 3 GiB of headroom, minus the e2e staging buffer (one input batch)
        budget = int(free - (3 << 30) - synth_bytes(W) - peer_reserve)
    if world > 1:  # one budget for all ranks (free HBM can differ by a few MB): identical plans
        t = torch.tensor([budget], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        budget = int(t.item())
    run = Run(W, budget, host, streams, rank, local, args.precision)
    ctx = run.ctx
    comm = None
    if world > 1 and args.comm == "nccl":
        ctx.set_comm(dp.broadcast_unique_id(rank, device="cuda"), rank, world)
        comm = ctx.comm_info()
        print("[rank %d] NCCL communicator: nranks %d, rank %d, cuda device %d, numa node %d" % (
            rank, comm[0], comm[1], comm[2], numa), file=sys.stderr, flush=True)
    elif world > 1:   # the library's own allreduce over NVLink peer memory (peer.cu)
        nb = dp.setup_peers(ctx, rank, world)
        comm = ctx.comm_info()
        print("[rank %d] peer-memory allreduce: nranks %d, rank %d, cuda device %d, exchange buffer %d B, "
              "numa node %d" % (rank, comm[0], comm[1], comm[2], nb, numa), file=sys.stderr, flush=True)

    # ---- profile (Sec. 4.2; median of --profile-repeats) + plan (Sec. 4.4); max over ranks
    t0 = time.time()
    prof = median_profile(ctx, args.profile_iters, args.profile_repeats)
    if world > 1:
        agreed = dp.agree_profile(prof, device="cuda")
        ctx.set_profile(agreed["fwd"], agreed["bwd"], agreed["rec"], agreed["d2h"], agreed["h2d"], agreed["tail"])
        ctx.set_link(agreed["d2h_gbs"], agreed["h2d_gbs"], agreed["duplex_gbs"])
        prof.update(d2h_gbs=agreed["d2h_gbs"], h2d_gbs=agreed["h2d_gbs"], duplex_gbs=agreed["duplex_gbs"])
    prof_s = time.time() - t0
    paper = None
    if not args.no_paper and world == 1:
        try:   # the paper's own PoocH (one search, no grid / refinement), measured on the executor
            pc, pr = plan_paper(ctx, args.li_cap)
            ctx.train_step(0.01, sync_loss=False)
            pms, _ = timed(run, 3, world, barrier)
            paper = {"ms_per_step": pms, "images_per_s": W.batch * 1000.0 / pms, "counts": counts_of(pc),
                     "simulated_ms": pr["makespan_ns"] / 1e6, "classes": pc}
        except Exception as e:  # infeasible is a result
            paper = {"feasible": False, "why": str(e)[:200]}
    cls, rep = ctx.plan("pooch", li_cap=args.li_cap)
    counts = {"keep": cls.count(0), "swap": cls.count(1), "recompute": cls.count(2)}
    if args.dump_profile and rank == 0:
        with open(args.dump_profile, "w") as f:
            json.dump({"workload": W.name, "batch": W.batch, "budget": run.budget, "profile": prof, "classes": cls,
                       "report": {k: (v if isinstance(v, (int, float)) else str(v)) for k, v in rep.items()}}, f)

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
    with Clocks(local) as clk:
        ms, _ = timed(run, args.steps, world, barrier)
    graph_used = ctx.step_was_graph()
    ms_e2e, e2e_mode = timed(run, max(3, args.steps // 2), world, barrier, e2e=True)
    # every rank must hold the same weights after the same steps (identical init, summed gradients)
    ident = dp.ranks_identical(dp.digest(run.params_now()))
    # instrumented step: per kernel family times (CUDA events on the launching streams)
    ctx.set_timing(True)
    ctx.train_step(0.01, sync_loss=True)
    fam = ctx.family_stats()
    segs = ctx.timing_segments()
    if args.trace and rank == 0:
        from paper_1907_05013_b200.planning import chrome_trace
        names = [l.name.decode() for l in ctx.layers]
        with open(args.trace, "w") as f:
            json.dump(chrome_trace(ctx.last_trace(simulated=True), names, 0, "simulated") +
                      chrome_trace(ctx.last_trace(), names, 1, "measured"), f)
    ctx.set_timing(False)
    launches = kernel_launches(ctx, args.steps)

    ablation = None
    if args.ablation:
        ablation = {}
        for strat in ("swap_all_naive", "swap_all", "swap_opt", "superneurons", "pooch"):
            try:
                c2, r2 = ctx.plan(strat, li_cap=args.li_cap)
            except Exception as e:  # infeasible plans are a result (superneurons OOM)
                ablation[strat] = {"feasible": False, "why": str(e)[:160]}
                continue
            ctx.train_step(0.01, sync_loss=False)
            ms_s, _ = timed(run, 2, world, barrier)
            ablation[strat] = {"feasible": True, "ms_per_step": ms_s, "images_per_s": W.batch * world * 1000.0 / ms_s,
                               "simulated_ms": r2["makespan_ns"] / 1e6, "counts": counts_of(c2)}

    # ---- correctness at the benchmarked size: one step of the adopted plan and one of another plan
    # from identical parameters and batch must agree bit for bit (north_star), and the loss is finite
    check = None
    if not args.no_check and world == 1:
        run.put_batch()
        a = one_step_bits(run, "fixed", cls)
        check = {"loss": float(a[3]), "loss_finite": bool(np.isfinite(a[3])), "plan_a": counts_of(cls)}
        alts = []
        if paper and paper.get("classes") and paper["classes"] != cls:
            alts.append(("paper PoocH", "fixed", paper["classes"]))
        alts += [("swap-opt", "swap_opt", None), ("in-core", "incore", None)]
        for name, strat, fx in alts:
            try:
                b = one_step_bits(run, strat, fx)
            except Exception:
                continue
            if b[0] == cls:
                continue
            check.update(plan_b=name + " " + counts_of(b[0]), bitexact=same_bits(a, b))
            break
        ctx.plan("pooch", li_cap=args.li_cap)

    value = W.batch * world * 1000.0 / ms
    pk = peaks()
    roof = roofline(fam, pk, segs, args.precision, W.name)
    line = {
        "metric": W.metric, "value": value, "unit": W.unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (%s tensor-core contractions, fp32 accumulate/storage)" % ("3xtf32" if args.precision else "tf32"),
        "data": "synthetic (x ~ N(0,1), labels U[0,%d), He-normal weights; seeded)" % W.classes,
        "config": {"workload": W.name, "global_batch": W.batch * world, "seq_len": None,
                   "parallelism": "dp%d" % world, "budget_bytes_per_gpu": run.budget,
                   "host_arena_bytes": host_bytes, "numa_node": numa, "l2": "inputs > L2 (maps are GBs)",
                   "profile_mode": prof.get("mode"), "profile_s": prof_s,
                   "plan_counts": counts, "planner_ms": rep["wall_ms"], "planner_sims": rep["n_sims"],
                   "simulated_ms_per_step": rep["makespan_ns"] / 1e6,
                   "arena_high_water_bytes": rep["arena_bytes"], "L_O": rep["lo_size"], "L_I": rep["li_size"]},
        "clocks": clk.summary(),
        "e2e": {"value": W.batch * world * 1000.0 / ms_e2e, "unit": W.unit, "input": e2e_mode,
                "h2d_bytes_per_step": int(run.x_host.numel() * 4 + run.l_host.numel() * 4), "d2h_bytes_per_step": 4},
        "gpu_launches": launches,
        "roofline": roof,
        "swap": swap_stats(fam, prof),
        "families": families_table(fam, peaks(), segs, args.precision),
        "ranks_identical": ident,
        "cuda_graph": graph_used,
    }
    if comm is not None:
        line["comm"] = {"kind": args.comm, "nranks": comm[0], "comm_nranks_ok": comm[0] == world}
    if paper is not None:
        line["pooch_paper"] = {k: v for k, v in paper.items() if k != "classes"}
    if check is not None:
        line["loss_finite"] = check["loss_finite"]
        line["bitexact"] = check
    if ablation is not None:
        line["ablation"] = ablation
    if W.three:
        line["voxels_per_s"] = value * W.voxels

    # ---- the in-core comparison and the secondary cfg2 line (after the arenas are released)
    if world == 1:
        run.close()
        run = ctx = None
        torch.cuda.empty_cache()
        if not args.no_incore:
            incore, cfg2 = incore_and_cfg2(W, args, host, streams)
            if incore is not None:
                line["incore"] = incore
                if W.three and incore.get("voxels_per_s"):
                    line["overhead_vs_incore"] = 1.0 - line["voxels_per_s"] / incore["voxels_per_s"]
                elif incore.get("images_per_s"):
                    line["overhead_vs_incore"] = 1.0 - value / incore["images_per_s"]
            if cfg2 is not None:
                line["cfg2"] = cfg2
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = (cpu_sample_rx(15.0) if W.rx else cpu_sample_3d(15.0) if W.three else
                                cpu_sample_alex(15.0) if W.net == "alexnet" else cpu_sample(15.0, batch=1))
    if rank == 0:
        print(json.dumps(line, default=lambda o: o.item() if hasattr(o, "item") else str(o)), flush=True)
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
    if W.rx:
        n = W.voxels
        x = np.zeros((n, 4), np.float32)                     # 3 channels padded to 4
        x[:, :3] = synthdata.rng(0 + rank).standard_normal((n, 3), dtype=np.float32)
        lab = synthdata.rng(1 + rank).integers(0, W.classes, 1).astype(np.int32)
        return torch.from_numpy(x.reshape(-1)).pin_memory(), torch.from_numpy(lab).pin_memory()
    if W.three:
        e = W.in_hw
        x = np.zeros((e * e * e, 32), np.float32)          # 1 channel padded to 32
        x[:, 0] = synthdata.rng(0 + rank).standard_normal(e * e * e, dtype=np.float32)
        lab = synthdata.rng(1 + rank).integers(0, W.classes, e * e * e).astype(np.int32)
        return torch.from_numpy(x.reshape(-1)).pin_memory(), torch.from_numpy(lab).pin_memory()
    x = torch.from_numpy(np.ascontiguousarray(pad4(synthdata.images(W.batch, W.in_hw, W.in_hw, 3, seed=0 + rank))))
    return x.reshape(-1).pin_memory(), torch.from_numpy(synthdata.labels(W.batch, 1000, seed=1 + rank)).pin_memory()


def ctx_map_bytes(ctx):
    return [ctx.batch * l.cout * max(l.dout, 1) * l.hout * l.wout * 4 for l in ctx.layers]


def name_out_channels(ctx, pname):
    task = pname.rsplit(".", 1)[0]
    for l in ctx.layers:
        name = l.name.decode()
        if name == task or (l.kind == 9 and name.split("+", 1)[1] == task):   # 9: BNRELU_CONV "<bn>+<conv>"
            return l.cout if l.kind in (0, 9, 10, 12) else ((l.cout + 3) // 4 * 4)
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


def alu_peak():
    """FP32 FMA roof of the CUDA cores (grouped conv3d, DESIGN.md Reading 47): 148 SMs x 128 FMA
    lanes x 2 flop x the SM clock (the boost clock, 1.965 GHz; B200_PROFILING.md unit counts)."""
    return 148 * 128 * 2 * 1.965e9


def seg_roof(segs, pk, precision):
    """Per family: sum of launch times, of per-launch roofline times max(F / P, B / BW) -- P the
    tensor roof, or the ALU roof for the grouped-conv families -- and of the time in launches
    whose binding roof is the compute pipe."""
    BW = pk["hbm_gbs"] * 1e9
    out = {}
    for f, ms, fl, by in segs:
        if f in ("other", "stall", "swap_out", "swap_in", "allreduce") or ms <= 0:
            continue
        P = alu_peak() if f.startswith("gconv") else tensor_peak(pk, precision)
        e = out.setdefault(f, {"t": 0.0, "bound": 0.0, "t_tensor": 0.0, "flops": 0.0, "bytes": 0.0})
        t = ms / 1e3
        tt, tb = fl / P, by / BW
        e["t"] += t
        e["bound"] += max(tt, tb)
        e["t_tensor"] += t if tt >= tb and fl > 0 else 0.0
        e["flops"] += fl
        e["bytes"] += by
    return out


def roofline(fam, pk, segs=None, precision=1, workload=""):
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
    if tensor and k.startswith("gconv"):
        ach = e["flops"] / e["t"] / 1e12
        return {"kernel": k, "bound": "alu", "achieved": ach, "peak": alu_peak() / 1e12, "unit": "TFLOP/s",
                "frac": ach / (alu_peak() / 1e12), "roofline_time_frac": e["bound"] / e["t"],
                "traffic": traffic_for(k, workload), "launches": launches,
                "peak_src": "148 SMs x 128 FP32 FMA/clk x 2 x 1.965 GHz (B200_PROFILING.md unit counts)"}
    if tensor:
        ach = e["flops"] / e["t"] / 1e12
        return {"kernel": k, "bound": "tensor", "achieved": ach, "peak": P / 1e12, "unit": "TFLOP/s",
                "frac": ach / (P / 1e12), "roofline_time_frac": e["bound"] / e["t"], "traffic": traffic_for(k, workload),
                "launches": launches, "peak_src": src}
    ach = e["bytes"] / e["t"] / 1e9
    return {"kernel": k, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": ach / pk["hbm_gbs"], "roofline_time_frac": e["bound"] / e["t"], "traffic": traffic_for(k, workload),
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
            alu = k.startswith("gconv")
            e["bound"] = ("alu" if alu else "tensor") if tensor else "hbm"
            Pk = alu_peak() if alu else P
            e["frac"] = round((r["flops"] / r["t"] / Pk) if tensor else (r["bytes"] / r["t"] / bw), 4)
            e["roofline_time_frac"] = round(r["bound"] / r["t"], 4)
        out[k] = e
    return out


def traffic_for(family, workload=""):
    """DRAM bytes per launch of `family` from the committed ncu capture of the same workload
    (profiles/ncu_traffic.json), else None."""
    try:
        d = json.load(open(os.path.join(HERE, "profiles", "ncu_traffic.json")))
        e = d.get(family)
        if e is None or not workload.startswith(e.get("workload", "?")):
            return None
        return e["dram_bytes_per_launch"]
    except Exception:
        return None


def swap_stats(fam, prof):
    out = {"probe_d2h_gbs": prof["d2h_gbs"], "probe_h2d_gbs": prof["h2d_gbs"], "probe_duplex_gbs": prof["duplex_gbs"]}
    # the planner's shared-link model (DESIGN.md Reading 51; executor make_problem): each direction's
    # rate while both copy lanes are busy, per mille of its one-way rate
    if prof["duplex_gbs"] > 0 and prof["d2h_gbs"] > 0 and prof["h2d_gbs"] > 0 and os.environ.get("POOCH_DUPLEX", "1") != "0":
        out["link_model_permille"] = {"d2h": max(1, min(1000, int(1000 * prof["duplex_gbs"] / prof["d2h_gbs"]))),
                                      "h2d": max(1, min(1000, int(1000 * prof["duplex_gbs"] / prof["h2d_gbs"])))}
    else:
        out["link_model_permille"] = None
    for k in ("swap_out", "swap_in"):
        v = fam[k]
        out[k + "_gbs"] = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else None
        out[k + "_bytes"] = v["bytes"]
    return out


def incore_and_cfg2(W, args, host, streams):
    """The same kernels with every map kept, at the largest batch that fits (the paper's per-image
    convention): ResNet-50 at batch 640, the 3D U-Net at half the volume edge. For ResNet-50
    also the secondary cfg2 line (BASELINE config 2: batch 640 under a 16 GiB budget): one step
    of its plan against the in-core step from identical parameters and batch (bit-exact at the
    full benchmarked size, north_star), and the plan from each profiling mode (Sec. 4.2, all-swap
    iterations vs isolated timing) with its simulated and measured step time."""
    import numpy as np
    import torch
    if W.rx:   # in-core fits at the benchmarked volume: the same step, every map kept
        Wi = Workload(W.net, 1, None, "in-core " + W.name.split(",")[0], W.in_hw, W.classes, W.width)
    elif W.three:
        Wi = Workload(W.net, 1, None, W.name, W.in_hw // 2, W.classes, W.width)
    elif W.net == "alexnet":   # in-core fits at the benchmarked batch: the same step, every map kept
        Wi = Workload(W.net, W.batch, None, "in-core AlexNet batch %d" % W.batch, W.in_hw, W.classes)
    else:
        Wi = Workload(W.net, 640, None, "in-core ResNet-50 v1.5 batch 640", 224, W.classes)
    Wi.fuse = W.fuse
    incore, cfg2 = None, None
    try:
        probe = Wi.context()
        need = int(probe.resident_bytes() + sum(ctx_map_bytes(probe)) * 1.4)
        probe.close()
        free_now, _ = torch.cuda.mem_get_info()
        if need > free_now - (2 << 30):
            return {"images_per_s": None, "note": "in-core does not fit (%d GB needed)" % (need >> 30)}, None
        ri = Run(Wi, need, None, streams, precision=args.precision)
        ri.ctx.set_profile_mode("isolated")
        ri.ctx.profile(1)
        ref = one_step_bits(ri, "incore")
        for _ in range(2):
            ri.ctx.train_step(0.01, sync_loss=False)
        ms, _ = timed(ri, max(3, args.steps // 2), 1, torch.cuda.synchronize)
        graph_in = ri.ctx.step_was_graph()
        ri.ctx.set_timing(True)
        ri.ctx.train_step(0.01, sync_loss=False)
        torch.cuda.synchronize()
        fam = families_table(ri.ctx.family_stats(), peaks(), ri.ctx.timing_segments(), args.precision)
        ri.ctx.set_timing(False)
        if W.three:
            e = Wi.in_hw
            incore = {"volume_edge": e, "voxels_per_s": Wi.voxels * 1000.0 / ms, "ms_per_step": ms, "families": fam,
                      "cuda_graph": graph_in}
            if W.rx:
                incore = {"volume": [Wi.width, e, e], "volumes_per_s": 1000.0 / ms,
                          "voxels_per_s": Wi.voxels * 1000.0 / ms, "ms_per_step": ms, "families": fam,
                          "cuda_graph": graph_in}
            ri.close()
            return incore, None
        incore = {"batch": Wi.batch, "images_per_s": Wi.batch * 1000.0 / ms, "ms_per_step": ms, "families": fam,
                  "cuda_graph": graph_in}
        if not args.no_cfg2 and W.net == "resnet50":
            W2 = Workload("resnet50", 640, 16 << 30, "cfg2: ResNet-50 v1.5 batch 640 224^2, device budget 16 GiB",
                          224, W.classes)
            W2.fuse = W.fuse
            r2 = Run(W2, W2.budget, host, streams, precision=args.precision)
            cfg2 = {"workload": W2.name}
            for mode in ("auto", "isolated"):
                r2.ctx.set_profile_mode(mode)
                r2.init_params()
                prof = r2.ctx.profile(args.profile_iters)
                cls, rep = r2.ctx.plan("pooch", li_cap=args.li_cap)
                for _ in range(2):
                    r2.ctx.train_step(0.01, sync_loss=False)
                ms2, _ = timed(r2, max(3, args.steps // 2), 1, torch.cuda.synchronize)
                e = {"profile_mode": prof["mode"], "images_per_s": 640 * 1000.0 / ms2, "ms_per_step": ms2,
                     "simulated_ms_per_step": rep["makespan_ns"] / 1e6, "plan_counts": counts_of(cls),
                     "overhead_vs_incore": 1.0 - (640 * 1000.0 / ms2) / incore["images_per_s"]}
                if mode == "auto":   # per kernel family, against the in-core step's (same batch)
                    r2.ctx.set_timing(True)
                    r2.ctx.train_step(0.01, sync_loss=False)
                    torch.cuda.synchronize()
                    e["families"] = families_table(r2.ctx.family_stats(), peaks(), r2.ctx.timing_segments(),
                                                   args.precision)
                    r2.ctx.set_timing(False)
                if prof["mode"] == "all_swap":
                    e["all_swap_profile_step_ms"] = prof["step_ns"] / 1e6
                r2.put_batch()
                b = one_step_bits(r2, "fixed", cls)
                e["loss_finite"] = bool(np.isfinite(b[3]))
                e["bitexact_vs_incore"] = same_bits(b, ref)
                if mode == "auto":
                    cfg2.update(e)
                else:
                    cfg2["isolated_profile"] = e
            r2.close()
        ri.close()
    except Exception as e:  # report, never fake
        incore = incore or {"images_per_s": None, "note": "in-core run failed: %s" % str(e)[:200]}
        if cfg2 is not None:
            cfg2["error"] = str(e)[:200]
    torch.cuda.empty_cache()
    return incore, cfg2


def synth_bytes(W):
    """Bytes of one input batch (+ labels) as the GPU stores it (the e2e staging buffer)."""
    if W.rx:
        return W.voxels * 4 * 4 + 4
    if W.three:
        return W.in_hw ** 3 * (32 + 1) * 4
    return W.batch * (W.in_hw * W.in_hw * 4 + 1) * 4


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # the driver launches N > 1 under torch.distributed.run; run by hand, relaunch the same way
        import torch
        from paper_1907_05013_b200.dp import relaunch_argv
        have = torch.cuda.device_count()
        if have < args.gpus and os.environ.get("POOCH_BENCH_SHARE_GPU") != "1":
            print("bench.py --gpus %d needs %d visible GPUs, found %d" % (args.gpus, args.gpus, have),
                  file=sys.stderr, flush=True)
            sys.exit(2)
        port = 29500 + os.getpid() % 1000
        sys.exit(subprocess.call(relaunch_argv(os.path.abspath(__file__), sys.argv[1:], args.gpus, port)))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print("bench.py: WORLD_SIZE %s != --gpus %d" % (os.environ["WORLD_SIZE"], args.gpus), file=sys.stderr)
        sys.exit(2)
    our_arm(args)


if __name__ == "__main__":
    main()
