"""One-off box probe: host RAM/cores, PCIe pinned bandwidth, TF32 matmul peak."""
import os, time, json, subprocess
import torch
out = {}
out["cores"] = len(os.sched_getaffinity(0))
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["nvsmi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,memory.free,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max", "--format=csv"], capture_output=True, text=True).stdout
out["numa"] = subprocess.run(["bash", "-c", "nvidia-smi topo -m; lscpu | head -30"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
torch.cuda.init()
free, total = torch.cuda.mem_get_info()
out["mem_get_info"] = [free, total]
# pinned bandwidth sweep
res = {}
for sz in [1 << 20, 16 << 20, 256 << 20, 1 << 30]:
    h = torch.empty(sz, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(sz, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for direction in ["h2d", "d2h"]:
        with torch.cuda.stream(s):
            for _ in range(2):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            n = 5
            for _ in range(n):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            e1.record(s)
        s.synchronize()
        res[f"{direction}_{sz}"] = sz * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    # duplex
    h2 = torch.empty(sz, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(sz, dtype=torch.uint8, device=dev)
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s.wait_event(e0); s2.wait_event(e0)
    with torch.cuda.stream(s):
        for _ in range(5): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(5): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    res[f"duplex_each_{sz}"] = sz * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del h, d, h2, d2
out["link_gbs"] = res
# big pinned alloc test
t0 = time.time()
try:
    big = torch.empty(64 << 30, dtype=torch.uint8, pin_memory=True)
    out["pin64g_s"] = time.time() - t0
    del big
except Exception as e:
    out["pin64g_err"] = str(e)
# tf32 peak
torch.backends.cuda.matmul.allow_tf32 = True
a = torch.randn(8192, 8192, device=dev); b = torch.randn(8192, 8192, device=dev)
for _ in range(3): a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
out["tf32_tflops_burst"] = 2 * 8192**3 / (best * 1e-3) / 1e12
t_end = time.time() + 4; n = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() < t_end:
    for _ in range(20): c = a @ b
    n += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
out["tf32_tflops_sustained"] = 2 * 8192**3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
