"""One-off probe of the GPU box: host cores/RAM, PCIe link bandwidth, HBM copy."""
import os, time, json, subprocess
import torch
out = {}
out["cpu_count"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    out["meminfo"] = [l.strip() for l in f.readlines()[:4]]
with open("/proc/cpuinfo") as f:
    for l in f:
        if l.startswith("model name"):
            out["cpu_model"] = l.split(":", 1)[1].strip(); break
p = torch.cuda.get_device_properties(0)
out["gpu"] = p.name; out["sms"] = p.multi_processor_count; out["mem"] = p.total_memory
out["l2"] = getattr(p, "L2_cache_size", None)
def bw(src, dst, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): dst.copy_(src, non_blocking=True)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps): dst.copy_(src, non_blocking=True)
        e1.record(s)
    s.synchronize()
    return src.numel() * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
out["d2h_GBs_1GiB"] = bw(d, h)
out["h2d_GBs_1GiB"] = bw(h, d)
d2 = torch.empty_like(d)
out["d2d_GBs_rw"] = 2 * bw(d, d2)
t0 = time.time(); hh = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin_8GiB_s"] = time.time() - t0
try:
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
    out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,pcie.link.gen.max,pcie.link.width.max,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
    out["numa"] = subprocess.run(["bash", "-c", "lscpu | head -30"], capture_output=True, text=True).stdout
except Exception as e:
    out["err"] = str(e)
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
