"""One-off GPU box probe: host RAM, CPU, PCIe link, pinned H2D bandwidth."""
import os, subprocess, time, json
out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["free"] = sh("free -g")
out["nproc"] = sh("nproc")
out["lscpu"] = sh("lscpu | head -30")
out["ulimit_l"] = sh("ulimit -l")
out["numa"] = sh("ls /sys/devices/system/node/ | grep node; cat /sys/fs/cgroup/memory.max 2>/dev/null")
out["smi"] = sh("nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max,memory.total,clocks.max.sm --format=csv")
out["topo"] = sh("nvidia-smi topo -m")
import torch
dev = torch.device("cuda:0")
res = {}
for mb in [9, 38, 75, 256, 1024]:
    n = mb * (1 << 20)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = max(2, 2048 // mb)
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res[mb] = n * reps / (ms * 1e-3) / 1e9
    del h, d
out["h2d_GBps"] = res
# D2H
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device=dev)
torch.cuda.synchronize(); t = time.time()
for _ in range(8): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); out["d2h_GBps"] = 8 * n / (time.time() - t) / 1e9
# pinned alloc speed for 8 GB
t = time.time(); big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin8GB_s"] = time.time() - t
del big
from cuda.bindings import driver as cu
cu.cuInit(0)
_, dv = cu.cuDeviceGet(0)
for a in ["CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR", "CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS", "CU_DEVICE_ATTRIBUTE_CAN_USE_HOST_POINTER_FOR_REGISTERED_MEM", "CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT", "CU_DEVICE_ATTRIBUTE_ASYNC_ENGINE_COUNT"]:
    try:
        out[a] = cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, a), dv)[1]
    except Exception as e:
        out[a] = str(e)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps(out, indent=1))
