import os, torch
torch.cuda.init(); torch.zeros(1, device="cuda")
print("ENV", {k: v for k, v in os.environ.items() if "INJECT" in k or k.startswith("NV") or "PRELOAD" in k})
maps = open("/proc/self/maps").read()
libs = sorted({l.split()[-1] for l in maps.splitlines() if len(l.split()) >= 6 and ("nject" in l or "sanitizer" in l.lower() or "nsight" in l.lower() or "nvperf" in l.lower())})
print("MAPS", libs)
