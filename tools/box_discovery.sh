#!/bin/bash
# One-shot box discovery: host/GPU topology + host-link microbenchmarks.
out=gpurun_out/box
mkdir -p $out
nvidia-smi -q > $out/nvidia_smi_q.txt 2>&1
nvidia-smi topo -m > $out/topo.txt 2>&1
nvidia-smi --query-gpu=index,name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,memory.total,clocks.max.sm --format=csv > $out/gpu.csv 2>&1
lscpu > $out/lscpu.txt 2>&1
nproc > $out/nproc.txt
free -g > $out/free.txt
cat /proc/meminfo > $out/meminfo.txt
numactl -H > $out/numa.txt 2>&1 || ls /sys/devices/system/node > $out/numa.txt
ulimit -a > $out/ulimit.txt
python - <<'PY' > $out/h2d.txt 2>&1
import torch, time
torch.cuda.init()
dev = torch.device('cuda:0')
for mb in [1, 8, 64, 256, 1024, 4096]:
    n = mb * 1024 * 1024
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    reps = max(3, min(50, 4096 // mb))
    s.record()
    for _ in range(reps): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3 / reps
    s.record()
    for _ in range(reps): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    t2 = s.elapsed_time(e) / 1e3 / reps
    print(f"{mb} MiB  H2D {n/t/1e9:.2f} GB/s  D2H {n/t2/1e9:.2f} GB/s")
# how much can we pin?
avail_gib = int([l for l in open('/proc/meminfo') if l.startswith('MemAvailable')][0].split()[1]) // (1 << 20)
print("MemAvailable GiB:", avail_gib)
tot = 0; bufs = []
try:
    for i in range(int(avail_gib * 0.4) // 8):
        bufs.append(torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)); tot += 8
except Exception as ex:
    print("pin stopped:", repr(ex)[:200])
print("pinned GiB ok:", tot)
PY
echo done
