set -x
nvidia-smi; nvidia-smi topo -m; free -g; nproc; lscpu | head -30; numactl -H 2>/dev/null | head; cat /proc/meminfo | head -5
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for gb in (1, 4):
    n = gb << 30
    t0=time.time(); h = torch.empty(n, dtype=torch.uint8, pin_memory=True); print("pin alloc", gb, "GB s", time.time()-t0)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for i in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best=0
    for i in range(5):
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); d.copy_(h, non_blocking=True); e.record(); e.synchronize()
        best=max(best, n/ (s.elapsed_time(e)/1e3)/1e9)
    print("H2D GB/s", gb, best)
    best=0
    for i in range(5):
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); h.copy_(d, non_blocking=True); e.record(); e.synchronize()
        best=max(best, n/ (s.elapsed_time(e)/1e3)/1e9)
    print("D2H GB/s", gb, best)
    # two streams concurrent H2D halves
    s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
    torch.cuda.synchronize(); t0=time.perf_counter()
    with torch.cuda.stream(s1): d[:n//2].copy_(h[:n//2], non_blocking=True)
    with torch.cuda.stream(s2): d[n//2:].copy_(h[n//2:], non_blocking=True)
    torch.cuda.synchronize(); print("2-stream H2D GB/s", n/(time.perf_counter()-t0)/1e9)
    del h, d
PY
