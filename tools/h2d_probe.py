import torch, time
for nb in (655360, 1310720, 131072, 262144):
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for k in range(30):
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
        torch.cuda.synchronize()
        if k >= 5: ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    tsd = []
    for k in range(30):
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            e0.record(s); h.copy_(d, non_blocking=True); e1.record(s)
        torch.cuda.synchronize()
        if k >= 5: tsd.append(e0.elapsed_time(e1) * 1e3)
    tsd.sort()
    print(f"{nb} B: H2D {ts[len(ts)//2]:.1f} us ({nb/ts[len(ts)//2]/1e3:.1f} GB/s), D2H {tsd[len(tsd)//2]:.1f} us")
