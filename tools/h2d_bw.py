import torch, time
n = 154140672 // 4
h = torch.rand(n).pin_memory()
d = torch.empty(n, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0) if False else s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{k} streams: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
