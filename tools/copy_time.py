import torch, time
dev = torch.device("cuda")
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
n = 314112 // 4
d = torch.empty(n, device=dev); h = torch.empty(n).pin_memory()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(100): fn()
    b.record(); torch.cuda.synchronize()
    print(name, a.elapsed_time(b) / 100 * 1000, "us per 314 KB copy")
