import torch, time, json
n = 4 << 30  # 4 GiB
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2): d.copy_(h, non_blocking=True); torch.cuda.synchronize()
res = {}
for name in ("h2d", "d2h", "both"):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3):
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2): h2.copy_(d, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    res[name] = round(n / dt / 1e9, 1)
print(json.dumps(res))
