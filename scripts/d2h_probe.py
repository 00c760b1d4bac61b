import time, torch
x = torch.empty(265_420_800 // 4, dtype=torch.int32, device="cuda").fill_(1)
torch.cuda.synchronize()
for kind in ("pageable", "pinned"):
    for rep in range(3):
        t0 = time.perf_counter()
        if kind == "pageable":
            y = x.cpu()
        else:
            y = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); y.copy_(x)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(kind, rep, round(dt * 1e3, 2), "ms", round(x.numel() * 4 / dt / 1e9, 1), "GB/s", flush=True)
