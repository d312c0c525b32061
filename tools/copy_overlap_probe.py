import time, numpy as np, torch
n, mp1 = 1 << 20, 31
hn = torch.randint(0, n, (n, mp1), dtype=torch.int64).pin_memory()
view = torch.from_numpy(hn.numpy())           # non-owning view of pinned memory, as the engine sees it
print("pinned view:", view.is_pinned())
dev = torch.device("cuda", 0)
def t(): torch.cuda.synchronize(); return time.perf_counter()
for src, name in ((hn, "owning pinned tensor"), (view, "from_numpy view of pinned memory")):
    for rep in range(3):
        d = torch.empty((n, mp1), dtype=torch.int64, device=dev)
        side = torch.cuda.Stream(device=dev)
        t0 = t()
        with torch.cuda.stream(side):
            for a in range(0, n, n // 8):
                d[a:a + n // 8].copy_(src[a:a + n // 8], non_blocking=True)
        t1 = time.perf_counter()
        torch.cuda.synchronize(); t2 = time.perf_counter()
        print(f"{name}: enqueue {1e3*(t1-t0):.2f} ms, complete {1e3*(t2-t0):.2f} ms")
