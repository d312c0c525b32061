import sys, time, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2407_02740_b200 import _cabi
lib = _cabi.load()
n, mp1, p, d = 1 << 20, 31, 1, 2
dev = torch.device("cuda", 0)
hn = torch.randint(0, n, (n, mp1), dtype=torch.int64).pin_memory()
hy = torch.randn(n, dtype=torch.float64).pin_memory(); hX = torch.ones((n, 1), dtype=torch.float64).pin_memory()
hl = torch.rand((n, 2), dtype=torch.float64).pin_memory()
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dy, dX, dl = hy.to(dev, non_blocking=True), hX.to(dev, non_blocking=True), hl.to(dev, non_blocking=True)
    t1 = time.perf_counter()
    dn = torch.empty((n, mp1), dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(device=dev); dn.record_stream(side)
    with torch.cuda.stream(side):
        for a in range(0, n, n // 8):
            dn[a:a + n // 8].copy_(hn[a:a + n // 8], non_blocking=True)
    t2 = time.perf_counter()
    h = ctypes.c_void_p()
    rc = lib.vb200_create(0, n, p, d, mp1, dy.data_ptr(), dX.data_ptr(), dl.data_ptr(), dn.data_ptr(), 0, n, None, ctypes.byref(h))
    t3 = time.perf_counter()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    lib.vb200_destroy(h); t5 = time.perf_counter()
    print(f"small uploads {1e3*(t1-t0):.2f}  enqueue nn {1e3*(t2-t1):.2f}  vb200_create {1e3*(t3-t2):.2f}  sync {1e3*(t4-t3):.2f}  destroy {1e3*(t5-t4):.2f}  rc={rc}")
