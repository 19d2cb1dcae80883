"""Host->device bandwidth for the e2e path: torch pinned tensor vs numpy view of it."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D
dev = torch.device("cuda", 0)
n = 20000
src = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
src.fill_(1.0)
dst = torch.empty((n, n), dtype=torch.complex128, device=dev)
for name, fn in [("torch pinned copy_", lambda: dst.copy_(src, non_blocking=True)),
                 ("numpy view -> to_device", lambda: D.to_device(src.numpy().T, dev)),
                 ("from_numpy.to", lambda: torch.from_numpy(src.numpy()).to(dev))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{name:28s} {16 * n * n / dt / 1e9:7.1f} GB/s", flush=True)
out = torch.empty((2200, n), dtype=torch.complex128, device=dev)
t = time.perf_counter(); h = D.to_host(out); dt = time.perf_counter() - t
print(f"{'to_host (pageable) 704 MB':28s} {16 * n * 2200 / dt / 1e9:7.1f} GB/s")
pin = torch.empty((2200, n), dtype=torch.complex128, pin_memory=True)
t = time.perf_counter(); pin.copy_(out); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"{'D2H into pinned 704 MB':28s} {16 * n * 2200 / dt / 1e9:7.1f} GB/s")
