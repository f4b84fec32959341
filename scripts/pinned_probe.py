"""Dev aid: H2D bandwidth of pinned host buffers by allocation time/method."""
import os, sys, time
import numpy as np
import torch

N = 64 << 20
cudart = torch.cuda.cudart()
d = torch.empty(N, dtype=torch.uint8, device="cuda")


def bw(tag, t):
    for _ in range(3):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    print(f"{tag:50s} {N / ((time.perf_counter() - t0) / 10) / 1e9:6.1f} GB/s", flush=True)


a = torch.empty(N, dtype=torch.uint8).pin_memory()
bw("torch pin #1", a)
b = torch.empty(N, dtype=torch.uint8).pin_memory()
bw("torch pin #2", b)
c = torch.empty(N, dtype=torch.uint8).pin_memory()
bw("torch pin #3", c)
x = np.ones(N, dtype=np.uint8)
cudart.cudaHostRegister(x.ctypes.data, N, 0)
bw("numpy + cudaHostRegister", torch.from_numpy(x))
y = np.ones(N + 4096, dtype=np.uint8)
cudart.cudaHostRegister(y.ctypes.data, N, 0)
bw("numpy + cudaHostRegister #2", torch.from_numpy(y[:N]))
big = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(8)]
for i, t in enumerate(big):
    bw(f"torch pin batch #{i}", t)
regs = []
for i in range(8):
    z = np.ones(N, dtype=np.uint8)
    cudart.cudaHostRegister(z.ctypes.data, N, 0)
    regs.append(z)
    bw(f"numpy(THP) + cudaHostRegister batch #{i}", torch.from_numpy(z))
