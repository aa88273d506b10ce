import torch, time
x = torch.empty(170_000_000, dtype=torch.float64).pin_memory()
y = torch.empty_like(x, device='cuda')
torch.cuda.synchronize()
for i in range(3):
    t = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"H2D 1.36GB: {dt*1e3:.1f} ms = {1.36/dt:.1f} GB/s")
import ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
t = time.perf_counter(); z = torch.empty(170_000_000, dtype=torch.float64, device='cuda'); torch.cuda.synchronize(); print("torch alloc (cached?)", (time.perf_counter()-t)*1e3)
