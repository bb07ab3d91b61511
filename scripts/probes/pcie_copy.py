import torch, time
n = 133432831
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("H2D GB/s", n * 8 / e0.elapsed_time(e1) / 1e6)
e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H GB/s", n * 8 / e0.elapsed_time(e1) / 1e6)
