import torch, time
h = torch.empty(1 << 20, dtype=torch.int64).pin_memory(); d = torch.empty(1 << 20, dtype=torch.int64, device='cuda')
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(20): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); print('H2D GB/s', 20*8e6/(time.perf_counter()-t)/1e9)
t=time.perf_counter()
for _ in range(20): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print('D2H GB/s', 20*8e6/(time.perf_counter()-t)/1e9)
