import torch, time
x = torch.empty(1 << 28, dtype=torch.float32).pin_memory()  # 1 GB pinned
y = torch.empty(1 << 28, dtype=torch.float32, device='cuda')
for _ in range(2):
    torch.cuda.synchronize(); t = time.time(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); print('pinned H2D GB/s', 1.0737 / (time.time() - t))
p = torch.empty(1 << 28, dtype=torch.float32)
p.fill_(1.0)
for _ in range(2):
    torch.cuda.synchronize(); t = time.time(); y.copy_(p); torch.cuda.synchronize(); print('pageable H2D GB/s', 1.0737 / (time.time() - t))
import numpy as np
a = np.ones(1 << 28, np.float32); b = x.numpy()
for _ in range(2):
    t = time.time(); np.copyto(b, a); print('host memcpy to pinned GB/s (1 thread)', 1.0737 / (time.time() - t))
