import torch
a = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
b = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize()
