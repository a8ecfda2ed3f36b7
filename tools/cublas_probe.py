import torch
A = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
B = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(3):
    C = A @ B
torch.cuda.synchronize()
