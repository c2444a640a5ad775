import torch
from torch.profiler import profile, ProfilerActivity
for m in (8192, 16384):
    a = torch.randn(m, m, dtype=torch.bfloat16, device="cuda"); b = torch.randn(m, m, dtype=torch.bfloat16, device="cuda")
    torch.matmul(a, b); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        torch.matmul(a, b); torch.cuda.synchronize()
    for e in p.events():
        if e.device_type == torch.autograd.DeviceType.CUDA: print(m, e.name)
