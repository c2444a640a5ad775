import torch, time
n = 2 * 1024**3 // 8
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
ho = torch.empty(n, dtype=torch.float64).pin_memory()
do = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); torch.cuda.synchronize(); e1.record(); e1.synchronize(); return e0.elapsed_time(e1)
for _ in range(2):
    a = t(lambda: [d[i].copy_(h[i], non_blocking=True) for i in range(3)])
    b = t(lambda: ho.copy_(do, non_blocking=True))
    def both():
        with torch.cuda.stream(s1):
            for i in range(3): d[i].copy_(h[i], non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
    c = t(both)
    print(f"H2D 6.4GB {a:.1f} ms ({6.44e9/a/1e6:.1f} GB/s)  D2H 2.1GB {b:.1f} ms ({2.15e9/b/1e6:.1f} GB/s)  both {c:.1f} ms")
