"""Host->device bandwidth of every rank at once (torchrun, one rank per GPU), with and
without binding the process to its GPU's NUMA-local CPUs (NVML affinity) before the
pinned buffers are allocated.  Prints one line per rank and mode."""
import os
import sys

import torch
import torch.distributed as dist


def nvml_cpus(dev):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(dev)
    n = (os.cpu_count() + 63) // 64
    masks = pynvml.nvmlDeviceGetCpuAffinity(h, n)
    cpus = {w * 64 + b for w, m in enumerate(masks) for b in range(64) if m >> b & 1}
    return cpus & set(range(os.cpu_count()))


def main():
    bind = len(sys.argv) > 1 and sys.argv[1] == "bind"
    rank, lr = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr)
    if bind:
        cpus = nvml_cpus(lr)
        if cpus:
            os.sched_setaffinity(0, cpus)
    dist.init_process_group("gloo")
    n = 1600 * 1024**2 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    best = 0.0
    for _ in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print(f"rank {rank} bind={bind} cpus={len(os.sched_getaffinity(0))} H2D {best:.1f} GB/s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
