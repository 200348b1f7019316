"""Device-timeline cost of a small pinned H2D copy between two dependent
kernels (diagnostic for the upload ring)."""
import torch
torch.cuda.init()
h = torch.zeros(64, dtype=torch.float64).pin_memory()
d = torch.zeros(64, dtype=torch.float64, device='cuda')
for size in (1 << 10, 1 << 20, 1 << 23):
    x = torch.zeros(size, device='cuda')
    def run(n, with_copy):
        torch.cuda.synchronize()
        big = torch.empty(1 << 28, device='cuda'); big.add_(1)   # queue ahead: GPU-bound
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            if with_copy:
                d.copy_(h, non_blocking=True)
            x.add_(1.0)
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / n
    run(200, False)
    a = run(1000, False); b = run(1000, True)
    print(f"elems={size}: kernel only {a:.2f} us/iter, with copy {b:.2f} us/iter")
