"""Pure-write and copy bandwidth on this B200 (torch fill_ / copy_ over 8 GiB, CUDA events, best
of 10): the denominator for write-dominated kernels such as k_correct."""
import json

import torch

n = 2 * 1024 ** 3                      # floats (8 GiB)
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
out = {}
for name, fn, nbytes in (("write_fill", lambda: a.fill_(1.0), 4 * n), ("copy", lambda: b.copy_(a), 8 * n)):
    fn()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[name] = {"GBps": nbytes / (best / 1e3) / 1e9, "ms": best}
print(json.dumps(out))
