"""Debug (not product): pinned host <-> device copy bandwidth of the e2e arm's per-step volume
(Q, K, V, dO in; O, dQ, dK, dV out: 4 x 40960 x 32 x 128 bf16 = 1.34 GB each way), each direction
alone and both at once on two streams."""
import torch

n = 40960 * 32 * 128
hin = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
hout = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
dev = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
dev2 = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nbytes = 4 * n * 2


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def h2d():
    with torch.cuda.stream(s1):
        for d, h in zip(dev, hin):
            d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        for h, d in zip(hout, dev2):
            h.copy_(d, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.1f} ms for {nbytes / 1e9:.2f} GB per direction -> {nbytes / ms / 1e6:.1f} GB/s per direction")
