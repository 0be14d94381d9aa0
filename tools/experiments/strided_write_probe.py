"""Does writing C (233k x 256 float32) as four strided 64-column panels cost
more DRAM time than four contiguous panels?  (hw variant 10 writes C in
column panels; the contiguous-panel probe does not.)  Writes with the L2
flushed between reps; median of 20 reps each."""
import statistics
import torch

M, N, P = 232965, 256, 64
dev = torch.device("cuda", 0)
c = torch.empty((M, N), device=dev)
src = [torch.rand((M, P), device=dev) for _ in range(N // P)]
cp = [torch.empty((M, P), device=dev) for _ in range(N // P)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn):
    ts = []
    for _ in range(20):
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def strided():
    for p in range(N // P):
        c[:, p * P:(p + 1) * P].copy_(src[p])


def contiguous():
    for p in range(N // P):
        cp[p].copy_(src[p])


for name, fn in (("strided panels", strided), ("contiguous panels", contiguous)):
    t = timed(fn)
    print(f"{name:18s} {t:.3f} ms  ({2 * M * N * 4 / t / 1e6:.0f} GB/s read+write)")
