"""Pinned host <-> device copy bandwidth, each direction alone and both at
once (the e2e path's bound)."""
import torch

dev = torch.device("cuda", 0)
up = torch.empty(670_000_000 // 4, dtype=torch.float32).pin_memory()
down = torch.empty(537_000_000 // 4, dtype=torch.float32).pin_memory()
d_up = torch.empty(up.shape, dtype=torch.float32, device=dev)
d_down = torch.empty(down.shape, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


h2d = t(lambda: d_up.copy_(up, non_blocking=True))
d2h = t(lambda: down.copy_(d_down, non_blocking=True))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_up.copy_(up, non_blocking=True)
    with torch.cuda.stream(s2):
        down.copy_(d_down, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


bi = t(both)
print(f"H2D 670 MB: {h2d:.2f} ms ({670 / h2d:.1f} GB/s); D2H 537 MB: {d2h:.2f} ms ({537 / d2h:.1f} GB/s); "
      f"both at once: {bi:.2f} ms ({1207 / bi:.1f} GB/s combined)")
