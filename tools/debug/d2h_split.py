"""D2H of a 20 MB output block: one copy vs row-part copies (debug)."""
import torch, time
dev = torch.device("cuda", 0)
n, D = 65536, 37
nbytes = n * (8 + 8 * D + 3)
src = torch.empty(nbytes, dtype=torch.uint8, device=dev)
dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
cs = torch.cuda.Stream(dev)
def one():
    dst.copy_(src, non_blocking=True)
def parts(P):
    rowf = 4 * D
    for p in range(P):
        r0, r1 = n * p // P, n * (p + 1) // P
        k = r1 - r0
        segs = [(8 * r0, 8 * k), (8 * n + rowf * r0, rowf * k), (8 * n + rowf * (n + r0), rowf * k),
                (8 * n + 2 * rowf * n + r0, k), (8 * n + 2 * rowf * n + n + r0, k),
                (8 * n + 2 * rowf * n + 2 * n + r0, k)]
        for off, b in segs:
            dst[off:off + b].copy_(src[off:off + b], non_blocking=True)
for name, f in (("one copy", one), ("2 parts x 6", lambda: parts(2)), ("4 parts x 6", lambda: parts(4))):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        f()
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name}: {ms * 1e3:.0f} us, {nbytes / ms / 1e6:.1f} GB/s")
