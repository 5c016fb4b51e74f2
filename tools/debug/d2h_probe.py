"""D2H copy probe (debug): one 20 MB device->pinned copy vs the same bytes in
pieces, and a copy overlapped with a busy kernel on another stream."""
import torch, time
dev = torch.device("cuda")
nbytes = 20119552
src = torch.empty(nbytes, dtype=torch.uint8, device=dev)
dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts) // 2]
print("one copy   %.3f ms" % timed(lambda: dst.copy_(src, non_blocking=True)))
for parts in (6, 12, 24):
    step = nbytes // parts
    def f():
        for i in range(parts):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    print(f"{parts:3d} pieces %.3f ms" % timed(f))
x = torch.randn(4096, 4096, device=dev)
def busy():
    for _ in range(3): x @ x
print("busy gemm  %.3f ms" % timed(busy))
def overlap():
    ev = torch.cuda.Event()
    with torch.cuda.stream(s1):
        busy()
    with torch.cuda.stream(s2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
print("gemm || copy %.3f ms" % timed(overlap))
