"""PCIe copy-rate probe (pinned host <-> device, 1.2 GB): one copy vs chunks on several streams,
and H2D + D2H concurrently.  Prints GB/s."""
import torch

n = 151_000_000  # 1.2 GB of fp64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
B = n * 8


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def chunked(dst, src, k, streams):
    m = (n + k - 1) // k
    cur = torch.cuda.current_stream()
    for i in range(k):
        s = streams[i % len(streams)]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            dst[i * m:(i + 1) * m].copy_(src[i * m:(i + 1) * m], non_blocking=True)
    for s in streams:
        cur.wait_stream(s)


ss = [torch.cuda.Stream() for _ in range(4)]
print("h2d single  GB/s", B / timed(lambda: d.copy_(h_in, non_blocking=True)) / 1e6)
print("d2h single  GB/s", B / timed(lambda: h_out.copy_(d, non_blocking=True)) / 1e6)
for k, ns in ((4, 2), (8, 4)):
    print(f"h2d {k} chunks/{ns} streams GB/s", B / timed(lambda: chunked(d, h_in, k, ss[:ns])) / 1e6)
    print(f"d2h {k} chunks/{ns} streams GB/s", B / timed(lambda: chunked(h_out, d, k, ss[:ns])) / 1e6)
a, b = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    a.wait_stream(cur)
    b.wait_stream(cur)
    with torch.cuda.stream(a):
        d.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(b):
        h_out.copy_(d2, non_blocking=True)
    cur.wait_stream(a)
    cur.wait_stream(b)


print("h2d+d2h concurrent, per direction GB/s", B / timed(both) / 1e6)
