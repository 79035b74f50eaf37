"""Dev probe: pinned H2D / D2H bandwidth for the e2e leg's copy patterns."""
import torch

MB = 12582912  # 8192 x 768 bf16
h = [torch.empty(MB, dtype=torch.uint8).pin_memory() for _ in range(3)]
hb = torch.empty(2 * MB, dtype=torch.uint8).pin_memory()
d = [torch.empty(MB, dtype=torch.uint8, device="cuda") for _ in range(3)]
db = torch.empty(2 * MB, dtype=torch.uint8, device="cuda")
s = [torch.cuda.Stream() for _ in range(3)]


def timeit(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    cur = torch.cuda.current_stream()
    for x in s:
        cur.wait_stream(x)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def one_big():
    with torch.cuda.stream(s[0]):
        db.copy_(hb, non_blocking=True)


def two_streams():
    for i in range(2):
        s[i].wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s[i]):
            d[i].copy_(h[i], non_blocking=True)


def big_plus_d2h():
    with torch.cuda.stream(s[0]):
        db.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s[2]):
        h[2].copy_(d[2], non_blocking=True)


def two_plus_d2h():
    two_streams()
    with torch.cuda.stream(s[2]):
        h[2].copy_(d[2], non_blocking=True)


for name, fn, by in (("one 25MB H2D", one_big, 2 * MB), ("two 12.6MB H2D streams", two_streams, 2 * MB),
                     ("one 25MB H2D + 12.6MB D2H", big_plus_d2h, 2 * MB), ("two H2D + D2H", two_plus_d2h, 2 * MB)):
    ms = timeit(fn)
    print(f"{name:30s} {ms:7.3f} ms  H2D {by / ms / 1e6:6.1f} GB/s")
