"""PCIe probe: page-locked H2D and D2H of one 332 MB latent, alone / concurrent, one stream vs split streams."""
import torch, time
n = 81000 * 1024
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, device="cuda")
d_b = torch.empty(n, device="cuda")


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def copies(k, up=True, down=True):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    def f():
        step = n // k
        for i in range(k):
            sl = slice(i * step, n if i == k - 1 else (i + 1) * step)
            if up:
                with torch.cuda.stream(ss[i]):
                    d_a[sl].copy_(h_in[sl], non_blocking=True)
            if down:
                with torch.cuda.stream(ss[k + i]):
                    h_out[sl].copy_(d_b[sl], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
    return f


gb = n * 4 / 1e9
for k in (1, 2, 4, 8):
    up = timed(copies(k, True, False)); dn = timed(copies(k, False, True)); both = timed(copies(k, True, True))
    print(f"streams/dir {k}: H2D {gb / up * 1e3:.1f} GB/s  D2H {gb / dn * 1e3:.1f} GB/s  both {both:.2f} ms "
          f"({2 * gb / both * 1e3:.1f} GB/s total)")
