import torch, time
n = 1 << 26
h_in = torch.empty(n * 16, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n * 24, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n * 16, dtype=torch.uint8, device='cuda')
d_out = torch.empty(n * 24, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, k=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
bo = t(both)
print(f"H2D 1 GiB {h2d:.2f} ms ({n*16/h2d/1e6:.1f} GB/s)  D2H 1.5 GiB {d2h:.2f} ms ({n*24/d2h/1e6:.1f} GB/s)  both {bo:.2f} ms")
# chunked D2H 16 MiB pieces
def chunked():
    c = 1 << 24
    for o in range(0, n * 24, c * 24):
        h_out[o:o + c * 24].copy_(d_out[o:o + c * 24], non_blocking=True)
print("chunked d2h", t(chunked))
