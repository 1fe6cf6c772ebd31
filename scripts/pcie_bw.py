"""Host<->device copy bandwidth on this box (pinned memory): the bound of bench.py's e2e number."""
import torch, time
n = 1_592_524_800 // 4  # the c3 batch (64 x 3 x 1080 x 1920 fp32)
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best
gb = n * 4 / 1e9
t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
t_both = timed(both)
print(f"H2D {gb / t_h2d:.1f} GB/s, D2H {gb / t_d2h:.1f} GB/s, concurrent H2D+D2H {2 * gb / t_both:.1f} GB/s "
      f"({t_both * 1e3:.1f} ms for {gb:.2f} GB each way)")

# several copy streams per direction (one DMA engine per stream may not fill PCIe Gen5)
for k in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    step = n // k

    def split():
        for i in range(k):
            with torch.cuda.stream(ss[i]):
                d_a[i * step:(i + 1) * step].copy_(h_in[i * step:(i + 1) * step], non_blocking=True)
            with torch.cuda.stream(ss[k + i]):
                h_out[i * step:(i + 1) * step].copy_(d_b[i * step:(i + 1) * step], non_blocking=True)
    t_k = timed(split)
    print(f"{k} streams per direction: concurrent {2 * gb / t_k:.1f} GB/s ({t_k * 1e3:.1f} ms)")
