"""PCIe copy ceiling on the GPU box: pinned H2D, D2H and both directions at once."""
import torch, time, json
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
h2d = timeit(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timeit(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
bo = timeit(both)
print(json.dumps({"h2d_GBs": n / h2d / 1e9, "d2h_GBs": n / d2h / 1e9, "both_each_GBs": n / bo / 1e9}))
