# PCIe duplex probe: H2D alone, D2H alone, both at once (pinned, 1 GiB each)
import time, torch
n = 1 << 27
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=4):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    gb = reps * n * 8 / 1e9 * (h2d + d2h)
    return gb / dt
for _ in range(2): run(1, 1)
print("H2D GB/s %.1f" % run(1, 0)); print("D2H GB/s %.1f" % run(0, 1)); print("both GB/s (sum) %.1f" % run(1, 1))
