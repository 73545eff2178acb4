"""PCIe probe: 1D / 2D (column-chunk) H2D and D2H rates, alone and concurrent (pinned host)."""
import torch, time
N, B = 65536, 4096
x = torch.empty((N, B), dtype=torch.float64).pin_memory()
y = torch.empty((N, B), dtype=torch.float64).pin_memory()
dx = torch.empty((N, B), dtype=torch.float64, device="cuda")
dy = torch.empty((N, B), dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = N * B * 8 / 1e9
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
for _ in range(2):
    h2d = t(lambda: dx.copy_(x, non_blocking=True))
    d2h = t(lambda: y.copy_(dy, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): dx.copy_(x, non_blocking=True)
        with torch.cuda.stream(s2): y.copy_(dy, non_blocking=True)
    bt = t(both)
    # 2D: 512-column chunk (strided host rows of 4 KB)
    c = 512
    h2d2 = t(lambda: [dx[:, i:i + c].copy_(x[:, i:i + c], non_blocking=True) for i in range(0, B, c)])
    d2h2 = t(lambda: [y[:, i:i + c].copy_(dy[:, i:i + c], non_blocking=True) for i in range(0, B, c)])
print(f"H2D 1D {gb/h2d:.1f} GB/s  D2H 1D {gb/d2h:.1f} GB/s  both-concurrent {2*gb/bt:.1f} GB/s total ({bt*1e3:.1f} ms)")
print(f"H2D 2D(512) {gb/h2d2:.1f} GB/s  D2H 2D(512) {gb/d2h2:.1f} GB/s")
