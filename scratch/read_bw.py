# pure-read HBM bandwidth on this B200 (torch reductions, CUDA events, L2-flushed by size):
# the ceiling a read-only streaming kernel (config 2) can reach, next to the copy-based peak
import torch
torch.cuda.set_device(0)
def bw(fn, nbytes, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(it):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / (best * 1e-3) / 1e9
for n in (1 << 24, 1 << 26, 1 << 28):
    x = torch.rand(n, device="cuda"); y = torch.rand(n, device="cuda")
    print(f"n=2^{n.bit_length()-1}: sum(x) {bw(lambda: x.sum(), 4*n):.0f} GB/s   dot(x,y) {bw(lambda: torch.dot(x, y), 8*n):.0f} GB/s   copy {bw(lambda: y.copy_(x), 8*n):.0f} GB/s")
