"""Reference copy rates for the condensation's dense blocks (torch kernels, CUDA
events, L2 flushed): the M_yx = J_d block copy into the ldm-strided M and a flat
copy of the same bytes."""
import torch

n_d, m = 4096, 4096
N = n_d + m
M = torch.empty((N, N), dtype=torch.float64, device="cuda")      # row-major view of col-major M (ld = N)
Jd = torch.randn((n_d, m), dtype=torch.float64, device="cuda")    # col-major J_d as rows = columns
H = torch.randn((n_d, n_d), dtype=torch.float64, device="cuda")
flat_a = torch.empty(2 * n_d * m // 2 * 3 // 2, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        flush.zero_()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return sorted(ts)[len(ts) // 2]


def blocks():
    M[:n_d, n_d:].copy_(Jd)      # columns j < n_d of col-major M, rows n_d.. : M^T view
    M[:n_d, :n_d].copy_(H)


nbytes = 2 * 8 * (n_d * m + n_d * n_d)
ms = t(blocks)
print(f"torch block copies (J_d + full H_dd -> M): {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s")
src = torch.empty(nbytes // 16, dtype=torch.float64, device="cuda")
dst = torch.empty_like(src)
ms = t(lambda: dst.copy_(src))
print(f"flat copy of the same bytes: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s")
