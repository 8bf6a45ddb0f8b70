"""Band-pruned 3-D transforms as GEMMs (cuBLAS, FP64): time of the forward
(grid -> band) and inverse (band -> grid) for 10 windows of 64^3 vs cuFFT D2Z/Z2D."""
import math

import torch

n, m, P = 64, 32, 10
h = m // 2
dev = "cuda"
g = torch.randn(P, n, n, n, dtype=torch.float64, device=dev)
z = torch.arange(n, dtype=torch.float64, device=dev)
kz = torch.arange(h, dtype=torch.float64, device=dev)
band = torch.cat([torch.arange(h), torch.arange(n - h, n)]).to(dev).double()
# forward matrices
Ez = torch.exp(-2j * math.pi * torch.outer(z, kz) / n)            # [n, h]
Dz = torch.view_as_real(Ez).reshape(n, 2 * h).contiguous()       # real [n, 2h] (re, im interleaved)
Ey = torch.exp(-2j * math.pi * torch.outer(band, z) / n)         # [m, n]
Ex = Ey.clone()                                                  # [m, n]


def forward():
    F1 = (g.reshape(P * n * n, n) @ Dz).view(P, n, n, h, 2)          # [P, x, y, kz] complex
    F1c = torch.view_as_complex(F1)                                   # [P, x, y, h]
    F2 = torch.matmul(Ey, F1c)                                        # [P, x, m(ky), h]
    F3 = torch.matmul(Ex, F2.permute(0, 2, 1, 3).reshape(P, m, n, h).permute(0, 2, 1, 3).reshape(P, n, m * h))
    return F3


def fftref():
    return torch.fft.rfftn(g, dim=(1, 2, 3))


def t(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print("rfftn 10 x 64^3 (torch / cuFFT)   us", t(fftref))
print("pruned forward as GEMMs (cuBLAS)  us", t(forward))
A = g.reshape(P * n * n, n)
print("  P1 DGEMM [40960x64]x[64x32]      us", t(lambda: A @ Dz))
F1c = torch.view_as_complex((A @ Dz).view(P, n, n, h, 2))
print("  P2 batched ZGEMM                 us", t(lambda: torch.matmul(Ey, F1c)))
