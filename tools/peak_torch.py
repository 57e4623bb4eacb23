"""cuBLAS DGEMM sanity ceiling (torch float64 matmul), for the roofline notes only."""
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"cuBLAS DGEMM 8192^3 best: {2*8192**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
e0.record()
for _ in range(40):
    c = a @ b
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
print(f"cuBLAS DGEMM sustained x40: {40*2*8192**3/t/1e9:.2f} TFLOP/s")
L = torch.linalg.cholesky(a @ a.T / 8192 + torch.eye(8192, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
x = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2):
    y = torch.linalg.solve_triangular(L, x, upper=False)
torch.cuda.synchronize()
e0.record(); y = torch.linalg.solve_triangular(L, x, upper=False); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
print(f"cuBLAS DTRSM 8192x8192: {8192**3/t/1e9:.2f} TFLOP/s ({t:.2f} ms)")
