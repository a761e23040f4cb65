"""cuBLAS DGEMM 16384^3 (torch.matmul, float64) for an ncu DRAM-traffic
comparison with dgemm_tma_kernel:
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -s 1 -c 1 python tools/cublas_traffic.py
"""
import torch

n = 16384
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    c = a @ b
torch.cuda.synchronize()
print("done", float(c[0, 0]))
