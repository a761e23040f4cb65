import ctypes as C, sys, torch
sys.path.insert(0, ".")
from paper_2203_08069_b200 import _native as nat
lib = nat.load()
torch.cuda.set_device(0)
a = torch.ones(64, 64, dtype=torch.float64, device="cuda:1"); c = torch.zeros(64, 64, dtype=torch.float64, device="cuda:1")
s1 = torch.cuda.Stream(device="cuda:1")
print("cur", torch.cuda.current_device())
for name, fn in [("fill", lambda: lib.td_fill(C.c_void_p(s1.cuda_stream), C.c_void_p(c.data_ptr()), 64, C.c_double(2.0))),
                 ("dgemm", lambda: lib.td_dgemm(C.c_void_p(s1.cuda_stream), 64, 64, 64, C.c_void_p(a.data_ptr()), 64, C.c_void_p(a.data_ptr()), 64, C.c_void_p(c.data_ptr()), 64, 0))]:
    rc = fn()
    print(name, rc, lib.td_last_error())
torch.cuda.synchronize("cuda:1")
print(c[0, :4])
