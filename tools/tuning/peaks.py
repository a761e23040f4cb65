import torch, time, subprocess, json
torch.cuda.init()
d = torch.device("cuda:0")
def timeit(fn, it=10):
    fn(); torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(it):
        s.record(); fn(); e.record(); e.synchronize(); best=min(best, s.elapsed_time(e))
    return best
res={}
for n in (4096, 8192, 16384):
    a=torch.randn(n,n,dtype=torch.float64,device=d); b=torch.randn(n,n,dtype=torch.float64,device=d)
    ms=timeit(lambda: torch.matmul(a,b), 5 if n==16384 else 10)
    res[f"dgemm_{n}_tflops"]=2*n**3/ms/1e9
    print(n, ms, 2*n**3/ms/1e9, flush=True)
# sustained 4 s dgemm 8192
n=8192
a=torch.randn(n,n,dtype=torch.float64,device=d); b=torch.randn(n,n,dtype=torch.float64,device=d)
p=subprocess.Popen("nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 200 > gpurun_out/dgemm_clocks.csv", shell=True)
t0=time.time(); cnt=0
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True); s.record()
while time.time()-t0<4:
    torch.matmul(a,b); cnt+=1
    if cnt%4==0: torch.cuda.synchronize()
e.record(); e.synchronize(); p.terminate()
res["dgemm_8192_sustained_tflops"]=cnt*2*n**3/s.elapsed_time(e)/1e9
print(res, flush=True)
x=torch.empty(2**30//8*8, dtype=torch.float64, device=d); y=torch.empty_like(x)
ms=timeit(lambda: y.copy_(x))
res["copy_gbs"]=2*x.numel()*8/ms/1e6
print(res)
json.dump(res, open("gpurun_out/peaks.json","w"))
