import time, ctypes as C
cr = C.CDLL("libcudart.so.12") if False else None
import torch
torch.cuda.init(); torch.cuda.synchronize()
cudart = C.CDLL(torch._C.__file__.replace('_C.cpython-312-x86_64-linux-gnu.so','lib/libcudart.so.12')) if False else None
from cuda.bindings import runtime as rt
for gb in (1, 10, 45):
    t0=time.perf_counter(); err, p = rt.cudaMalloc(int(gb*1e9)); t1=time.perf_counter()
    rt.cudaMemset(p, 0, int(gb*1e9)); rt.cudaDeviceSynchronize(); t2=time.perf_counter()
    rt.cudaMemset(p, 0, int(gb*1e9)); rt.cudaDeviceSynchronize(); t3=time.perf_counter()
    rt.cudaFree(p); t4=time.perf_counter()
    print(f"{gb} GB: malloc {1e3*(t1-t0):.1f} ms, first memset {1e3*(t2-t1):.1f} ms, second memset {1e3*(t3-t2):.1f} ms, free {1e3*(t4-t3):.1f} ms", flush=True)
# many chunks
t0=time.perf_counter(); ps=[rt.cudaMalloc(int(2e9))[1] for _ in range(20)]; t1=time.perf_counter()
print(f"20 x 2 GB malloc {1e3*(t1-t0):.1f} ms")
