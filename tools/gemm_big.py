"""Large square products (the SUMMA sweep sizes) against cuBLAS, with SM clock / power samples."""
import sys, torch, subprocess, threading, time
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K
def bench(fn, iters=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
def clocks():
    return subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,power.draw","--format=csv,noheader"],capture_output=True,text=True).stdout.strip()
for N in (16384, 32768):
    a = torch.randn(N, N, device="cuda").bfloat16(); b = torch.randn(N, N, device="cuda").bfloat16(); o = torch.empty(N, N, device="cuda").bfloat16()
    fl = 2.0 * N**3
    samp = []
    stop = False
    def sampler():
        while not stop:
            samp.append(clocks()); time.sleep(0.2)
    th = threading.Thread(target=sampler); th.start()
    ms = bench(lambda: K.gemm(a, b, o))
    ms2 = bench(lambda: torch.matmul(a, b, out=o))
    stop = True; th.join()
    print(f"N={N}: sg {ms:.2f} ms {fl/ms/1e9:.0f} TF/s | cublas {ms2:.2f} ms {fl/ms2/1e9:.0f} TF/s | clocks {samp[len(samp)//4]} .. {samp[-2] if len(samp)>1 else ''}", flush=True)
    del a, b, o
