import sys
import torch
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


b, s, nh, d = 32, 512, 16, 64
hb = nh * d
qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
dout = torch.randn(b * s, hb, device="cuda").bfloat16()
out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, nh, s, device="cuda")
drow = torch.empty(b, nh, s, device="cuda")
dq = torch.zeros(b * s, hb, device="cuda")
dqkv = torch.empty(b * s, 3 * hb, device="cuda", dtype=torch.bfloat16)
fl = 4.0 * b * nh * s * s * d
t = timeit(lambda: K.flash_attn_fwd(qkv, b, s, nh, d, out, lse))
print(f"flash fwd b={b} s={s} nh={nh} d={d}: {t*1e3:.1f} us, {fl/t/1e9:.1f} TF/s")
t = timeit(lambda: K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv))
print(f"flash bwd kernel: {t*1e3:.1f} us, {2.5*fl/t/1e9:.1f} TF/s")
t = timeit(lambda: K.attn_rowdot(dout, out, nh, d, s, drow))
print(f"rowdot: {t*1e3:.1f} us")
# s = 2048 (GPT-shaped heads, d = 64 slice) for the forward
b2, s2 = 4, 2048
qkv2 = torch.randn(b2 * s2, 3 * hb, device="cuda").bfloat16()
out2 = torch.empty(b2 * s2, hb, device="cuda", dtype=torch.bfloat16)
lse2 = torch.empty(b2, nh, s2, device="cuda")
fl2 = 4.0 * b2 * nh * s2 * s2 * d
t = timeit(lambda: K.flash_attn_fwd(qkv2, b2, s2, nh, d, out2, lse2))
print(f"flash fwd b={b2} s={s2} nh={nh} d={d}: {t*1e3:.1f} us, {fl2/t/1e9:.1f} TF/s")
dout2 = torch.randn(b2 * s2, hb, device="cuda").bfloat16()
drow2 = torch.empty(b2, nh, s2, device="cuda")
dq2 = torch.zeros(b2 * s2, hb, device="cuda")
dqkv2 = torch.empty(b2 * s2, 3 * hb, device="cuda", dtype=torch.bfloat16)
K.flash_attn_fwd(qkv2, b2, s2, nh, d, out2, lse2)
t = timeit(lambda: K.flash_attn_bwd(qkv2, dout2, lse2, drow2, b2, s2, nh, d, dq2, dqkv2))
print(f"flash bwd b={b2} s={s2}: {t*1e3:.1f} us, {2.5*fl2/t/1e9:.1f} TF/s")
