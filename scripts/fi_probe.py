import torch, time
import flashinfer
print(flashinfer.__version__)
T, Hq, Hkv, D = 32768, 32, 8, 128
q = torch.randn(Hq, D, device="cuda", dtype=torch.bfloat16)
k = torch.randn(Hkv, T, D, device="cuda", dtype=torch.bfloat16)
v = torch.randn(Hkv, T, D, device="cuda", dtype=torch.bfloat16)
o = flashinfer.single_decode_with_kv_cache(q, k, v, kv_layout="HND")
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(8):
        o = flashinfer.single_decode_with_kv_cache(q, k, v, kv_layout="HND")
g.replay(); torch.cuda.synchronize()
a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): g.replay()
b.record(); b.synchronize()
us = a.elapsed_time(b)*1e3/80
print("flashinfer single_decode us", us, "GB/s", Hkv*T*D*2*2/us/1e3)
# reference check
import math
ref = torch.softmax((k.float().repeat_interleave(4,0) @ q.float()[:, :, None]).squeeze(-1)/math.sqrt(D), -1)
ref = (ref[:, :, None] * v.float().repeat_interleave(4,0)).sum(1)
print("max err", (o.float()-ref).abs().max().item())
