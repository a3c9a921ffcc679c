"""Compare every ap_gemm_tc call of a batch-8 engine step with torch.matmul on the same operands."""
import torch

from paper_2502_04077_b200 import decode as Dm
from paper_2502_04077_b200.decode import DecodeEngine, ModelShape

sh = ModelShape("tiny", n_layers=2, hidden=1024, n_q_heads=8, n_kv_heads=2, ffn=2816, vocab=4096, rope_theta=5e5)
a = DecodeEngine(sh, 8, 2048, 8, mode="dense", seed=3)
orig = DecodeEngine._mm


def mm(self, x, W, y):
    orig(self, x, W, y)
    torch.cuda.synchronize()
    want = x.float() @ W.float().t()
    err = (y.float() - want).abs().max().item()
    print(tuple(W.shape), tuple(x.shape), x.is_contiguous(), x.stride(), "err", err, "max", want.abs().max().item(),
          flush=True)


DecodeEngine._mm = mm
a.tok.copy_(torch.arange(8, device="cuda"))
a.step(use_graph=False)
