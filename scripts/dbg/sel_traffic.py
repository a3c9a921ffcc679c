"""One ap_sel_step on the engine's real decode state (LLaMA-3.1-8B, 32K, KV-group maps) inside an NVTX
range "sel", for `ncu --nvtx --nvtx-include sel/ --metrics dram__bytes_read.sum,dram__bytes_write.sum`."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2502_04077_b200.decode import SHAPES, DecodeEngine
from paper_2502_04077_b200.selector import SelectorConfig

group = int(sys.argv[1]) if len(sys.argv) > 1 else 4
eng = DecodeEngine(SHAPES["llama-3.1-8b"], 1, 32768, max_new=64, cfg=SelectorConfig(budget=1024), group=group)
eng.init_history()
eng.step(use_graph=False)
eng.capture_all()
for _ in range(6):
    eng.step()
eng._step_body(eng.variant_for_next(), selector=False)
torch.empty(256 << 20, dtype=torch.uint8, device="cuda").zero_()  # cold L2, as after the LM head
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("sel")
eng.sel.step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
