"""Replay a reference-written .att1 trace through the device selector: the native reader gathers
each step's rows for every (layer, head) into the push staging layout (ap_trace_gather_step), the
batched selector runs the evaluation loop's predictor branch on the GPU (evaluation.py:90-115:
prefill rows, then dense rows masked to each map's previous selection, dense rows on calibration
steps), and every step's middle blocks must equal those the reference recorded on the same trace
(tests/golden/trace_tiny.npz, gen_golden.py::gen_trace_fixture)."""

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_trace_replay_matches_reference_selections():
    import torch
    from paper_2502_04077_b200 import predictor
    from paper_2502_04077_b200.batched import PUSH_DENSE, PUSH_PREFILL, BatchedSelector
    from paper_2502_04077_b200.selector import SelectorConfig
    from paper_2502_04077_b200.trace import TraceReader

    d = np.load(GOLDEN / "trace_tiny.npz")
    b, bs, hist, calib, sink, local, ui = d["cfg"].tolist()
    cfg = SelectorConfig(budget=b, block_size=bs, history=hist, calibration_period=calib, sink_tokens=sink,
                         local_tokens=local, update_interval=ui)
    predictor.install_weights(predictor.PredictorWeights.from_flat(d["weights"]))
    with TraceReader(GOLDEN / "trace_tiny.att1") as r:
        h = r.header
        n_maps = h.num_layers * h.num_heads
        sel = BatchedSelector(cfg, n_maps, w_max=-(-h.total_len // bs) + 4, precision="fp16x3")
        for s in range(h.first_step_offset, 0):  # prompt rows kept for the history window
            rows = r.gather_step(s)
            sel.push_rows(torch.from_numpy(rows).cuda(), rows.shape[1], mode=PUSH_PREFILL)
        for t in range(h.num_decode_steps):
            rows = r.gather_step(t)
            sel.push_rows(torch.from_numpy(rows).cuda(), rows.shape[1], mode=PUSH_DENSE)
            sel.step()
            sel.check_status()
            for layer in range(h.num_layers):
                for head in range(h.num_heads):
                    f, o = d[f"mid_{layer}_{head}"], d[f"mid_{layer}_{head}_off"]
                    want = f[o[t]:o[t + 1]].tolist()
                    got = sorted(sel.middle(layer * h.num_heads + head))
                    assert got == want, f"step {t} (layer {layer}, head {head}): {got} != {want}"
