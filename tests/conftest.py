"""Shared test plumbing.

Markers: ``gpu`` — needs a B200 and the in-tree native library; everything
else runs on the CPU-only build container (oracle vs golden vectors, host
logic, C-ABI symbol table, gloo multi-process paths).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libattnpred.so")


def unragged(flat, off):
    return [flat[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def loop_case(name: str) -> dict:
    """A recorded reference selector run: rows, cfg, weights, per-step selections and forecasts."""
    z = load_golden(f"loop_{name}")
    heads = []
    for h in range(int(z["num_heads"])):
        heads.append({
            "prefill": unragged(z[f"prefill_{h}"], z[f"prefill_{h}_off"]),
            "decode": unragged(z[f"decode_{h}"], z[f"decode_{h}_off"]),
            "sel": unragged(z[f"sel_{h}"], z[f"sel_{h}_off"]),
            "pred": unragged(z[f"pred_{h}"], z[f"pred_{h}_off"]),
        })
    keys = ("budget", "block_size", "history", "calibration_period", "sink_tokens", "local_tokens",
            "update_interval")
    cfg = dict(zip(keys, (int(v) for v in z["cfg"])))
    return {"cfg": cfg, "weights": z["weights"], "heads": heads}


LOOP_CASES = ("h8_b256", "h64_b1024", "h16_ui4", "h64_short")


def _cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
