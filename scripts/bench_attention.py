"""Micro-benchmark of the decode-attention kernels at the bench shape (LLaMA-3.1-8B layer, 32K).

sparse: one layer's selection (sink + local + 56 middle blocks per map), with emission;
dense:  full attention (output) and the K-only calibration pass.
Reports µs per launch (CUDA events, warm L2 excluded by rotating 8 layers' KV) and GB/s of
algorithmic bytes (selected K+V blocks, or all K[+V]).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_04077_b200.attention import DecodeAttention  # noqa: E402
from paper_2502_04077_b200.batched import BatchedSelector  # noqa: E402
from paper_2502_04077_b200.selector import SelectorConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, default=32768)
    ap.add_argument("--group", choices=["head", "kv"], default="kv")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--splits", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dense-splits", type=int, default=0, help="0: attention.dense_splits rule")
    args = ap.parse_args()
    S, Hq, Hkv, L = args.batch, 32, 8, args.layers
    t_max = -(-(args.t + 16) // 1024) * 1024
    G = 1 if args.group == "head" else Hq // Hkv
    maps = Hq // G
    k = torch.randn(L, S, Hkv, t_max, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(L, S, Hkv, t_max, 128, device="cuda", dtype=torch.bfloat16)
    q = torch.randn(S, Hq, 128, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(S, Hq, 128, device="cuda", dtype=torch.bfloat16)
    seq_len = torch.full((S,), args.t, dtype=torch.int32, device="cuda")
    cfg = SelectorConfig(budget=1024)
    sel = BatchedSelector(cfg, S * L * maps, t_max // 16)
    rng = np.random.default_rng(0)
    st = sel.states().copy()
    W = -(-args.t // 16)
    for m in range(S * L * maps):
        blk = sorted(rng.choice(np.arange(4, W - 6), cfg.middle_blocks, replace=False).tolist())
        st[m]["n_mid"] = len(blk)
        st[m]["mid_clip"] = args.t - 1
        sel.mid_blocks[m, : len(blk)] = torch.tensor(blk, dtype=torch.int32)
    sel.state.copy_(torch.from_numpy(st.view(np.uint8).copy()))
    from paper_2502_04077_b200 import _lib
    from paper_2502_04077_b200.attention import dense_splits
    nsd = args.dense_splits or dense_splits(S * Hkv, _lib.fn("ap_device_sm_count")(), t_max)
    att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_dense=nsd, n_splits_sparse=args.splits)

    def timeit(fn):
        """GPU time per launch: the L launches (one per layer) captured in a CUDA graph, replayed."""
        for i in range(L):
            fn(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(L):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
        for i in range(args.reps):
            ev[i][0].record()
            g.replay()
            ev[i][1].record()
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) * 1e3 for a, b in ev])) / L

    res = {}
    n_units = 4 + 5 + cfg.middle_blocks
    sparse_bytes = S * (maps * n_units * 4096 * 2 if G > 1 else Hq * n_units * 4096 * 2)
    res["sparse_emit_us"] = timeit(lambda l: att.sparse(q, k[l], v[l], seq_len, out, sel, emit=True, map_base=l * maps,
                                                         maps_per_seq=L * maps, group=G))
    res["sparse_noemit_us"] = timeit(lambda l: att.sparse(q, k[l], v[l], seq_len, out, sel, emit=False,
                                                           map_base=l * maps, maps_per_seq=L * maps, group=G))
    res["sparse_GBps"] = sparse_bytes / (res["sparse_noemit_us"] * 1e-6) / 1e9
    dense_bytes = S * Hkv * args.t * 256 * 2
    res["dense_us"] = timeit(lambda l: att.dense(q, k[l], v[l], seq_len, out, with_v=True))
    res["dense_GBps"] = dense_bytes / (res["dense_us"] * 1e-6) / 1e9
    res["calib_us"] = timeit(lambda l: att.dense(q, k[l], k[l], seq_len, None, with_v=False, emit=True, selector=sel,
                                                 map_base=l * maps, maps_per_seq=L * maps, group=G))
    res["calib_GBps"] = dense_bytes / 2 / (res["calib_us"] * 1e-6) / 1e9
    res.update(batch=S, dense_splits=nsd, t=args.t, group=args.group, sparse_bytes=sparse_bytes, dense_bytes=dense_bytes)
    print(json.dumps({k_: (round(v_, 2) if isinstance(v_, float) else v_) for k_, v_ in res.items()}))


if __name__ == "__main__":
    main()
