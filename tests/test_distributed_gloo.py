"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

* sequence sharding covers every sequence exactly once;
* KV-head split: each rank computes decode attention for its KV heads (the
  float64 oracle math stands in for the CUDA kernel, which is tested on the
  GPU), the outputs are all-gathered — by ``gather_heads`` and by the engine's
  own ``gather_heads_into`` (all_gather_into_tensor + head-major permute) — and
  the result equals the unsplit computation; the fused-QKV row slice selects exactly the rank's heads;
* max-over-ranks timing takes the slowest rank.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import attention as A


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, ret):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_04077_b200.distributed import (HeadSplit, gather_heads, gather_heads_into, max_over_ranks,
                                                       seq_shard)
        rng = np.random.default_rng(0)  # same data on every rank
        S, Hq, Hkv, D, t = 2, 8, 4, 16, 50
        qv = rng.standard_normal((S, Hq, D))
        K = rng.standard_normal((S, Hkv, t, D))
        V = rng.standard_normal((S, Hkv, t, D))
        split = HeadSplit(rank, world, Hq, Hkv)
        G = Hq // Hkv
        local = np.zeros((S, split.q_per_rank, D))
        for s in range(S):
            for i, h in enumerate(split.q_range):
                out, _, _ = A.dense_decode(qv[s, h], K[s, h // G], V[s, h // G])
                local[s, i] = out
        full = gather_heads(torch.from_numpy(local), split).numpy()
        want = np.stack([[A.dense_decode(qv[s, h], K[s, h // G], V[s, h // G])[0] for h in range(Hq)]
                         for s in range(S)])
        ok_heads = bool(np.allclose(full, want))
        # the decode engine's exchange (DecodeEngine._layer, KV-head split): all_gather_into_tensor + permute
        eng_full = gather_heads_into(torch.empty(S, Hq, D, dtype=torch.float64), torch.from_numpy(local), split)
        ok_heads = ok_heads and bool(np.allclose(eng_full.numpy(), want))
        rows = split.qkv_rows(D)
        ok_rows = len(rows) == (split.q_per_rank + 2 * split.kv_per_rank) * D and rows[0] == rank * split.q_per_rank * D
        starts = [seq_shard(7, r, world) for r in range(world)]
        cover = sorted(i for st, n in starts for i in range(st, st + n)) == list(range(7))
        slowest = max_over_ranks(float(rank + 1))
        ret.put((rank, ok_heads, ok_rows, cover, slowest))
    finally:
        dist.destroy_process_group()


def test_head_split_and_sharding_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, ret)) for r in range(2)]
    for p in procs:
        p.start()
    results = [ret.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_heads, ok_rows, cover, slowest in results:
        assert ok_heads, f"rank {rank}: gathered heads differ from the unsplit attention"
        assert ok_rows and cover
        assert slowest == 2.0


def test_seq_shard_balanced():
    from paper_2502_04077_b200.distributed import seq_shard
    for n in (1, 7, 64):
        for world in (1, 2, 4, 8):
            counts = [seq_shard(n, r, world)[1] for r in range(world)]
            assert sum(counts) == n and max(counts) - min(counts) <= 1


def test_head_split_rejects_bad_world():
    from paper_2502_04077_b200.distributed import HeadSplit
    from paper_2502_04077_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        HeadSplit(0, 3, 32, 8)
