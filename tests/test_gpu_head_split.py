"""KV-head split through the decode engine itself, on the one B200 gpurun exposes:
two processes, each owning one of TINY's two KV heads (its q-heads, KV cache, selector maps), exchange
their per-layer attention outputs with the engine's own ``distributed.gather_heads_into`` (gloo,
host-staged here; NCCL over NVLink on a multi-GPU box) and must produce the same logits as the unsplit
engine.  Eager steps (no CUDA graphs), so no kernel of one rank waits on the other rank's kernels."""

from __future__ import annotations

import os
import socket

import pytest

pytestmark = pytest.mark.gpu

CTX, STEPS = 700, 6


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _engine(split, group):
    from paper_2502_04077_b200.decode import DecodeEngine, ModelShape
    from paper_2502_04077_b200.selector import SelectorConfig
    tiny = ModelShape("tiny", n_layers=3, hidden=512, n_q_heads=4, n_kv_heads=2, ffn=1024, vocab=1000,
                      rope_theta=10000.0)
    cfg = SelectorConfig(budget=256, calibration_period=3)  # a real selection: 8 middle blocks of ~44
    return DecodeEngine(tiny, 2, CTX, max_new=STEPS + 4, cfg=cfg, group=group, seed=3, head_split=split,
                        attn_splits=(4, 2))


def _run(eng):
    import torch
    eng.init_history()
    out = []
    for _ in range(STEPS):
        eng.step(use_graph=False)
        torch.cuda.synchronize()
        out.append(eng.logits.float().cpu())
    return out


def _worker(rank, world, port, group, ret):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_04077_b200.distributed import HeadSplit
        split = HeadSplit(rank, world, 4, 2)
        got = _run(_engine(split, group))
        if rank == 0:
            want = _run(_engine(None, group))
            worst = max(float((a - b).abs().max()) for a, b in zip(got, want))
            exact = all(torch.equal(a, b) for a, b in zip(got, want))
            ret.put((worst, exact, max(float(b.abs().max()) for b in want)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("group", [1, 2], ids=["per_head_maps", "kv_group_maps"])
def test_head_split_engine_equals_unsplit(group):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, group, ret)) for r in range(2)]
    for p in procs:
        p.start()
    worst, exact, scale = ret.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    print(f"head split vs unsplit (group={group}): worst |logit diff| = {worst} (scale {scale}), exact={exact}")
    assert exact, f"split logits differ from the unsplit engine: {worst} (scale {scale})"
