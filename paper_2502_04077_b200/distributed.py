"""Multi-GPU plumbing for the critical-token path.

The reference has no parallelism.  Every (sequence, layer,
head) forecaster state is independent and the 4833 weights are replicated, so
the path shards two ways:

* **sequence sharding** (primary, no collective): rank r decodes sequences
  ``seq_shard(n_total, r, world)``; each GPU holds its sequences' KV, history
  rings and r-maps.  ``bench.py --gpus N`` under torchrun is this mode
  (replicas, weak scaling).
* **KV-head split** (one long sequence, or to fit a large batch): rank r owns
  KV heads ``HeadSplit.kv_range`` and their q-heads, their KV cache and their
  selector maps; after attention the per-layer outputs are all-gathered over
  NCCL (NVLink) so the replicated o_proj / MLP see every head.  The gathered
  payload is n_seq x n_q_heads x 128 bf16 per layer (8 KiB per sequence for
  LLaMA-3.1-8B) — latency-bound, one collective per layer.

Both are exercised with the ``gloo`` backend on CPU in
``tests/test_distributed_gloo.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


def seq_shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced sequence range (start, count) of ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError("bad rank/world")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class HeadSplit:
    """Ownership of KV heads (and their GQA q-heads) across ``world`` ranks."""

    rank: int
    world: int
    n_q_heads: int
    n_kv_heads: int

    def __post_init__(self):
        if self.n_kv_heads % self.world:
            raise ConfigError("n_kv_heads must be divisible by the head-split world size")
        if self.n_q_heads % self.n_kv_heads:
            raise ConfigError("n_q_heads must be a multiple of n_kv_heads")

    @property
    def kv_per_rank(self) -> int:
        return self.n_kv_heads // self.world

    @property
    def q_per_rank(self) -> int:
        return self.n_q_heads // self.world

    @property
    def kv_range(self) -> range:
        return range(self.rank * self.kv_per_rank, (self.rank + 1) * self.kv_per_rank)

    @property
    def q_range(self) -> range:
        return range(self.rank * self.q_per_rank, (self.rank + 1) * self.q_per_rank)

    def qkv_rows(self, head_dim: int = 128):
        """Row indices of this rank's slice of a fused [q | k | v] projection weight."""
        q = [h * head_dim + i for h in self.q_range for i in range(head_dim)]
        k0 = self.n_q_heads * head_dim
        k = [k0 + h * head_dim + i for h in self.kv_range for i in range(head_dim)]
        v0 = k0 + self.n_kv_heads * head_dim
        v = [v0 + h * head_dim + i for h in self.kv_range for i in range(head_dim)]
        return q + k + v


def gather_heads(local_out, split: HeadSplit, group=None):
    """All-gather per-rank attention outputs [S, q_per_rank, D] -> [S, n_q_heads, D] (rank order = head order)."""
    import torch
    import torch.distributed as dist
    if split.world == 1:
        return local_out
    parts = [torch.empty_like(local_out) for _ in range(split.world)]
    dist.all_gather(parts, local_out.contiguous(), group=group)
    return torch.cat(parts, dim=1)


def gather_heads_into(out_full, local_out, split: HeadSplit, group=None):
    """The engine's per-layer exchange (decode.py, KV-head split): every rank's [S, q_per_rank, D]
    attention output -> ``out_full`` [S, n_q_heads, D] in head order.  One
    ``all_gather_into_tensor`` (a single NCCL collective over NVLink, capturable in the step's CUDA
    graph) into a rank-major buffer, then a head-major copy."""
    import torch
    import torch.distributed as dist
    if split.world == 1:
        out_full.copy_(local_out)
        return out_full
    S, hq, D = local_out.shape
    if dist.get_backend(group) == "gloo" and local_out.is_cuda:  # host-staged (CPU tests; never on the NCCL path)
        parts = torch.empty(split.world * S, hq, D, dtype=local_out.dtype)
        dist.all_gather_into_tensor(parts, local_out.contiguous().cpu(), group=group)
        parts = parts.to(local_out.device)
    else:
        parts = torch.empty(split.world * S, hq, D, dtype=local_out.dtype, device=local_out.device)  # rank-major
        dist.all_gather_into_tensor(parts, local_out.contiguous(), group=group)
    out_full.copy_(parts.view(split.world, S, hq, D).permute(1, 0, 2, 3).reshape(S, split.world * hq, D))
    return out_full


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (timing) over the default process group."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
