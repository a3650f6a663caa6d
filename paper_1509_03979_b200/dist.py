"""Multi-GPU plumbing for batched recovery.

Independent problems shard across ranks (one process per GPU) in contiguous
blocks; each rank recovers its block with cs_recover_batched and the only
collective is one all-gather of fixed-size result records (support, values,
report) — NCCL over NVLink on GPUs, gloo in the CPU tests.  No data-path
collective: the recovery itself never communicates.
"""
from __future__ import annotations

from typing import Tuple


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block (b0, count) of `total` problems owned by `rank`; the first
    total % world ranks get one extra problem."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    b0 = rank * base + min(rank, extra)
    return b0, base + (1 if rank < extra else 0)


def record_bytes(K: int, value_itemsize: int, report_bytes: int = 40) -> int:
    return K * 4 + K * value_itemsize + report_bytes


def pack_records(support, values, report):
    """[B, K] int32 support, [B, K] values, [B, 40] uint8 report -> [B, rec] uint8."""
    import torch
    B = support.shape[0]
    return torch.cat([support.contiguous().view(torch.uint8).reshape(B, -1),
                      values.contiguous().view(torch.uint8).reshape(B, -1),
                      report.contiguous().reshape(B, -1)], dim=1)


def unpack_records(rec, K: int, value_dtype):
    import torch
    B = rec.shape[0]
    vs = torch.empty((), dtype=value_dtype).element_size()
    supp = rec[:, :4 * K].contiguous().view(torch.int32).reshape(B, K)
    vals = rec[:, 4 * K:4 * K + vs * K].contiguous().view(value_dtype).reshape(B, K)
    rep = rec[:, 4 * K + vs * K:].contiguous()
    return supp, vals, rep


def gather_records(rec, world: int, total: int = 0, out=None, group=None):
    """All-gather every rank's [B_r, rec] block into [total, rec] in rank order (= problem
    order for `shard`).  Blocks may differ by one problem (total % world != 0): each rank's
    block is padded to ceil(total / world) records for the collective and the padding is
    dropped afterwards.  total = 0 means world * B_r (equal blocks)."""
    import torch
    import torch.distributed as dist
    B_r, R = rec.shape
    if total <= 0:
        total = world * B_r
    per = -(-total // world)
    if B_r != per:
        pad = torch.zeros((per, R), dtype=rec.dtype, device=rec.device)
        pad[:B_r] = rec
        rec = pad
    flat = rec.contiguous().reshape(-1)
    if out is None or out.numel() != world * flat.numel():
        out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, flat, group=group)
    else:  # gloo: list form
        parts = list(out.chunk(world))
        dist.all_gather(parts, flat, group=group)
        out = torch.cat(parts)
    full = out.reshape(world, per, R)
    if per * world == total:
        return full.reshape(total, R)
    keep = [shard(total, r, world)[1] for r in range(world)]
    return torch.cat([full[r, :keep[r]] for r in range(world)])
