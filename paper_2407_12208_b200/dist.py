"""Host-side logic of the point-sharded multi-GPU path.

One process per GPU. Rows are split into contiguous shards; the library's handles
(kmeans_create_dist) own an NCCL communicator created from a unique id that rank 0 generates and
this module broadcasts over the torch.distributed process group. Per Lloyd iteration the library
exchanges, with fp32 work (the exact fixed-point update, R9), the int64 totals of the
grid integers (two k*d arrays) and the int32 counts in one NCCL group, plus [SSE_t, #changed] in
fp64; with fp64 work one fp64 allreduce of the packed buffer
    [ sums (k*d) | counts (k) | SSE_t | #changed | reserved (2) ]
(AccLayout in csrc/internal.h). Every rank then finalises identical centroids. The same exchange
can run between virtual ranks on one GPU (kmeans_vgroup_create / kmeans_create_virtual).
This module only moves bytes and indices; every numeric step runs in the CUDA library.
"""
from __future__ import annotations

import torch
import torch.distributed as tdist

NCCL_ID_BYTES = 128


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous rows [r0, r1) of rank `rank`: ceil(n / world) rows per rank, the last shorter."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = (n + world - 1) // world
    r0 = min(n, rank * per)
    return r0, min(n, r0 + per)


def packed_layout(k: int, d: int) -> dict:
    """Offsets (in fp64 elements) of the per-iteration allreduce buffer (mirrors AccLayout)."""
    return {"sums": 0, "counts": k * d, "sse": k * d + k, "changed": k * d + k + 1,
            "total": k * d + k + 4}


def _device_for_backend() -> torch.device:
    if tdist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_nccl_id(nccl_id: bytes | None, src: int = 0) -> bytes:
    """Broadcast rank `src`'s 128-byte ncclUniqueId to every rank of the default group."""
    buf = bytearray(nccl_id if nccl_id is not None else bytes(NCCL_ID_BYTES))
    if len(buf) != NCCL_ID_BYTES:
        raise ValueError("ncclUniqueId is 128 bytes")
    t = torch.tensor(list(buf), dtype=torch.uint8, device=_device_for_backend())
    tdist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def max_over_ranks(x: float) -> float:
    """Max of a per-rank scalar (timings are reported as the max over ranks)."""
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for_backend())
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for_backend())
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    return float(t.item())
