"""Multi-view rendering across GPUs: one process per GPU, the scene
replicated through one broadcast, the views block-partitioned across ranks.

The path has no data-path collective: every rank renders its own views from the
replicated scene. NCCL (torch.distributed, backend "nccl" over NVLink) carries the
scene blob once and, optionally, the frames back to a root. The host logic here is
device-agnostic so it is also exercised with the gloo backend on CPU
(tests/test_multiview_gloo.py).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as C


def shard_views(n_views: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [begin, end) of the views owned by `rank` (deterministic,
    sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_views, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def ring_views_per_rank(views_per_rank: int, world: int, rank: int, ring: int) -> List[int]:
    """Weak-scaling assignment used by bench.py: rank r renders ring cameras
    [(r * v + j) mod ring for j < v]."""
    return [(rank * views_per_rank + j) % ring for j in range(views_per_rank)]


def _global_rank(group, rank: int) -> int:
    import torch.distributed as dist

    return rank if group is None else dist.get_global_rank(group, rank)


def broadcast_scene_blob(scene, device, src: int = 0, group=None):
    """Ship the scene's device layout from `src` (a rank within `group`) to every rank.

    `scene` is a paper_2501_00342_b200.Scene on `src` (ignored elsewhere). Returns
    (meta, blob) where blob is a uint8 torch tensor on `device` holding the packed
    planes on every rank. On GPUs the blob is bound without a copy
    (Renderer.bind); on CPU (gloo) it is what the tests compare.
    """
    import torch
    import torch.distributed as dist

    from . import Renderer

    rank = dist.get_rank(group)
    holder = [None]
    host = None
    if rank == src:
        meta, host = Renderer.pack(scene)
        holder[0] = bytes(meta)
    gsrc = _global_rank(group, src)  # (the collectives take global ranks)
    dist.broadcast_object_list(holder, src=gsrc, group=group)
    meta = C.sgs_scene_meta.from_buffer_copy(holder[0])
    blob = torch.empty(meta.blob_bytes, dtype=torch.uint8, device=device)
    if rank == src:
        blob.copy_(torch.from_numpy(host))
    dist.broadcast(blob, src=gsrc, group=group)
    return meta, blob


def gather_frames(frames, dst: int = 0, group=None):
    """Gather each rank's frames (a tensor whose leading dimension is the rank's view
    count, which may differ by rank: shard_views blocks differ by one) to `dst`, a
    rank within `group`: a list of per-rank tensors on dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # leading sizes first, then equal-size (padded) buffers for the collective
    n = torch.tensor([frames.shape[0]], dtype=torch.int64, device=frames.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(x.item()) for x in sizes]
    most = max(sizes)
    send = frames
    if frames.shape[0] < most:
        send = torch.zeros((most,) + tuple(frames.shape[1:]), dtype=frames.dtype, device=frames.device)
        send[: frames.shape[0]] = frames
    recv = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send.contiguous(), recv, dst=_global_rank(group, dst), group=group)
    return [r[: k] for r, k in zip(recv, sizes)] if rank == dst else None
