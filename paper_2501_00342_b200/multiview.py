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


def broadcast_scene_blob(scene, device, src: int = 0, group=None):
    """Ship the scene's device layout from `src` to every rank.

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
    dist.broadcast_object_list(holder, src=src, group=group)
    meta = C.sgs_scene_meta.from_buffer_copy(holder[0])
    blob = torch.empty(meta.blob_bytes, dtype=torch.uint8, device=device)
    if rank == src:
        blob.copy_(torch.from_numpy(host))
    dist.broadcast(blob, src=src, group=group)
    return meta, blob


def gather_frames(frames, dst: int = 0, group=None):
    """Gather each rank's frame tensor to `dst` (list on dst, None elsewhere)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    recv = [torch.empty_like(frames) for _ in range(world)] if rank == dst else None
    dist.gather(frames, recv, dst=dst, group=group)
    return recv
