"""Multi-view rendering across GPUs: one rank per GPU, the scene
replicated through one broadcast, the views block-partitioned across ranks.

The path has no data-path collective: every rank renders its own views from the
replicated scene. Two ways in:

* RenderGroup -- the C-ABI's own multi-GPU path (sgs_group_*, include/sgs.h): NCCL
  ranks made by the library (one process per GPU with a shipped unique id, or one
  process driving every GPU), scene broadcast over NVLink, frames gathered to a root
  with grouped send/recv overlapped with rendering. What bench.py --gpus N times and
  what a C++ caller (the CLI, the trainer) uses.
* broadcast_scene_blob / gather_frames -- the same steps through torch.distributed,
  device-agnostic so the multi-rank host logic is also exercised with the gloo
  backend on CPU (tests/test_multiview_gloo.py).
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


def _load_nccl_first():
    """The library binds the NCCL already in the process; when torch is installed,
    import it first so that is torch's (one NCCL per process)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


class RenderGroup:
    """One rank of an sgs_group (include/sgs.h): every method is collective -- each
    rank calls it, with the same arguments (the scene only on the root)."""

    def __init__(self, handle: int, renderer, rank: int):
        self.handle = ctypes.c_void_p(handle)
        self.renderer = renderer  # the rank's render context
        self.rank = rank

    @staticmethod
    def unique_id() -> bytes:
        from . import _check, _lib

        _load_nccl_first()
        buf = (ctypes.c_uint8 * C.GROUP_ID_BYTES)()
        _check(_lib().sgs_group_unique_id(buf))
        return bytes(buf)

    @classmethod
    def init_rank(cls, renderer, nranks: int, rank: int, uid: bytes) -> "RenderGroup":
        """Rank `rank` of `nranks`, one process per GPU (ncclCommInitRank)."""
        from . import _check, _lib

        _load_nccl_first()
        h = ctypes.c_void_p()
        idb = (ctypes.c_uint8 * C.GROUP_ID_BYTES).from_buffer_copy(uid)
        _check(_lib().sgs_group_init_rank(renderer.handle, nranks, rank, idb, ctypes.byref(h)))
        return cls(h.value, renderer, rank)

    @classmethod
    def create(cls, devices: Sequence[int]) -> List["RenderGroup"]:
        """Every rank in this process (ncclCommInitAll); drive each from its own thread."""
        from . import Renderer, _check, _lib

        _load_nccl_first()
        n = len(devices)
        devs = (ctypes.c_int32 * n)(*devices)
        hs = (ctypes.c_void_p * n)()
        _check(_lib().sgs_group_create(n, devs, hs))
        out = []
        for r, (d, h) in enumerate(zip(devices, hs)):
            ctx = ctypes.c_void_p()
            _check(_lib().sgs_group_context(h, ctypes.byref(ctx)))
            out.append(cls(h, Renderer._wrap(ctx.value, d), r))
        return out

    def close(self):
        from . import _lib

        if self.handle:
            _lib().sgs_group_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def broadcast_scene(self, scene, root: int = 0):
        """The root's scene on every rank (NCCL broadcast of its device layout)."""
        from . import DeviceScene, _check, _lib

        h = ctypes.c_void_p()
        desc = None
        keep = None
        if scene is not None:
            desc, keep = scene._desc()
        _check(_lib().sgs_group_broadcast_scene(self.handle, ctypes.byref(desc) if desc is not None else None,
                                                root, ctypes.byref(h)))
        del keep
        return DeviceScene(self.renderer, h.value)

    def render_views(self, dscene, cams, root: int = 0, tile_size=16, thresholds=(2.0, 8.0), degree_override=-1,
                     early_stop=1e-4, rgb=None, T=None, device_out=False, with_T=True):
        """Views [0, len(cams)): this rank renders its block; the root receives every
        frame (numpy host arrays, or device pointers with device_out=True). with_T
        (the same on every rank; T=False on the root means the same) says whether
        transmittance frames travel. Returns (rgb, T) on the root."""
        import numpy as np

        from . import _check, _config, _lib

        n = len(cams)
        carr = (C.sgs_camera * max(n, 1))(*[c._c() for c in cams])
        cfg = _config(tile_size, thresholds, 0, degree_override, early_stop)
        with_T = with_T and T is not False
        if self.rank != root:  # off the root only T's null-ness matters: 1 stands for "T travels"
            _check(_lib().sgs_group_render_views(self.handle, dscene.handle, carr, n, ctypes.byref(cfg), root,
                                                 None, 1 if with_T else None,
                                                 C.SGS_DEVICE if device_out else C.SGS_HOST, None))
            return None, None
        if device_out:
            if with_T and not T:
                raise ValueError("with_T on the root needs a device T buffer")
            rgb_p, T_p, mem = rgb, T if with_T else None, C.SGS_DEVICE
        else:
            H, W = (cams[0].height, cams[0].width) if n else (0, 0)
            if rgb is None:
                rgb = np.empty((n, H, W, 3), dtype=np.float32)
            if T is None:
                T = np.empty((n, H, W, 1), dtype=np.float32)
            rgb_p = rgb.ctypes.data
            T_p = T.ctypes.data if with_T else None
            mem = C.SGS_HOST
        _check(_lib().sgs_group_render_views(self.handle, dscene.handle, carr, n, ctypes.byref(cfg), root,
                                             rgb_p, T_p, mem, None))
        return rgb, T
