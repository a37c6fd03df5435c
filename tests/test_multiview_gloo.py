"""Multi-rank host logic of the multi-view path on CPU (gloo, world size 2):
view sharding, scene-blob broadcast (the NCCL path on GPUs), frame gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2501_00342_b200 as sg
from paper_2501_00342_b200 import multiview


def test_shard_views_partitions_exactly():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                b, e = multiview.shard_views(n, world, r)
                covered.extend(range(b, e))
            assert covered == list(range(n))
    assert multiview.ring_views_per_rank(32, 8, 7, 256) == list(range(224, 256))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene = sg.synth_scene(5000, "mixed", 20260003, log_scale_range=(-5.5, -4.0)) if rank == 0 else None
        meta, blob = multiview.broadcast_scene_blob(scene, "cpu", src=0)
        # every rank can reproduce the layout locally: the broadcast bytes must match
        mine, host = sg.Renderer.pack(sg.synth_scene(5000, "mixed", 20260003,
                                                     log_scale_range=(-5.5, -4.0)))
        ok_meta = bytes(meta) == bytes(mine)
        ok_blob = np.array_equal(blob.numpy(), host)
        frames = torch.full((4, 3), float(rank))
        got = multiview.gather_frames(frames, dst=0)
        ok_gather = rank != 0 or all(torch.all(g == i) for i, g in enumerate(got))
        # ragged shards (shard_views of 5 views over 2 ranks: 3 + 2), gathered to rank 1
        b, e = multiview.shard_views(5, world, rank)
        rag = torch.arange(b, e, dtype=torch.float32).reshape(-1, 1).repeat(1, 3)
        got = multiview.gather_frames(rag, dst=1)
        if rank == 1:
            ok_gather = ok_gather and [g.shape[0] for g in got] == [3, 2] and \
                torch.equal(torch.cat(got)[:, 0], torch.arange(5, dtype=torch.float32))
        # src / dst are ranks within the group: group rank 1 (global rank 1) sends
        sub = dist.new_group([0, 1])
        src_scene = sg.synth_scene(5000, "mixed", 20260003, log_scale_range=(-5.5, -4.0)) if rank == 1 else None
        sub_meta, sub_blob = multiview.broadcast_scene_blob(src_scene, "cpu", src=1, group=sub)
        ok_blob = ok_blob and np.array_equal(sub_blob.numpy(), host)
        out.put((rank, ok_meta, ok_blob, bool(ok_gather), int(meta.blob_bytes)))
    finally:
        dist.destroy_process_group()


def test_scene_broadcast_and_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert len(results) == 2
    for rank, ok_meta, ok_blob, ok_gather, nbytes in results:
        assert ok_meta and ok_blob and ok_gather, (rank, ok_meta, ok_blob, ok_gather)
        assert nbytes >= 5000 * 16 * 13
