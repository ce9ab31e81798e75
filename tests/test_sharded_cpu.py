"""Sort-first multi-GPU partition and gather logic (render/sharded.py) on
CPU: strip ownership covers every frame row exactly once, re-interleaving
is the inverse of the partition, and the gather + counter all-reduce over a
world_size-2 gloo group assembles the frame on the root rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_2074_b200.render.core import RenderCounters
from paper_1407_2074_b200.render.sharded import (SortFirstRenderer, assemble,
                                                  frame_rows_of_part, part_rows)


@pytest.mark.parametrize("H,strip,G", [(1080, 8, 2), (1080, 8, 3), (1080, 8, 8), (17, 4, 4),
                                        (5, 8, 2), (2160, 16, 8), (1, 1, 1)])
def test_strips_cover_each_row_once(H, strip, G):
    rows = np.concatenate([frame_rows_of_part(H, strip, G, p) for p in range(G)])
    rows = rows[rows >= 0]
    assert np.array_equal(np.sort(rows), np.arange(H))
    for p in range(G):
        assert len(frame_rows_of_part(H, strip, G, p)) == part_rows(H, strip, G)


@pytest.mark.parametrize("H,W,strip,G", [(1080, 6, 8, 8), (37, 3, 4, 3), (64, 2, 16, 2)])
def test_assemble_inverts_partition(H, W, strip, G):
    img = torch.arange(H * W * 4, dtype=torch.int64).reshape(H, W, 4)
    parts = []
    for p in range(G):
        fr = frame_rows_of_part(H, strip, G, p)
        part = torch.zeros((len(fr), W, 4), dtype=torch.int64)
        ok = fr >= 0
        part[torch.as_tensor(np.flatnonzero(ok))] = img[torch.as_tensor(fr[ok])]
        parts.append(part)
    assert torch.equal(assemble(torch.stack(parts), H, strip), img)


class _FakeRenderer(SortFirstRenderer):
    """render_part paints each row with its frame-row index (CPU tensors)."""

    def __init__(self, H, W, strip):
        super().__init__(None, strip_rows=strip)
        self.H, self.W = H, W

    def render_part(self, scene, out_kind=None):
        fr = frame_rows_of_part(self.H, self.strip_rows, self.world, self.rank)
        part = torch.from_numpy(np.repeat(np.maximum(fr, 0)[:, None, None], self.W * 4, axis=1)
                                .reshape(len(fr), self.W, 4).astype(np.int32))
        part[torch.as_tensor(fr < 0)] = 0
        return part, RenderCounters(samples=100 + self.rank, tf_lookups=3)


class _Cam:
    def __init__(self, H):
        self.height = H


class _Scene:
    def __init__(self, H):
        self.camera = _Cam(H)


def _worker(rank, world, port, H, W, strip, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = _FakeRenderer(H, W, strip)
        img, cnt = r.render_fullframe(_Scene(H))
        if rank == 0:
            expect = np.repeat(np.arange(H)[:, None, None], W * 4, axis=1).reshape(H, W, 4)
            q.put(("img", bool(np.array_equal(img.numpy(), expect))))
        else:
            q.put(("img", img is None))
        q.put(("cnt", (cnt.samples, cnt.tf_lookups)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_assembles_frame(world):
    H, W, strip = 45, 5, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, strip, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get(timeout=5) for _ in range(2 * world)]
    assert all(v for k, v in res if k == "img")
    assert all(v == (sum(100 + r for r in range(world)), 3 * world) for k, v in res if k == "cnt")
