"""Multi-process path on CPU (world_size 2, gloo): every rank renders its block-cyclic shard of every
(technique, side) index range and the images are summed on rank 0 by the one collective of the path
(SURVEY 8(e)).  The per-rank renderer here is the CPU oracle (test infrastructure); the GPU kernels' own
index mapping is checked against the unsharded render in tests/test_gpu_parity.py."""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_16302_b200.shard import SHARD_BLOCK, reduce_image, shard_ranges
from rr_inputs import scenes as S


def _workload():
    w = S.config1(64, 64, spp=32, max_depth=3)  # one-way: 64*64*32 = 2 blocks of 2^16 per technique
    return w, dataclasses.replace(w.args, flags=0, technique_mask=0x43)


def _render(w, args, ranges_of):
    from oracle import binding as B
    o = B.Oracle(w.scene, w.edits)
    mask = o.effective_mask(args.technique_mask)
    img = np.zeros((w.scene.camera.height, w.scene.camera.width, 3), np.float64)
    n = o.sample_range(args)
    for l in range(1, 8):
        if (mask >> (l - 1)) & 1:
            for i0, i1 in ranges_of(n):
                o.residual(args, l, 0, i0, i1, image=img)
    return img


def _rank(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, args = _workload()
    img = torch.from_numpy(_render(w, args, lambda n: shard_ranges(n, rank, world)))
    reduce_image(img, dst=0)
    if rank == 0:
        np.save(out, img.numpy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_partition():
    for n in (1, SHARD_BLOCK - 1, SHARD_BLOCK, 5 * SHARD_BLOCK + 17):
        for world in (1, 2, 3, 8):
            seen = np.zeros(n, np.int32)
            for r in range(world):
                for i0, i1 in shard_ranges(n, r, world):
                    assert i0 % SHARD_BLOCK == 0 and (i0 // SHARD_BLOCK) % world == r
                    seen[i0:i1] += 1
            assert np.all(seen == 1)
    with pytest.raises(ValueError):
        shard_ranges(10, 2, 2)


def test_two_rank_gloo_reduce_matches_unsharded(tmp_path):
    out = str(tmp_path / "img.npy")
    mp.spawn(_rank, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    w, args = _workload()
    full = _render(w, args, lambda n: [(0, n)])
    assert np.abs(full).sum() > 0
    np.testing.assert_allclose(got, full, rtol=1e-12, atol=1e-15)
