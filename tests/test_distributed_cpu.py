"""N>1 host path on CPU: world_size-2 gloo processes run the bin-sharded and
frame-sharded partitions and the optional slab gather.  The per-rank compute
is the oracle standing in for the device kernel (no GPU here); what is under
test is the partition + assembly logic of paper_1711_01919_b200.sharding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, bins, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from paper_1711_01919_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img = O.synth_image(37, 23, 5)
    lut = O.np_uniform_table(bins)
    full = O.compute_sequential(img, lut, bins)

    def compute(lo, hi):  # oracle stand-in for the device slab kernel
        return torch.from_numpy(full[lo:hi].copy()).view(torch.uint32)

    (lo, hi), slab = sharding.local_bin_slab(compute, bins, rank, world)
    got = sharding.gather_slabs(slab, bins, 23, 37, rank, world)
    if rank == 0:
        np.save(os.path.join(outdir, f"full_{bins}.npy"), got.view(torch.int32).numpy())
    # frame sharding: each rank takes its contiguous frames; all-gather the checksums
    shards = sharding.frame_shards(6, world)
    f0, f1 = shards[rank]
    mine = [int(O.tensor_checksum(O.compute_sequential(O.synth_image(16, 9, k), lut, bins)), 16)
            for k in range(f0, f1)]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        np.save(os.path.join(outdir, f"frames_{bins}.npy"),
                np.array([c for part in gathered for c in part], dtype=np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("bins", [5, 1, 16])
def test_bin_and_frame_sharding_gloo(tmp_path, bins):
    from oracle import oracle as O

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), bins, str(tmp_path)), nprocs=world, join=True)
    full = np.load(tmp_path / f"full_{bins}.npy").view(np.uint32)
    expect = O.compute_sequential(O.synth_image(37, 23, 5), O.np_uniform_table(bins), bins)
    assert np.array_equal(full, expect)
    frames = np.load(tmp_path / f"frames_{bins}.npy")
    lut = O.np_uniform_table(bins)
    want = [int(O.tensor_checksum(O.compute_sequential(O.synth_image(16, 9, k), lut, bins)), 16)
            for k in range(6)]
    assert frames.tolist() == want
