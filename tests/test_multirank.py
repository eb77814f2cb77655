"""N>1 path on CPU: world_size-2 (and 3) gloo runs of the stripe sharding,
bookkeeping collectives, gather and .strf merge (tests/multirank_worker.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import multirank_worker as W
from paper_2005_05826_b200 import shard
from paper_2005_05826_b200 import stripefrac as sf


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_rank_ranges_tile_and_match_reference_split():
    for S in (1, 2, 7, 12500, 56860):
        for world in (1, 2, 3, 4, 8):
            ranges = shard.all_ranges(0, S, world)
            shard.check_tiling(ranges, 0, S)
            # kernels.hpp:302-303: start + span*g/G
            assert ranges == [(S * g // world, S * (g + 1) // world) for g in range(world)]
    assert shard.rank_range(5, 17, 1, 2) == (11, 17)
    with pytest.raises(ValueError):
        shard.rank_range(0, 10, 2, 2)
    with pytest.raises(ValueError):
        shard.check_tiling([(0, 3), (4, 10)], 0, 10)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_gather_and_merge(tmp_path, world):
    seed, n, leaves, dens = 77, 41, 90, 0.1
    port = _free_port()
    mp.start_processes(W.run, args=(world, port, str(tmp_path), seed, n, leaves, dens),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(tmp_path / "gathered.npy")
    want = np.load(tmp_path / "want.npy")
    assert np.array_equal(got, want)
    # the per-rank .strf partials (stripes.cpp:179-201) read back and tile the
    # full range; merging them into a matrix condenses on device (GPU tests)
    parts = sorted((sf.read_stripe_file(str(tmp_path / f"part{r}.strf")) for r in range(world)),
                   key=lambda p: p.start)
    shard.check_tiling([(p.start, p.stop) for p in parts], 0, n // 2)
    assert np.array_equal(np.concatenate([p.distances for p in parts]), want)
