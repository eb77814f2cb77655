"""Worker for tests/test_multirank.py: one rank of a gloo world on CPU.

Exercises the N>1 host path exactly as bench.py / a multi-process user runs
it: the reference's stripe split per rank (shard.rank_range), each rank's
stripe block (here from the CPU oracle — test infrastructure — since the
device kernels need a B200), max/sum reductions, gathering on rank 0, and the
per-rank `.strf` partial files + merge of the reference's multi-process flow
(stripes.cpp:179-297)."""
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))


def run(rank, world, port, outdir, seed, n, leaves, dens):
    import numpy as np
    import torch.distributed as dist

    import oracle_port as op
    from paper_2005_05826_b200 import shard
    from paper_2005_05826_b200 import stripefrac as sf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        a, b = shard.rank_range(0, S, rank, world)
        d, t = op.compute_stripes(problem, 1, 8, a, b)  # finalized distances
        # bookkeeping collectives of the bench
        assert shard.max_over_ranks(float(rank)) == world - 1
        assert shard.sum_over_ranks(1.0) == world
        full = shard.gather_stripes(d, n, 0, S)
        # per-rank partial file (the reference's `compute --stripes a:b`)
        part = sf.StripeSet(n_samples=n, start=a, stop=b, metric=sf.Metric.Unweighted, finalized=True,
                            distances=d, totals=t)
        sf.write_stripe_file(os.path.join(outdir, f"part{rank}.strf"), part)
        dist.barrier()
        if rank == 0:
            want_d, _ = op.compute_stripes(problem, 1, 8, 0, S)
            np.save(os.path.join(outdir, "gathered.npy"), full)
            np.save(os.path.join(outdir, "want.npy"), want_d)
    finally:
        dist.destroy_process_group()
