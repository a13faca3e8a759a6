"""The N>1 replica path on CPU: world_size-2 gloo process group.

Each rank solves its shard of the right-hand sides of a small case with the
oracle (the GPU solve is the same per rank; no data-path collective), the
timing reduction is the max over ranks and the work count the sum.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1410_5910_b200.replicas import shard


def test_shard_is_a_balanced_partition():
    for n in (0, 1, 7, 64):
        for w in (1, 2, 3, 8):
            parts = [list(shard(n, w, r)) for r in range(w)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world_size, port, out_dir):
    import torch.distributed as dist

    from conftest import golden_path
    from oracle import ref_port as O
    from paper_1410_5910_b200.operator import load_case_arrays
    from paper_1410_5910_b200.replicas import gather_counts, max_over_ranks, shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world_size), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    meta, arr = load_case_arrays(golden_path("fx_uneven"))
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    rng = np.random.default_rng(5)
    rhs = [rng.standard_normal(pol.n_block_rows * pol.m) + 0j for _ in range(5)]
    mine = shard(len(rhs), world_size, rank)
    for s in mine:
        x, rep = O.gmres_solve(pol.matvec, lambda v: O.preconditioner_apply(2, d, r, perm, v),
                               rhs[s], rel_tol=1e-10)
        np.save(os.path.join(out_dir, f"x{s}.npy"), x)
    t = max_over_ranks(10.0 + rank)
    n = gather_counts(len(mine))
    np.save(os.path.join(out_dir, f"red{rank}.npy"), np.array([t, n]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gloo(tmp_path):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for rank in range(2):
        t, n = np.load(tmp_path / f"red{rank}.npy")
        assert t == 11.0 and n == 5
    # every right-hand side solved exactly once, and equal to a 1-rank solve
    from conftest import golden_path
    from oracle import ref_port as O
    from paper_1410_5910_b200.operator import load_case_arrays
    meta, arr = load_case_arrays(golden_path("fx_uneven"))
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    rng = np.random.default_rng(5)
    rhs = [rng.standard_normal(pol.n_block_rows * pol.m) + 0j for _ in range(5)]
    for s in range(5):
        x, _ = O.gmres_solve(pol.matvec, lambda v: O.preconditioner_apply(2, d, r, perm, v),
                             rhs[s], rel_tol=1e-10)
        assert np.array_equal(np.load(tmp_path / f"x{s}.npy"), x)
