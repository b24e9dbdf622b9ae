"""World-size-2 gloo test of the multi-GPU host path on CPU: cyclic A-block shard
assignment + hit gathering.  Each rank computes its shard with the CPU oracle (the
GPU kernel honours the same ranges, see tests/test_gpu.py::test_shard_invariance);
rank 0's gathered list must equal the single-process search."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle
    from paper_2109_14814_b200 import device as D

    z = np.load(os.path.join(GOLD, "c4ii.npz"))
    A, B = z["A"], z["B"]
    n_tri = 2 * A.shape[2] * (A.shape[1] - 1)
    parts = []
    for a0, a1 in D.shard_ranges(n_tri, rank, world, a_block=1024):
        r = c_oracle.search(A, B, a_range=(a0, a1), sweep=True)
        h = np.zeros(len(r["ia"]), dtype=D.HIT_DTYPE)
        for k in ("ia", "ib", "s", "t", "a", "b"):
            h[k] = r[k]
        parts.append(h)
    mine = np.concatenate(parts) if parts else np.zeros(0, D.HIT_DTYPE)
    merged = D.gather_hits(mine[::-1].copy(), dst=0)
    if rank == 0:
        np.save(out_path, merged)
    else:
        assert merged is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_gather_equals_single(tmp_path, world):
    from oracle import c_oracle
    from paper_2109_14814_b200 import device as D

    c_oracle.build()
    out = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    merged = np.load(out)
    z = np.load(os.path.join(GOLD, "c4ii.npz"))
    assert np.array_equal(merged["ia"], z["ia"]) and np.array_equal(merged["ib"], z["ib"])
    for f in "stab":
        assert np.array_equal(merged[f].view(np.uint64), z[f])
    # the ranges tile [0, n_tri) exactly once
    n = 2 * z["A"].shape[2] * (z["A"].shape[1] - 1)
    rs = sorted(r for k in range(world) for r in D.shard_ranges(n, k, world, a_block=1024))
    assert rs[0][0] == 0 and rs[-1][1] == n and all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
