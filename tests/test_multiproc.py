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


# ------------------------------------------------------------ plan sharding across ranks
def _oracle_run_part(halves, plan, mine, device, mode, pipeline, dedup, text):
    """CPU stand-in for layers.run_part (same output format): the SPEC-literal serial
    backend's hits per task → host records → the runtime's record rows and text."""
    from oracle import serial
    from paper_2109_14814_b200 import device as D, isect, runtime
    rows, chunks, stats = [], [], []
    for j, k in enumerate(mine):
        n1, s1, n2, s2 = plan.tasks[k]
        hu, hs = halves[("u", n1, s1)], halves[("s", n2, s2)]
        ca, cb = np.ascontiguousarray(hu.coords), np.ascontiguousarray(hs.coords)
        r = serial.find_intersections(ca, cb)
        h = np.zeros(len(r["ia"]), dtype=D.HIT_DTYPE)
        for f in ("ia", "ib", "s", "t", "a", "b"):
            h[f] = r[f]
        recs = isect.hits_to_records(ca, hu.s_values, cb, hs.s_values, h, layer=plan.tasks[k], dedup=dedup)
        arr = np.zeros(len(recs), runtime.RECORD_DTYPE)
        for i, rec in enumerate(recs):
            arr[i] = (rec.pair.gid, rec.tri_index[0], rec.tri_index[1], rec.point, rec.bary, rec.params, j, 0)
        rows.append(arr)
        chunks.append("".join(rec.to_line() + "\n" for rec in recs).encode())
        stats.append({"n_hits": len(h)})
    return np.concatenate(rows), b"".join(chunks), stats


def _plan_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_14814_b200 import layers
    from paper_2109_14814_b200.mesh import layered_mesh
    layers.run_part = _oracle_run_part  # CPU: the oracle stands in for the GPU part
    u = layered_mesh(48, "unstable", 3, 1.6, 0.1, 1)
    s = layered_mesh(48, "stable", 3, 1 / 1.6, 0.1, 2)
    plan = layers.enumerate_layer_pairs(u, s, 3, include_core=True)
    res = layers.search_plan_distributed(u, s, plan, device=rank, text=True)
    if rank == 0:
        single = layers.merge_parts(plan, *layers.plan_parts(u, s, plan, 1)[:1],
                                    [list(range(len(plan)))],
                                    [_oracle_run_part(layers.plan_parts(u, s, plan, 1)[0], plan,
                                                      list(range(len(plan))), 0, 0, 0, True, True)], [0], True)
        ok = (res.text == single.text and [r.to_line() for r in res.records] == [r.to_line() for r in single.records]
              and [st["layer"] for st in res.stats] == plan.tasks and len(res.records) > 0
              and sorted({st["device"] for st in res.stats}) == [0, 1])
        with open(out_path, "w") as fh:
            fh.write("ok" if ok else "mismatch")
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


def test_plan_sharding_gathers_single_device_records(tmp_path):
    """World size 2 (gloo, CPU): layers.search_plan_distributed deals whole layer-pair
    tasks over the ranks, gathers the record lists to rank 0 and merges them in plan
    order — the records and records text equal a single-device run of the same plan."""
    out = tmp_path / "plan.txt"
    mp.spawn(_plan_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"
