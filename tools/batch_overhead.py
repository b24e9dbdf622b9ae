"""Where the host time of one batched search call goes (the paper's 108-task plan):
wall time of device.search_batch vs its kernel time, and of its host-side pieces."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.layers import enumerate_layer_pairs  # noqa: E402
from paper_2109_14814_b200.mesh import half_layer, layered_mesh  # noqa: E402

um = layered_mesh(1024, "unstable", 14, 1.6, 0.1, 1, K=17, per_layer=34)
sm = layered_mesh(2048, "stable", 14, 1 / 1.6, 0.1, 2, K=17, per_layer=34)
plan = enumerate_layer_pairs(um, sm, 14)
dm = {}


def half(mesh, key, n, sg):
    if key not in dm:
        dm[key] = D.DeviceMesh(np.ascontiguousarray(half_layer(mesh, n, 1 if sg == "+" else -1).coords), 0)
    return dm[key]


pairs = [(half(um, ("u", n1, s1), n1, s1), half(sm, ("s", n2, s2), n2, s2)) for n1, s1, n2, s2 in plan.tasks]
for mode in ("cull", "prefilter"):
    m = _lib.MODE_NAMES[mode]
    for _ in range(3):
        D.search_batch(pairs, mode=m)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        res = D.search_batch(pairs, mode=m, timing=True)
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    for _ in range(10):
        [(p[0].struct(), p[1].struct()) for p in pairs]
    t_structs = (time.perf_counter() - t0) / 10
    print(f"{mode}: wall {1e3 * np.median(ts):.3f} ms, kernels {res[0].stats['kernel_ms']:.3f} ms, "
          f"ctypes structs {1e3 * t_structs:.3f} ms, hits {sum(len(r.hits) for r in res)}")

# finer split of the cull call
m = _lib.MODE_CULL
L = _lib.load()
W = D._Workspace.get(0)
s = torch.cuda.current_stream(0)
n = len(pairs)
for rep in range(3):
    t0 = time.perf_counter()
    tasks = (_lib.Task * n)()
    for k, p in enumerate(pairs):
        tasks[k].A, tasks[k].B = p[0].struct_ptr(), p[1].struct_ptr()
    t1 = time.perf_counter()
    opts = _lib.Opts(0, s.cuda_stream, 0, 0, 0, 1, m, 1, None, 0)
    need = L.mcx_batch_workspace_bytes(tasks, n, opts)
    ws = W.workspace(need)
    opts.workspace, opts.workspace_bytes = ws.data_ptr(), ws.numel()
    stats = (_lib.Stats * n)()
    buf = W.hit_buffer(1 << 16)
    tb = W.task_buffer(buf.numel() // 5)
    t2 = time.perf_counter()
    rc = L.mcx_search_batch(tasks, n, opts, buf.data_ptr(), tb.data_ptr(), buf.numel() // 5, stats)
    t3 = time.perf_counter()
    total = sum(int(stats[k].n_hits) for k in range(n))
    hits = buf[: total * 5].cpu().numpy()
    owner = tb[:total].cpu().numpy()
    t4 = time.perf_counter()
    print(f"split: structs+tasks {1e3*(t1-t0):.3f}  ws/opts {1e3*(t2-t1):.3f}  mcx_search_batch {1e3*(t3-t2):.3f} "
          f"(kernels {stats[0].kernel_ms:.3f})  D2H+numpy {1e3*(t4-t3):.3f} ms")
