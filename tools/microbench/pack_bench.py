"""Pack kernel time per config: mcx_pack on a device-resident grid, CUDA events on the
launching stream, L2 flushed (256 MB memset) before every timed launch, median of 20.
Prints one JSON line per config with the algorithmic bytes (16 B of grid +
64 B box + 4 B perm + level boxes per record) and the achieved HBM rate.  With --check,
also compares the packed arrays against a pack of the same grid done by DeviceMesh.
    python tools/microbench/pack_bench.py [C3 C5 ...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402

names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["C2", "C3", "C5", "C5hd"]
L = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
for name in names:
    A, _, B, _ = config_pair(name)
    for tag, X in (("A", A), ("B", B)):
        m = D.DeviceMesh(X, 0)
        s = torch.cuda.current_stream(0)
        outs = [torch.empty_like(t) for t in (m.box, m.perm, m.gbox, m.tbox, m.bbox, m.status)]
        ts = []
        for it in range(23):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            rc = L.mcx_pack(m.coords.data_ptr(), m.N, m.M, _lib.ORDER_TILED, *(o.data_ptr() for o in outs), 0,
                            s.cuda_stream)
            e1.record(s)
            _lib.check(rc, "mcx_pack")
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        same = all(torch.equal(a, b) for a, b in zip(outs[:5], (m.box, m.perm, m.gbox, m.tbox, m.bbox)))
        n = m.n_tri
        alg = m.coords.numel() * 8 + n * (64 + 4) + (m.gbox.numel() + m.tbox.numel() + m.bbox.numel()) * 8
        us = statistics.median(ts)
        print(json.dumps({"config": name, "mesh": tag, "n_tri": n, "us": round(us, 2), "alg_bytes": alg,
                          "GBps": round(alg / us * 1e-3, 1), "same_as_devicemesh": same}), flush=True)
