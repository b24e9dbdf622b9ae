"""Break down one end-to-end search step (host grids -> hits) by phase with CUDA events
and host timers, for the e2e optimisation work."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2109_14814_b200 import device as D, _lib
from paper_2109_14814_b200.mesh import config_pair

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
A, _, B, _ = config_pair(name)
pa = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
pb = torch.from_numpy(np.ascontiguousarray(B)).pin_memory()
s = torch.cuda.current_stream()
for mode in (_lib.MODE_CULL,):
    for it in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Am = D.DeviceMesh(pa, 0)
        t1 = time.perf_counter()
        Bm = D.DeviceMesh(pb, 0)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        r = D.search_device(Am, Bm, mode=mode)
        t3 = time.perf_counter()
        print(f"iter {it}: meshA(host) {1e3*(t1-t0):.3f} ms, meshA+B(sync) {1e3*(t2-t0):.3f} ms, search {1e3*(t3-t2):.3f} ms, total {1e3*(t3-t0):.3f} ms, hits {len(r.hits)}")
