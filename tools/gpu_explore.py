"""Ad-hoc GPU exploration: parity on small configs + variant timing on C2/C3."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2109_14814_b200 import device as D, _lib
from paper_2109_14814_b200.mesh import config_pair
from oracle import c_oracle as C, canonical as O

def same(r, h):
    return (np.array_equal(r['ia'], h['ia']) and np.array_equal(r['ib'], h['ib']) and
            all(np.array_equal(r[k].view(np.uint64), h[k].view(np.uint64)) for k in 'stab'))

out = {}
for name in ['C1', 'C4i', 'C4ii']:
    A, sa, B, sb = config_pair(name)
    ref = C.search(A, B, sweep=True)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    box, geo = C.pack(A)
    pk_ok = np.array_equal(Am.box.cpu().numpy(), box) and np.array_equal(Am.geo.cpu().numpy()[:, :19], geo)
    for v in range(4):
        os.environ['MCX_VARIANT'] = str(v)
        r = D.search_device(Am, Bm)
        ok = same(ref, r.hits) and r.stats['n_aabb_pass'] == ref['n_aabb_pass'] and r.stats['n_singular'] == ref['n_singular']
        print(name, 'variant', v, 'pack_ok', pk_ok, 'parity', ok, len(r.hits), r.stats, flush=True)

for name in ['C2', 'C3']:
    A, sa, B, sb = config_pair(name)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    for v in range(4):
        os.environ['MCX_VARIANT'] = str(v)
        D.search_device(Am, Bm)
        ts = []
        for k in range(3):
            r = D.search_device(Am, Bm, timing=True)
            ts.append(r.stats['kernel_ms'])
        ms = min(ts)
        pairs = r.stats['n_pairs']
        print(json.dumps({'cfg': name, 'variant': v, 'ms': ms, 'pairs_per_s': pairs / ms * 1e3,
                          'lane_ops_per_s': 8 * pairs / ms * 1e3, 'hits': int(r.stats['n_hits']),
                          'pass': int(r.stats['n_aabb_pass'])}), flush=True)
