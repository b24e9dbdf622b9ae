#!/usr/bin/env python
"""Benchmark: triangle-pair tests/s and full-search wall time of the 4D
mesh-intersection search (BASELINE.json metric) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One step = one complete search of mesh A against mesh B (every triangle pair
is tested, the AABB survivors get the canonical FP64 solve, hits are compacted)
for the named synthetic configuration (default C3: 1024×512 vs 1024×512 grids,
1,046,528 triangles each, 1.095e12 pairs).  `value` uses MCX_MODE_PREFILTER
(every pair tested by a conservative quantised-box integer test, its passes by
the exact FP64 test); the FP64 brute-force kernel and the culled search of the
same workload are measured in the same run and reported beside it.  Under
torchrun each rank owns one GPU and searches its cyclic share of A's
1024-triangle blocks (no collective on the data path); timing is the max over
ranks of CUDA-event device time.

``--impl reference`` times the reference's CPU search (the C port of the
SPEC's all-pairs "parallel" backend, oracle/mcx_oracle.c, all host threads) on the
deterministic slice A triangles [0, 8192) × all of B per step, plus
the NumPy "parallel" backend (multiprocessing over A-row chunks) and the SPEC-literal
serial NumPy backend on smaller slices; see DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "triangle-pair tests/s"
UNIT = "pair-tests/s"
FP64_LANES_PER_CLK_PER_SM = 64  # B200 FP64 pipe; verified by tools/microbench/pipes.cu (dadd 63.5)


def hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling
    guide's fallback."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write bytes)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--mode", default="prefilter", choices=["prefilter", "brute", "cull"],
                    help="primary mode for `value` (the others are measured too and reported alongside)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper's 14-layer workload block")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[4] (C5hd) hit-compaction / balance block")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets several ranks share one GPU (logic test of the N>1 path on a 1-GPU box)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload_desc(name, A, B):
    nA = 2 * A.shape[2] * (A.shape[1] - 1)
    nB = 2 * B.shape[2] * (B.shape[1] - 1)
    return {"workload": f"{name}: synthetic 4D mesh pair, A {A.shape[2]}x{A.shape[1]} grid ({nA} tri) vs "
                        f"B {B.shape[2]}x{B.shape[1]} grid ({nB} tri), float64",
            "triangles_a": nA, "triangles_b": nB, "pairs_per_step": nA * nB}


# ------------------------------------------------------------------ CPU baseline
REF_ROWS = 8192  # A triangles [0, 8192) x all of B per timed step


_REF_PACKED = {}


def cpu_reference_sample(A, B, rows=REF_ROWS, threads=0):
    """The C port of the SPEC all-pairs search (brute force, all threads) on the fixed slice
    A[0, rows) × all of B.  Both meshes are packed once per process, untimed (the oracle's
    mcxo_pack_new), so a step times exactly the search."""
    from oracle import c_oracle
    c_oracle.build()
    key = (id(A), id(B))
    if key not in _REF_PACKED:
        _REF_PACKED.clear()
        _REF_PACKED[key] = (c_oracle.Packed(A), c_oracle.Packed(B))
    PA, PB = _REF_PACKED[key]
    n = min(PA.n, rows)
    t0 = time.perf_counter()
    hits, pairs = c_oracle.search_packed(PA, PB, a_range=(0, n), sweep=False, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": pairs / dt, "seconds": dt, "a_triangles": n, "pairs": pairs, "hits": hits,
            "threads": c_oracle.max_threads() if threads == 0 else threads}


_NP_PACKED = None  # packed meshes shared with the forked workers (copy-on-write)


def _numpy_rows(rng):
    from oracle import canonical
    r = canonical.search(None, None, a_range=rng, packed=_NP_PACKED)
    return len(r["ia"])


def cpu_numpy_parallel_sample(A, B, rows=2048):
    """the canonical NumPy oracle in the SPEC's "parallel" mode —
    multiprocessing over A-row chunks on all cores — on A[0, rows) × all of B (both
    meshes packed once in the parent, untimed, and shared with the forked workers)."""
    global _NP_PACKED
    import multiprocessing as mp
    from oracle import canonical
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    cores = len(os.sched_getaffinity(0))
    nB = 2 * B.shape[2] * (B.shape[1] - 1)
    n = min(rows, 2 * A.shape[2] * (A.shape[1] - 1))
    _NP_PACKED = (canonical.pack(A), canonical.pack(B))
    cuts = np.linspace(0, n, cores + 1).astype(int)
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_numpy_rows, [(0, 0)] * cores)  # workers up
        t0 = time.perf_counter()
        hits = sum(pool.map(_numpy_rows, [(int(cuts[k]), int(cuts[k + 1])) for k in range(cores)]))
        dt = time.perf_counter() - t0
    _NP_PACKED = None
    return {"value": n * nB / dt, "unit": UNIT, "cores": cores, "seconds": dt, "hits": hits,
            "sample": f"A triangles [0, {n}) x all {nB} B triangles, NumPy canonical oracle (oracle/canonical.py), "
                      f"multiprocessing over {cores} A-row chunks, packing excluded"}


def cpu_spec_literal_sample(A, B, target_s=3.0):
    """The SPEC-literal serial backend (oracle/serial.py: quad AABB + Möller + precise,
    NumPy, one process) on a slice of A's quads — the reference's own 'serial' path."""
    from oracle import serial
    _, MA, NA = A.shape
    n_cols = 1
    while True:
        sub = np.ascontiguousarray(A[:, :n_cols + 1, :])
        t0 = time.perf_counter()
        serial.pair_candidates(sub, B)
        dt = time.perf_counter() - t0
        if dt > target_s / 4 or n_cols + 1 >= MA:
            break
        n_cols = min(MA - 1, n_cols * 2)
    nq_a = NA * n_cols
    nq_b = B.shape[2] * (B.shape[1] - 1)
    return {"value": 4.0 * nq_a * nq_b / dt, "seconds": dt, "a_quads": nq_a, "cores": 1,
            "note": "SPEC-literal serial backend (NumPy, 1 process): quad AABB + Moller, triangle-pair "
                    "equivalents (4 per quad pair) per second"}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def bench_config(desc, mode, world):
    """The `config` object both arms print (same workload, same keys)."""
    return {**desc, "mode": mode, "parallelism": f"A-block cyclic shards x{world}, B replicated",
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2109_14814_b200.mesh import config_pair
    A, _, B, _ = config_pair(args.config)
    desc = workload_desc(args.config, A, B)
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    for _ in range(max(0, args.warmup)):
        cpu_reference_sample(A, B, rows=1024)
    secs, pairs = [], 0
    for _ in range(max(1, args.steps)):
        s = cpu_reference_sample(A, B)
        secs.append(s["seconds"])
        pairs += s["pairs"]
    v = pairs / sum(secs)
    ms = 1e3 * sum(secs) / len(secs)
    sample = (f"A triangles [0, {s['a_triangles']}) x all {desc['triangles_b']} B triangles per step "
              f"({s['pairs']:.3e} pairs, brute force, packing excluded); ms_per_step is that slice")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(desc, args.mode, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": s["threads"], "kind": "port",
                             "sample": sample, "cpu": cpu_model(),
                             "algorithm": "the SPEC's all-pairs search (every pair through the FP64 AABB test, "
                                          "canonical solve of the passes), C port, OpenMP over A"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "full_search_s_extrapolated": desc["pairs_per_step"] / v,
            "numpy_parallel": None if args.no_cpu_baseline else cpu_numpy_parallel_sample(A, B),
            "spec_literal_serial": None if args.no_cpu_baseline else cpu_spec_literal_sample(A, B)}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() in ("active", "1"):
                    reasons.add(n)
        load = [v for v in sm if v > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ our arm
# our kernels per search call: brute = box sweep + solve (which also checks the meshes'
# non-finite flags); cull = 2 cull levels + solve; prefilter = fp32 boxes + box sweep + solve
KERNEL_LAUNCHES = {"brute": 2, "cull": 3, "prefilter": 3}
INT_LANES_PER_CLK_PER_SM = 64  # B200 fma-heavy (IMAD) and alu (LOP3) pipes, each; IMAD measured 62.7 lanes/clk/SM
                               # (tools/microbench/hprefilter.cu swar3_mix0); issue: 4 SMSP x 32 = 128 lanes/clk/SM
# SASS of the prefilter inner loop (half words, accumulated folds), per 16 pair tests: 8
# subtractions (each tests two pairs): 4 IMAD + 2 IMAD.X (fma-heavy pipe) + 2 IADD3 (alu pipe),
# and 4 LOP3.LUT (alu pipe; each folds two subtraction results into an accumulator) - 12
# instructions, 6 per pipe
PREFILTER_IMAD_PER_PAIR = 6.0 / 16.0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2109_14814_b200 import _lib, device as D
    from paper_2109_14814_b200.mesh import config_pair

    rank, world, local = dist_env()
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    local = local % torch.cuda.device_count()  # ranks may share a GPU under --dist-backend gloo
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    A, sa, B, sb = config_pair(args.config)
    desc = workload_desc(args.config, A, B)
    modes = dict(_lib.MODE_NAMES)
    shard = (rank, world)

    stream = torch.cuda.current_stream(dev)
    Am, Bm = D.DeviceMesh(A, local), D.DeviceMesh(B, local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def reduce(x, op):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    MAX = dist.ReduceOp.MAX if world > 1 else None
    SUM = dist.ReduceOp.SUM if world > 1 else None

    def measure(mode_name, with_clocks):
        mode = modes[mode_name]
        for _ in range(args.warmup):
            D.search_device(Am, Bm, mode=mode, shard=shard, stream=stream)
        barrier()
        clk = ClockSampler(local) if (with_clocks and rank == 0) else None
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        my_pairs = my_tested = 0
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[k][0].record(stream)
            res = D.search_device(Am, Bm, mode=mode, shard=shard, stream=stream)
            ev[k][1].record(stream)
            my_pairs += res.stats["n_pairs"]
            my_tested += res.stats["n_tested"]
        barrier()
        clocks = clk.stop() if clk else None
        dev_ms = sum(s.elapsed_time(e) for s, e in ev)
        t_max = reduce(dev_ms, MAX)
        hits = res.hits
        if world > 1:
            hits = D.gather_hits(hits)
        st = D.search_device(Am, Bm, mode=mode, shard=shard, stream=stream, timing=True).stats
        return {"t_max_ms": t_max, "ms_per_step": t_max / args.steps,
                "pairs": reduce(my_pairs, SUM), "tested": reduce(my_tested, SUM),
                "value": reduce(my_pairs, SUM) / (t_max * 1e-3), "hits": None if hits is None else len(hits),
                "kernel_ms": reduce(st["kernel_ms"], MAX), "stats": st, "clocks": clocks,
                "launches": KERNEL_LAUNCHES[mode_name] * args.steps}

    from paper_2109_14814_b200 import runtime
    pin_a = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
    pin_b = torch.from_numpy(np.ascontiguousarray(B)).pin_memory()
    h2d_bytes = (pin_a.numel() + pin_b.numel() + len(sa) + len(sb)) * 8

    def h2d_floor():
        """The same grids copied host→device alone (pinned, CUDA events): the PCIe time
        any implementation of the call pays."""
        da, db = torch.empty_like(pin_a, device=dev), torch.empty_like(pin_b, device=dev)
        ts = []
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            da.copy_(pin_a, non_blocking=True)
            db.copy_(pin_b, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
        return min(ts[1:])

    def measure_e2e(mode_name, pipeline, pairs_per_step, steps):
        """The reference-facing call end to end: isect.find_intersections' C-ABI entry
        (mcx_find_intersections) from pinned HOST grids — H2D of both grids, packing, the
        search, records, (gid, τ) sort, 1e-9 dedup and the records text on the device, D2H
        of records + text — timed on the host around synchronous calls, max over ranks."""
        ctx = runtime.context(local)
        mode, pipe = modes[mode_name], _lib.PIPELINE_NAMES[pipeline]

        def step():  # this rank's cyclic share of the larger mesh's blocks (all of it at N = 1)
            return ctx.find(pin_a, sa, pin_b, sb, mode=mode, pipeline=pipe, text=True, shard=shard)

        for _ in range(max(1, args.warmup)):
            step()
        barrier()
        d2h = 0
        t0 = time.perf_counter()
        for _ in range(steps):
            recs, text, _ = step()
            d2h += 8 * (8 + 8) + recs.nbytes + len(text)
        t_ms = reduce((time.perf_counter() - t0) * 1e3, MAX)
        barrier()
        return {"value": pairs_per_step * steps / (t_ms * 1e-3), "unit": UNIT, "ms_per_step": t_ms / steps,
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h // steps, "records": len(recs),
                "path": "runtime.Context.find -> mcx_find_intersections(host grids): H2D in column chunks (8 per "
                        "grid from 2^20 triangles) on two streams, each chunk packed as it lands (when one mesh is "
                        ">= 4x the other, the larger one's chunks are also searched as they land), solve, "
                        "records + sort + dedup + %.17g text on the device, D2H of records + text",
                "mode": mode_name, "pipeline": pipeline}

    primary = args.mode
    others = [m for m in ("prefilter", "brute", "cull") if m != primary]
    res_by_mode = {primary: measure(primary, True)}
    for m in others:
        res_by_mode[m] = measure(m, False)
    m1 = res_by_mode[primary]
    brute, cull, pre = res_by_mode["brute"], res_by_mode["cull"], res_by_mode["prefilter"]
    hit_counts = {k: v["hits"] for k, v in res_by_mode.items() if v["hits"] is not None}
    if len(set(hit_counts.values())) > 1:
        raise SystemExit(f"hit counts differ between modes: {hit_counts}")

    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    clocks = m1["clocks"] or {}
    f_max = clocks.get("sm_max_mhz") or 1965.0
    f_run = clocks.get("sm_mhz") or f_max

    # ---- roofline of the FP64 pair-test kernel (MCX_MODE_BRUTE, kernel-only events)
    st = brute["stats"]
    lane_ops = 8.0 * st["n_tested"] + 100.0 * st["n_aabb_pass"]
    achieved = lane_ops / (st["kernel_ms"] * 1e-3) / 1e12
    peak = sms * FP64_LANES_PER_CLK_PER_SM * f_max * 1e6 / 1e12
    peak_run = sms * FP64_LANES_PER_CLK_PER_SM * f_run * 1e6 / 1e12
    fp64_roofline = {
        "bound": "fp64_pipe", "kernel": "search_brute_kernel (MCX_MODE_BRUTE, the FP64 pair-test kernel)",
        "achieved": achieved, "peak": peak, "unit": "Tlane-op/s", "frac": achieved / peak,
        "frac_at_observed_clock": achieved / peak_run,
        "peak_source": f"{sms} SMs x {FP64_LANES_PER_CLK_PER_SM} FP64 lanes/clk x {f_max:.0f} MHz "
                       "(pipe rate measured: DADD 63.5 lanes/clk/SM, profiles/r01_pipes.jsonl; "
                       "MEASURED_PEAKS.json has no FP64 entry)",
        "work_per_launch": "8 FP64 compare lane-ops per pair + ~100 FP64 lane-ops per AABB survivor",
        "kernel_ms": st["kernel_ms"],
        "traffic": (1935119000.0 + 16355584.0) if args.config == "C3" else None,
        "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of one C3 launch, ncu --set full "
                        "(profiles/r02_ncu_brute_c3.txt): 1.95 GB vs 68 GB of algorithmic L2->SMEM tile "
                        "traffic; B's 67 MB of boxes are re-read from HBM ~29x per launch (L2 is split "
                        "over two dies) at ~4 GB/s - negligible against the FP64 bound"}
    # ---- roofline of the prefilter kernel: every pair = 6/16 IMAD-class op (fma-heavy pipe, 64
    # lanes/clk/SM) + 2/16 IADD3 + 1/4 LOP3 (alu pipe, 64 lanes/clk/SM): 0.75 instructions per
    # pair, so the fma pipe, the alu pipe and instruction issue all bind at 170.7 pairs/clk/SM
    pst = pre["stats"]
    pf_peak = sms * INT_LANES_PER_CLK_PER_SM / PREFILTER_IMAD_PER_PAIR * f_max * 1e6
    pf_achieved = pst["n_tested"] / (pst["kernel_ms"] * 1e-3)
    pf_roofline = {
        "bound": "int_pipes+issue", "kernel": "search_local_kernel (MCX_MODE_PREFILTER: quantised-box packed "
                                              "integer test of every pair, exact FP64 test of its passes)",
        "achieved": pf_achieved, "peak": pf_peak, "unit": "pair-tests/s", "frac": pf_achieved / pf_peak,
        "peak_source": f"{sms} SMs x {INT_LANES_PER_CLK_PER_SM} IMAD lanes/clk (fma-heavy pipe) / "
                       f"{PREFILTER_IMAD_PER_PAIR:.4f} IMAD-class ops per pair x {f_max:.0f} MHz (IMAD rate "
                       "measured 62.7 lanes/clk/SM, tools/microbench/hprefilter.cu); the alu pipe (6/16 per "
                       "pair) and issue (0.75 instructions per pair, 4 SMSP x 32 lanes/clk) bind at the same rate",
        "work_per_launch": "n_pairs quantised pair tests (4 of the 8 box compares at 3-bit resolution in the "
                           "warp's frame; 1/2 subtraction + 1/4 LOP3 each: two pairs per 32-bit subtraction "
                           "of 16-bit half words, four per accumulating LOP3) + per voting 64-record group "
                           "the per-record half test and the full 8-compare word test of its passes + "
                           "n_exact_tests FP64 box tests",
        "exact_tests_per_step": pst["n_exact_tests"], "kernel_ms": pst["kernel_ms"],
        "kernel_ms_note": "CUDA events around the whole call: fp32 box kernel (~0.03 ms) + search",
        "traffic": (68039680.0 + 3686144.0) if args.config == "C3" else None,
        "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of one C3 launch, ncu --set full "
                        "(profiles/r02_ncu_prefilter_c3.txt): B's 33 MB of fp32 boxes + A's, read ~once; the "
                        "1.1e12 pair tests touch only registers and shared memory"}
    roofline = pf_roofline if primary == "prefilter" else fp64_roofline
    fp64_block = {"mode": "brute", "value": brute["value"], "unit": UNIT, "ms_per_step": brute["ms_per_step"],
                  "kernel_ms": brute["kernel_ms"], "roofline": fp64_roofline,
                  "note": "every pair gets the 8-compare FP64 AABB test (the north star's FP64 kernel)"}
    pre_block = {"mode": "prefilter", "value": pre["value"], "unit": UNIT, "ms_per_step": pre["ms_per_step"],
                 "kernel_ms": pre["kernel_ms"], "roofline": pf_roofline,
                 "speedup_vs_fp64_brute": brute["ms_per_step"] / pre["ms_per_step"]}
    cst = cull["stats"]
    cull_block = {"mode": "cull", "value": cull["value"], "unit": UNIT + " (logical)",
                  "ms_per_step": cull["ms_per_step"], "search_wall_s": cull["ms_per_step"] / 1e3,
                  "kernel_ms": cull["kernel_ms"], "logical_pairs_per_step": cst["n_pairs"],
                  "executed_pair_tests_per_step": cst["n_tested"], "aabb_pass": cst["n_aabb_pass"],
                  "speedup_vs_brute": brute["ms_per_step"] / cull["ms_per_step"],
                  "speedup_vs_prefilter": pre["ms_per_step"] / cull["ms_per_step"], "hits": cull["hits"],
                  "executed_fp64_frac": (8.0 * cst["n_tested"] + 100.0 * cst["n_aabb_pass"]) /
                                        (cst["kernel_ms"] * 1e-3) / 1e12 / peak,
                  "note": "identical hit set / AABB-pass / singular counts; exact union-box culling over the "
                          "tiled storage order skips only provably disjoint pairs"}

    # ---- roofline of the fused pack kernel (mcx_pack of A: boxes + perm + level boxes)
    def measure_pack(reps=10):
        L = _lib.load()
        outs = [torch.empty_like(t) for t in (Am.box, Am.perm, Am.gbox, Am.tbox, Am.bbox, Am.status)]
        ts = []
        for it in range(reps + 2):
            flush.zero_()  # the pack reads its grid from HBM, not from the L2 copy a previous launch left
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rc = L.mcx_pack(Am.coords.data_ptr(), Am.N, Am.M, _lib.ORDER_TILED, *(o.data_ptr() for o in outs), local,
                            stream.cuda_stream)
            e1.record(stream)
            _lib.check(rc, "mcx_pack")
            torch.cuda.synchronize(dev)
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        n = Am.n_tri
        alg = Am.coords.numel() * 8 + n * (64 + 4) + (Am.gbox.numel() + Am.tbox.numel() + Am.bbox.numel()) * 8
        peak, src = hbm_peak()
        return {"bound": "hbm", "kernel": "pack_kernel (mcx_pack of A: exact triangle boxes in the tiled order, "
                                           "perm, group/tile/block union boxes; persistent CTAs, cp.async grid window)",
                "achieved": alg / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": alg / (ms * 1e-3) / 1e9 / peak, "peak_source": src,
                "work_per_launch": f"{alg} algorithmic bytes: grid 32 B/vertex read once, 64 B box + 4 B perm per "
                                   "record, 64 B per 32/512/1024-record union box written",
                "kernel_ms": ms, "timing": "CUDA events on the launching stream around one mcx_pack, L2 flushed "
                                           "(256 MB write) before each, median of 10",
                "traffic": (16805120.0 + 17992704.0) if args.config == "C3" else None,
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of one C3 launch, ncu --set full "
                                "(profiles/r02_ncu_pack_c3.txt): the 71 MB of boxes stay in the 126 MB L2 during the "
                                "launch and are written back later",
                "note": "in find_intersections every chunk's pack overlaps the next chunk's PCIe copy, so only the "
                        "last chunk's pack is on the e2e critical path"}

    pack_roofline = measure_pack()

    e2e = None
    if not args.no_e2e:
        floor_ms = reduce(h2d_floor(), MAX)
        e2e = measure_e2e(primary, "triangle", m1["pairs"] // args.steps, args.steps)
        e2e["h2d_floor_ms"] = floor_ms
        cull_spec = measure_e2e("cull", "spec", m1["pairs"] // args.steps, max(args.steps, 10))
        cull_spec["over_h2d_floor_ms"] = cull_spec["ms_per_step"] - floor_ms
        cull_spec["note"] = ("the product default (isect.find_intersections: SPEC-literal pipeline on the culling "
                             "kernels); logical pair tests per second")
        e2e["other_modes"] = {"cull_spec": cull_spec,
                              "brute_triangle": measure_e2e("brute", "triangle", m1["pairs"] // args.steps, min(args.steps, 3))}
        if world > 1:  # per-rank fixed costs (every rank uploads and packs both grids) vs its shard's kernel
            mine = {"rank": rank, "h2d_floor_ms": h2d_floor(), "e2e_ms": e2e["ms_per_step"],
                    "kernel_ms": m1["stats"]["kernel_ms"], "cull_spec_e2e_ms": cull_spec["ms_per_step"]}
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            e2e["per_rank"] = allr

    # ---- the paper's own benchmark shape: 14-layer search, 108 layer-pair tasks of
    # N1 = 1024 x N2 = 2048 grids with 35 s-values per half-layer (PAPER.md "Computational
    # Results": 2,424,307,712 quad pairs / 9,697,230,848 triangle pairs per task), one batch.
    paper = None
    if not args.no_paper:
        from paper_2109_14814_b200.layers import enumerate_layer_pairs
        from paper_2109_14814_b200.mesh import half_layer, layered_mesh
        um = layered_mesh(1024, "unstable", 14, 1.6, 0.1, 1, K=17, per_layer=34)
        sm = layered_mesh(2048, "stable", 14, 1 / 1.6, 0.1, 2, K=17, per_layer=34)
        plan = enumerate_layer_pairs(um, sm, 14)
        dm = {}

        def half(mesh, key, n, sg):
            if key not in dm:
                dm[key] = D.DeviceMesh(np.ascontiguousarray(half_layer(mesh, n, 1 if sg == "+" else -1).coords), local)
            return dm[key]

        pairs = [(half(um, ("u", n1, s1), n1, s1), half(sm, ("s", n2, s2), n2, s2)) for n1, s1, n2, s2 in plan.tasks]
        paper = {"workload": "synthetic layered meshes, U 1024 x S 2048 theta points, 14 layers, 35 s-values per "
                             "half-layer, all 108 layer-pair tasks in one mcx_search_batch job",
                 "tasks": len(pairs), "published": {"dgx_v100_full_search_s": 16.0, "laptop_full_search_s": 62.0,
                                                    "dgx_v100_bbox_kernel_per_task_s": 0.03}}
        for mname in ("prefilter", "brute", "cull"):
            for _ in range(max(1, args.warmup)):
                res = D.search_batch(pairs, mode=modes[mname], shard=shard, stream=stream)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                res = D.search_batch(pairs, mode=modes[mname], shard=shard, stream=stream)
            e1.record(stream)
            barrier()
            ms = reduce(e0.elapsed_time(e1), MAX) / args.steps
            pairs_total = reduce(sum(r.stats["n_pairs"] for r in res), SUM)
            paper[mname] = {"full_search_s": ms / 1e3, "pair_tests_per_s": pairs_total / (ms * 1e-3),
                            "pairs": pairs_total, "executed_pair_tests": reduce(sum(r.stats["n_tested"] for r in res), SUM),
                            "hits": reduce(sum(len(r.hits) for r in res), SUM),
                            "speedup_vs_dgx_v100_full_search": 16.0 / (ms / 1e3)}
        # the whole plan through the reference-facing task loop: layers.search_plan (each distinct
        # half-layer uploaded and packed once, one batched search, records + text on the device)
        if rank == 0 and world == 1:
            from paper_2109_14814_b200 import layers as LY
            for pipe in ("spec", "triangle"):
                LY.search_plan(um, sm, plan, pipeline=pipe, text=True)
                ts = []
                for _ in range(3):
                    t0 = time.perf_counter()
                    pr = LY.search_plan(um, sm, plan, pipeline=pipe, text=True)
                    ts.append(time.perf_counter() - t0)
                paper[f"search_plan_e2e_{pipe}"] = {
                    "wall_s": min(ts), "records": len(pr.records), "text_bytes": len(pr.text),
                    "h2d_bytes": int(um.coords.nbytes + sm.coords.nbytes + um.s_values.nbytes + sm.s_values.nbytes),
                    "speedup_vs_dgx_v100_full_search": 16.0 / min(ts),
                    "path": "layers.search_plan: the two host meshes uploaded once each (pageable NumPy), 56 "
                            "half-layers as zero-copy column views packed in place, one mcx_intersect (108 tasks "
                            "in one batched search), records + text on the device"}
        # the paper's own GPU stage per task: quad-level bbox + Moller candidates (pair_candidates)
        if rank == 0:
            busiest = max(range(len(res)), key=lambda k: res[k].stats["n_aabb_pass"])
            n1, s1, n2, s2 = plan.tasks[busiest]
            hu = np.ascontiguousarray(half_layer(um, n1, 1 if s1 == "+" else -1).coords)
            hs = np.ascontiguousarray(half_layer(sm, n2, 1 if s2 == "+" else -1).coords)
            nq = (hu.shape[2] * (hu.shape[1] - 1)) * (hs.shape[2] * (hs.shape[1] - 1))
            D.pair_candidates_device(hu, hs, device=local)
            torch.cuda.synchronize(dev)
            reps = 5
            t0 = time.perf_counter()
            for _ in range(reps):
                cand = D.pair_candidates_device(hu, hs, device=local)
            torch.cuda.synchronize(dev)
            dt = (time.perf_counter() - t0) / reps
            Hu, Hs = dm[("u", n1, s1)], dm[("s", n2, s2)]
            D.pair_candidates_mesh(Hu, Hs, stream=stream)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(reps):
                cand2, pst = D.pair_candidates_mesh(Hu, Hs, stream=stream)
            torch.cuda.synchronize(dev)
            dt2 = (time.perf_counter() - t0) / reps
            paper["pair_candidates_one_task"] = {
                "task": f"(U{n1}{s1}, S{n2}{s2}) (the plan's busiest task) quad pairs, SPEC-literal bbox + "
                        "Moller + compaction",
                "quad_pairs": nq, "candidates": int(len(cand)),
                "brute": {"seconds": dt, "quad_pairs_per_s": nq / dt, "speedup_vs_dgx_v100_bbox_kernel": 0.03 / dt,
                          "path": "host grids -> mcx_pair_candidates (every quad pair tested)"},
                "cull": {"seconds": dt2, "quad_pairs_per_s": nq / dt2, "speedup_vs_dgx_v100_bbox_kernel": 0.03 / dt2,
                         "quad_box_tests": int(pst["n_tested"]), "same_candidates": bool(np.array_equal(cand, cand2)),
                         "path": "packed meshes -> mcx_pair_candidates_mesh (exact union-box culling)"}}

    # ---- the 8-GPU partition of the headline workload, run shard by shard on this GPU
    # (world == 1 only): per-shard device time of the primary mode; the max over shards is
    # what an 8-GPU run's max-over-ranks timing would see for the kernel alone
    shards8 = None
    if world == 1 and not args.no_c5:
        mode = modes[primary]
        ms8 = []
        for g in range(8):
            D.search_device(Am, Bm, mode=mode, shard=(g, 8), stream=stream)
            ms8.append(min(D.search_device(Am, Bm, mode=mode, shard=(g, 8), stream=stream, timing=True)
                           .stats["kernel_ms"] for _ in range(2)))
        shards8 = {"mode": primary, "per_shard_kernel_ms": ms8, "max_over_mean": max(ms8) / statistics.mean(ms8),
                   "sum_over_unsharded": sum(ms8) / m1["kernel_ms"],
                   "pairs_per_s_if_8_gpus": desc["pairs_per_step"] / (max(ms8) * 1e-3),
                   "note": "NOT a multi-GPU measurement: the 8 cyclic A-block shards of this workload timed one "
                           "after another on one GPU (kernel events); the last field is the pair rate 8 GPUs "
                           "would reach if each ran its shard as fast, with no host or copy overhead"}

    # ---- configs[4]: unbalanced high-hit-density pair (C5hd: 4.2M x 65k triangles, 13,226
    # hits clustered in A's first quarter) - hit compaction, and the 8-GPU cyclic partition's
    # balance measured shard by shard on this GPU (world == 1 only)
    c5 = None
    if world == 1 and not args.no_c5:
        A5, _, B5, _ = config_pair("C5hd")
        A5m, B5m = D.DeviceMesh(A5, local), D.DeviceMesh(B5, local)
        c5 = {"workload": workload_desc("C5hd", A5, B5)["workload"] + " (configs[4], high-hit-density variant)"}
        for mname in ("prefilter", "brute", "cull"):
            for _ in range(max(1, args.warmup)):
                D.search_device(A5m, B5m, mode=modes[mname], stream=stream)
            ts = [D.search_device(A5m, B5m, mode=modes[mname], stream=stream, timing=True) for _ in range(args.steps)]
            ms = statistics.median(r.stats["kernel_ms"] for r in ts)
            c5[mname] = {"kernel_ms": ms, "pair_tests_per_s": ts[0].stats["n_pairs"] / (ms * 1e-3),
                         "hits": int(ts[0].stats["n_hits"]), "aabb_pass": int(ts[0].stats["n_aabb_pass"])}
        shards = []
        for g in range(8):
            r = D.search_device(A5m, B5m, mode=modes["prefilter"], shard=(g, 8), stream=stream, timing=True)
            shards.append({"kernel_ms": r.stats["kernel_ms"], "hits": int(r.stats["n_hits"]),
                           "aabb_pass": int(r.stats["n_aabb_pass"])})
        kms = [x["kernel_ms"] for x in shards]
        hs = [x["hits"] for x in shards]
        c5["prefilter_8_cyclic_shards"] = {
            "per_shard": shards, "time_max_over_mean": max(kms) / statistics.mean(kms),
            "hits_max_over_mean": max(hs) / statistics.mean(hs), "hits_total": sum(hs),
            "note": "the 8-GPU partition (A blocks dealt cyclically) run shard by shard on one GPU"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_reference_sample(A, B, rows=1024)  # warm-up, as the reference arm does
        cpu_steps = min(max(args.steps, 1), 5)
        runs = [cpu_reference_sample(A, B) for _ in range(cpu_steps)]
        s = runs[-1]
        cpu = {"value": sum(r["pairs"] for r in runs) / sum(r["seconds"] for r in runs), "unit": UNIT,
               "cores": s["threads"], "kind": "port",
               "sample": f"C port of the SPEC all-pairs search, A triangles [0, {s['a_triangles']}) x all B "
                         f"({s['pairs']:.3e} pairs per step, packing excluded), mean of {cpu_steps} steps after a "
                         "warm-up - the same slice, code and protocol as --impl reference",
               "step_values": [r["value"] for r in runs], "cpu": cpu_model(),
               "numpy_parallel": cpu_numpy_parallel_sample(A, B),
               "spec_literal_serial": cpu_spec_literal_sample(A, B)}
        # the culling counterpart on the CPU: the C oracle's exact x-sweep-and-prune over the
        # whole workload (all threads, packing included) - the CPU analogue of `cull`
        from oracle import c_oracle
        t0 = time.perf_counter()
        rs = c_oracle.search(A, B, sweep=True)
        sw = time.perf_counter() - t0
        cpu["sweep_and_prune_full_search"] = {
            "seconds": sw, "hits": int(len(rs["ia"])), "threads": c_oracle.max_threads(),
            "vs_gpu_cull_step": sw / (cull["ms_per_step"] * 1e-3),
            "note": "exact CPU culling search of the full workload (C oracle x-sweep), packing included"}

    if rank == 0:
        line = {"metric": METRIC, "value": m1["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": m1["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": bench_config(desc, primary, world),
                "search_wall_s": m1["ms_per_step"] / 1e3, "hits": m1["hits"], "kernel_ms": m1["kernel_ms"],
                "roofline": roofline, "fp64_brute": fp64_block, "prefilter": pre_block, "cull": cull_block,
                "pack": pack_roofline,
                "e2e": e2e, "cpu_baseline": cpu, "paper_workload": paper, "c5_unbalanced": c5, "shards8": shards8, "clocks": m1["clocks"],
                "gpu_launches": m1["launches"], "gpu": props.name, "sms": sms}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
