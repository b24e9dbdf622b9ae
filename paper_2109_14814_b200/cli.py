"""Command line for the search stages of the reference pipeline.

Only the two stages on the mesh-search path are provided, with the reference's
flags and files:

    python -m paper_2109_14814_b200.cli layers --umesh U.mnf --smesh S.mnf --nmax N --plan plan.txt \
        [--include-core]
    python -m paper_2109_14814_b200.cli intersect --umesh U.mnf --smesh S.mnf --plan plan.txt \
        --backend cuda --out records.txt [--pipeline spec|triangle] [--mode cull|brute|prefilter] \
        [--devices 0,1,...]

Meshes are MNF1 files, the plan is ``n1 sign1 n2 sign2 tof`` per
line, records are ``n1 sign1 n2 sign2 gid x y px py a b c d theta_u
s_u theta_s s_s``.  Exit codes: 0 ok, 2 config error,
3 numerical / backend failure, 4 I/O error.
"""
from __future__ import annotations

import argparse
import json
import sys

from .errors import ConfigError, FileFormatError, ManiconnError, exit_code


def _parser():
    ap = argparse.ArgumentParser(prog="maniconn-b200")
    ap.add_argument("--log-level", default="warning")
    sub = ap.add_subparsers(dest="cmd", required=True)
    la = sub.add_parser("layers", help="enumerate the layer-pair plan")
    la.add_argument("--umesh", required=True)
    la.add_argument("--smesh", required=True)
    la.add_argument("--nmax", type=int, required=True)
    la.add_argument("--omega-p", type=float, default=1.0, help="perturbation frequency Ω_p for the TOF")
    la.add_argument("--plan", required=True)
    la.add_argument("--include-core", action="store_true",
                    help="also search the fundamental-domain cores |s| < D as layer 0 (SPEC.md:398)")
    it = sub.add_parser("intersect", help="search every planned layer pair for mesh intersections")
    it.add_argument("--umesh", required=True)
    it.add_argument("--smesh", required=True)
    it.add_argument("--plan", required=True)
    it.add_argument("--backend", default="cuda")
    it.add_argument("--mode", default="cull", choices=["cull", "brute", "prefilter"])
    it.add_argument("--pipeline", default="spec", choices=["spec", "triangle"],
                    help="spec: quad AABB + Moller + 4 precise tests (the reference's serial backend); "
                         "triangle: every triangle pair's boxes, then the precise test")
    it.add_argument("--device", type=int, default=0)
    it.add_argument("--devices", default=None, help="comma-separated GPU list; tasks are dealt out whole")
    it.add_argument("--out", required=True)
    it.add_argument("--manifest", default=None, help="optional JSON with per-layer-pair counters")
    return ap


def main(argv=None) -> int:
    from . import layers
    from .mesh import read_mesh

    try:
        args = _parser().parse_args(argv)
    except SystemExit as exc:
        return 2 if exc.code else 0
    try:
        if args.cmd == "layers":
            u, s = read_mesh(args.umesh), read_mesh(args.smesh)
            layers.write_plan(args.plan, layers.enumerate_layer_pairs(u, s, args.nmax, args.omega_p,
                                                                      include_core=args.include_core))
            return 0
        u, s = read_mesh(args.umesh), read_mesh(args.smesh)
        plan = layers.read_plan(args.plan)
        try:
            devices = [int(d) for d in args.devices.split(",")] if args.devices else [args.device]
        except ValueError:
            raise ConfigError(f"--devices must be a comma-separated list of integers, got {args.devices!r}") from None
        res = layers.search_plan(u, s, plan, backend=args.backend, mode=args.mode, pipeline=args.pipeline,
                                 devices=devices, text=True)
        with open(args.out, "wb") as fh:  # formatted on the device, byte-identical to write_records
            fh.write(res.text)
        if args.manifest:
            with open(args.manifest, "w") as fh:
                json.dump({"records": len(res.records), "tasks": res.stats}, fh, indent=1)
        return 0
    except (OSError, ConfigError, FileFormatError, ManiconnError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exit_code(exc)


if __name__ == "__main__":
    sys.exit(main())
