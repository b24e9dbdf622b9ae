#!/bin/bash
# Regenerate every file under profiles/ on a B200 box (run from the repo root, e.g.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash tools/reproduce_profiles.sh'
# then copy gpurun_out/profiles/* into profiles/).  ~5 GPU-minutes.
set -euo pipefail
out=gpurun_out/profiles
mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build(); g.smoke()"
python bench.py > "$out/r01_bench_c3.json"
python - "$out" <<'PY'
import json, sys
d = json.loads(open(f"{sys.argv[1]}/r01_bench_c3.json").read().strip().splitlines()[-1])
json.dump(d["paper_workload"], open(f"{sys.argv[1]}/r01_paper_workload.json", "w"), indent=1)
json.dump(d["c5_unbalanced"], open(f"{sys.argv[1]}/r01_c5hd.json", "w"), indent=1)
PY
python tools/mode_table.py > "$out/r01_modes.jsonl"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c5 > /dev/null
python tools/ncu_summary.py list "$out/launches.csv" > "$out/r01_launches_bench_c3.txt"
ncu_rep() {  # name, kernel regex, launch count, mode
  ncu --set full --import-source on --clock-control none -k regex:"$2" -c "$3" \
      -o "$out/ncu_$1" python tools/profile_run.py --config C3 --mode "$4" --iters 1 > /dev/null
  python tools/ncu_summary.py rep "$out/ncu_$1.ncu-rep" > "$out/r01_ncu_$1_c3.txt"
}
ncu_rep prefilter "search_local|fbox" 2 prefilter
ncu_rep brute "search_brute" 1 brute
ncu_rep cull "cull_" 2 cull
ncu_rep pack "pack_kernel|levels_kernel" 2 cull
make -C tools/microbench > /dev/null 2>&1 || nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
    -o tools/microbench/hprefilter tools/microbench/hprefilter.cu
tools/microbench/hprefilter > "$out/r01_microbench_pairtest.jsonl"
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"; compute-sanitizer --tool $t --error-exitcode 7 python tools/sanitize_run.py 2>&1 | grep -E "SUMMARY|workload"
done > "$out/r01_sanitizer.txt"
