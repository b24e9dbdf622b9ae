#!/bin/bash
# Regenerate the round-2 files under profiles/ on a B200 box (run from the repo root, e.g.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/reproduce_profiles.sh'
# then copy gpurun_out/profiles/* into profiles/).  ~10 GPU-minutes.
set -uo pipefail
out=gpurun_out/profiles
mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$out/r02_smoke.txt" 2>&1
python bench.py > "$out/r02_bench_c3.json" 2> "$out/r02_bench_c3.err"
python bench.py --impl reference --steps 5 --warmup 2 > "$out/r02_reference_c3.json" 2> /dev/null
python tools/e2e_runtime.py C3 C2 C5 C5hd > "$out/r02_e2e_runtime.jsonl" 2>&1
python tools/microbench/pack_bench.py C2 C3 C5 > "$out/r02_pack.jsonl" 2>&1
python tools/mode_table.py > "$out/r02_modes.jsonl" 2>&1
# launch lists: a short bench run, and one find_intersections call (C3, cull, spec pipeline)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c5 --no-paper > /dev/null 2>&1
python tools/ncu_summary.py list "$out/launches.csv" > "$out/r02_launches_bench_c3.txt"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/find.csv" \
    python tools/debug/trace_find.py C3 > /dev/null 2>&1
python tools/ncu_summary.py list "$out/find.csv" > "$out/r02_launches_find_c3.txt"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/find5.csv" \
    python tools/debug/trace_find.py C5hd > /dev/null 2>&1
python tools/ncu_summary.py list "$out/find5.csv" > "$out/r02_launches_find_c5hd.txt"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/find5s.csv" \
    python tools/debug/trace_find.py C5 > /dev/null 2>&1
python tools/ncu_summary.py list "$out/find5s.csv" > "$out/r02_launches_find_c5.txt"
MCX_TRACE=1 python tools/debug/trace_find.py C3 > "$out/r02_trace_find_c3.txt" 2>&1
MCX_TRACE=1 python tools/debug/trace_find.py C5 > "$out/r02_trace_find_c5.txt" 2>&1
MCX_TRACE=1 python tools/debug/trace_find.py C5hd > "$out/r02_trace_find_c5hd.txt" 2>&1
ncu_rep() {  # name, kernel regex, launch count, config, mode
  ncu --set full --import-source on --clock-control none -k regex:"$2" -c "$3" \
      -o "$out/ncu_$1" python tools/profile_run.py --config "$4" --mode "$5" --iters 1 > /dev/null 2>&1
  python tools/ncu_summary.py rep "$out/ncu_$1.ncu-rep" > "$out/r02_ncu_$1.txt" 2>&1
}
ncu_rep prefilter_c3 "search_local|fbox|solve" 3 C3 prefilter
ncu_rep brute_c3 "search_brute|solve" 2 C3 brute
ncu_rep cull_c3 "cull_|solve" 3 C3 cull
ncu_rep pack_c3 "pack_kernel" 1 C3 cull
ncu_rep cull_c5hd "cull_|solve" 3 C5hd cull
python tools/ncu_opmix.py "$out/ncu_prefilter_c3.ncu-rep" > "$out/r02_opmix_prefilter_c3.txt" 2>&1
python tools/ncu_opmix.py "$out/ncu_pack_c3.ncu-rep" > "$out/r02_opmix_pack_c3.txt" 2>&1
rm -f "$out"/*.ncu-rep  # the merge back is capped at 64 MiB
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"; timeout 600 compute-sanitizer --tool $t --error-exitcode 7 python tools/sanitize_run.py 2>&1 \
    | grep -E "SUMMARY|workload"
done > "$out/r02_sanitizer.txt"
rm -f "$out"/*.csv
