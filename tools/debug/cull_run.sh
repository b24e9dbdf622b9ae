# cull-path experiment: GPU tests, mode table, device-stamp trace of find_intersections,
# ncu of the culling kernels (C3, C5hd) and the source-line stall table of level 1
set -uo pipefail
out=gpurun_out/cull
mkdir -p $out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -2 $out/gputest.log
python tools/mode_table.py > $out/modes.jsonl 2>&1
MCX_TRACE=2 python tools/debug/trace_find.py C3 > $out/trace_c3.txt 2>&1
for cfg in C3 C5hd; do
ncu --set full --import-source on --clock-control none -k regex:"cull_|solve" -c 3 -o $out/ncu_cull_$cfg python tools/profile_run.py --config $cfg --mode cull --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py rep $out/ncu_cull_$cfg.ncu-rep > $out/ncu_cull_$cfg.txt 2>&1
done
ncu -i $out/ncu_cull_C3.ncu-rep -k regex:cull_blocks --page source --csv --print-source sass > $out/src_blocks.csv 2>&1
rm -f $out/*.ncu-rep
