#!/bin/bash
# One GPU-box pass of the round's evidence (run under gpurun from the repo root):
#   pytest -m gpu, smoke(), bench.py for every config + the reference arm, the
#   ncu launch list of the default bench command and one --set full capture of
#   the headline kernel.  Everything lands in gpurun_out/ with prefix $1.
set -u
P=${1:-r02}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${P}_gpu_tests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.txt 2>&1
# the ms-scale steps of cfg1 / cfg3 get more steps: one NVML sample landing in a 0.6 ms step costs it ~1 ms
for k in 1 2 3 5 4; do
  case $k in 1) S="--steps 50";; 3) S="--steps 20";; *) S="";; esac
  timeout 900 python bench.py --config $k $S > gpurun_out/${P}_bench_cfg$k.json 2> gpurun_out/${P}_bench_cfg$k.err
done
timeout 900 python bench.py --impl reference > gpurun_out/${P}_bench_cfg4_reference.json 2> gpurun_out/${P}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${P}_launches_cfg4.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${P}_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lse_tc -s 1 -c 1 \
  -o gpurun_out/${P}_lse_tc_cfg4 python tools/prof_half_step.py --config 4 --reps 3 > gpurun_out/${P}_ncu_full.log 2>&1
# summaries are made on the box and the reports dropped (gpurun_out/ is capped at 64 MiB)
summarize() {  # $1 = report stem, $2 = summary name
  if [ -f gpurun_out/$1.ncu-rep ]; then
    python profiles/summarize_ncu.py gpurun_out/$1.ncu-rep > gpurun_out/$2.txt 2>&1
    ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_src.csv 2>/dev/null \
      && python tools/ncu_stalls.py gpurun_out/$1_src.csv > gpurun_out/$2_stalls.txt 2>&1
    rm -f gpurun_out/$1.ncu-rep gpurun_out/$1_src.csv
  fi
}
summarize ${P}_lse_tc_cfg4 ${P}_ncu_lse_tc_anchored_cfg4
for k in 2 5; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lse_tc -s 1 -c 1 \
    -o gpurun_out/${P}_lse_tc_cfg$k python tools/prof_half_step.py --config $k --reps 3 > gpurun_out/${P}_ncu_full_cfg$k.log 2>&1
  summarize ${P}_lse_tc_cfg$k ${P}_ncu_lse_tc_anchored_cfg$k
done
# cfg1 (persistent small solve) and cfg3 (K3c): launch list of the bench command + one full capture each
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${P}_launches_cfg1.csv python bench.py --config 1 --steps 2 --warmup 1 > gpurun_out/${P}_ncu_launches_cfg1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:solve_small -s 2 -c 1 \
  -o gpurun_out/${P}_solve_small_cfg1 python tools/small_builds.py > gpurun_out/${P}_ncu_full_cfg1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dense_cluster -s 1 -c 1 \
  -o gpurun_out/${P}_dense_cluster_cfg3 python tools/dense_prof.py > gpurun_out/${P}_ncu_full_cfg3.log 2>&1
summarize ${P}_solve_small_cfg1 ${P}_ncu_solve_small_cfg1
summarize ${P}_dense_cluster_cfg3 ${P}_ncu_dense_cluster_cfg3
timeout 300 python tools/small_trace.py > gpurun_out/${P}_small_trace_cfg1.txt 2>&1
timeout 300 python tools/cfg1_profile.py > gpurun_out/${P}_cfg1_profile.txt 2>&1
tail -3 gpurun_out/${P}_gpu_tests.txt; tail -1 gpurun_out/${P}_smoke.txt
for k in 1 2 3 5 4; do python -c "
import json,sys
for l in open('gpurun_out/${P}_bench_cfg$k.json'):
    if l.startswith('{'):
        d=json.loads(l); r=d.get('roofline') or {}
        print('cfg$k', '%.3e'%d['value'], 'e2e %.3e'%d.get('e2e',{}).get('value',0), 'frac %.3f'%r.get('frac',0), 'ttt %.2f ms'%d['run']['time_to_tolerance_ms'], d['clocks'])
"; done
