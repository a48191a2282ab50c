#!/bin/bash
# Turn the gpurun_out/ artefacts of tools/refresh_profiles.sh into the committed profiles/ files.
# usage: tools/summarize_round.sh [ROUND=r1] [TRACE_SRC=paper_2410_14128_b200/csrc/trace.cu]
cd "$(dirname "$0")/.."
R=${1:-r1}
SRC=${2:-paper_2410_14128_b200/csrc/trace.cu}
REP=gpurun_out/full_cfg4.ncu-rep
ncu -i $REP --page source --csv --print-source cuda,sass > gpurun_out/full_cfg4_src.csv 2>/dev/null
ncu -i $REP --page source --csv --print-source sass > gpurun_out/full_cfg4_sass.csv 2>/dev/null
{
  python tools/summarize_ncu.py $REP 2073600 "round ${R#r}, cfg4 2048^3 city, R(4,4,4) G(7), stack, one thread per ray (tools/prof_trace.py)"
  echo; echo "## code regions (tools/ncu_regions.py; \`start\` includes the iteration prologue)"; echo; echo '```'
  python tools/ncu_regions.py $SRC gpurun_out/full_cfg4_src.csv 2073600
  echo '```'; echo "## stall reasons"; echo; echo '```'
  python tools/ncu_sass_summary.py gpurun_out/full_cfg4_sass.csv 0
  echo '```'
} > profiles/${R}_cfg4_trace_kernel.md
python tools/summarize_launches.py gpurun_out/launches_cfg4.csv > profiles/${R}_cfg4_launches.csv
for c in cfg4 cfg2 cfg3 cfg5 cfg4i t512 cfg1; do
  [ -f gpurun_out/traffic_$c.csv ] && python tools/traffic_json.py gpurun_out/traffic_$c.csv gpurun_out/traffic_$c.out
  [ -f gpurun_out/bench_$c.json ] || continue
  cp gpurun_out/bench_$c.json profiles/${R}_bench_$c.json
  python tools/sweep_table.py gpurun_out/bench_$c.json > profiles/${R}_${c}_sweep.md
done
{ echo "# Pareto frontiers, round ${R#r} (tools/pareto.py over profiles/${R}_bench_*.json)"; echo
  for c in cfg4 t512 cfg2 cfg3 cfg5; do python tools/pareto.py profiles/${R}_bench_$c.json; echo; done; } > profiles/${R}_pareto.md
echo "profiles/ updated for $R"
