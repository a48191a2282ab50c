#!/bin/bash
# Shrink gpurun_out/ below gpurun's 64 MiB copy-back limit: export every .ncu-rep to csv pages
# (raw metrics, details, source) and drop reports larger than 12 MiB.
cd "$(dirname "$0")/.."
for r in gpurun_out/*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i "$r" --page raw --csv > "${b}_raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${b}_details.csv" 2>/dev/null
  ncu -i "$r" --page source --csv --print-source sass > "${b}_source.csv" 2>/dev/null
  gzip -f "${b}_source.csv"
  [ $(stat -c %s "$r") -gt 12000000 ] && rm -f "$r"
done
du -sh gpurun_out
