#!/bin/bash
# usage: tools/ncu_export.sh <report-stem>  — raw + SASS source pages as CSV next to the report, then drop the report
# (gpurun brings back at most 64 MiB; a --set full report of several kernels exceeds it)
rep="$1.ncu-rep"
ncu -i "$rep" --page raw --csv > "$1_raw.csv" 2>/dev/null
ncu -i "$rep" --page source --csv --print-source sass > "$1_src.csv" 2>/dev/null
gzip -f "$1_src.csv"
rm -f "$rep"
