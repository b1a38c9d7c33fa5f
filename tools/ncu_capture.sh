#!/bin/bash
# One `ncu --set full` capture of the first launch of a kernel, exported on
# the GPU box as CSV (raw counters + per-source-line page), report deleted so
# gpurun_out/ stays small.  usage: tools/ncu_capture.sh NAME KERNEL_REGEX cmd...
name=$1; kre=$2; shift 2
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$kre" -c 1 -o "gpurun_out/$name" "$@" > "gpurun_out/$name.log" 2>&1
ncu -i "gpurun_out/$name.ncu-rep" --page raw --csv > "gpurun_out/${name}_raw.csv" 2>/dev/null
ncu -i "gpurun_out/$name.ncu-rep" --page source --csv --print-source sass > "gpurun_out/${name}_sass.csv" 2>/dev/null
ncu -i "gpurun_out/$name.ncu-rep" --page details --csv > "gpurun_out/${name}_details.csv" 2>/dev/null
rm -f "gpurun_out/$name.ncu-rep"
tail -n 2 "gpurun_out/$name.log"
