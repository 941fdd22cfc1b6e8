#!/bin/bash
# ncu full capture of the (skip+1)-th run_kernel launch: $1 = tag, $2 = launches to skip, $3.. = bench.py args
tag=$1; skip=$2; shift 2
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:run_kernel --launch-skip $skip -c 1 -f -o /tmp/prof_$tag python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e "$@" > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_${tag}_src.csv.gz
