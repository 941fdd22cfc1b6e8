#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -f -o /tmp/prof_c2 python bench.py --steps 1 --warmup 0 --trace-steps 1000 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv
ncu -i /tmp/prof_c2.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_c2_src.csv.gz
