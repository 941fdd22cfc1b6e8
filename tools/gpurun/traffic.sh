#!/bin/bash
# DRAM bytes + duration of every run_kernel launch of ONE bench step at the bench shape
# (c2 65,536 x 10,000; c3 2^20 x 1,000; c4 / c5 262,144-scenario grid sample x 1,000), and the
# launch list of a default c2 bench run; CSVs under gpurun_out/, summarised by tools/ncu_traffic.py
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:run_kernel --csv --log-file gpurun_out/traffic_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:run_kernel --csv --log-file gpurun_out/traffic_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:run_kernel --csv --log-file gpurun_out/traffic_c4.csv python bench.py --config c4 --total-streams 262144 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:run_kernel --csv --log-file gpurun_out/traffic_c5.csv python bench.py --config c5 --total-streams 262144 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out/traffic_*.csv gpurun_out/launches_c2.csv
