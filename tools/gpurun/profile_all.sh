#!/bin/bash
# Round-end evidence: launch list of the default bench, full ncu captures of
# run_kernel for c2 / c3 / c4 (exported as CSV on the box), DRAM traffic.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --trace-steps 1000 --no-cpu --no-e2e > /dev/null 2>&1
for cfg in c2 c3 c4; do
  case $cfg in
    c2) extra="--trace-steps 1000";;
    c3) extra="--config c3 --streams 65536 --trace-steps 200";;
    c4) extra="--config c4 --streams 65536 --trace-steps 100";;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -f -o /tmp/prof_$cfg python bench.py --steps 1 --warmup 0 $extra --no-cpu --no-e2e > gpurun_out/ncu_$cfg.log 2>&1
  ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_${cfg}_raw.csv
  ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_${cfg}_src.csv.gz
done
ls -la gpurun_out | tail -12
