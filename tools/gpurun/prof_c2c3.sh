#!/bin/bash
# ncu full captures (with SASS source counters) of run_kernel for c2 and c3;
# exported to CSV on the box (the .ncu-rep files are too large to bring back).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in c2 c3; do
  if [ $cfg = c2 ]; then extra="--trace-steps 200"; else extra="--config c3 --streams 131072 --trace-steps 100"; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -f -o /tmp/prof_$cfg python bench.py --steps 1 --warmup 0 $extra --no-cpu --no-e2e > gpurun_out/ncu_$cfg.log 2>&1
  ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_${cfg}_raw.csv
  ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_${cfg}_src.csv.gz
  ls -la /tmp/prof_$cfg.ncu-rep
done
ls -la gpurun_out
