#!/bin/bash
# Evidence pass: default bench (c2), reference arm, c3/c4/c5 lines, launch list, ncu captures.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
timeout 900 python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err
timeout 900 python bench.py --config c4 --streams 262144 --steps 2 --warmup 3 --no-e2e > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err
timeout 900 python bench.py --config c5 --streams 262144 --steps 2 --warmup 3 --no-e2e > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --trace-steps 1000 --no-cpu --no-e2e > /dev/null 2>&1
for cfg in c2 c3 c4; do
  case $cfg in
    c2) extra="--trace-steps 1000";;
    c3) extra="--config c3 --streams 1048576 --trace-steps 30";;
    c4) extra="--config c4 --streams 65536 --trace-steps 300";;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -f -o /tmp/prof_$cfg python bench.py --steps 1 --warmup 0 $extra --no-cpu --no-e2e > gpurun_out/ncu_$cfg.log 2>&1
  ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_${cfg}_raw.csv
  ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_${cfg}_src.csv.gz
done
for f in gpurun_out/f_*.json; do echo $f; head -c 400 $f; echo; done
