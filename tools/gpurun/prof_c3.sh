#!/bin/bash
# ncu full capture (SASS source counters) of run_kernel for c3 (65,536 x 200),
# exported to CSV on the box; optional $1 = tag for the output names.
tag=${1:-c3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -f -o /tmp/prof_$tag python bench.py --steps 1 --warmup 0 --config c3 --streams ${STREAMS:-65536} --trace-steps ${TSTEPS:-200} --no-cpu --no-e2e > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_${tag}_src.csv.gz
timeout 300 python bench.py --config c3 --no-cpu > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
tail -1 gpurun_out/b_$tag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
