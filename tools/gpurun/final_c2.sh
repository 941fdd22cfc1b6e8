#!/bin/bash
# c2 evidence with the final build: default bench line, launch list, ncu capture
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --trace-steps 1000 --no-cpu --no-e2e > /dev/null 2>&1
bash tools/gpurun/prof_cfg.sh c2 --trace-steps 1000
tail -1 gpurun_out/f_c2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
