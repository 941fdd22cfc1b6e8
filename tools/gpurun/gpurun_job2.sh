#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -rA 2>&1 | tail -60 > gpurun_out/pytest_gpu.log
for L in 1 2 4; do timeout 300 python bench.py --steps 3 --warmup 2 --trace-steps 2000 --no-cpu --no-e2e --lanes $L > gpurun_out/bench_l$L.json 2>/dev/null; done
timeout 300 python bench.py --steps 3 --warmup 2 --trace-steps 2000 --no-cpu --no-e2e --tpb 64 > gpurun_out/bench_tpb64.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --trace-steps 1000 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -o gpurun_out/prof_run python bench.py --steps 1 --warmup 0 --trace-steps 200 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -c 2500 gpurun_out/pytest_gpu.log
for f in gpurun_out/bench_l*.json gpurun_out/bench_tpb64.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms_per_launch'])"; done
ls -la gpurun_out
