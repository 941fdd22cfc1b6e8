#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 2 --trace-steps 2000 --no-cpu --no-e2e > gpurun_out/b11_c2.json 2>/dev/null
timeout 600 python bench.py --config c4 --streams 262144 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/b11_c4.json 2> /dev/null
timeout 600 python bench.py --config c5 --streams 262144 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/b11_c5.json 2> gpurun_out/b11_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -o gpurun_out/prof_c5 python bench.py --config c5 --streams 16384 --steps 1 --warmup 0 --trace-steps 100 --no-cpu --no-e2e > gpurun_out/ncu_c5.log 2>&1
cat gpurun_out/pytest_gpu.log | tail -12
for f in gpurun_out/b11_*.json; do echo $f $(python -c "import json; d=json.load(open('$f')); print(round(d['value']/1e9,4), round(d['roofline']['frac'],3), d['config']['lanes_per_stream'], d['quality'])" 2>&1 | tail -1); done
