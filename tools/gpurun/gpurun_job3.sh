#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -rf 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
for cfg in "1 32" "1 64" "1 128" "2 64" "2 128" "4 64"; do set -- $cfg
  timeout 300 python bench.py --steps 3 --warmup 2 --trace-steps 2000 --no-cpu --no-e2e --lanes $1 --tpb $2 > gpurun_out/bench_l$1_t$2.json 2>/dev/null; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -o gpurun_out/prof_run3 python bench.py --steps 1 --warmup 0 --trace-steps 200 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/pytest_gpu.log | tail -12
for f in gpurun_out/bench_l*_t*.json; do echo $f $(python -c "import json; d=json.load(open('$f')); print(round(d['value']/1e9,3), round(d['roofline']['frac'],3), d['quality']['fp64_rerank_fraction'])"); done
