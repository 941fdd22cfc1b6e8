#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -rf 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
for cfg in "1 64" "1 128"; do set -- $cfg
  timeout 300 python bench.py --steps 3 --warmup 2 --trace-steps 2000 --no-cpu --no-e2e --lanes $1 --tpb $2 > gpurun_out/b7_c2_l$1_t$2.json 2>/dev/null; done
timeout 600 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/b7_c3.json 2> gpurun_out/b7_c3.err
for L in 4 8 16; do timeout 600 python bench.py --config c4 --streams 262144 --steps 2 --warmup 1 --no-cpu --no-e2e --lanes $L > gpurun_out/b7_c4_l$L.json 2> /dev/null; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -o gpurun_out/prof_run7 python bench.py --steps 1 --warmup 0 --trace-steps 200 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -o gpurun_out/prof_run7_c3 python bench.py --config c3 --streams 65536 --steps 1 --warmup 0 --trace-steps 200 --no-cpu --no-e2e > gpurun_out/ncu_full_c3.log 2>&1
cat gpurun_out/pytest_gpu.log | tail -8
for f in gpurun_out/b7_*.json; do echo $f $(python -c "import json; d=json.load(open('$f')); print(round(d['value']/1e9,4), round(d['roofline']['frac'],3), d['config']['lanes_per_stream'], d['quality']['fp64_rerank_fraction'])" 2>&1 | tail -1); done
