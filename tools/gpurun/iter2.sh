#!/bin/bash
# iteration: selected GPU tests, c2 A/B, c4, ncu source capture of c2 (exported as CSV on the box)
mkdir -p gpurun_out
K=${1:-}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "$K" ]; then timeout 900 python -m pytest tests -q -m gpu -x -k "$K" 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
else timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; fi
timeout 300 python bench.py --steps 3 --warmup 3 --trace-steps 2000 --no-cpu --no-e2e > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 300 python bench.py --steps 3 --warmup 3 --trace-steps 2000 --no-cpu --no-e2e --flags 4 > gpurun_out/b_c2_nofast.json 2> /dev/null
timeout 600 python bench.py --config c4 --streams 262144 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_c4.json 2> /dev/null
timeout 600 python bench.py --config c4 --streams 262144 --steps 2 --warmup 3 --no-cpu --no-e2e --flags 4 > gpurun_out/b_c4_nofast.json 2> /dev/null
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_c3.json 2> /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:run_kernel -c 1 -f -o /tmp/prof_c2 python bench.py --steps 1 --warmup 0 --trace-steps 1000 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv
ncu -i /tmp/prof_c2.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/prof_c2_src.csv.gz
tail -4 gpurun_out/pytest_gpu.log
for f in gpurun_out/b_c2.json gpurun_out/b_c2_nofast.json gpurun_out/b_c4.json gpurun_out/b_c4_nofast.json gpurun_out/b_c3.json; do echo $f $(python -c "import json; d=json.load(open('$f')); print('%.4g' % d['value'], round(d['roofline']['frac'],3), d['quality']['fp64_rerank_fraction'], d['quality'].get('full_scan_fraction'), d['quality']['mean_energy_j'])" 2>&1 | tail -1); done
