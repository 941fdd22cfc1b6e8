#!/bin/bash
# Iteration job: GPU tests (optionally a -k filter), then c2 bench A/B (fast scan vs --flags 4).
mkdir -p gpurun_out
K=${1:-}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "$K" ]; then timeout 900 python -m pytest tests -q -m gpu -x -k "$K" 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
else timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; fi
timeout 300 python bench.py --steps 3 --warmup 3 --trace-steps 2000 --no-cpu --no-e2e > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 300 python bench.py --steps 3 --warmup 3 --trace-steps 2000 --no-cpu --no-e2e --flags 4 > gpurun_out/b_c2_nofast.json 2> /dev/null
timeout 600 python bench.py --config c4 --streams 262144 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_c4.json 2> /dev/null
tail -4 gpurun_out/pytest_gpu.log
for f in gpurun_out/b_c2.json gpurun_out/b_c2_nofast.json gpurun_out/b_c4.json; do echo $f $(python -c "import json; d=json.load(open('$f')); print('%.4g' % d['value'], round(d['roofline']['frac'],3), d['quality']['fp64_rerank_fraction'], d['quality']['mean_energy_j'])" 2>&1 | tail -1); done
