#!/bin/bash
# A/B of a flag on c2 in one process family on one box (alternating runs)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
F=${1:-16}
for r in 1 2 3; do
  for fl in 0 $F; do
    timeout 300 python bench.py --steps 3 --warmup 3 --trace-steps 3000 --no-cpu --no-e2e --flags $fl 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flags $fl', '%.4g' % d['value'], round(d['roofline']['frac'],3))"
  done
done
