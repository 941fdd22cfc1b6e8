#!/bin/bash
# min-energy parity tests + c4 / c5 bench (prebuilt .so from the snapshot)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "fast_scan or c4 or grid or golden or parity or large" 2>&1 | tail -3 > gpurun_out/pytest_c4.log
for c in c4 c5; do timeout 600 python bench.py --config $c --streams 262144 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_${c}it.json 2> /dev/null; done
cat gpurun_out/pytest_c4.log
for c in c4 c5; do tail -1 gpurun_out/b_${c}it.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '%.4g' % d['value'], round(d['roofline']['frac'],3), d['quality'].get('full_scan_fraction'))"; done
