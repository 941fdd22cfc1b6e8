#!/bin/bash
# iteration: GPU tests (optional -k filter $1) + c3 / c4 / c2 bench lines (no CPU baseline)
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 1200 python -m pytest tests -q -m gpu -x -k "$1" > gpurun_out/pytest_iter.log 2>&1
else timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1; fi
tail -3 gpurun_out/pytest_iter.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 3 --no-cpu --no-e2e > gpurun_out/it_$cfg.json 2> gpurun_out/it_$cfg.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/it_$cfg.json').read().strip().split('\n')[-1]); print('$cfg', d['value'], d['roofline']['frac'], d['quality'].get('full_scan_fraction'))"
done
timeout 600 python bench.py --config c4 --total-streams 262144 --steps 2 --no-cpu --no-e2e > gpurun_out/it_c4.json 2> gpurun_out/it_c4.err
python -c "import json,sys; d=json.loads(open('gpurun_out/it_c4.json').read().strip().split('\n')[-1]); print('c4', d['value'], d['roofline']['frac'])"
