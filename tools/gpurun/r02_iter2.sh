#!/bin/bash
# GPU tests + c3 ncu capture + bench lines + sanitizers
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1
tail -2 gpurun_out/pytest_iter.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpurun/prof_cfg.sh c3n --config c3 --total-streams 1048576 --trace-steps 100
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 3 --no-cpu --no-e2e > gpurun_out/it_$cfg.json 2> gpurun_out/it_$cfg.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/it_$cfg.json').read().strip().split('\n')[-1]); print('$cfg', d['value'], d['roofline']['frac'], d['quality'].get('full_scan_fraction'), d['gpu_launches'])"
done
bash tools/gpurun/sanitize.sh
