#!/bin/bash
# GPU tests + smoke + bench lines for c3 / c2 / c4 / c5 (sampled grid)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1
tail -2 gpurun_out/pytest_iter.log; grep -E "^FAILED|Error" gpurun_out/pytest_iter.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 3 --no-cpu --no-e2e > gpurun_out/it_$cfg.json 2> gpurun_out/it_$cfg.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/it_$cfg.json').read().strip().split('\n')[-1]); print('$cfg', d['value'], d['roofline']['frac'], d['quality'].get('full_scan_fraction'), d['gpu_launches'])" || tail -3 gpurun_out/it_$cfg.err
done
for cfg in c4 c5; do
  timeout 900 python bench.py --config $cfg --total-streams 262144 --steps 2 --no-cpu --no-e2e > gpurun_out/it_$cfg.json 2> gpurun_out/it_$cfg.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/it_$cfg.json').read().strip().split('\n')[-1]); print('$cfg', d['value'], d['roofline']['frac'])" || tail -3 gpurun_out/it_$cfg.err
done
