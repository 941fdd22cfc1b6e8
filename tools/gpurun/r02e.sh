#!/bin/bash
# After the HostStreamer ring / cross-pass changes: GPU suite + smoke, c2 (default and the driver's K/W), c3
mkdir -p gpurun_out
bash tools/gpurun/tests.sh
timeout 900 python bench.py > gpurun_out/e_c2def.json 2> gpurun_out/e_c2def.err; tail -1 gpurun_out/e_c2def.json | cut -c1-120
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/e_c2.json 2> gpurun_out/e_c2.err; tail -1 gpurun_out/e_c2.json | cut -c1-120
timeout 900 python bench.py --config c3 > gpurun_out/e_c3.json 2> gpurun_out/e_c3.err; tail -1 gpurun_out/e_c3.json | cut -c1-120
for c in c2def c2 c3; do python -c "
import json; d=json.loads(open('gpurun_out/e_$c.json').read().strip().split('\n')[-1]); print('$c', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], d['clocks'])"; done
