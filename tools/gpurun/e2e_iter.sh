#!/bin/bash
# HostStreamer pipeline check: its GPU tests, the pinned copy rates, c2 / c3 bench lines with e2e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "host_streamer" 2>&1 | tail -5
timeout 300 python tools/h2d_probe.py > gpurun_out/h2d_probe.json 2>&1; cat gpurun_out/h2d_probe.json
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/e_c2.json 2> gpurun_out/e_c2.err
timeout 900 python bench.py --config c3 --no-cpu > gpurun_out/e_c3.json 2> gpurun_out/e_c3.err
for c in c2 c3; do python -c "
import json; d=json.loads(open('gpurun_out/e_$c.json').read().strip().split('\n')[-1]); print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks'])" || tail -3 gpurun_out/e_$c.err; done
