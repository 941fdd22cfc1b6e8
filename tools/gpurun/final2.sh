#!/bin/bash
# Evidence refresh after the c3 / c4 changes: full GPU tests + smoke, c2 / c3 /
# c4 / c5 / reference lines, c3 ncu capture at its bench shape.
mkdir -p gpurun_out
bash tools/gpurun/tests.sh
timeout 900 python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err
timeout 900 python bench.py --config c4 --streams 262144 --steps 2 --warmup 3 --no-e2e > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err
timeout 900 python bench.py --config c5 --streams 262144 --steps 2 --warmup 3 --no-e2e > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err
bash tools/gpurun/prof_cfg.sh c3 --config c3 --streams 1048576 --trace-steps 30
for f in gpurun_out/f_c*.json gpurun_out/f_ref.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', '%.4g' % d['value'], d.get('roofline', {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks'))"; done
