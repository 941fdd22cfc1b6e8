#!/bin/bash
# max-accuracy parity tests + c3 bench (prebuilt .so from the snapshot)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "max_accuracy or c3 or golden or baselines or parity" 2>&1 | tail -5 > gpurun_out/pytest_c3.log
timeout 300 python bench.py --config c3 --no-cpu > gpurun_out/b_c3it.json 2> gpurun_out/b_c3it.err
cat gpurun_out/pytest_c3.log
tail -1 gpurun_out/b_c3it.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d.get('full_scan_fraction'))"
