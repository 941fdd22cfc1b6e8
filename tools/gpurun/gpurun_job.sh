#!/bin/bash
# one GPU session: tests, smoke, bench, launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --trace-steps 2000 --no-cpu > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/pytest_gpu.log
cat gpurun_out/smoke.log gpurun_out/bench_small.json gpurun_out/bench.json
tail -5 gpurun_out/bench.err
