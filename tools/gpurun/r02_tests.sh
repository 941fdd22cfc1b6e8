#!/bin/bash
# GPU tests (optionally -k filter), smoke; logs under gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "$1" ]; then timeout 1800 python -m pytest tests -q -m gpu -x -k "$1" > gpurun_out/pytest_gpu.log 2>&1
else timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -30 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
