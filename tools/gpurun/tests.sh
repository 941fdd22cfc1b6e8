#!/bin/bash
# GPU test suite (optionally -k filter) + smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "$1" ]; then timeout 1500 python -m pytest tests -q -m gpu -k "$1" 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
else timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.log; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
cat gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|error|FAILED" | head -20; cat gpurun_out/smoke.log | tail -2
