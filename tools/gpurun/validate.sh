#!/bin/bash
# Full validation pass on a gpurun box: build, GPU tests, smoke, default bench, reference arm, launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
timeout 1500 python -m pytest tests -q -m gpu -x -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/bench_full.json gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_full.err
