#!/bin/bash
# new GPU tests (records, goals, bench grid, 2 ranks) + c2/c3/c4-sample bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "bench_grid or records or two_ranks" > gpurun_out/pytest_new.log 2>&1
tail -5 gpurun_out/pytest_new.log
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -1 gpurun_out/b_c2.json | cut -c1-600
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; tail -1 gpurun_out/b_c3.json | cut -c1-300
timeout 900 python bench.py --config c4 --total-streams 262144 --steps 2 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; tail -1 gpurun_out/b_c4.json | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; tail -1 gpurun_out/b_ref.json | cut -c1-300
