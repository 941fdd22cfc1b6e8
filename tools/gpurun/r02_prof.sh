#!/bin/bash
# ncu full captures of run_kernel (SASS source counters exported as CSV on the box):
# c3 at 1M streams x 100 steps, c2 at 65,536 x 200, c5 (ALERT + oracle) at 65,536 grid items x 100 steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/gpurun/prof_cfg.sh c3 --config c3 --total-streams 1048576 --trace-steps 100
bash tools/gpurun/prof_cfg.sh c2 --trace-steps 200
bash tools/gpurun/prof_cfg.sh c5 --config c5 --total-streams 65536 --trace-steps 100
bash tools/gpurun/prof_cfg.sh c4 --config c4 --total-streams 65536 --trace-steps 100
ls -la gpurun_out
