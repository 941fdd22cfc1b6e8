#!/bin/bash
# Round-2 verification: full GPU suite + smoke, then c2/c3/c4/c5/reference bench lines
mkdir -p gpurun_out
bash tools/gpurun/tests.sh
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -1 gpurun_out/b_c2.json | cut -c1-400
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; tail -1 gpurun_out/b_c3.json | cut -c1-400
timeout 900 python bench.py --config c4 --total-streams 262144 --steps 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; tail -1 gpurun_out/b_c4.json | cut -c1-400
timeout 900 python bench.py --config c5 --total-streams 262144 --steps 3 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; tail -1 gpurun_out/b_c5.json | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; tail -1 gpurun_out/b_ref.json | cut -c1-400
