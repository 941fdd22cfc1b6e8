#!/bin/bash
# Round-2 closing evidence after the HostStreamer pipeline change (kernels unchanged since the r02c
# ncu captures): GPU suite + smoke, bench lines for every config, the reference arm.
mkdir -p gpurun_out
bash tools/gpurun/tests.sh
timeout 900 python bench.py > gpurun_out/d_c2def.json 2> gpurun_out/d_c2def.err; tail -1 gpurun_out/d_c2def.json | cut -c1-160
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/d_c2.json 2> gpurun_out/d_c2.err; tail -1 gpurun_out/d_c2.json | cut -c1-160
timeout 900 python bench.py --config c3 > gpurun_out/d_c3.json 2> gpurun_out/d_c3.err; tail -1 gpurun_out/d_c3.json | cut -c1-160
timeout 1500 python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/d_c4.json 2> gpurun_out/d_c4.err; tail -1 gpurun_out/d_c4.json | cut -c1-160
timeout 1800 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/d_c5.json 2> gpurun_out/d_c5.err; tail -1 gpurun_out/d_c5.json | cut -c1-160
timeout 900 python bench.py --config c1 > gpurun_out/d_c1.json 2> gpurun_out/d_c1.err; tail -1 gpurun_out/d_c1.json | cut -c1-160
timeout 900 python bench.py --config c2 --goal-changes 4 --steps 3 > gpurun_out/d_c2g.json 2> gpurun_out/d_c2g.err; tail -1 gpurun_out/d_c2g.json | cut -c1-160
timeout 600 python bench.py --impl reference > gpurun_out/d_ref.json 2> gpurun_out/d_ref.err; tail -1 gpurun_out/d_ref.json | cut -c1-160
