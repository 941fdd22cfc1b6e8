#!/bin/bash
# Round-2 start: GPU tests + smoke, c2 and c3 bench lines on the unchanged round-1 build.
mkdir -p gpurun_out
bash tools/gpurun/tests.sh
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
tail -1 gpurun_out/b_c2.json; tail -1 gpurun_out/b_c3.json
