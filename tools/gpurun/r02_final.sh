#!/bin/bash
# Round-2 evidence: GPU tests + smoke, bench lines for every config (c4/c5 on the full 2^24 grid),
# the reference arm, the launch list, ncu captures of run_kernel (c2, c3, c5 max-accuracy launch),
# DRAM traffic at the bench shapes, compute-sanitizer.
mkdir -p gpurun_out
bash tools/gpurun/tests.sh
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; tail -1 gpurun_out/f_c2.json | cut -c1-200
timeout 900 python bench.py --config c3 > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err; tail -1 gpurun_out/f_c3.json | cut -c1-200
timeout 1500 python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err; tail -1 gpurun_out/f_c4.json | cut -c1-200
timeout 1800 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err; tail -1 gpurun_out/f_c5.json | cut -c1-200
timeout 900 python bench.py --config c1 > gpurun_out/f_c1.json 2> gpurun_out/f_c1.err; tail -1 gpurun_out/f_c1.json | cut -c1-200
timeout 900 python bench.py --config c2 --goal-changes 4 --steps 3 > gpurun_out/f_c2g.json 2> gpurun_out/f_c2g.err; tail -1 gpurun_out/f_c2g.json | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; tail -1 gpurun_out/f_ref.json | cut -c1-200
bash tools/gpurun/traffic.sh
bash tools/gpurun/prof_cfg.sh c2f --trace-steps 1000
bash tools/gpurun/prof_cfg.sh c3f --config c3 --total-streams 1048576 --trace-steps 100
bash tools/gpurun/prof_skip.sh c5maxf 1 --config c5 --total-streams 65536 --trace-steps 100
bash tools/gpurun/prof_skip.sh c4maxf 1 --config c4 --total-streams 65536 --trace-steps 100
# compute-sanitizer is closed on the GPU pool since the round-2 logs in profiles/r02_sanitizer_*.log
