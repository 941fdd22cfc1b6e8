#!/bin/bash
# A/B bench lines: each argument line "TAG|ENV|bench args" -> value, frac
mkdir -p gpurun_out
while IFS='|' read -r tag envs args; do
  [ -z "$tag" ] && continue
  env $envs timeout 900 python bench.py $args --no-cpu --no-e2e > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().split('\n')[-1]); print('$tag', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'], d['config'].get('threads_per_block'), d['quality'].get('full_scan_fraction'))" 2>/dev/null || { echo "$tag FAILED"; tail -2 gpurun_out/ab_$tag.err; }
done < "${1:-tools/gpurun/ab.txt}"
