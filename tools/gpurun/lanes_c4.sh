# c4 / c5 throughput by lanes per stream
for c in c4 c5; do for l in ${LANES:-8 16 32}; do timeout 600 python bench.py --config $c --streams 262144 --steps 2 --warmup 3 --no-cpu --no-e2e --lanes $l 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c lanes $l', '%.4g' % d['value'])"; done; done
