# c2 / c3 throughput by lanes per stream
for l in ${LANES:-1 2}; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --lanes $l 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 lanes $l', '%.4g' % d['value'])"; done
for l in ${LANES3:-1 2}; do timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e --lanes $l 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 lanes $l', '%.4g' % d['value'])"; done
