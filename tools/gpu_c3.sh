#!/bin/bash
# C3 line + GPU parity tests + random stress (team-shape changes)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --config c3 --steps 3 --warmup 2 --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], '%.3g'%d['value'], d['parity'], 'cpu %.3g'%d['cpu_baseline']['value'])"
timeout 600 python tools/stress_parity.py 18 48 | tail -1
