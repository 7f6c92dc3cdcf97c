#!/bin/bash
# quick GPU iteration: parity tests + one bench line (+ optional phase profile)
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
python -c "
import json; d=json.load(open('$OUT/bench.json'))
print('ms/step', d['ms_per_step'], 'value %.3g'%d['value'], 'frac %.4f'%d['roofline']['frac'], d['parity'])"
if [ -n "$PHASES" ]; then
  timeout 600 python tools/profile_phases.py 64 $OUT/phases.json > $OUT/phases.log 2>&1
  python -c "
import json; d=json.load(open('$OUT/phases.json')); print(json.dumps(d['phase_cycles_per_epoch'])); print('mean/max', d['mean_cycles_per_scenario'], d['max_cycles_per_scenario'])"
fi
echo done
