#!/bin/bash
# per-epoch phase cycles vs scenarios per GPU (i-cache / co-residency study)
OUT=gpurun_out/${1:-psweep}
mkdir -p $OUT
for s in 8 32 64; do
  timeout 600 python tools/profile_phases.py $s $OUT/phases_$s.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('$OUT/phases_$s.json')); print('seeds $s', d['scenarios'], 'step_ms %.1f'%d['step_ms'], {k: int(v) for k,v in d['phase_cycles_per_epoch'].items()}, 'max', int(d['max_cycles_per_scenario']/3600))"
done
