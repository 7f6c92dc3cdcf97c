mkdir -p gpurun_out/r02d
for U in 2 8; do
  sed -i "s/^#define EC_SWEEP_UNROLL .*/#define EC_SWEEP_UNROLL $U \/* tmp *\//" paper_2604_16682_b200/csrc/engine_core.h
  ASB_PROFILE_SWEEP=1 timeout 600 python tools/profile_phases.py 64 gpurun_out/r02d/sweep_u$U.json > gpurun_out/r02d/sweep_u$U.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/r02d/sweep_u$U.json')); print('U=$U', d['step_ms'], {k: round(v) for k, v in d['phase_cycles_per_epoch'].items()})"
done
