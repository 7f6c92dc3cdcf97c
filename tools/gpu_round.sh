#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, the ncu launch list and
# one full ncu capture of the engine kernel.  Outputs land in gpurun_out/.
#   gpurun --timeout 2400 -- bash tools/gpu_round.sh [tag]
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:asb_engine -s 1 -c 1 \
    -o $OUT/engine python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
echo done
# the other BASELINE configs (reported in DESIGN.md; the driver's headline is the default, c5full)
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 900 python tools/time_batch_api.py 64 $OUT/batch_api.json > $OUT/batch_api.log 2>&1
echo done2
