#!/bin/bash
# full ncu capture of the engine on a small shard (8 seeds = 64 scenarios, 1 CTA/SM)
TAG=${1:-ncus}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:asb_engine -s 1 -c 1 \
    -o $OUT/engine python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --seeds-per-gpu ${SEEDS:-8} > $OUT/ncu_full.log 2>&1
ncu -i $OUT/engine.ncu-rep --page source --csv --print-source=cuda,sass > $OUT/source_cuda_sass.csv 2>/dev/null
ncu -i $OUT/engine.ncu-rep --page source --csv --print-source=sass > $OUT/source_sass.csv 2>/dev/null
echo done
