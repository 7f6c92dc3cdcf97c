#!/bin/bash
# Compile engine variants (extra -D flags) and time each on the C5 shard.
#   gpurun -- bash tools/variant_bench.sh TAG "-DA=1" "-DB=2 -DC" ...
# The first variant "" is the default build.  Output: gpurun_out/TAG/variants.txt
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
CONFIG=${ASB_CONFIG:-c5}
for DEFS in "$@"; do
  SO=/tmp/asb_var_$RANDOM.so
  nvcc $DEFS -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
    -shared -o $SO paper_2604_16682_b200/csrc/engine.cu paper_2604_16682_b200/csrc/unit_ops.cu || { echo "[$DEFS] build failed" >> $OUT/variants.txt; continue; }
  for rep in 1 2; do
    ASB_DEBUG_LAUNCH=1 ASB_LIB=$SO timeout 900 python bench.py --config $CONFIG --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/v.json 2>>$OUT/variants.err
    python -c "
import json,sys; d=json.load(open('$OUT/v.json')); print('[$DEFS] rep $rep ms/step %.2f kernel %.2f' % (d['ms_per_step'], d['roofline']['kernel_ms']))" >> $OUT/variants.txt
  done
done
cat $OUT/variants.txt
