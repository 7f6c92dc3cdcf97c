#!/bin/bash
# Same-box A/B of engine source trees: tmp_v/<name>/{paper_2604_16682_b200/csrc,include}
# (engine.cu + engine_core.h per tree; unit_ops.cu from the working tree).
#   gpurun -- bash tools/ab_engine.sh "c5 c3" [reps]
CONFIGS=${1:-c5}
REPS=${2:-2}
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in $(ls tmp_v); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared \
    -o /tmp/ab_$v.so tmp_v/$v/paper_2604_16682_b200/csrc/engine.cu paper_2604_16682_b200/csrc/unit_ops.cu &
done
wait
for C in $CONFIGS; do
  for r in $(seq $REPS); do
    for v in $(ls tmp_v); do
      ASB_LIB=/tmp/ab_$v.so timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline \
        > gpurun_out/ab/b.json 2>gpurun_out/ab/b.err
      python -c "import json; d=json.load(open('gpurun_out/ab/b.json')); print('$C $v rep $r', round(d['ms_per_step'],1))"
    done
  done
done
