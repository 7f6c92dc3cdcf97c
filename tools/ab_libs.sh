#!/bin/bash
# Same-box A/B of prebuilt engine libraries tmp_v/*.so (bench with ASB_LIB).
#   gpurun -- bash tools/ab_libs.sh "c5 c3" [reps]
CONFIGS=${1:-c5}
REPS=${2:-2}
OUT=gpurun_out/ab
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for C in $CONFIGS; do
  for r in $(seq $REPS); do
    for lib in tmp_v/*.so; do
      v=$(basename $lib .so)
      ASB_LIB=$lib timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-e2e ${PARITY:+} $([ -z "$PARITY" ] && echo --no-cpu-baseline) \
        > $OUT/$C.$v.$r.json 2>$OUT/$C.$v.$r.err
      python -c "import json; d=json.load(open('$OUT/$C.$v.$r.json')); print('$C $v rep $r', round(d['ms_per_step'],1), round(d['roofline']['kernel_ms'],1), d.get('parity'))" || tail -3 $OUT/$C.$v.$r.err
    done
  done
done
