for v in _prev "" _prev "" _prev ""; do
  L=paper_2604_16682_b200/_lib/libagentsim_b200$v.so
  r=$(ASB_LIB=$L timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f'%d['ms_per_step'])" 2>&1 | tail -1)
  echo "lib$v: $r ms"
done
