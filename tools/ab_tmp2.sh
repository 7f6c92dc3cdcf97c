for t in quad solo quad solo; do
  r=$(ASB_TEAM=$t timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f'%d['ms_per_step'], d['parity'])" 2>&1 | tail -1)
  echo "team $t: $r"
done
