for i in 1 2; do
  for v in old new; do
    if [ $v = old ]; then d=_ab/old; else d=.; fi
    (cd $d && timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-comparator 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))")
  done
done
