# A/B of tuning environment variables on the default bench (one line per setting)
for v in "X=1" "X=2"; do
  echo "== $v"; env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['value'],1), round(d['ms_per_step'],2), k['warp']['ms_per_step_serialized'], k['mid']['ms_per_step_serialized'])"
done
