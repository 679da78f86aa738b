for v in "" "FIND_B200_PANEL=warp" "FIND_B200_PANEL=reg" "FIND_B200_PDL=1" "FIND_B200_PRIO=0"; do
  echo "== $v"; env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],2))"
done
