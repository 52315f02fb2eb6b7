for dbg in 0 1 2 3; do for v in 0 4; do
  r=$(IXB_BG_DEBUG=$dbg IXB_BG_VARIANT=$v python bench.py --no-cpu-baseline --steps 30 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2))" 2>&1 | tail -1)
  echo "debug=$dbg variant=$v us=$r"
done; done
