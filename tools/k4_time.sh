#!/bin/bash
# cfg2 K4 bench value for the shipped library and scratch_libs variants
for v in main "$@"; do
  if [ "$v" = main ]; then lp=""; else lp="$PWD/scratch_libs/$v/libixb.so"; fi
  IXB_LIB_PATH=$lp timeout 300 python bench.py --workload cfg2 --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e3,1), 'TFLOP/s')"
done
