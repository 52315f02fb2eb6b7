#!/bin/bash
# cfg5 K6 kernel time for the shipped library and each scratch_libs variant given
for v in main "$@"; do
  if [ "$v" = main ]; then lp=""; else lp="$PWD/scratch_libs/$v/libixb.so"; fi
  IXB_LIB_PATH=$lp timeout 300 python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],4), 'ms')"
done
