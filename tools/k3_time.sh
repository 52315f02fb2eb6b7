#!/bin/bash
# cfg1 / cfg3 K3 bench value for the shipped library and scratch_libs variants
for v in main "$@"; do
  if [ "$v" = main ]; then lp=""; else lp="$PWD/scratch_libs/$v/libixb.so"; fi
  for w in ${K3_WORKLOADS:-cfg1 cfg3_d0.02}; do
    IXB_LIB_PATH=$lp timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --workloads none --no-sharded-records 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3))"
  done
done
