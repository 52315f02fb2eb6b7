#!/bin/bash
# bench lines + ncu captures of the K3 workloads only (after a K3 change)
mkdir -p gpurun_out
for w in cfg1 cfg3_d0.30 cfg3_d0.02; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for w in cfg1 cfg3_d0.30; do
  ncu --set full --clock-control none --import-source on -k regex:spmm_groupcoo -s 3 -c 1 \
      -o gpurun_out/prof_$w python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_$w.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$w.ncu-rep $w gpurun_out > /dev/null 2>&1
done
