#!/bin/bash
# GPU-side profiling session (run under gpurun): bench lines, launch lists and
# one ncu --set full capture of each workload's hot kernel.
set -u
mkdir -p gpurun_out
for w in cfg2 cfg1 cfg3_d0.30 cfg3_d0.02 cfg5 cfg4; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
prof() {  # workload kernel-regex
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
      -o gpurun_out/prof_$1 python bench.py --workload $1 --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_$1.log 2>&1
}
prof cfg2 bgcoo_tc
prof cfg1 spmm_groupcoo
prof cfg3_d0.30 spmm_groupcoo
prof cfg5 conv_tc
ncu --set full --clock-control none --import-source on -k regex:tp_tc -s 1 -c 1 \
    -o gpurun_out/prof_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_cfg4.log 2>&1
ls -la gpurun_out
