set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2_r2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workloads none --no-sharded-records > /dev/null 2>&1
prof() {  # workload kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-3} -c 1 \
      -o gpurun_out/prof_$1 python bench.py --workload $1 --steps 3 --warmup 3 --no-cpu-baseline --workloads none --no-sharded-records \
      > gpurun_out/ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$1.ncu-rep $1 gpurun_out > /dev/null 2>&1
}
prof cfg2 bgcoo_tc
prof cfg5 conv_unit
prof cfg4 tp_tc 1
ls gpurun_out
