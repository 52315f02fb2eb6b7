#!/bin/bash
# GPU-side profiling session (run under gpurun): the GPU test suite, bench
# lines for every workload, the cfg2 launch list and one ncu --set full
# capture of each workload's hot kernel (summarised by tools/ncu_summary.py).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
for w in cfg2 cfg1 cfg3_d0.30 cfg3_d0.02 cfg5 cfg4; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
prof() {  # workload kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-3} -c 1 \
      -o gpurun_out/prof_$1 python bench.py --workload $1 --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$1.ncu-rep $1 gpurun_out > /dev/null 2>&1
}
prof cfg2 bgcoo_tc
prof cfg1 spmm_groupcoo
prof cfg3_d0.30 spmm_groupcoo
prof cfg5 conv_unit
prof cfg4 tp_tc 1
ls -la gpurun_out
