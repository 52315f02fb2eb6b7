#!/bin/bash
# K4 cfg2 timing of the shipped library and every scratch_libs/ variant
# (perf experiment; build variants with tools/build_variant.sh)
mkdir -p gpurun_out
for v in main $(ls scratch_libs 2>/dev/null); do
  if [ $v = main ]; then lp=""; else lp=$PWD/scratch_libs/$v/libixb.so; fi
  echo -n "$v "; IXB_LIB_PATH=$lp timeout 120 python tools/k4_time.py --reps 30 2>&1 | tail -1
done
