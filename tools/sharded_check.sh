set -x
python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -5
for w in cfg2 cfg3_d0.30 cfg4 cfg5; do
  timeout 300 python bench.py --workload $w --sharded --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/sh1_$w.json
done
for w in cfg2 cfg3_d0.30 cfg4 cfg5; do
  IXB_DIST_BACKEND=gloo timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $w --sharded --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sh2_$w.json 2> gpurun_out/sh2_$w.err; echo rc=$?
done
tail -c 600 gpurun_out/sh1_*.json
