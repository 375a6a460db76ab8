# Smoke test of bench.py's multi-rank path on ONE GPU with host-side (gloo)
# collectives: 2 ranks share the device, no kernel waits on another rank.
mkdir -p gpurun_out
V2D_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 \
  --no-cpu-baseline > gpurun_out/multirank.log 2>&1; echo multirank=$?
grep "^{" gpurun_out/multirank.log | tail -1 | cut -c1-400
tail -5 gpurun_out/multirank.log | cut -c1-300
